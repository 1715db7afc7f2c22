import json, sys, time
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
from paper_2412_18169_b200.ttft import measure
# default: the bench's p99_ttft configuration (bench.py); argv[1]: JSON kwargs
kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {"kv_gib": 1.25, "base_rps": 3.0,
                                                        "output_mean": 128}
t0 = time.time()
print(json.dumps(measure(**kw)), flush=True)
print("wall", time.time() - t0)
