import json, sys, time
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
from paper_2412_18169_b200.ttft import measure
kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
t0 = time.time()
print(json.dumps(measure(**kw)), flush=True)
print("wall", time.time() - t0)
