"""Wall-clock TTFT run that keeps the event logs (gpurun_out/wall_logs_<tag>.json)."""
import json, sys, time
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
from paper_2412_18169_b200.ttft import measure
tag = sys.argv[1] if len(sys.argv) > 1 else "x"
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
kw = {"kv_gib": 1.25, "base_rps": 3.0, "output_mean": 128, **kw}
t0 = time.time()
res = measure(keep_logs=True, **kw)
logs = {p: res[p].pop("_log") for p in res if isinstance(res[p], dict) and "_log" in res[p]}
json.dump(logs, open(f"gpurun_out/wall_logs_{tag}.json", "w"))
print(json.dumps(res), flush=True)
print("wall", time.time() - t0)
