import sys, json, collections
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
from paper_2412_18169_b200.core import SHAPES
from paper_2412_18169_b200.serving import DeviceEngine, device_config
from paper_2412_18169_b200.metrics import collect, parse_line
from paper_2412_18169_b200.ttft import burst_trace, run_policy
shape = SHAPES["llama3_8b"]
trace = burst_trace(base_rps=3.0, output_mean=128)
cfg = device_config(shape, instances=2, kv_bytes=int(1.25 * (1 << 30)))
cfg.policy.kind = "recompute"
cfg.report.drain_s = 60.0
eng = DeviceEngine(cfg, trace)
res = eng.run()
st = collect(res.log_lines)
served = set()
kinds = collections.Counter()
per = collections.defaultdict(list)
for l in res.log_lines:
    t, k, f = parse_line(l)
    kinds[k] += 1
    r = f.get("req")
    if r is not None:
        per[int(r)].append((t, k))
    if k == "FIRST_TOKEN":
        served.add(int(f["req"]))
print(dict(kinds))
miss = [i for i in range(len(trace)) if i not in served]
print("unserved", miss[:10], "n", len(miss))
for r in miss[:3]:
    print(r, per[r][:12])
print("last log time", parse_line(res.log_lines[-1])[0])
for pool in eng.pools.values():
    pool.close()
