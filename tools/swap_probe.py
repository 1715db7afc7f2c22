"""Why a wall-clock swap run leaves requests unserved: run one policy on one
bench-style trace and report the end state of every request without a first
token (state, home, queue position, swap bookkeeping).  Debug tool.

    python tools/swap_probe.py [policy] [seed] [rps]
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import importlib  # noqa: E402

from paper_2412_18169_b200 import build  # noqa: E402
from paper_2412_18169_b200.core import SHAPES  # noqa: E402
from paper_2412_18169_b200.metrics import collect  # noqa: E402
from paper_2412_18169_b200.serving import device_config  # noqa: E402

ttft = importlib.import_module("paper_2412_18169_b200.ttft")
build.build()
policy = sys.argv[1] if len(sys.argv) > 1 else "swap"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rps = float(sys.argv[3]) if len(sys.argv) > 3 else 3.0
clock = sys.argv[4] if len(sys.argv) > 4 else "wall"
trace = ttft.burst_trace(base_rps=rps, output_mean=128, seed=seed)
shape = SHAPES["llama3_8b"]
cfg = device_config(shape, instances=2, kv_bytes=int(1.25 * (1 << 30)))
cfg.policy.kind = policy
cfg.report.drain_s = 60.0
if len(sys.argv) > 5 and sys.argv[5] == "fit":  # plan with the warm-up refit, as ttft.measure
    from paper_2412_18169_b200.costmodel import CostCoefficients
    warm = ttft.burst_trace(duration_s=4.0, base_rps=4.0, input_mean=1660, output_mean=8, seed=11)
    w, _ = ttft.run_policy("kunserve", warm, shape, int(0.25 * (1 << 30)), clock=clock)
    f = w["cost_fit"]
    cfg.cost = CostCoefficients(alpha=f["alpha"], beta=f["beta"], gamma=f["gamma"])
if clock == "wall":
    from paper_2412_18169_b200.realtime import WallClockEngine
    eng = WallClockEngine(cfg, trace)
else:
    from paper_2412_18169_b200.serving import DeviceEngine
    eng = DeviceEngine(cfg, trace)
res = eng.run()
st = collect(res.log_lines)
served = {rid for rid, r in st.requests.items() if r.first_token_us is not None}
kinds = collections.Counter(l.split(" ", 2)[1] for l in res.log_lines)
stuck = []
for rid, req in sorted(eng.requests.items()):
    if rid in served:
        continue
    stuck.append({"rid": rid, "state": req.state.value, "home": req.home_instance,
                  "in": req.input_len, "out": req.output_len, "prefilled": req.tokens_prefilled,
                  "decoded": req.tokens_decoded,
                  "swap_inflight": rid in getattr(eng, "swap_inflight", ()),
                  "host_kv": rid in getattr(eng.te, "host_kv", {})})
print(json.dumps({"policy": policy, "clock": clock, "requests": len(trace), "created": len(eng.requests),
                  "served": len(served), "kinds": dict(kinds), "stuck": stuck[:40]}, indent=0))
last = res.log_lines[-15:]
print("\n".join(last))
