"""Stress the wall-clock serving engine: the bench's TTFT measurement
(ttft.measure, all four policies) repeated over trace seeds and rates, each
run's outcome printed -- timing-dependent interleavings of monitor ticks and
in-flight rounds differ run to run.  Measurement / test tool.

    python tools/wall_stress.py [runs]
"""
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import importlib  # noqa: E402

from paper_2412_18169_b200 import build  # noqa: E402

ttft = importlib.import_module("paper_2412_18169_b200.ttft")

build.build()
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fails = 0
for i in range(runs):
    kw = dict(kv_gib=1.25, base_rps=3.0 + 0.5 * (i % 3), output_mean=128, seed=100 + i)
    try:
        r = ttft.measure(**kw)
        print(json.dumps({"run": i, "ok": True, **{p: {"p99": v["p99_ttft_s"], "served": v.get("served")}
                                                   for p, v in r.items() if isinstance(v, dict) and "p99_ttft_s" in v}}),
              flush=True)
    except Exception:
        fails += 1
        print(json.dumps({"run": i, "ok": False, "kw": kw}), flush=True)
        traceback.print_exc()
print("FAILS", fails)
