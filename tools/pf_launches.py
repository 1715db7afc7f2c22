"""One pass of the bench's chunked config-4 prefill layer (16 chunks) for an
ncu launch list: per-chunk attention and split-combine kernel durations.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/pf_launches.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2412_18169_b200 import runtime  # noqa: E402

bench.prefill_measure(runtime.Runtime(0), 1637.1, iters=1)
