"""Paged decode over the merged bench state (bench.decode_measure) without
the rest of the bench: two Llama-3-8B replicas, 16 GiB KV each, 90% full."""
import json
import sys
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
import bench
from paper_2412_18169_b200 import runtime
from paper_2412_18169_b200.core import SHAPES
from paper_2412_18169_b200.cycle import OverloadCycle
rt = runtime.Runtime(0, max_slots=512, max_pages_per_seq=256)
cyc = OverloadCycle([rt, rt], SHAPES["llama3_8b"], 16 << 30)
cyc.pause_merged = True
cyc.step()
for _ in range(2):
    d = bench.decode_measure(cyc, 10, 6548.2)
print(json.dumps({"tok_s": d["value"], "frac": d["roofline"]["frac"], "ms": d["ms_per_token_step"]}))
