"""Prefill A/B probe for the library KB_LIB_PATH names (default: the in-tree
_kb.so): the bench's chunked config-4 layer (Qwen2.5-14B heads, 32k prompt in
2048-token chunks) and one causal square chunk (KB_PF_SQ tokens, default
8192), TFLOP/s and fraction of the measured bf16 peak.  Measurement only."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2412_18169_b200 import runtime  # noqa: E402

peak = bench.load_peaks()[1]
if os.environ.get("KB_PF_OLD_SPLITS") == "1":  # the round-2 split rule, for A/B
    def _old(nseq, n_q_heads, max_q_len, max_kv_len, n_sm=148):
        units = nseq * -(-max_q_len // 256) * n_q_heads
        tiles = -(-max_kv_len // 128)
        best, best_score = 1, units / (n_sm * -(-units // n_sm))
        for s in range(2, 9):
            if tiles < 16 * s:
                break
            score = units * s / (n_sm * -(-(units * s) // n_sm)) - 0.03 * (s - 1)
            if score > best_score:
                best, best_score = s, score
        return best
    runtime.prefill_splits = _old
rt = runtime.Runtime(0)
out = {"lib": os.path.basename(os.environ.get("KB_LIB_PATH", "_kb.so")), "old_splits": os.environ.get("KB_PF_OLD_SPLITS") == "1"}
ch = bench.prefill_measure(rt, peak)
out["chunked"] = {"ms": ch["ms_per_layer"], "frac": ch["roofline"]["frac"]}
sq = int(os.environ.get("KB_PF_SQ", 8192))
s = bench.prefill_measure(rt, peak, ctx=sq, chunk=sq, kv_splits=1)
out[f"square{sq}"] = {"ms": s["ms_per_layer"], "frac": s["roofline"]["frac"]}
print(json.dumps(out), flush=True)
