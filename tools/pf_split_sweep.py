"""Per-chunk KV-split sweep of the config-4 prefill layer (Qwen2.5-14B
heads, 32k prompt, 2048-token chunks): device time of every chunk for each
split count, beside what runtime.prefill_splits picks.  Tuning tool.

    python tools/pf_split_sweep.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2412_18169_b200 import build, runtime  # noqa: E402
from paper_2412_18169_b200.core import SHAPES  # noqa: E402

build.build()
ctx, chunk = 32768, 2048
shape = SHAPES["qwen25_14b"]
model = shape.spec()
rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=ctx // shape.block_tokens)
pool = rt.create_pool(0, model, model.param_bytes + (1 << 30), shape)
B, Hq, Hkv = shape.block_tokens, shape.n_q_heads, shape.n_kv_heads
assert pool.grow([(0, 0, 1, ctx // B)])
g = torch.Generator(device="cuda").manual_seed(21)
dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
for s in range(0, ctx, 4096):
    k = torch.randn((4096, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
    runtime.kv_append(pool, 0, k, k, dev([0] * 4096), torch.arange(s, s + 4096, dtype=torch.int32,
                                                                   device="cuda"))
q = torch.randn((chunk, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
out = torch.empty_like(q)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
for p in range(0, ctx, chunk):
    args = (dev([0]), dev([0]), dev([chunk]), dev([p]))
    auto = runtime.prefill_splits(1, Hq, chunk, p + chunk)
    row = {"auto": auto}
    for ks in (1, 2, 3, 4, 5, 6, 8):
        def call():
            runtime.paged_prefill(pool, 0, q, *args, chunk, out, 128 ** -0.5, kv_splits=ks)
        call()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for _ in range(5):
            call()
        b.record()
        b.synchronize()
        row[ks] = round(a.elapsed_time(b) / 5 * 1e3, 1)
    best = min((k for k in row if k != "auto"), key=lambda k: row[k])
    row["best"] = best
    res[p] = row
    print(p, json.dumps(row), flush=True)
tot_auto = sum(r[r["auto"]] for r in res.values())
tot_best = sum(r[r["best"]] for r in res.values())
print(json.dumps({"total_us_auto": round(tot_auto, 1), "total_us_best": round(tot_best, 1)}))
