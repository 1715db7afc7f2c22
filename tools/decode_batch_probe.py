"""Paged decode device time per layer (CUDA-graph replay, 16 layers per
plan) at serving batch sizes (Llama-3-8B heads, ShareGPT-like contexts): the small batches a pipeline stage decodes, where
the split merge sits on the kernel's critical path.  A/B builds through
KB_LIB_PATH."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2412_18169_b200 import build  # noqa: E402
build.build()
from paper_2412_18169_b200 import runtime  # noqa: E402
from paper_2412_18169_b200.core import ModelShape  # noqa: E402

shape = ModelShape("g4", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                   ffn=1024, vocab=1024, block_tokens=64)
rt = runtime.Runtime(0, max_slots=256, max_pages_per_seq=128, slack_pages=256)
model = shape.spec()
pool = rt.create_pool(0, model, model.param_bytes + (12 << 30), shape)
rng = np.random.default_rng(int(os.environ.get("KB_PROBE_SEED", "5")))
MS = int(os.environ.get("KB_PROBE_MAX_SPLITS", "16"))
APPEND = os.environ.get("KB_PROBE_APPEND", "0") == "1"
# KB_PROBE_MERGE=1: force the combine launch, 0: force the in-kernel merge
KW = {"combine": os.environ["KB_PROBE_MERGE"] == "1"} if "KB_PROBE_MERGE" in os.environ else {}
out = {}
SIZES = ([int(x) for x in os.environ["KB_PROBE_NSEQ"].split(",")] if "KB_PROBE_NSEQ" in os.environ
         else [4, 16, 32, 64, 147])
for nseq in SIZES:
    ctx = np.clip(rng.lognormal(np.log(1500), 0.6, nseq), 16, 8000).astype(int)
    slots = list(range(nseq))
    for s, c in zip(slots, ctx):
        pool.release([s], 0, 2)
        assert pool.grow([(s, 0, 2, (int(c) + 63) // 64)])
    q = torch.randn((nseq, 32, 128), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    sl = torch.tensor(slots, dtype=torch.int32, device="cuda")
    cl = torch.tensor(ctx, dtype=torch.int32, device="cuda")
    ws = torch.empty(runtime.decode_workspace_bytes(nseq, 32, 16), dtype=torch.uint8, device="cuda")

    kn = torch.randn((nseq, 8, 128), device="cuda").to(torch.bfloat16)
    pos = torch.tensor(ctx - 1, dtype=torch.int32, device="cuda")

    def step():
        for i in range(16):
            if APPEND:  # the new token's K/V first, as a decode stage does
                runtime.kv_append(pool, i % 2, kn, kn, sl, pos)
            runtime.paged_decode(pool, i % 2, q, sl, cl, int(ctx.max()), o, ws, 128 ** -0.5,
                                 max_splits=MS, reuse_plan=i > 0, **KW)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    # captured in a CUDA graph, as the device engine replays decode-only
    # stages: device time, not the host's per-call launch cost
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / 20 / 16 * 1000  # per layer
    # algorithmic bytes per layer: every context token's K and V of every kv
    # head (2 x 8 x 128 x 2 B) plus q and out rows
    algo = int(ctx.sum()) * 2 * 8 * 128 * 2 + 2 * nseq * 32 * 128 * 2
    out[nseq] = {"us_per_layer": round(us, 2), "hbm_gbs": round(algo / us / 1e3, 1)}
peak = None
try:
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except Exception:
    pass
if peak:
    for v in out.values():
        v["frac"] = round(v["hbm_gbs"] / peak, 4)
print(json.dumps({"decode": out, "hbm_peak_gbs": peak}))
