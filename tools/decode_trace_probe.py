"""Phase timeline of one decode_tc_kernel launch (per-CTA %globaltimer stamps,
variant build with -DKB_DEC_TRACE) at a pipeline stage's batch sizes.

    python tools/decode_trace_probe.py            # builds tools/var/_kb_trace.so, re-execs

Slots: 0 entry, 1 after griddepcontrol.wait, 2 producer has item 0,
3 first TMA issued, 4 first tile landed (MMA warp), 5 first S in TMEM
(softmax), 6/7/8 items 0/1/2 done, 9 last item done, 10 exit; 11 items, 12 tiles.
Times in us relative to the earliest CTA entry."""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "tools", "var", "_kb_trace.so")

if os.environ.get("KB_LIB_PATH") != VAR:
    from paper_2412_18169_b200 import build
    os.makedirs(os.path.dirname(VAR), exist_ok=True)
    build.build_variant(VAR, ["-DKB_DEC_TRACE"] + sys.argv[1:])
    env = dict(os.environ, KB_LIB_PATH=VAR)
    sys.exit(subprocess.call([sys.executable, os.path.abspath(__file__)], env=env))

import torch  # noqa: E402

from paper_2412_18169_b200 import runtime  # noqa: E402
from paper_2412_18169_b200.core import ModelShape  # noqa: E402

shape = ModelShape("g4", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                   ffn=1024, vocab=1024, block_tokens=64)
rt = runtime.Runtime(0, max_slots=256, max_pages_per_seq=128, slack_pages=256)
model = shape.spec()
pool = rt.create_pool(0, model, model.param_bytes + (12 << 30), shape)
rng = np.random.default_rng(5)
fn = runtime._lib.kb_debug_dec_trace
fn.argtypes = [C.c_void_p, C.c_int32]
SL = 16
res = {}
for nseq in [int(x) for x in os.environ.get("KB_PROBE_SIZES", "4,16,32,147").split(",")]:
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
    for i in range(6):
        runtime.paged_decode(pool, i % 2, q, sl, cl, int(ctx.max()), o, ws, 128 ** -0.5,
                             max_splits=16, reuse_plan=i > 0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    runtime.paged_decode(pool, 1, q, sl, cl, int(ctx.max()), o, ws, 128 ** -0.5,
                         max_splits=16, reuse_plan=True)
    b.record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (148 * SL))()
    assert fn(C.addressof(buf), 148 * SL) == 0
    t = np.array(buf, dtype=np.uint64).reshape(148, SL).astype(np.int64)
    t0 = t[:, 0].min()
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    names = {0: "entry", 1: "post_wait", 2: "item0", 3: "tma0", 4: "land0", 5: "s0",
             6: "item0_done", 7: "item1_done", 8: "item2_done", 9: "last_done", 10: "exit"}
    row = {}
    for k, nm in names.items():
        v = rel(k)
        v = v[(v >= 0) & (v < 1e4)]
        if len(v):
            row[nm] = {"min": round(float(v.min()), 2), "med": round(float(np.median(v)), 2),
                       "max": round(float(v.max()), 2)}
    row["items_per_cta"] = np.bincount(t[:, 11].clip(0, 20)).tolist()
    row["tiles_per_cta"] = {"min": int(t[:, 12].min()), "med": float(np.median(t[:, 12])),
                            "max": int(t[:, 12].max())}
    row["event_us"] = round(a.elapsed_time(b) * 1e3, 2)
    algo = int(ctx.sum()) * 2 * 8 * 128 * 2
    row["kv_mb"] = round(algo / 1e6, 1)
    row["ideal_us_at_6.5TBs"] = round(algo / 6.5e6, 2)
    res[nseq] = row
    print(nseq, json.dumps(row), flush=True)
