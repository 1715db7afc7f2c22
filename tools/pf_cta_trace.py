"""Per-CTA timeline of one config-4 prefill chunk launch (Qwen2.5-14B heads,
2048 new tokens at a given prefix, the runtime's KV split): ramp (entry ->
first S), body, drain (last P -> exit), and per-SM idle between
consecutive CTAs.  Variant build with -DKB_PF_CTA_TRACE
(tools/var/_kb_pfcta.so).

    python tools/pf_cta_trace.py [prefix] [splits]
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "tools", "var", "_kb_pfcta.so")

if os.environ.get("KB_LIB_PATH") != VAR:
    from paper_2412_18169_b200 import build
    os.makedirs(os.path.dirname(VAR), exist_ok=True)
    build.build_variant(VAR, ["-DKB_PF_CTA_TRACE"])
    env = dict(os.environ, KB_LIB_PATH=VAR)
    sys.exit(subprocess.call([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))

import torch  # noqa: E402

from paper_2412_18169_b200 import runtime  # noqa: E402
from paper_2412_18169_b200.core import SHAPES  # noqa: E402

pre = int(sys.argv[1]) if len(sys.argv) > 1 else 30720
ks = int(sys.argv[2]) if len(sys.argv) > 2 else None
chunk, ctx = 2048, pre + 2048
shape = SHAPES["qwen25_14b"]
model = shape.spec()
rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=-(-ctx // shape.block_tokens))
pool = rt.create_pool(0, model, model.param_bytes + (1 << 30), shape)
B, Hq, Hkv = shape.block_tokens, shape.n_q_heads, shape.n_kv_heads
assert pool.grow([(0, 0, 1, -(-ctx // B))])
g = torch.Generator(device="cuda").manual_seed(21)
dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
for s in range(0, ctx, 2048):
    k = torch.randn((2048, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
    runtime.kv_append(pool, 0, k, k, dev([0] * 2048), torch.arange(s, s + 2048, dtype=torch.int32,
                                                                   device="cuda"))
q = torch.randn((chunk, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
out = torch.empty_like(q)
args = (dev([0]), dev([0]), dev([chunk]), dev([pre]))
splits = ks or runtime.prefill_splits(1, Hq, chunk, ctx)
for _ in range(3):
    runtime.paged_prefill(pool, 0, q, *args, chunk, out, 128 ** -0.5, kv_splits=splits)
torch.cuda.synchronize()
fn = runtime._lib.kb_debug_pf_cta_trace
fn.argtypes = [C.c_void_p, C.c_int32]
buf = (C.c_ulonglong * (8192 * 5))()
assert fn(C.addressof(buf), 8192 * 5) == 0
ncta = -(-chunk // 256) * Hq * splits
t = np.array(buf, dtype=np.uint64).reshape(8192, 5)[:ncta].astype(np.int64)
t0 = t[:, 0].min()
e, s1, p2, x = [(t[:, i] - t0) / 1e3 for i in range(4)]
sm = t[:, 4]
span = x.max()
res = {"prefix": pre, "splits": splits, "ctas": int(ncta), "span_us": round(float(span), 1),
       "cta_us_med": round(float(np.median(x - e)), 1),
       "ramp_us (entry->first S) med/p90": [round(float(np.median(s1 - e)), 2), round(float(np.percentile(s1 - e, 90)), 2)],
       "drain_us (last P->exit) med/p90": [round(float(np.median(x - p2)), 2), round(float(np.percentile(x - p2, 90)), 2)],
       "body_us med": round(float(np.median(p2 - s1)), 1)}
busy = np.zeros(int(sm.max()) + 1)
gaps = []
for m in np.unique(sm):
    idx = np.where(sm == m)[0]
    idx = idx[np.argsort(e[idx])]
    busy[m] = float((x[idx] - e[idx]).sum())
    gaps += list(e[idx][1:] - x[idx][:-1])
    res.setdefault("first_entry_max", 0.0)
res["sm_busy_frac"] = round(float(busy.sum() / (len(np.unique(sm)) * span)), 4)
res["gap_between_ctas_us med/p90"] = [round(float(np.median(gaps)), 2), round(float(np.percentile(gaps, 90)), 2)]
res["last_exit_minus_median_last_exit_per_sm"] = round(float(span - np.median(
    [x[sm == m].max() for m in np.unique(sm)])), 2)
# the time the tensor pipe could have been fed: sum of bodies / (SMs x span)
res["body_frac"] = round(float((p2 - s1).sum() / (len(np.unique(sm)) * span)), 4)
print(json.dumps(res))
