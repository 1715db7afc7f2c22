"""One square (32k causal, Qwen2.5-14B heads) prefill launch of this repo's
kernel and one of FlashAttention-4 (vllm.vllm_flash_attn.cute), for a side by
side `ncu --set full` capture.  Measurement only.

    ncu --set full -k regex:'prefill_tc|flash|Flash' -c 2 python tools/fa4_ncu_pair.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_18169_b200 import build, runtime  # noqa: E402

build.build()
rt = runtime.Runtime(0)
bench.prefill_measure(rt, 1637.1, ctx=8192, chunk=8192, kv_splits=1, iters=1)
from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402
ctx = int(os.environ.get("KB_SQ", 8192))
g = torch.Generator(device="cuda").manual_seed(21)
k = torch.randn((1, ctx, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn((1, ctx, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
q = torch.randn((1, ctx, 40, 128), device="cuda", generator=g).to(torch.bfloat16)
flash_attn_func(q, k, v, softmax_scale=128 ** -0.5, causal=True)
torch.cuda.synchronize()
