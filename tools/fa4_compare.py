"""Library ceiling for the config-4 prefill: FlashAttention-4 (the CuTe-DSL
sm100 forward vllm ships, vllm.vllm_flash_attn.cute) on the bench's
workload -- one Qwen2.5-14B layer (40 q / 8 kv heads, d 128), a 32k prompt
in 2048-token chunks, each chunk causal over its prefix + itself -- with
contiguous (non-paged) K/V, beside this repo's paged kernel
(bench.prefill_measure).  Measurement only; nothing here is on a product
path.

    python tools/fa4_compare.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def fa4(ctx=32768, chunk=2048, Hq=40, Hkv=8, iters=3):
    from vllm.vllm_flash_attn.cute.interface import flash_attn_func
    g = torch.Generator(device="cuda").manual_seed(21)
    k = torch.randn((1, ctx, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((1, ctx, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
    q = torch.randn((1, chunk, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
    flops = 0
    calls = []
    for p in range(0, ctx, chunk):
        flops += 4 * Hq * 128 * (p * chunk + chunk * (chunk + 1) // 2)
        calls.append((k[:, :p + chunk], v[:, :p + chunk]))

    def run():
        for kk, vv in calls:
            flash_attn_func(q, kk, vv, softmax_scale=128 ** -0.5, causal=True)
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        run()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / iters
    # dense square case as well: 32k x 32k causal, one call
    qf = torch.randn((1, ctx, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
    flash_attn_func(qf, k, v, softmax_scale=128 ** -0.5, causal=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(iters):
        flash_attn_func(qf, k, v, softmax_scale=128 ** -0.5, causal=True)
    b.record()
    b.synchronize()
    ms_sq = a.elapsed_time(b) / iters
    flops_sq = 4 * Hq * 128 * ctx * (ctx + 1) // 2
    return {"chunked_ms_per_layer": round(ms, 3), "chunked_tflops": round(flops / ms / 1e9, 1),
            "square_ms": round(ms_sq, 3), "square_tflops": round(flops_sq / ms_sq / 1e9, 1)}


if __name__ == "__main__":
    import bench
    from paper_2412_18169_b200 import build, runtime
    build.build()
    peak = bench.load_peaks()[1]
    rt = runtime.Runtime(0)
    ours = bench.prefill_measure(rt, peak)
    out = {"ours_paged": {"ms_per_layer": ours["ms_per_layer"],
                          "tflops": ours["roofline"]["achieved"], "frac": ours["roofline"]["frac"]}}
    # the same kernel on one 32k causal chunk (no prefix): 5,120 CTAs, so no
    # wave quantisation -- the kernel's own efficiency
    sq = bench.prefill_measure(rt, peak, chunk=32768, kv_splits=1)
    out["ours_square"] = {"ms": sq["ms_per_layer"], "tflops": sq["roofline"]["achieved"],
                          "frac": sq["roofline"]["frac"]}
    for ks in (1, 2, 4, 8):
        r = bench.prefill_measure(rt, peak, kv_splits=ks)
        out[f"ours_splits{ks}"] = {"ms": r["ms_per_layer"], "tflops": r["roofline"]["achieved"]}
    try:
        out["fa4_contiguous"] = fa4()
        out["fa4_contiguous"]["frac"] = round(out["fa4_contiguous"]["chunked_tflops"] / peak, 4)
    except Exception as e:  # library path unavailable on this box
        out["fa4_contiguous"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    out["peak_tflops"] = peak
    print(json.dumps(out))
