"""Library reference point for the small-batch paged decode: FlashInfer's
BatchDecodeWithPagedKVCacheWrapper (HND pages of 64 tokens -- the same
[K|V][kv head][64 tok][128] page this repo stores) on the workload of
tools/decode_batch_probe.py: Llama-3-8B heads (32 q / 8 kv), lognormal
contexts around 1,500 tokens (seed 5), 16 layer calls alternating over two
layer caches per CUDA-graph replay, device time per layer.  Measurement only
(library code, never on a product path).

    python tools/decode_lib_compare.py
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import flashinfer
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rng = np.random.default_rng(int(os.environ.get("KB_PROBE_SEED", "5")))
    sizes = [int(x) for x in os.environ.get("KB_PROBE_NSEQ", "4,16,32,64,147").split(",")]
    out = {}
    for nseq in sizes:
        ctx = np.clip(rng.lognormal(np.log(1500), 0.6, nseq), 16, 8000).astype(int)
        npg = (ctx + 63) // 64
        indptr = torch.tensor(np.concatenate([[0], np.cumsum(npg)]), dtype=torch.int32, device="cuda")
        total = int(npg.sum())
        indices = torch.arange(total, dtype=torch.int32, device="cuda")
        last = torch.tensor(ctx - (npg - 1) * 64, dtype=torch.int32, device="cuda")
        caches = [torch.randn((total, 2, 8, 64, 128), device="cuda").to(torch.bfloat16)
                  for _ in range(2)]
        q = torch.randn((nseq, 32, 128), device="cuda").to(torch.bfloat16)
        row = {}
        for tc in (False, True):
            ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(
                ws, kv_layout="HND", use_cuda_graph=True, use_tensor_cores=tc,
                paged_kv_indptr_buffer=indptr.clone(), paged_kv_indices_buffer=indices.clone(),
                paged_kv_last_page_len_buffer=last.clone())
            w.plan(indptr, indices, last, 32, 8, 128, 64, q_data_type=torch.bfloat16,
                   kv_data_type=torch.bfloat16, sm_scale=128 ** -0.5)
            o = torch.empty_like(q)

            def step():
                for i in range(16):
                    w.run(q, caches[i % 2], out=o)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
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
            us = a.elapsed_time(b) / 20 / 16 * 1000
            algo = int(ctx.sum()) * 2 * 8 * 128 * 2 + 2 * nseq * 32 * 128 * 2
            row["tensor_cores" if tc else "cuda_cores"] = {
                "us_per_layer": round(us, 2), "frac": round(algo / us / 1e3 / peak, 4)}
        out[nseq] = row
        print(nseq, json.dumps(row), flush=True)
    print(json.dumps({"flashinfer_decode": out, "hbm_peak_gbs": peak}))


if __name__ == "__main__":
    main()
