"""Headline bench: KunServe's parameter-centric overload path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1] on one GPU): two Llama-3-8B bf16 replicas
-- both resident on the GPU as independent VMM slab pools with their own
paged KV pools -- each filled to 90% of its KV budget with ShareGPT-shaped
residents (lognormal, mean 1660 tokens).  A step is one overload cycle
through the public API (cycle.OverloadCycle): plan_drop -> drop 16 layers
per replica (their aliased slabs join the paged KV pool) -> coordinated KV
exchange (page gather/scatter kernels) -> burst drains (untimed) -> restore
(device page compaction + peer slab pull of 16 layers per replica) ->
dissolve + KV consolidation.  Every step ends in the boot layout; the run
checks bit-exact weights and KV checksums after the timed steps.

metric   drop/restore GB/s = payload bytes moved per step / step device time
         (CUDA events on the transfer stream, remaps included)
paged_decode   tcgen05 paged-decode attention over the merged (enlarged)
         pools, all 32 layers per token, tok/s
p99_ttft  the reference's scheduler on real Llama-3-8B pools with measured
         stage times (serving.DeviceEngine), KunServe vs the reference's three
         baselines -- recompute, swap (pages to pinned host memory over PCIe)
         and migrate (pages to the other replica) -- on one 4x ShareGPT-shaped
         burst (ttft.py)
With --gpus N each rank runs its own pair of replicas on its GPU (the path
shards into independent groups: scaling "weak", no data-path collective).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "P99 TTFT under overload burst; drop/restore NVLink GB/s; paged decode tok/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p.get("bf16_tflops"), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        try:  # initialise NVML outside the timed region (the first init is slow)
            import pynvml
            pynvml.nvmlInit()
        except Exception:
            pass

    def start(self):
        # NVML when available: a query costs microseconds, so the timed region
        # (tens of ms) gets many samples; nvidia-smi (~50 ms per call) otherwise
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [("hw_slowdown", pynvml.nvmlClocksThrottleReasonHwSlowdown),
                    ("hw_thermal_slowdown", pynvml.nvmlClocksThrottleReasonHwThermalSlowdown),
                    ("sw_thermal_slowdown", pynvml.nvmlClocksThrottleReasonSwThermalSlowdown),
                    ("sw_power_cap", pynvml.nvmlClocksThrottleReasonSwPowerCap)]

            def sample():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(self.device), str(sm), str(mx), "", ""] +
                                 ["Active" if rs & b else "Not Active" for _, b in bits])
            period = 0.005
        except Exception:
            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            period = 0.2

        def run():
            while not self._stop.is_set():
                try:
                    sample()
                except Exception:
                    pass
                self._stop.wait(period)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        sm = sorted(int(float(r[1])) for r in self.rows if len(r) > 2 and r[1] not in ("", "[N/A]"))
        mx = max((int(float(r[2])) for r in self.rows if len(r) > 2 and r[2] not in ("", "[N/A]")),
                 default=None)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, n in enumerate(names):
                if len(r) > 5 + k and r[5 + k] == "Active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def arm_config(kv_gib: float, residents: int, ws: int) -> dict:
    """The workload both arms report (the reference arm times a bounded
    sample of it, described in its cpu_baseline.sample)."""
    return {"workload": "llama3_8b bf16, 2 replicas per GPU -> 1 PP-2 group; "
                        "ShareGPT-shaped residents at 90% KV; drop+exchange+"
                        "restore+consolidate per step",
            "model": "llama3_8b", "replicas_per_gpu": 2,
            "kv_budget_gib_per_replica": kv_gib,
            "residents": residents, "parallelism": f"pp2 x{ws} (replica pairs)",
            "l2": "inputs larger than L2 (GB-scale moves per step)"}


def host_residents(kv_gib: float) -> dict:
    """The GPU arm's resident list (cycle.resident_tokens over two host
    instances with the same KV budget): {rid: tokens}."""
    from paper_2412_18169_b200 import memory
    from paper_2412_18169_b200.core import SHAPES
    from paper_2412_18169_b200.cycle import resident_tokens
    model = SHAPES["llama3_8b"].spec()
    caps = {i: memory.build_instance(i, model, model.param_bytes + int(kv_gib * (1 << 30)),
                                     900_000_000_000).kv.capacity_tokens for i in range(2)}
    return resident_tokens(caps)[0]


def run_reference(args) -> None:
    """CPU arm: the reference's path executed by the oracle port on host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.cpu_cycle import CpuCycle
    from paper_2412_18169_b200.core import SHAPES
    shape = SHAPES["llama3_8b"]
    model = shape.spec()
    full = host_residents(args.kv_gib)
    res = [full[r] for r in sorted(full)[:32]]  # the sample: the first 32 residents
    cyc = CpuCycle(model.bytes_per_layer, shape.page_bytes, shape.block_tokens, 2,
                   model.num_layers, res, model.kv_bytes_per_token)
    for _ in range(max(1, args.warmup)):
        cyc.step()
    t0 = time.perf_counter()
    moved = 0
    for _ in range(args.steps):
        r = cyc.step()
        moved += r["bytes"]
    dt = time.perf_counter() - t0
    gbs = moved / dt / 1e9
    sample = (f"2 of 32 Llama-3-8B layer slabs + the first {len(res)} of the {len(full)} "
              f"residents' pages per step, control plane at full size, numpy copies on "
              f"{cyc.threads} threads")
    line = {"metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "impl": "reference",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": arm_config(args.kv_gib, len(full), ws),
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": cyc.threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def copy_sweep(rt, iters: int = 5) -> dict:
    """Config 5 on one GPU: KV-block migration (scattered 256 KiB pages named
    by block tables) and layer restore (contiguous slab ranges) at 64 KiB x
    2^k up to 2 GiB (16 points).  Same-GPU copies read and write HBM, so the
    payload roofline is half the copy bandwidth; NVLink (peer pools) is 900
    GB/s per direction nominal.  The sources hold a deterministic pattern of
    (page, offset), and after the sweep every copied byte is checked on the
    device: each page's position-sensitive hash against its source page's,
    each slab's against its source slab's."""
    import torch
    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.core import SHAPES
    shape = SHAPES["llama3_8b"]
    model = shape.spec()
    rt2 = runtime.Runtime(rt.device, max_slots=4, max_pages_per_seq=8192)
    a = rt2.create_pool(0, model, model.param_bytes + (2 << 30) + (64 << 20), shape)
    b = rt2.create_pool(1, model, model.param_bytes + (2 << 30) + (64 << 20), shape)
    pb = shape.page_bytes
    npg = (2 << 30) // pb
    assert a.grow([(0, 0, 1, npg)]) and b.grow([(0, 0, 1, npg)])
    # f(page, offset): int32 words = golden-ratio hash of their global index
    kv = a.kv_bytes().view(torch.int32)
    kv.copy_((torch.arange(kv.numel(), dtype=torch.int64, device="cuda") * 2654435761 % (1 << 31))
             .to(torch.int32))
    for l in range(5):
        w = a.weight_bytes(l).view(torch.int32)
        w.copy_((torch.arange(w.numel(), dtype=torch.int64, device="cuda") * 40503 + l)
                .remainder(1 << 31).to(torch.int32))
    torch.cuda.synchronize()
    b.drop_layers(0, 5)
    b.restore_begin(0, 5)  # a 5-slab (2.19 GB) pull target
    out = {"pages": [], "slabs": []}
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    size = 64 << 10
    while size <= (2 << 30):
        n = max(1, size // pb)
        for kind in ("pages", "slabs"):
            def run():
                if kind == "pages":
                    runtime.copy_pages(b, a, [(0, 0, 0, 1, npg, 0, n)], stream=st)
                else:
                    runtime.copy_slabs(b, a, 0, 5, 0, size, stream=st)
            run()
            ev0.record(st)
            for _ in range(iters):
                run()
            ev1.record(st)
            ev1.synchronize()
            ms = ev0.elapsed_time(ev1) / iters
            moved = n * pb if kind == "pages" else size
            out[kind].append([size, round(moved / (ms / 1e3) / 1e9, 1)])
        size *= 2
    b.restore_complete(0, 5)
    torch.cuda.synchronize()
    # every byte of the largest point (2 GiB of pages, 2 GiB of slabs)
    pa = torch.tensor(a.block_table(0, 0), dtype=torch.int64, device="cuda")
    pb_ = torch.tensor(b.block_table(0, 0), dtype=torch.int64, device="cuda")
    ha = runtime.hash_segments(a.info().kv_base, pb, npg, index=pa)
    hb = runtime.hash_segments(b.info().kv_base, pb, npg, index=pb_)
    pages_ok = bool(torch.equal(ha, hb))
    rem = 2 << 30
    slabs_ok = True
    for l in range(5):
        nb = min(rem, model.bytes_per_layer)
        if nb <= 0:
            break
        slabs_ok &= bool(torch.equal(runtime.hash_tensor(a.weight_bytes(l)[:nb]),
                                     runtime.hash_tensor(b.weight_bytes(l)[:nb])))
        rem -= nb
    a.close()
    b.close()
    out["unit"] = "payload GB/s (same GPU: read + write HBM)"
    out["verified"] = {"pages_2GiB_hash_equal": pages_ok, "slabs_2GiB_hash_equal": slabs_ok}
    return out


def prefill_measure(rt, tensor_peak: float, ctx: int = 32768, chunk: int = 2048,
                    iters: int = 3, kv_splits=None) -> dict:
    """Config 4 attention: one Qwen2.5-14B layer, a 32k-token prompt prefilled
    in 2048-token chunks over the paged pool (each chunk attends to its
    prefix + itself causally).  FLOPs = 4*Hq*d*(p*c + c(c+1)/2) per chunk
    (costmodel.attention_units)."""
    import torch
    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.core import SHAPES
    shape = SHAPES["qwen25_14b"]
    model = shape.spec()
    rt = runtime.Runtime(rt.device, max_slots=4, max_pages_per_seq=ctx // shape.block_tokens)
    pool = rt.create_pool(0, model, model.param_bytes + (1 << 30), shape)
    B, Hq, Hkv = shape.block_tokens, shape.n_q_heads, shape.n_kv_heads
    assert pool.grow([(0, 0, 1, ctx // B)])
    g = torch.Generator(device="cuda").manual_seed(21)
    dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
    for s in range(0, ctx, 4096):
        k = torch.randn((4096, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn((4096, Hkv, 128), device="cuda", generator=g).to(torch.bfloat16)
        runtime.kv_append(pool, 0, k, v, dev([0] * 4096), torch.arange(s, s + 4096, dtype=torch.int32,
                                                                       device="cuda"))
    q = torch.randn((chunk, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty_like(q)
    flops = 0
    calls = []
    for p in range(0, ctx, chunk):
        flops += 4 * Hq * 128 * (p * chunk + chunk * (chunk + 1) // 2)
        calls.append((dev([0]), dev([0]), dev([chunk]), dev([p]), p + chunk))

    def run():
        for sl, off, ln, pre, kvl in calls:
            runtime.paged_prefill(pool, 0, q, sl, off, ln, pre, chunk, out, 128 ** -0.5,
                                  max_kv_len=kvl if kv_splits is None else None,
                                  kv_splits=kv_splits)
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        run()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / iters
    tf = flops / (ms / 1e3) / 1e12
    pool.close()
    return {"value": round(ctx / (ms / 1e3), 1), "unit": "tok/s (one layer, 32k prompt)",
            "ms_per_layer": round(ms, 3), "chunks": len(calls),
            "roofline": {"bound": "tensor", "achieved": round(tf, 1), "peak": tensor_peak,
                         "unit": "TFLOP/s", "frac": round(tf / tensor_peak, 4),
                         "traffic": (_traffic("prefill_tc_kernel") or {}).get(
                             "dram_bytes_per_launch"),
                         "flops_per_layer": flops}}


def decode_measure(cyc, iters: int, hbm_peak: float):
    """tcgen05 paged decode over the merged pools: one token for every
    resident through all 32 layers (each member decodes its stage)."""
    import torch
    from paper_2412_18169_b200 import runtime
    layout = cyc.merged_decode_layout()
    shape = cyc.shape
    Hq = shape.n_q_heads
    work = []
    nres = 0
    algo_bytes = 0
    for iid, ((lo, hi), res) in sorted(layout.items()):
        pool = cyc.pools[iid]
        n = len(res)
        nres = max(nres, n)
        g = torch.Generator(device="cuda").manual_seed(5 + iid)
        q = torch.randn((n, Hq, 128), device="cuda", generator=g).to(torch.bfloat16)
        out = torch.empty_like(q)
        slots = torch.tensor([s for _, s, _ in res], dtype=torch.int32, device="cuda")
        ctx = torch.tensor([c for _, _, c in res], dtype=torch.int32, device="cuda")
        ws = torch.empty(runtime.decode_workspace_bytes(n, Hq, 16), dtype=torch.uint8,
                         device="cuda")
        work.append((pool, lo, hi, q, slots, ctx, max(c for _, _, c in res), out, ws))
        per_layer = sum(c for _, _, c in res) * shape.kv_bytes_per_token_layer + 2 * n * Hq * 256
        algo_bytes += per_layer * (hi - lo)
    st = torch.cuda.current_stream()

    def one_token():
        for pool, lo, hi, q, slots, ctx, mx, out, ws in work:
            for l in range(lo, hi):  # one plan per decode step, reused by every layer
                runtime.paged_decode(pool, l, q, slots, ctx, mx, out, ws, 128 ** -0.5,
                                     max_splits=16, reuse_plan=l > lo, stream=st)
    for _ in range(3):
        one_token()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(iters):
        one_token()
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / iters
    # per member: one plan, then per layer one attention launch (which
    # merges the KV splits itself at this batch size) or attention + combine
    # (kb_paged_decode fuses from half a (sequence, kv head) pair per SM up:
    # KB_DEC_FUSE_MIN_PAIRS_PER_SM_X4 = 2, kb_decode.cu)
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    launches = sum(1 + (hi - lo) * (1 if 4 * q.shape[0] * pool.shape.n_kv_heads >= 2 * sms else 2)
                   for pool, lo, hi, q, *_ in work)
    gbs = algo_bytes / (ms / 1e3) / 1e9
    stage = decode_stage_measure(work[0], shape, hbm_peak)
    return {"value": round(nres / (ms / 1e3), 1), "unit": "tok/s",
            "tokens_per_step": nres, "ms_per_token_step": round(ms, 4),
            "note": "attention only, one token per resident through 32 layers",
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                         "traffic": (_traffic("decode_tc_kernel") or {}).get(
                             "dram_bytes_per_launch")},
            "launches_per_step": launches,
            "stage16": stage}


def decode_batch_sweep(rt, hbm_peak: float, sizes=(4, 16, 32, 64, 147), seed: int = 5) -> dict:
    """tools/decode_batch_probe.py's measurement inside the bench line:
    Llama-3-8B heads, ShareGPT-like contexts (lognormal around 1,500
    tokens), 16 layer launches per CUDA-graph replay over one plan, device
    time per layer at each batch size."""
    import numpy as np
    import torch
    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.core import ModelShape
    shape = ModelShape("g4", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8,
                       head_dim=128, ffn=1024, vocab=1024, block_tokens=64)
    rt2 = runtime.Runtime(rt.device, max_slots=256, max_pages_per_seq=128, slack_pages=256)
    model = shape.spec()
    pool = rt2.create_pool(0, model, model.param_bytes + (12 << 30), shape)
    rng = np.random.default_rng(seed)
    out = {}
    for nseq in sizes:
        ctx = np.clip(rng.lognormal(np.log(1500), 0.6, nseq), 16, 8000).astype(int)
        for s_, c in enumerate(ctx):
            pool.release([s_], 0, 2)
            assert pool.grow([(s_, 0, 2, (int(c) + 63) // 64)])
        q = torch.randn((nseq, 32, 128), device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        sl = torch.arange(nseq, dtype=torch.int32, device="cuda")
        cl = torch.tensor(ctx, dtype=torch.int32, device="cuda")
        ws = torch.empty(runtime.decode_workspace_bytes(nseq, 32, 16), dtype=torch.uint8,
                         device="cuda")
        mx = int(ctx.max())

        def step():
            for i in range(16):
                runtime.paged_decode(pool, i % 2, q, sl, cl, mx, o, ws, 128 ** -0.5,
                                     max_splits=16, reuse_plan=i > 0)
        for _ in range(5):
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
        gbs = algo / us / 1e3
        out[str(nseq)] = {"us_per_layer": round(us, 2), "hbm_gbs": round(gbs, 1),
                          "frac": round(gbs / hbm_peak, 4)}
    pool.close()
    return {"seed": seed, "sizes": out,
            "note": "tools/decode_batch_probe.py in-line: 16 layer launches per graph replay "
                    "over one plan, two alternating layers' pools"}


def decode_stage_measure(member, shape, hbm_peak: float, nseq: int = 16):
    """A pipeline stage's decode: the first `nseq` residents of one member
    through its stage's layers, replayed as a CUDA graph (as the serving
    engine replays decode-only stages), device time per layer."""
    import torch
    from paper_2412_18169_b200 import runtime
    pool, lo, hi, q, slots, ctx, mx, out, _ = member
    q, slots, ctx, out = q[:nseq], slots[:nseq], ctx[:nseq], out[:nseq]
    Hq = shape.n_q_heads
    ws = torch.empty(runtime.decode_workspace_bytes(nseq, Hq, 16), dtype=torch.uint8,
                     device="cuda")
    st = torch.cuda.Stream()
    mx = int(ctx.max())

    def step():
        for l in range(lo, hi):
            runtime.paged_decode(pool, l, q, slots, ctx, mx, out, ws, 128 ** -0.5,
                                 max_splits=16, reuse_plan=l > lo, stream=st)
    with torch.cuda.stream(st):
        for _ in range(3):
            step()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step()
    pool.stream_begin(st)
    reps = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
    pool.stream_end(st)
    b.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps / (hi - lo)
    per_layer = int(ctx.sum().item()) * shape.kv_bytes_per_token_layer + 2 * nseq * Hq * 256
    gbs = per_layer / (us / 1e6) / 1e9
    return {"sequences": nseq, "layers": hi - lo, "us_per_layer": round(us, 2),
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(gbs / hbm_peak, 4)},
            "note": "CUDA-graph replay of one stage's decode (16 layers), device time"}


def nvlink_measure(rt, shape, args, pp: int = 2) -> dict:
    """BASELINE configs[2]/[3]: one replica per GPU (rank r owns instance r),
    plan_drop merges (0,1), (2,3), ... into PP-2 groups spanning two GPUs;
    a step is drop -> KV exchange -> restore -> consolidation where every
    byte a rank receives is pulled from its peer's pool through a peer view
    (dist_cycle.DistCycle) -- NVLink traffic.  value = payload summed over
    ranks / max-over-ranks step time."""
    import torch
    from paper_2412_18169_b200 import dist_cycle
    ws = torch.distributed.get_world_size()
    out = dist_cycle.run(rt, shape, int(args.kv_gib * (1 << 30)), steps=args.steps,
                         warmup=args.warmup, key=f"bench{pp}", pipeline=pp == 2, pp=pp)
    ms = out["ms_total_max"]
    gbs = out["bytes_total"] / (ms / 1e3) / 1e9
    peer_gbs_per_gpu = out["bytes_peer"] / ws / (out["peer_kernel_ms_max"] / 1e3) / 1e9 \
        if out["peer_kernel_ms_max"] else 0.0
    last = out["last"]
    return {"value": round(gbs, 1), "unit": "GB/s", "n_gpus": ws,
            "workload": f"{shape.name} bf16, {ws} replicas on {ws} GPUs -> {ws // pp} PP-{pp} "
                        f"groups spanning GPUs; exchange + restore + consolidation over NVLink",
            "ms_per_step": round(ms / args.steps, 3),
            "peer_bytes_per_step": int(out["bytes_peer"] / args.steps),
            "roofline": ({"bound": "nvlink", "achieved": round(peer_gbs_per_gpu, 1),
                          "peak": 900.0, "unit": "GB/s per GPU per direction",
                          "frac": round(peer_gbs_per_gpu / 900.0, 4),
                          "kernel": "copy_pages_kernel + copy_flat_kernel pulling from peer views"}
                         if not out["peers_on_same_gpu"] else
                         {"bound": "hbm", "note": "ranks share one GPU (KB_BENCH_BACKEND=gloo "
                          "test mode): peer pulls read the same HBM, no NVLink",
                          "achieved": round(peer_gbs_per_gpu, 1), "unit": "GB/s payload"}),
            "rank0_ms": {k: round(v, 3) for k, v in last.ms.items()},
            "parity_bit_exact": out["parity_fail"] == 0,
            # the merged groups decoding as real cross-GPU pipelines: stage 0
            # on one GPU, stage 1 on its peer, activations handed over by the
            # copy kernel into the peer's IPC-mapped slots (dist.ActChannel)
            "pipelined_decode": None if out["pipeline"] is None else
            {k: (round(v, 3) if isinstance(v, float) else v) for k, v in out["pipeline"].items()}}


def _traffic(kernel: str):
    """{dram_bytes_per_launch, source} of `kernel` from the committed ncu
    capture (profiles/ncu_traffic.json: which capture, when), or None.  ncu
    cannot run inside the timed bench, so this is the last capture's number,
    labelled with its date."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)[kernel]
        return {"dram_bytes_per_launch": d.get("dram_bytes_per_launch"),
                "source": d.get("source", "profiles/ncu_traffic.json")}
    except (OSError, KeyError, ValueError):
        return None


def _summary(line: dict) -> dict:
    """The numbers a reader needs, last in the line (the driver keeps its tail)."""
    t = line.get("p99_ttft") or {}
    dec = (line.get("paged_decode") or {}).get("roofline", {})
    pre = (line.get("paged_prefill") or {}).get("roofline", {})
    pol = {p: {"p99_ttft_s": (t.get(p) or {}).get("p99_ttft_s"),
               "p50_tpot_s": (t.get(p) or {}).get("p50_tpot_s"),
               "served": (t.get(p) or {}).get("served")}
           for p in ("kunserve", "recompute", "swap", "migrate") if t.get(p)}
    return {"payload_gbs_same_gpu_proxy": line["value"], "e2e_gbs": line["e2e"]["value"],
            "copy_pages_frac": line["roofline"]["frac"],
            "param_pull_frac": line["roofline_param_pull"]["frac"],
            "decode_frac": dec.get("frac"),
            "decode_stage16_frac": (((line.get("paged_decode") or {}).get("stage16") or {})
                                    .get("roofline") or {}).get("frac"),
            "decode_sweep_frac": {k: v["frac"] for k, v in
                                  (((line.get("paged_decode") or {}).get("batch_sweep") or {})
                                   .get("sizes") or {}).items()},
            "prefill_frac": pre.get("frac"),
            "parity": line["parity"]["weights_bit_exact"] and line["parity"]["kv_bit_exact"],
            "ttft_clock": t.get("clock"), "ttft": pol,
            "criterion_4": t.get("criterion_4"),
            "nvlink_frac": (line.get("roofline_nvlink") or {}).get("frac")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kv-gib", type=float, default=16.0)
    ap.add_argument("--decode-iters", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttft", action="store_true",
                    help="skip the device-engine P99 TTFT measurement (~90 s)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    ws, rank, local = dist_env()
    # one GPU per rank; KB_BENCH_BACKEND=gloo lets several ranks share one
    # GPU to exercise the multi-rank path on a single-GPU box (NCCL refuses
    # two ranks on one device)
    backend = os.environ.get("KB_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    hbm_peak, _, peak_src = load_peaks()

    from paper_2412_18169_b200 import build as _build
    if rank == 0 or ws == 1:
        _build.build()
    if ws > 1:
        torch.distributed.barrier()
    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.core import SHAPES
    from paper_2412_18169_b200.cycle import OverloadCycle

    shape = SHAPES["llama3_8b"]
    rt = runtime.Runtime(local, max_slots=512, max_pages_per_seq=256)
    cyc = OverloadCycle([rt, rt], shape, int(args.kv_gib * (1 << 30)))
    w0 = cyc.weight_checksums()
    k0 = cyc.kv_checksums()
    for _ in range(args.warmup):
        cyc.step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    reps = []
    launches0 = runtime.LAUNCHES[0]
    # the collector runs between steps, not inside them (a full collection
    # of this process's heap costs milliseconds; serving loops do the same)
    gc.collect()
    gc.disable()
    t_host = time.perf_counter()
    for _ in range(args.steps):
        reps.append(cyc.step())
    torch.cuda.synchronize()
    host_s = time.perf_counter() - t_host
    gc.enable()
    launches = runtime.LAUNCHES[0] - launches0
    if ws > 1:
        torch.distributed.barrier()
    clk = clocks.stop()

    dev_ms = sum(r.ms["total"] for r in reps)
    payload = sum(r.payload_bytes for r in reps)
    if ws > 1:
        t = torch.tensor([dev_ms, float(payload)], dtype=torch.float64, device="cuda")
        mx = t.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = t.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        dev_ms, payload = float(mx[0]), int(sm[1])
    # headline: the reference's payload (sum of TransferTask.size_bytes of the
    # exchange, restore and consolidation tasks) per device-timed step
    value = payload / (dev_ms / 1e3) / 1e9
    # parity at full size, position-sensitive: every slab's 64-bit content
    # hash equals its boot value AND the other replica's (identical weights);
    # every long-lived resident's per-page hashes, in block-table order, equal
    # their boot values
    w1 = cyc.weight_checksums()
    k1 = cyc.kv_checksums()
    L = shape.num_layers
    parity = {"weights_bit_exact": w0 == w1 and all(w1[(0, l)] == w1[(1, l)] for l in range(L)),
              "kv_bit_exact": set(k0) == set(k1) and all(torch.equal(k0[r], k1[r]) for r in k0),
              "check": "kb_hash_segments (position-sensitive 64-bit hash) of all "
                       f"{2 * L} slabs and {sum(v.numel() for v in k1.values())} resident KV pages"}
    # the copy launches alone (events around them, no grows or queueing):
    # KV page copies (copy_pages_kernel, the time-dominant kernel) and slab
    # pulls (copy_flat_kernel); same-GPU copies read + write HBM
    kv_ms = sum(r.kv_copy_ms for r in reps)
    kv_b = sum(r.kv_copy_bytes for r in reps)
    kv_achieved = 2 * kv_b / (kv_ms / 1e3) / 1e9 if kv_ms else 0.0
    pk_ms = sum(r.param_copy_ms for r in reps)
    pk_b = sum(r.param_copy_bytes for r in reps)
    pk_achieved = 2 * pk_b / (pk_ms / 1e3) / 1e9 if pk_ms else 0.0
    kv_launches = sum(r.kv_copy_launches for r in reps)

    # paged decode in the merged state
    cyc.pause_merged = True
    cyc.step()
    dec = decode_measure(cyc, args.decode_iters, hbm_peak)
    cyc.resume()

    # e2e through the public API: each step's input is a queued burst (the
    # request table per replica, host data: traceio.synth_burst lengths) from
    # which plan_drop sizes the merge; the plan reaches the device as
    # descriptors through the C-ABI (block-table grows, page moves, release
    # lists, slab ranges: h2d_bytes_per_step, counted by the runtime); the
    # step's result -- every long-lived resident's first page on its home
    # pool, plus the compactions' moved-page counts -- is read back D2H
    res = torch.empty(len(cyc.tokens), dtype=torch.int32).pin_memory()
    cyc.auto_refill = False
    e2e_s = 0.0
    e2e_steps = []
    e2e_dev = []  # the same steps' device span (first to last event of the cycle)
    gc.collect()
    gc.disable()
    e_payload = 0
    h2d = []
    for i in range(args.warmup + args.steps):  # the first W steps are warm-up
        burst = cyc.burst_for(seed=100 + i)
        torch.cuda.synchronize()
        h0 = runtime.H2D_BYTES[0]
        t0 = time.perf_counter()
        # the result read-back is queued right behind the cycle's last device
        # operation; the step's host-side accounting overlaps the device tail
        # (light: no per-launch kernel timing -- that is the device-timed
        # loop's instrumentation, not part of a cycle)
        r = cyc.step(burst=burst, light=True,
                     on_enqueued=lambda: res.copy_(cyc.home_first_pages(), non_blocking=True))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_dev.append(round(r.ms["total"], 2))
            e2e_steps.append(round(dt * 1e3, 2))
            e2e_s += dt
            e_payload += r.payload_bytes
            h2d.append(runtime.H2D_BYTES[0] - h0)
        cyc.refill()  # the next burst's arrivals: not part of the cycle
    gc.enable()
    cyc.auto_refill = True
    r_last = reps[-1]
    cyc.close()
    _, tensor_peak, _ = load_peaks()
    prefill = prefill_measure(rt, tensor_peak or 1590.0)
    dec["batch_sweep"] = decode_batch_sweep(rt, hbm_peak)

    sweep = copy_sweep(rt) if ws == 1 else None
    # P99 TTFT: the reference's scheduler on real pools, KunServe vs the
    # reference's three baselines on one 4x burst
    ttft = None
    if not args.no_ttft and ws == 1:  # a single-GPU measurement (two replicas per GPU)
        from paper_2412_18169_b200.ttft import measure
        ttft = measure(kv_gib=1.25, base_rps=3.0, output_mean=128)

    # configs[2] across GPUs: replica r on GPU r, PP-2 groups spanning GPU
    # pairs, every exchange / restore / consolidation byte pulled over NVLink
    nvl = nvl4 = sweep_n = None
    if ws > 1:
        nvl = nvlink_measure(rt, shape, args)
        from paper_2412_18169_b200.dist import nvlink_sweep  # config 5 across GPUs
        sweep_n = nvlink_sweep(rt)
    if ws >= 4 and ws % 4 == 0:  # configs[3]: Qwen2.5-14B replicas into PP-4 groups
        nvl4 = nvlink_measure(rt, SHAPES["qwen25_14b"], args, pp=4)

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            from oracle.cpu_cycle import CpuCycle
            model = shape.spec()
            res_toks = [cyc.tokens[r] for r in sorted(cyc.tokens)][:32]
            cc = CpuCycle(model.bytes_per_layer, shape.page_bytes, shape.block_tokens, 2,
                          model.num_layers, res_toks, model.kv_bytes_per_token)
            cc.step()
            t0 = time.perf_counter()
            cb = 0
            for _ in range(3):
                cb += cc.step()["bytes"]
            cdt = time.perf_counter() - t0
            cpu = {"value": round(cb / cdt / 1e9, 3), "unit": "GB/s", "cores": cc.threads,
                   "kind": "port",
                   "sample": f"3 CPU cycles of 2 of 32 layer slabs + {len(res_toks)} residents' "
                             f"pages, numpy copies on {cc.threads} threads"}
        r0 = r_last
        trf = _traffic("copy_pages_kernel")
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dev_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "value_label": ("drop/restore payload GB/s (sum of TransferTask.size_bytes per "
                            "device-timed step); at N=1 a SAME-GPU HBM PROXY -- both replicas "
                            "share one B200, so no byte crosses NVLink; cross-GPU numbers are "
                            "nvlink_* (N>1)"),
            "config": arm_config(args.kv_gib, len(cyc.tokens), ws),
            "breakdown": {"payload_bytes_per_step": r0.payload_bytes,
                          "payload": {"kv_exchange": r0.payload_kv_exchange,
                                      "param_restore": r0.payload_param,
                                      "kv_consolidate": r0.payload_kv_consolidate},
                          "device_bytes": {"kv_exchange_pages": r0.bytes_kv_exchange,
                                           "param_restore": r0.bytes_param,
                                           "kv_consolidate_pages": r0.bytes_kv_consolidate},
                          "compaction_bytes_not_in_value": r0.bytes_compaction,
                          "ms": {k: round(v, 3) for k, v in r0.ms.items()},
                          "remap_ms": round(r0.remap_ns / 1e6, 3), "tasks": r0.n_tasks,
                          "host_enqueue_ms": {k: round(v, 3) for k, v in r0.host_ms.items()}},
            "roofline": {"bound": "hbm", "achieved": round(kv_achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(kv_achieved / hbm_peak, 4),
                         "traffic": trf.get("dram_bytes_per_launch") if trf else None,
                         "traffic_source": trf.get("source") if trf else None,
                         "kernel": "copy_pages_kernel (KV exchange + consolidation page copies; "
                                   "the step's time-dominant kernel); achieved = 2 x page bytes "
                                   "(read + write HBM) / copy-launch time, events around the "
                                   "launches alone",
                         "algorithmic_bytes_per_launch": round(2 * kv_b / max(1, kv_launches)),
                         # the measured peak is torch's own copy_ (MEASURED_PEAKS.json);
                         # one-CTA-per-piece streaming copies beat it, so also
                         # against the HBM3e spec (B200_PROFILING.md: 7.7 TB/s HGX)
                         "frac_vs_spec_7700": round(kv_achieved / 7700.0, 4),
                         "kernel_ms_per_step": round(kv_ms / args.steps, 3),
                         "peak_source": peak_src},
            "roofline_param_pull": {"bound": "hbm", "achieved": round(pk_achieved, 1),
                                    "peak": hbm_peak, "unit": "GB/s",
                                    "frac": round(pk_achieved / hbm_peak, 4),
                                    "frac_vs_spec_7700": round(pk_achieved / 7700.0, 4),
                                    "kernel": "copy_flat_kernel (slab pulls)",
                                    "kernel_ms_per_step": round(pk_ms / args.steps, 3),
                                    "traffic": (_traffic("copy_flat_kernel") or {}).get(
                                        "dram_bytes_per_launch"),
                                    "traffic_source": (_traffic("copy_flat_kernel") or {}).get(
                                        "source")},
            "paged_decode": dec,
            "paged_prefill": prefill,
            "copy_sweep": sweep,
            "p99_ttft": ttft,
            "nvlink_cycle": nvl,
            "nvlink_cycle_pp4": nvl4,
            "nvlink_sweep": sweep_n,
            "roofline_nvlink": (nvl or {}).get("roofline"),
            "parity": parity,
            "e2e": {"value": round(e_payload / e2e_s / 1e9, 1), "unit": "GB/s",
                    "h2d_bytes_per_step": int(sum(h2d) / max(1, len(h2d))),
                    "d2h_bytes_per_step": res.numel() * 4 + 16 * 2,
                    "ms_per_step": e2e_steps,
                    "device_span_ms_per_step": e2e_dev,
                    "input": "queued burst per replica -> plan_drop -> C-ABI descriptors "
                             "(grows, page moves, releases, slab ranges)"},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "host_s_timed": round(host_s, 3),
        }
        line["summary"] = _summary(line)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
