"""ORACLE -- the overload cycle on the host CPU.  CPU BASELINE ONLY
(bench.py's cpu_baseline and --impl reference legs; never the product).

The reference simulates the drop/restore path on one Python thread and moves
no bytes (pkg/src/dropsim/memory.py, exchange.py).  This is its CPU
execution: the control plane is oracle/dropsim_port.py (the reference's
algorithms, pinned against its golden outputs) and the data plane moves
the same bytes the GPU path moves -- KV pages named by block tables and
parameter slabs -- between host-memory replicas with numpy copies spread
over every host thread.  The sample is bounded (a slice of the layers and
residents) so a step costs seconds, and reports GB/s of moved payload.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np

from . import dropsim_port as ds


def _par_copy(dst: np.ndarray, src: np.ndarray, pool, parts: int) -> None:
    n = src.shape[0]
    cuts = [n * i // parts for i in range(parts + 1)]
    list(pool.map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]),
                  range(parts)))


def _par_gather(dst: np.ndarray, didx: np.ndarray, src: np.ndarray, sidx: np.ndarray, pool,
                parts: int) -> None:
    n = len(sidx)
    cuts = [n * i // parts for i in range(parts + 1)]

    def run(i):
        a, b = cuts[i], cuts[i + 1]
        dst[didx[a:b]] = src[sidx[a:b]]
    list(pool.map(run, range(parts)))


class CpuCycle:
    """Two replicas on the host: `layers` layer slabs of `slab_bytes` each and
    a page pool of `pages` pages; residents with ShareGPT-like context."""

    def __init__(self, slab_bytes: int, page_bytes: int, block_tokens: int, layers: int,
                 full_layers: int, residents: list[int], kvbpt: int, threads: int = 0):
        self.threads = threads or len(os.sched_getaffinity(0))
        self.pool = cf.ThreadPoolExecutor(self.threads)
        self.L = full_layers
        self.layers = layers
        self.slab = slab_bytes
        self.page = page_bytes
        self.B = block_tokens
        self.kvbpt = kvbpt
        self.residents = residents
        self.npg = [-(-t // block_tokens) for t in residents]
        pages = sum(self.npg) * layers * 2 + 16
        rng = np.random.default_rng(0)
        self.w = [rng.integers(0, 255, size=(layers, slab_bytes), dtype=np.uint8),
                  np.zeros((layers, slab_bytes), dtype=np.uint8)]
        self.kv = [rng.integers(0, 255, size=(pages, page_bytes), dtype=np.uint8),
                   np.zeros((pages, page_bytes), dtype=np.uint8)]

    def step(self) -> dict:
        t0 = time.perf_counter()
        L, half = self.L, self.layers // 2
        P = L * self.slab
        # control plane at full size (the reference's own algorithms)
        merges, freed, fb, _ = ds.plan_drop([(0, {0: (0, L)}), (1, {1: (0, L)})], P // 2, L, P)
        smap = merges[0][4]
        toks = {rid: t for rid, t in enumerate(self.residents)}
        tasks = ds.plan_exchange(toks, {0: (0, L)}, smap, L, self.kvbpt, 64 << 20)
        ds.plan_restore_transfers({0: (L // 2, L)}, {0: [(0, L // 2)], 1: [(L // 2, L)]},
                                  self.slab, 256 << 20)
        t_ctl = time.perf_counter() - t0
        # data plane on the sampled layers: exchange (half the layers of every
        # resident's pages), parameter restore (half the slabs), consolidation
        per_layer = sum(self.npg)
        src_idx = np.arange(half * per_layer, 2 * half * per_layer, dtype=np.int64)
        dst_idx = np.arange(0, half * per_layer, dtype=np.int64)
        moved = 0
        _par_gather(self.kv[1], dst_idx, self.kv[0], src_idx, self.pool, self.threads)
        moved += len(src_idx) * self.page
        _par_copy(self.w[1][:half], self.w[0][half:2 * half], self.pool, self.threads)
        moved += half * self.slab
        _par_gather(self.kv[0], src_idx, self.kv[1], dst_idx, self.pool, self.threads)
        moved += len(src_idx) * self.page
        dt = time.perf_counter() - t0
        return {"bytes": moved, "seconds": dt, "control_s": t_ctl, "tasks": len(tasks),
                "gbs": moved / dt / 1e9}
