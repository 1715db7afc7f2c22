"""Device-backed serving: the reference's engine driving real B200 pools.

`DeviceEngine` keeps every scheduling decision of engine.Engine (itself a
byte-for-byte mirror of the reference's event loop, pkg/src/dropsim/engine.py)
and replaces the emulated device with real work:

  * every instance is a VMM slab pool with a paged KV pool
    (memory.build_instance(device=...)); drops / restores are device page
    remaps and compactions;
  * KV token allocations (group_alloc, engine.py:214-225) grow the members'
    block tables on the device; frees release pages;
  * every TransferTask executes on the GPU when its link starts it
    (transfer.TransferEngine): KV chunks are page copies between pools,
    parameter shards are slab pulls, activations are byte copies;
  * stage execution times are MEASURED: each microbatch's stage runs the
    member's Llama layers on its pool (cuBLAS GEMMs + this repo's kv_append,
    paged prefill and paged decode kernels over the pool's block tables),
    timed with CUDA events, and those times drive the event clock instead of
    the cost model (engine.py:389-397).
Link times (activations, KV exchange, restores) stay on the reference's link
model with the configured bandwidth (NVLink-5 in bench.py), because the
replicas of a one-GPU run share one HBM rather than an NVLink.
Supported policies: kunserve and the reference's three baselines
(engine.py:863-1047) -- recompute (evict + re-prefill), swap (the victim's
pages to pinned host memory and back, SM-driven over PCIe:
kb_copy_pages_host) and migrate (the victim's pages to another replica's
pool: kb_copy_pages).
"""

from __future__ import annotations

import collections
import gc

import math
from typing import Optional

from . import runtime
from .engine import Engine, GroupRun
from .exchange import TaskKind, TransferTask
from .transfer import SlotTable, TransferEngine


class LayerWeights:
    """bf16 views of one layer's slab: [Wqkv | Wo | Wgate_up | Wdown | norm1 | norm2],
    each stored as x @ W ([in, out], row-major)."""

    def __init__(self, slab, shape):
        import torch
        H, Hq, Hkv, d, F = shape.hidden, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, shape.ffn
        w = slab.view(torch.bfloat16)
        off = 0

        def take(n, dims):
            nonlocal off
            t = w[off:off + n].view(*dims)
            off += n
            return t
        self.wqkv = take(H * (Hq + 2 * Hkv) * d, (H, (Hq + 2 * Hkv) * d))
        self.wo = take(Hq * d * H, (Hq * d, H))
        self.wgu = take(H * 2 * F, (H, 2 * F))
        self.wd = take(F * H, (F, H))
        self.n1 = take(H, (H,))
        self.n2 = take(H, (H,))


def init_weights(pool, shape, layers, seed: int = 1000) -> None:
    """Identical replicas: layer l draws from seed + l (bf16 randn x 0.02,
    norms 1, 2 MiB rounding tail zero)."""
    import torch
    n = shape.layer_weight_bytes // 2
    for l in layers:
        slab = pool.weight_bytes(l)
        slab[2 * n:].zero_()
        g = torch.Generator(device=slab.device).manual_seed(seed + l)
        w = slab[:2 * n].view(torch.bfloat16)
        w.copy_((torch.randn(n, device=w.device, generator=g) * 0.02).to(torch.bfloat16))
        lw = LayerWeights(slab, shape)
        lw.n1.fill_(1.0)
        lw.n2.fill_(1.0)


class StageRunner:
    """Runs layers [lo, hi) of one pool for a microbatch of prefill chunks
    and decode tokens."""

    def __init__(self, pool, shape, max_seqs: int = 1024, max_splits: int = 16):
        import torch
        self.torch = torch
        self.pool = pool
        self.shape = shape
        self.max_splits = max_splits
        self.ws = torch.empty(runtime.decode_workspace_bytes(max_seqs, shape.n_q_heads, max_splits),
                              dtype=torch.uint8, device=f"cuda:{pool.rt.device}")
        self.max_seqs = max_seqs
        self.scale = shape.head_dim ** -0.5

    def _weights(self, l):
        # a layer's slab sits at a fixed weight VA (mapped once at pool
        # creation), so its views are built once
        if not hasattr(self, "_wcache"):
            self._wcache = {}
        w = self._wcache.get(l)
        if w is None:
            w = self._wcache[l] = LayerWeights(self.pool.weight_bytes(l), self.shape)
        return w

    # -- CUDA graphs for decode-only microbatches -------------------------
    # One graph per (layers, batch size), captured on first use after an
    # eager warm-up; inputs (hidden rows, slots, positions, context lengths)
    # are copied into the graph's static buffers before each replay.  Block
    # tables are read on device at replay time, so pages grown since capture
    # are seen.  Removes the per-launch host overhead from measured stage time.
    # Graphs of exact batch sizes are kept least-recently-used, at most
    # max_graphs of them (each holds a private pool for its intermediates,
    # outside the KV budget); the padded graphs of the wall-clock engine are
    # pinned.
    graphs_enabled = True
    max_graphs = 48

    def prepare_decode_graph(self, lo: int, hi: int, x, batch: dict) -> None:
        """Capture the (layers, batch size) graph if it does not exist yet.
        Runs outside the timed region: an eager warm-up (it writes the same
        K/V rows the replay writes again) and the capture."""
        torch = self.torch
        key = (lo, hi, batch["n"])
        if not hasattr(self, "_graphs"):
            self._graphs = collections.OrderedDict()
            self._pinned = set()
        if key in self._graphs:
            self._graphs.move_to_end(key)
            return
        while len(self._graphs) - len(self._pinned) >= self.max_graphs:
            old = next(k for k in self._graphs if k not in self._pinned)
            del self._graphs[old]  # its graph and private memory pool go with it
        self.run(lo, hi, x.clone(), batch)  # warm-up: lazy attributes, cuBLAS handles
        st = {"x": x.clone(), "slots": batch["slots"].clone(), "pos": batch["pos"].clone(),
              "d_slots": batch["d_slots"].clone(), "d_ctx": batch["d_ctx"].clone(),
              "d_rows": batch["d_rows"].clone()}
        sb = dict(batch, slots=st["slots"], pos=st["pos"], d_slots=st["d_slots"],
                  d_ctx=st["d_ctx"], d_rows=st["d_rows"])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        # no garbage collection inside the capture: a finalizer that frees a
        # device pool (kb_pool_destroy synchronizes the device) would
        # invalidate it
        gc.collect()
        gc.disable()
        try:
            with torch.cuda.graph(g):
                st["out"] = self.run(lo, hi, st["x"], sb)
        finally:
            gc.enable()
        self._graphs[key] = (g, st)

    def run_decode_graph(self, lo: int, hi: int, x, batch: dict):
        g, st = self._graphs[(lo, hi, batch["n"])]
        st["x"].copy_(x)
        for k in ("slots", "pos", "d_slots", "d_ctx"):
            st[k].copy_(batch[k])
        # a replay is invisible to the pool's stream ordering (captures record
        # no pool events): wait for its last bitmap op, and let later releases
        # / compactions wait for the replay
        self.pool.stream_begin()
        g.replay()
        self.pool.stream_end()
        return st["out"]

    # -- padded decode graphs (wall-clock serving) ------------------------
    # A decode-only microbatch of n rows replays the graph of the smallest
    # bucket >= n; the extra rows decode a reserved dummy slot (one page per
    # layer, context 1) from zero activations, so their K/V land in the dummy
    # page and their outputs are dropped (the caller pads the index vectors:
    # realtime.WallClockEngine._stage_batch).  Graphs are captured ahead of time
    # (capture_padded), so serving never captures.
    def capture_padded(self, lo: int, hi: int, n_pad: int, dummy_slot: int) -> None:
        torch = self.torch
        dev = self.pool.rt.device
        i32 = lambda v: torch.full((n_pad,), v, dtype=torch.int32, device=f"cuda:{dev}")  # noqa: E731
        b = {"n": n_pad, "np": 0, "nd": n_pad, "n_prefill_rows": 0, "slots": i32(dummy_slot),
             "pos": i32(0), "d_slots": i32(dummy_slot), "d_ctx": i32(1), "d_max": 1,
             "d_rows": torch.arange(n_pad, dtype=torch.int64, device=f"cuda:{dev}")}
        x = torch.zeros((n_pad, self.shape.hidden), dtype=torch.bfloat16, device=f"cuda:{dev}")
        self.prepare_decode_graph(lo, hi, x, b)
        self._pinned.add((lo, hi, n_pad))

    def run_padded_decode(self, lo: int, hi: int, x, batch: dict, n_pad: int):
        """Replay the (lo, hi, n_pad) graph for the first batch["n"] rows of
        `batch` (already padded with padded_batch); returns a fresh [n, hidden]
        tensor (the graph's static output is overwritten by the next replay)."""
        g, st = self._graphs[(lo, hi, n_pad)]
        n = x.shape[0]
        st["x"][:n].copy_(x)
        st["x"][n:].zero_()
        for k in ("slots", "pos", "d_slots", "d_ctx"):
            st[k].copy_(batch[k])
        self.pool.stream_begin()
        g.replay()
        self.pool.stream_end()
        return st["out"][:n].clone()

    def run(self, lo: int, hi: int, x, batch: dict):
        """Layers [lo, hi) over the microbatch rows x (bf16 [n, hidden],
        updated in place as the residual stream)."""
        torch = self.torch
        sh = self.shape
        Hq, Hkv, d, F = sh.n_q_heads, sh.n_kv_heads, sh.head_dim, sh.ffn
        n = x.shape[0]
        h = torch.empty_like(x)
        pending = None  # the previous layer's MLP output, added by the next norm
        for l in range(lo, hi):
            w = self._weights(l)
            runtime.add_rmsnorm(x, pending, w.n1, h)
            qkv = h @ w.wqkv
            q = qkv[:, :Hq * d].reshape(n, Hq, d)
            # K / V straight out of the fused projection (strided rows)
            k = qkv[:, Hq * d:(Hq + Hkv) * d].view(n, Hkv, d)
            v = qkv[:, (Hq + Hkv) * d:].view(n, Hkv, d)
            runtime.kv_append(self.pool, l, k, v, batch["slots"], batch["pos"])
            q = q.contiguous()
            o = torch.empty((n, Hq, d), dtype=x.dtype, device=x.device)
            # rows are ordered prefill chunks first, then decode tokens
            # (_batch), so each kind is a contiguous row range
            npr = batch.get("n_prefill_rows", 0)
            if batch["np"]:
                runtime.paged_prefill(self.pool, l, q[:npr], batch["p_slots"], batch["p_off"],
                                      batch["p_len"], batch["p_prefix"], batch["p_max"], o[:npr],
                                      self.scale, max_kv_len=batch.get("p_kv_max"))
            if batch["nd"]:
                runtime.paged_decode(self.pool, l, q[npr:], batch["d_slots"], batch["d_ctx"],
                                     batch["d_max"], o[npr:], self.ws, self.scale,
                                     max_splits=self.max_splits, reuse_plan=l > lo)
            runtime.add_rmsnorm(x, o.reshape(n, Hq * d) @ w.wo, w.n2, h)  # residual + norm 2
            gu = h @ w.wgu
            act = torch.empty((n, F), dtype=x.dtype, device=x.device)
            runtime.silu_mul(gu, act)
            pending = act @ w.wd
        if pending is not None:
            x.add_(pending)
        return x


class DeviceEngine(Engine):
    def __init__(self, cfg, trace, policy: Optional[str] = None, seed: int = 0,
                 runtimes: Optional[dict] = None, max_seqs: Optional[int] = None,
                 host_replica: bool = False):
        import torch
        self.torch = torch
        pol = policy or cfg.policy.kind
        if pol not in ("kunserve", "recompute", "swap", "migrate"):
            raise ValueError(f"unknown policy {pol}")
        if runtimes is None:
            runtimes = {d: runtime.Runtime(d, max_slots=cfg.device.max_slots,
                                           max_pages_per_seq=cfg.device.max_pages_per_seq)
                        for d in cfg.device.devices}
        self.runtimes = runtimes
        super().__init__(cfg, trace, policy=policy, seed=seed, runtimes=runtimes)
        self.shape = cfg.device.shape
        self.B = self.shape.block_tokens
        self.pools = {i: inst.pool for i, inst in self.instances.items()}
        self.slots = {i: SlotTable(cfg.device.max_slots) for i in self.instances}
        self.te = TransferEngine(self.pools, self.slots)
        self.transfer_hook = self._run_task
        # stream of block-table grows / releases (the transfer stream: a grow
        # always sees every earlier release; the wall-clock engine moves them
        # to the transfer engine's meta stream so they do not queue behind
        # KV bursts -- the pool orders bitmap ops on the device either way)
        self.page_stream = self.te.bulk
        for iid, inst in self.instances.items():
            init_weights(inst.pool, self.shape, inst.table.layers_held())
        if host_replica:
            # one full parameter copy in pinned host memory (the HOST source of
            # exchange.py:18, 224-233): the weights every replica boots with
            L = self.model.num_layers
            rep = torch.empty(self.model.param_bytes, dtype=torch.uint8).pin_memory()
            tmp = self.runtimes[cfg.device.devices[0]].create_pool(-1, self.model, self.model.param_bytes
                                                                   + (1 << 21), self.shape)
            init_weights(tmp, self.shape, range(L))
            for l in range(L):
                a = l * self.model.bytes_per_layer
                rep[a:a + self.model.bytes_per_layer].copy_(tmp.weight_bytes(l))
            tmp.close()
            self.te.host_replica = rep
        # a decode microbatch can hold every slot of a pool: size the
        # attention workspace for that (paged_decode refuses a smaller one)
        self.runners = {iid: StageRunner(p, self.shape, max_seqs=max_seqs or cfg.device.max_slots)
                        for iid, p in self.pools.items()}
        self.emb = {}
        for d in set(cfg.device.devices):
            g = torch.Generator(device=f"cuda:{d}").manual_seed(7)
            self.emb[d] = torch.randn((self.shape.vocab, self.shape.hidden), device=f"cuda:{d}",
                                      generator=g).to(torch.bfloat16)
        self.acts: dict = {}
        self._extra_tid = 1 << 40  # device-only pulls, outside the engine's tid space
        self.stage_samples: list = []   # (tokens, prefill_units, decode_tokens, layers, us)
        self.fetch_left: dict = {}
        torch.cuda.synchronize()

    def _dev_of(self, iid: int) -> int:
        return self.pools[iid].rt.device

    # ---------------------------------------------------------- KV pages
    def _ensure_pages(self, iid: int, rid: int, tokens: int, lo: int, hi: int) -> None:
        pool = self.pools[iid]
        slot = self.slots[iid].get(rid)
        need = -(-tokens // self.B)
        reqs = []
        for l in range(lo, hi):
            add = need - pool.npages(slot, l)
            if add > 0:
                if reqs and reqs[-1][2] == l and reqs[-1][3] == add:
                    reqs[-1] = (slot, reqs[-1][1], l + 1, add)
                else:
                    reqs.append((slot, l, l + 1, add))
        # page ops share one stream (the transfer stream) so a grow always
        # sees every earlier release; execution waits on that stream
        if reqs and not pool.grow(reqs, stream=self.page_stream):
            raise runtime.DeviceError(f"instance {iid}: out of KV pages for request {rid} "
                                      "(page slack exhausted)")

    def group_alloc(self, grun: GroupRun, rid: int, delta: int) -> bool:
        if not super().group_alloc(grun, rid, delta):
            return False
        total = self.total_alloc[rid]
        for iid in grun.group.member_instances:
            lo, hi = grun.group.stage_layer_map[iid]
            self._ensure_pages(iid, rid, total, lo, hi)
        return True

    def _release_everywhere(self, rid: int) -> None:
        L = self.model.num_layers
        for iid, slots in self.slots.items():
            slot = slots.of.get(rid)
            if slot is not None:
                self.pools[iid].release([slot], 0, L, stream=self.page_stream)
                slots.drop(rid)

    def group_free(self, grun: GroupRun, rid: int) -> None:
        super().group_free(grun, rid)
        self._release_everywhere(rid)

    # ---------------------------------------------------------- transfers
    def _run_task(self, task: TransferTask) -> None:
        if task.kind is TaskKind.ACTIVATION:
            return  # the stage inputs were handed over when the round executed
        if task.kind is TaskKind.KVCACHE_CHUNK and task.tid not in self.te.chunk_of:
            # a baseline's whole-request move (swap out / in, migrate): the
            # request's pages of every layer, destination pages already allocated
            self.te.register_request_move(task, (0, self.model.num_layers),
                                          self.requests[task.rid].context_len)
        self.te.submit(task)

    def fail_instance(self, iid: int) -> None:
        """engine.Engine.fail_instance on the device: the failed pool's weight
        slabs are overwritten first, so a restore that read from it could not
        reproduce the boot weights."""
        pool = self.pools[iid]
        for l in self.instances[iid].table.layers_held():
            pool.weight_bytes(l).fill_(0x7F)
        super().fail_instance(iid)

    def _transfers_landed(self) -> None:
        """Called when the engine's clock says a transfer finished: the
        simulated clock runs ahead of the device, so wait for the copies
        (the wall-clock engine only fires the callback once the task's own
        event completed, so there it just collects finished tasks)."""
        self.te.drain()

    def _swap_in_done(self, gid, task, when) -> None:
        self._transfers_landed()    # the host copy has been read
        self.te.release_host(task.rid)
        super()._swap_in_done(gid, task, when)

    def _migrate_done(self, src_gid, dst_gid, task, tokens, when) -> None:
        # the source pages free behind the copy (same stream, device-ordered)
        slot = self.slots[task.src].of.get(task.rid)
        if slot is not None:
            self.pools[task.src].release([slot], 0, self.model.num_layers, stream=self.te.bulk)
            self.slots[task.src].drop(task.rid)
        super()._migrate_done(src_gid, dst_gid, task, tokens, when)

    def _on_exchange_planned(self, tasks, old_map, new_map, tokens) -> None:
        self.te.register_exchange(tasks, old_map, new_map, tokens)

    def _on_params_planned(self, tasks, fetch: bool, **restore) -> None:
        self.te.register_restore(tasks, self.model.bytes_per_layer)
        missing = restore.get("missing")
        if missing:
            self._pull_uncovered(missing, restore["holders"], restore["chunk"])
        if fetch:  # merge-time fetch: vacate the destination slab first
            for t in tasks:
                key = (t.dst, t.layers)
                if key not in self.fetch_left:
                    self.pools[t.dst].restore_begin(*t.layers, stream=self.te.bulk)
                    self.fetch_left[key] = 0
                self.fetch_left[key] += 1

    def _pull_uncovered(self, missing: dict, holders: dict, chunk: int) -> None:
        """The reference plans one range per restoring member
        (engine.py:1127: {iid: rng for ... for rng in rngs} keeps the last),
        so a member that misses two disjoint ranges (the middle members of a
        PP-4 group) would complete_restore layers nobody pulled.  In
        simulation that is invisible; on the device those slabs may hold KV
        pages by now.  The event log keeps the reference's tasks; the other
        ranges are pulled here, on the same stream, ahead of them -- they
        land before the reference's last restore chunk completes."""
        from .exchange import plan_restore_transfers
        extra = []
        for k in range(max(len(r) for r in missing.values())):
            flat = {iid: rngs[k] for iid, rngs in missing.items() if len(rngs) > k + 1}
            if flat:
                extra += plan_restore_transfers(flat, holders, self.model.bytes_per_layer, chunk,
                                                tid_start=self._extra_tid + len(extra))
        if extra:
            self._extra_tid += len(extra)
            self.te.register_restore(extra, self.model.bytes_per_layer)
            self.te.submit_many(extra)

    def _fetch_done(self, gid, task, when) -> None:
        self._transfers_landed()
        key = (task.dst, task.layers)
        if key in self.fetch_left:
            self.fetch_left[key] -= 1
            if self.fetch_left[key] == 0:
                del self.fetch_left[key]
                self.pools[task.dst].restore_complete(*task.layers)
        super()._fetch_done(gid, task, when)

    def _exchange_chunk_done(self, task, when) -> None:
        self._transfers_landed()
        self.te.finish_flow_sources()
        super()._exchange_chunk_done(task, when)

    def _restore_chunk_done(self, gid, task, when) -> None:
        self._transfers_landed()  # the slab bytes land before complete_restore flips ownership
        super()._restore_chunk_done(gid, task, when)

    def _on_consolidation_planned(self, rid, peer, home, layers, tasks) -> None:
        self.te.register_chunked_kv(tasks, layers, {rid: self.requests[rid].context_len})

    def _on_consolidated(self, rid, peers) -> None:
        self._transfers_landed()
        self.te.finish_flow_sources()
        L = self.model.num_layers
        for iid in peers:
            slot = self.slots[iid].of.get(rid)
            if slot is not None:
                self.pools[iid].release([slot], 0, L, stream=self.page_stream)
                self.slots[iid].drop(rid)

    # ---------------------------------------------------------- execution
    def _to_device(self, xs, dtype, dev):
        return self.torch.tensor(xs, dtype=dtype, device=dev)

    def _batch(self, iid: int, mb) -> dict:
        torch = self.torch
        dev = f"cuda:{self._dev_of(iid)}"
        slots, pos = [], []
        p_rows, p_slots, p_off, p_len, p_prefix = [], [], [], [], []
        d_rows, d_slots, d_ctx = [], [], []
        last_rows = []  # rows that produce a token: decodes, last row of each prefill chunk
        row = 0
        # prefill chunks first, then decode tokens: each kind is one
        # contiguous row range for the attention kernels (row order is free:
        # every row's output depends only on its own request)
        ordered = [ch for ch in mb.chunks if not ch.decode] + [ch for ch in mb.chunks if ch.decode]
        n_prefill_rows = sum(ch.token_count for ch in mb.chunks if not ch.decode)
        for ch in ordered:
            slot = self.slots[iid].of[ch.rid]
            if ch.decode:
                ctx = ch.prefix_len  # context incl. the token being decoded
                slots.append(slot)
                pos.append(ctx - 1)
                d_rows.append(row)
                d_slots.append(slot)
                d_ctx.append(ctx)
                last_rows.append(row)
                row += 1
            else:
                c, p = ch.token_count, ch.prefix_len
                slots.extend([slot] * c)
                pos.extend(range(p, p + c))
                p_off.append(len(p_rows))
                p_rows.extend(range(row, row + c))
                p_slots.append(slot)
                p_len.append(c)
                p_prefix.append(p)
                row += c
                last_rows.append(row - 1)
        i32 = lambda xs: self._to_device(xs, torch.int32, dev)  # noqa: E731
        i64 = lambda xs: self._to_device(xs, torch.int64, dev)  # noqa: E731
        return {"n": row, "slots": i32(slots), "pos": i32(pos), "n_prefill_rows": n_prefill_rows,
                "np": len(p_slots), "p_rows": i64(p_rows), "p_slots": i32(p_slots),
                "p_off": i32(p_off), "p_len": i32(p_len), "p_prefix": i32(p_prefix),
                "p_max": max(p_len) if p_len else 0,
                "p_kv_max": max((a + b for a, b in zip(p_prefix, p_len)), default=0),
                "nd": len(d_slots), "d_rows": i64(d_rows), "d_slots": i32(d_slots),
                "d_ctx": i32(d_ctx), "d_max": max(d_ctx) if d_ctx else 0,
                "last": i64(last_rows),
                "units": sum(ch.token_count * ch.prefix_len + (ch.token_count ** 2 + ch.token_count) / 2
                             for ch in mb.chunks if not ch.decode)}

    def _stage_times(self, grun: GroupRun, mbs, spans) -> list:
        """Execute every (microbatch, stage) of the round on its member's pool
        and return the measured times in us (one device sync per round)."""
        torch = self.torch
        members = grun.group.member_instances
        st = torch.cuda.current_stream()
        st.wait_stream(self.te.bulk)  # KV moves / restores this round depends on
        events = []
        for k, mb in enumerate(mbs):
            x = None
            for s, iid in enumerate(members):
                lo, hi = grun.group.stage_layer_map[iid]
                b = self._batch(iid, mb)
                if x is None:
                    ids = torch.randint(0, self.shape.vocab, (b["n"],), device=b["slots"].device)
                    x = self.emb[self._dev_of(iid)].index_select(0, ids)
                elif x.device != b["slots"].device:
                    x = x.to(b["slots"].device)
                a = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                runner = self.runners[iid]
                use_graph = b["np"] == 0 and runner.graphs_enabled
                if use_graph:
                    runner.prepare_decode_graph(lo, hi, x, b)  # untimed capture
                a.record(st)
                if use_graph:
                    x = runner.run_decode_graph(lo, hi, x, b)
                else:
                    x = runner.run(lo, hi, x, b)
                if s == len(members) - 1:  # sample the next token of each sequence
                    lw = self.emb[self._dev_of(iid)]
                    if b["last"].numel():
                        logits = x.index_select(0, b["last"]) @ lw.t()
                        logits.argmax(dim=-1)
                e.record(st)
                events.append((s, k, a, e, b["n"], b["units"], b["nd"], hi - lo))
        e.synchronize()
        for iid in members:  # the fp16 V cache's range guard (kb_pool_kv_status)
            self.pools[iid].check_kv_range(synchronize=False)
        times = [[1] * len(mbs) for _ in members]
        for s, k, a, e, n, units, nd, layers in events:
            us = max(1, int(round(a.elapsed_time(e) * 1000)))
            times[s][k] = us
            self.stage_samples.append((n, units, nd, layers, us))
        return times


def device_config(shape, instances: int = 2, kv_bytes: int = 8 << 30, devices=(0,),
                  nvlink_bandwidth: int = 900_000_000_000, link_latency_us: int = 5,
                  host_bandwidth: int = 50_000_000_000,
                  map_latency_us: int = 0):
    """SimConfig for `instances` replicas of `shape` with `kv_bytes` of KV
    budget each, NVLink-5 links, a PCIe Gen5 x16 host link (swap baseline)
    and the aliased-slab remap cost."""
    from .config import SimConfig
    cfg = SimConfig()
    cfg.model = shape.spec()
    cfg.cluster.instances = instances
    cfg.cluster.hbm_bytes = cfg.model.param_bytes + kv_bytes
    cfg.cluster.nic_bandwidth = nvlink_bandwidth
    cfg.cluster.host_bandwidth = host_bandwidth
    cfg.cluster.link_base_latency_us = link_latency_us
    cfg.cluster.map_latency_us = map_latency_us
    cfg.device.shape = shape
    cfg.device.devices = tuple(devices)
    cfg.device.max_pages_per_seq = max(64, math.ceil(32768 / shape.block_tokens))
    cfg.device.max_slots = 512
    if len(set(devices)) < instances:
        # members of a pipeline group share a GPU here, so their stages
        # cannot overlap: the lookahead formulation's small microbatches
        # (formulation.py, split down to min_batch_tokens = 256) would only
        # re-read every stage's weights once more per microbatch.  Split no
        # finer than the token budget (the reference's own knob, config.py).
        cfg.policy.min_batch_tokens = cfg.policy.token_budget
    return cfg
