"""Device execution of TransferTasks (N4 / N5 / N6 / N7).

The reference times every task on a serialized link model
(pkg/src/dropsim/exchange.py:49-101) and the engine consumes them through
`enqueue_task(task, cb)` / `cb(task, done_us)` (engine.py:279-302).  Here the
same task lists run on the GPU:

  KVCACHE_CHUNK  -> kb_copy_pages over a slice of the flow's pages.  A flow
                    is (rid, src -> dst) over the layer overlap of the old and
                    new stage maps (exchange.py:146-205); chunk k of n covers
                    flattened pages [k*P//n, (k+1)*P//n) of the flow's
                    P = layers x pages, so the chunks tile the flow exactly.
                    The destination's pages are grown on the first chunk,
                    the source's released after the last one lands.
  PARAM_SHARD    -> kb_copy_slabs over consecutive byte ranges of the run's
                    layers (exchange.py:208-249); HOST sources come from a
                    pinned host replica (kb_copy_slabs_from_host).
  ACTIVATION     -> kb_copy_bytes (stage s -> s+1 hand-off, engine.py:428-448).

Scheduling (N6): activations go on a high-priority stream, KV chunks and
parameter shards on a low-priority stream in FIFO order -- the device
version of `_PRIO` (exchange.py:27-28).  Chunks are the preemption points,
as in the reference; completion is a CUDA event the engine polls.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Optional

from . import runtime
from .exchange import HOST, TaskKind, TransferTask


class SlotTable:
    """rid -> block-table slot on one pool (lowest free slot first)."""

    def __init__(self, max_slots: int):
        self.max_slots = max_slots
        self.of: dict[int, int] = {}
        self._free = list(range(max_slots - 1, -1, -1))

    def get(self, rid: int) -> int:
        s = self.of.get(rid)
        if s is None:
            if not self._free:
                raise RuntimeError("out of block-table slots")
            s = self._free.pop()
            self.of[rid] = s
        return s

    def drop(self, rid: int) -> Optional[int]:
        s = self.of.pop(rid, None)
        if s is not None:
            self._free.append(s)
            self._free.sort(reverse=True)
        return s


@dataclass
class KVFlow:
    rid: int
    src: int
    dst: int
    layers: tuple[int, int]
    npages: int
    n_chunks: int
    done_chunks: int = 0
    submitted: int = 0
    grown: bool = False
    release_src: bool = True  # False: the engine frees the source itself (baseline moves)

    @property
    def total(self) -> int:
        return (self.layers[1] - self.layers[0]) * self.npages


@dataclass
class Pending:
    task: TransferTask
    event: object
    cb: Optional[Callable]
    bytes_moved: int
    start_event: object = None


@dataclass
class TransferStats:
    kv_bytes: int = 0
    param_bytes: int = 0
    act_bytes: int = 0
    tasks: int = 0
    param_launches: int = 0


class TransferEngine:
    """Runs transfer tasks between device pools of one process.

    pools: iid -> DevicePool; slots: iid -> SlotTable; host_replica: optional
    pinned host tensor holding one full parameter copy (layer l at
    l * bytes_per_layer) for HOST-sourced restores.

    Ordering contract: copies run on the engine's own streams (bulk, urgent,
    meta) and are ordered after the pools' page-table operations
    (kb::pool_enter), not after arbitrary work on other streams -- the bytes
    a task moves must have landed before it is submitted (the engines submit
    only after observing the writers' completion events; a caller that just
    wrote pages on its own stream synchronizes first).  Waiting on the
    caller's stream here would serialize KV exchange behind serving compute.
    """

    def __init__(self, pools: dict, slots: dict, host_replica=None, timing: bool = False):
        import torch
        self.torch = torch
        self.pools = pools
        self.slots = slots
        self.host_replica = host_replica
        lo, hi = torch.cuda.Stream.priority_range()
        self.bulk = torch.cuda.Stream(priority=lo)   # KV chunks + param shards, FIFO
        self.urgent = torch.cuda.Stream(priority=hi)  # activations
        # block-table growth for the next burst runs here while the previous
        # burst's copies stream on `bulk`; the pool's device ordering makes
        # the copies into the new pages wait for it (kb::pool_enter)
        self.meta = torch.cuda.Stream(priority=lo)
        self.flows: dict[tuple[int, int, int], KVFlow] = {}
        self.chunk_of: dict[int, tuple[tuple[int, int, int], int]] = {}
        self.param_off: dict[int, int] = {}
        self.pending: deque[Pending] = deque()
        self.stats = TransferStats()
        self.timing = timing
        # timing=True: (kind, start, end, bytes) events around the copy
        # launches alone of every burst (the roofline's kernel time: no grow
        # or queueing inside), kind "kv" (copy_pages) or "param" (slab pulls)
        self.kernel_spans: list = []
        # swapped-out KV (HOST endpoint): rid -> (pinned tensor, layers, npages)
        self.host_kv: dict[int, tuple] = {}

    # -------------------------------------------------------------- planning
    def register_exchange(self, tasks: list[TransferTask], old_map: dict, new_map: dict,
                          context_tokens: dict[int, int]) -> None:
        """Attach device geometry to a plan_exchange task list."""
        per_flow: dict[tuple[int, int, int], list[TransferTask]] = {}
        for t in tasks:
            per_flow.setdefault((t.rid, t.src, t.dst), []).append(t)
        for key, chunks in per_flow.items():
            rid, j, k = key
            lo = max(old_map[j][0], new_map[k][0])
            hi = min(old_map[j][1], new_map[k][1])
            npages = self._flow_pages(j, rid, context_tokens[rid], lo)
            self.flows[key] = KVFlow(rid, j, k, (lo, hi), npages, len(chunks))
            for idx, t in enumerate(chunks):
                self.chunk_of[t.tid] = (key, idx)

    def _flow_pages(self, src: int, rid: int, tokens: int, layer: int) -> int:
        """Pages a flow moves: the request's context in pages, capped by what
        the source holds.  (The reference's context_len counts the token just
        emitted, whose KV is written only when its decode round allocates it,
        engine.py:335-345 -- so the source may hold one page fewer.)"""
        B = self.pools[src].shape.block_tokens
        want = -(-tokens // B)
        slot = self.slots[src].of.get(rid)
        have = self.pools[src].npages(slot, layer) if slot is not None else 0
        return min(want, have)

    def register_restore(self, tasks: list[TransferTask], bytes_per_layer: int) -> None:
        """Byte offsets of every PARAM_SHARD chunk inside its layer run."""
        run_off: dict[tuple[int, int, tuple[int, int]], int] = {}
        for t in tasks:
            key = (t.src, t.dst, t.layers)
            off = run_off.get(key, 0)
            self.param_off[t.tid] = off
            run_off[key] = off + t.size_bytes

    def register_chunked_kv(self, tasks: list[TransferTask], layers: tuple[int, int],
                            context_tokens: dict[int, int]) -> None:
        """Consolidation-style KV moves (dissolve, engine.py:1211-1239): every
        task of (rid, src, dst) moves the request's pages of `layers`."""
        per_flow: dict[tuple[int, int, int], list[TransferTask]] = {}
        for t in tasks:
            per_flow.setdefault((t.rid, t.src, t.dst), []).append(t)
        for key, chunks in per_flow.items():
            rid, j, _ = key
            npages = self._flow_pages(j, rid, context_tokens[rid], layers[0])
            self.flows[key] = KVFlow(rid, j, key[2], layers, npages, len(chunks))
            for idx, t in enumerate(chunks):
                self.chunk_of[t.tid] = (key, idx)

    def register_request_move(self, task: TransferTask, layers: tuple[int, int],
                              context_tokens: int) -> None:
        """A baseline policy's whole-request KV move as one task (swap out /
        swap in / migrate, engine.py:906-1047): every page of `layers`.  The
        destination's pages already exist (the engine allocated them before
        enqueueing), so the flow is not grown here; a HOST destination gets
        a pinned buffer, a HOST source is the buffer of the swap-out."""
        rid, j, k = task.rid, task.src, task.dst
        if j == HOST:
            buf, hl, npages = self.host_kv[rid]
            if hl != layers:
                raise ValueError(f"rid {rid}: swapped out layers {hl}, swap-in asks {layers}")
        else:
            npages = self._flow_pages(j, rid, context_tokens, layers[0])
        key = (rid, j, k)
        self.flows[key] = KVFlow(rid, j, k, layers, npages, 1, grown=True, release_src=False)
        self.chunk_of[task.tid] = (key, 0)

    def _run_host_flow(self, fl: KVFlow, stream) -> int:
        """Swap out (device -> pinned host) or swap in (host -> device)."""
        lo, hi = fl.layers
        if fl.dst == HOST:
            pool = self.pools[fl.src]
            buf = self.torch.empty((hi - lo) * fl.npages * pool.page_bytes, dtype=self.torch.uint8,
                                   pin_memory=True)
            self.host_kv[fl.rid] = (buf, fl.layers, fl.npages)
            if fl.npages:
                runtime.copy_pages_host(pool, self.slots[fl.src].get(fl.rid), lo, hi, fl.npages,
                                        buf, True, stream=stream)
            return (hi - lo) * fl.npages * pool.page_bytes
        pool = self.pools[fl.dst]
        buf, _, npages = self.host_kv[fl.rid]
        slot = self.slots[fl.dst].get(fl.rid)
        have = min(pool.npages(slot, l) for l in range(lo, hi))
        if have >= npages:
            if npages:
                runtime.copy_pages_host(pool, slot, lo, hi, npages, buf, False, stream=stream)
        else:  # fewer pages re-allocated than swapped out: per layer, the first `have`
            per = npages * pool.page_bytes
            for l in range(lo, hi):
                view = buf[(l - lo) * per:(l - lo + 1) * per]
                if have:
                    runtime.copy_pages_host(pool, slot, l, l + 1, have, view, False,
                                            stream=stream)
            npages = have
        return (hi - lo) * npages * pool.page_bytes

    def release_host(self, rid: int) -> None:
        """Drop a swapped-in request's host copy (after its copy landed)."""
        self.host_kv.pop(rid, None)

    # -------------------------------------------------------------- execution
    def submit(self, task: TransferTask, cb: Optional[Callable] = None) -> None:
        torch = self.torch
        stream = self.urgent if task.kind is TaskKind.ACTIVATION else self.bulk
        start = torch.cuda.Event(enable_timing=True) if self.timing else None
        if start is not None:
            start.record(stream)
        moved = 0
        if task.kind is TaskKind.KVCACHE_CHUNK:
            moved = self._run_kv_chunk(task, stream)
            self.stats.kv_bytes += moved
        elif task.kind is TaskKind.PARAM_SHARD:
            moved = self._run_param_shard(task, stream)
            self.stats.param_bytes += moved
        else:
            raise ValueError("activation tasks go through submit_activation")
        ev = torch.cuda.Event(enable_timing=self.timing)
        ev.record(stream)
        self.stats.tasks += 1
        self.pending.append(Pending(task, ev, cb, moved, start))

    def submit_many(self, tasks: list[TransferTask], cb: Optional[Callable] = None) -> None:
        """Submit a burst of KV / parameter tasks on the bulk stream with one
        block-table growth per destination pool, one page-copy launch per
        (src, dst) pair (up to 256 moves per launch) and one completion event
        for the burst.  Used when nothing needs per-chunk completion times
        (exchange right after a drop, restore pulls, consolidation)."""
        torch = self.torch
        stream = self.bulk
        start = torch.cuda.Event(enable_timing=True) if self.timing else None
        if start is not None:
            start.record(stream)
        grows: dict[int, list] = {}
        for t in tasks:
            if t.kind is TaskKind.KVCACHE_CHUNK:
                fl = self.flows[self.chunk_of[t.tid][0]]
                if not fl.grown:
                    if fl.npages:
                        grows.setdefault(fl.dst, []).append(
                            (self.slots[fl.dst].get(fl.rid), fl.layers[0], fl.layers[1],
                             fl.npages))
                    fl.grown = True
        for dst, reqs in grows.items():
            if not self.pools[dst].grow(reqs, stream=self.meta):
                raise runtime.DeviceError(f"instance {dst} out of KV pages for an exchange")
        pairs: dict[tuple[int, int], list] = {}
        runs: list = []
        moved = {}
        for t in tasks:
            if t.kind is TaskKind.KVCACHE_CHUNK:
                key, idx = self.chunk_of.pop(t.tid)
                fl = self.flows[key]
                fl.submitted += 1
                P = fl.total
                a, b = idx * P // fl.n_chunks, (idx + 1) * P // fl.n_chunks
                if b > a:
                    pairs.setdefault((fl.src, fl.dst), []).append(
                        (self.slots[fl.src].get(fl.rid), self.slots[fl.dst].get(fl.rid),
                         fl.layers[0], fl.layers[1], fl.npages, a, b))
                moved[t.tid] = (b - a) * self.pools[fl.src].page_bytes
                self.stats.kv_bytes += moved[t.tid]
            elif t.kind is TaskKind.PARAM_SHARD:
                # consecutive shards of one run coalesce into one pull launch
                off = self.param_off.pop(t.tid)
                key = (t.src, t.dst, t.layers)
                if runs and runs[-1][0] == key and runs[-1][2] == off:
                    runs[-1][2] += t.size_bytes
                else:
                    runs.append([key, off, off + t.size_bytes])
                moved[t.tid] = t.size_bytes
                self.stats.param_bytes += t.size_bytes
            else:
                raise ValueError("activation tasks go through submit_activation")
        def span(kind, nbytes, launch):
            if not self.timing:
                launch()
                return
            a_ev = torch.cuda.Event(enable_timing=True)
            b_ev = torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            launch()
            b_ev.record(stream)
            self.kernel_spans.append((kind, a_ev, b_ev, nbytes))
        if self.timing and grows:
            stream.wait_stream(self.meta)  # the grows land before the span starts
        if pairs:
            def kv_launch():
                for (s, d), moves in pairs.items():
                    runtime.copy_pages(self.pools[d], self.pools[s], moves, stream=stream)
            span("kv", sum((m[6] - m[5]) * self.pools[s].page_bytes
                           for (s, _), ms in pairs.items() for m in ms), kv_launch)
        if runs:
            def param_launch():
                for (src, dst, layers), a, b in runs:
                    self._copy_param(src, dst, layers, a, b, stream)
            span("param", sum(b - a for _, a, b in runs), param_launch)
        self.stats.param_launches += len(runs)
        ev = torch.cuda.Event(enable_timing=self.timing)
        ev.record(stream)
        self.stats.tasks += len(tasks)
        for t in tasks:
            self.pending.append(Pending(t, ev, cb, moved[t.tid], start))

    def submit_activation(self, task: TransferTask, dst_ptr: int, src_ptr: int,
                          cb: Optional[Callable] = None) -> None:
        runtime.copy_bytes(dst_ptr, src_ptr, task.size_bytes, stream=self.urgent)
        ev = self.torch.cuda.Event()
        ev.record(self.urgent)
        self.stats.act_bytes += task.size_bytes
        self.pending.append(Pending(task, ev, cb, task.size_bytes))

    def _run_kv_chunk(self, task: TransferTask, stream) -> int:
        key, idx = self.chunk_of.pop(task.tid)
        fl = self.flows[key]
        fl.submitted += 1
        if fl.src == HOST or fl.dst == HOST:
            return self._run_host_flow(fl, stream)
        src, dst = self.pools[fl.src], self.pools[fl.dst]
        s_slot = self.slots[fl.src].get(fl.rid)
        d_slot = self.slots[fl.dst].get(fl.rid)
        lo, hi = fl.layers
        if not fl.grown:
            if fl.npages and not dst.grow([(d_slot, lo, hi, fl.npages)], stream=stream):
                raise runtime.DeviceError(f"instance {fl.dst} out of KV pages for rid {fl.rid}")
            fl.grown = True
        P = fl.total
        a, b = idx * P // fl.n_chunks, (idx + 1) * P // fl.n_chunks
        if b > a:
            runtime.copy_pages(dst, src, [(s_slot, d_slot, lo, hi, fl.npages, a, b)],
                               stream=stream)
        return (b - a) * src.page_bytes

    def _run_param_shard(self, task: TransferTask, stream) -> int:
        off = self.param_off.pop(task.tid)
        self._copy_param(task.src, task.dst, task.layers, off, off + task.size_bytes, stream)
        self.stats.param_launches += 1
        return task.size_bytes

    def _copy_param(self, src: int, dst_iid: int, layers: tuple[int, int], a: int, b: int,
                    stream) -> None:
        """Bytes [a, b) of the layer run `layers` (slab-contiguous) into dst."""
        lo, hi = layers
        dst = self.pools[dst_iid]
        if src == HOST:
            if self.host_replica is None:
                raise runtime.DeviceError("HOST-sourced restore without a host replica")
            base = self.host_replica.data_ptr() + lo * dst.model.bytes_per_layer
            runtime.copy_slabs_from_host(dst, base, lo, hi, a, b, stream=stream)
        else:
            runtime.copy_slabs(dst, self.pools[src], lo, hi, a, b, stream=stream)

    def finish_flow_sources(self, ordered: bool = False) -> list[KVFlow]:
        """Release source pages of every flow whose chunks all landed: one
        release launch per (source pool, layer range).  ordered=True also
        takes flows whose chunks are all submitted but maybe not landed: the
        release goes on the bulk stream behind the copies (and the pool
        orders it after every other stream's readers), so the host never
        waits for the transfer."""
        done = []
        batches: dict[tuple[int, tuple[int, int]], list[int]] = {}
        for key, fl in list(self.flows.items()):
            if fl.done_chunks == fl.n_chunks or (ordered and fl.submitted == fl.n_chunks):
                slot = self.slots[fl.src].of.get(fl.rid) if fl.release_src else None
                if slot is not None:
                    batches.setdefault((fl.src, fl.layers), []).append(slot)
                del self.flows[key]
                done.append(fl)
        for (src, (lo, hi)), slots in batches.items():
            self.pools[src].release(slots, lo, hi, stream=self.bulk)
        return done

    def poll(self, block: bool = False) -> list[Pending]:
        """Completed tasks in submission order; runs their callbacks."""
        out = []
        done_ev = None  # a burst shares one event: check / wait for it once
        while self.pending:
            p = self.pending[0]
            if p.event is not done_ev:
                if not block and not p.event.query():
                    break
                p.event.synchronize()
                done_ev = p.event
            self.pending.popleft()
            if p.task.kind is TaskKind.KVCACHE_CHUNK:
                fl = self.flows.get((p.task.rid, p.task.src, p.task.dst))
                if fl is not None:
                    fl.done_chunks += 1
            out.append(p)
            if p.cb is not None:
                p.cb(p.task)
        return out

    def drain(self) -> list[Pending]:
        return self.poll(block=True)
