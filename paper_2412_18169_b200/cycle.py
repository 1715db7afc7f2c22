"""One parameter-centric overload cycle on real device pools.

drop -> KV exchange -> (burst drains) -> restore -> consolidate, driven
through the same public calls the reference's engine makes
(pkg/src/dropsim/engine.py):

  plan     compute_demand + plan_drop               engine.py:616-648
  drop     member_moves + memory.drop_layers         engine.py:751-807
  re-share stage_share allocations                   engine.py:823-830
  exchange plan_exchange per original-map cohort     engine.py:690-726
  drain    half the residents finish: occupancy falls under the restore
           threshold (0.5), the gate of engine.py:1051-1059
  restore  memory.restore_layers + plan_restore_transfers +
           complete_restore                          engine.py:1093-1157
  dissolve consolidation of peer KV back home        engine.py:1159-1254
  refill   the finished residents are re-admitted (next burst)

Every byte movement runs on the GPU through transfer.TransferEngine.  The
drain and refill phases are bookkeeping + synthetic KV writes and are not
part of the timed path; the long-lived residents' KV must survive every
cycle bit for bit (checked by kv_checksums()).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from . import memory, runtime
from .core import Group, ModelShape
from .exchange import TaskKind, TransferTask, plan_exchange, plan_restore_transfers, share_bytes
from .planner import compute_demand, member_moves, plan_drop
from .traceio import synth_burst
from .transfer import SlotTable, TransferEngine


def _span_ms(done) -> float:
    """Device time of completed submissions (each (start, end) event pair once)."""
    seen = {}
    for p in done:
        if p.start_event is not None and id(p.event) not in seen:
            seen[id(p.event)] = p.start_event.elapsed_time(p.event)
    return sum(seen.values())


@dataclass
class CycleReport:
    # device bytes copied (whole pages for KV; slab bytes for parameters)
    bytes_kv_exchange: int = 0
    bytes_param: int = 0
    bytes_kv_consolidate: int = 0
    # restore-time page compaction inside one pool (not a TransferTask)
    bytes_compaction: int = 0
    # the reference's payload: sum of TransferTask.size_bytes (exchange.py
    # share_bytes per flow, plan_restore_transfers shards, consolidation)
    payload_kv_exchange: int = 0
    payload_param: int = 0
    payload_kv_consolidate: int = 0
    # copy launches alone (events around them, transfer.kernel_spans)
    kv_copy_ms: float = 0.0
    kv_copy_bytes: int = 0
    kv_copy_launches: int = 0
    param_copy_ms: float = 0.0
    param_copy_bytes: int = 0
    pages_compacted: int = 0
    remap_ns: int = 0
    n_tasks: int = 0
    ms: dict = field(default_factory=dict)
    param_kernel_ms: float = 0.0   # device time of the parameter-pull launches
    kv_kernel_ms: float = 0.0      # device time of the KV page-copy launches
    host_ms: dict = field(default_factory=dict)  # host enqueue time per phase
    tid_marks: list = field(default_factory=list)  # first tid of restore / consolidation
    param_launches: int = 0        # parameter-pull launches (coalesced runs)

    @property
    def payload_bytes(self) -> int:
        """Sum of the step's TransferTask.size_bytes: the headline's bytes."""
        return self.payload_kv_exchange + self.payload_param + self.payload_kv_consolidate

    @property
    def bytes_moved(self) -> int:
        """Device bytes the transfer kernels copied (pages, slabs); the
        compaction is reported separately (bytes_compaction)."""
        return self.bytes_kv_exchange + self.bytes_param + self.bytes_kv_consolidate


def resident_tokens(capacity_tokens: dict, fill: float = 0.9, seed: int = 3,
                    input_mean: int = 1660):
    """The bench's residents: a ShareGPT-shaped trace (traceio.synth_burst)
    dealt round-robin to the replicas until each is `fill` full (host-only;
    the CPU reference arm samples the same list).  Returns ({rid: tokens},
    {rid: home replica})."""
    trace = synth_burst(10_000.0, 4.0, 16.0, 0.0, 10_000.0, input_mean, 373, seed=seed)
    tokens: dict[int, int] = {}
    home: dict[int, int] = {}
    used = {i: 0 for i in capacity_tokens}
    full = {i: False for i in capacity_tokens}
    ids = sorted(capacity_tokens)
    rid = 0
    for rec in trace:
        if all(full.values()):
            break
        iid = ids[rid % len(ids)]
        rid += 1
        if full[iid]:
            continue
        if used[iid] + rec.input_len > fill * capacity_tokens[iid]:
            full[iid] = True
            continue
        tokens[rid] = rec.input_len
        home[rid] = iid
        used[iid] += rec.input_len
    return tokens, home


class OverloadCycle:
    """Replicas (one per entry of `runtimes`; several may share a GPU), each
    filled to `fill` of its KV budget with ShareGPT-shaped residents; every
    other resident is transient (finishes during the drain)."""

    def __init__(self, runtimes: list, shape: ModelShape, kv_budget_bytes: int,
                 fill: float = 0.9, seed: int = 3, kv_chunk_bytes: int = 64 << 20,
                 param_chunk_bytes: int = 256 << 20, input_mean: int = 1660):
        import torch
        self.torch = torch
        self.shape = shape
        self.model = shape.spec()
        self.L = self.model.num_layers
        self.kv_chunk = kv_chunk_bytes
        self.param_chunk = param_chunk_bytes
        self.instances = {}
        for iid, rt in enumerate(runtimes):
            self.instances[iid] = memory.build_instance(
                iid, self.model, self.model.param_bytes + kv_budget_bytes, 900_000_000_000,
                device=rt, shape=shape)
        self.pools = {i: inst.pool for i, inst in self.instances.items()}
        self.slots = {i: SlotTable(runtimes[i].max_slots) for i in self.instances}
        self.te = TransferEngine(self.pools, self.slots, timing=True)
        self.tokens, self.home = resident_tokens(
            {i: inst.kv.capacity_tokens for i, inst in self.instances.items()}, fill, seed,
            input_mean)
        for rid in sorted(self.tokens):
            self._admit(rid)
        self.transient = set(sorted(self.tokens)[1::2])
        for iid, pool in self.pools.items():
            # synthetic KV content on the head pages (the residents live there;
            # the slab pages alias the weights and are filled next)
            g = torch.Generator(device=f"cuda:{pool.rt.device}").manual_seed(77 + iid)
            head = pool.info().extent_pages * pool.page_bytes
            kv = pool.kv_bytes()[:head].view(torch.int32)
            kv.copy_(torch.randint(-2**31, 2**31 - 1, (kv.numel(),), dtype=torch.int32,
                                   device=kv.device, generator=g))
        self._fill_weights()
        torch.cuda.synchronize()
        self.exchange_batch = 8    # residents in the first plan_exchange / submission batch
        self.pause_merged = False  # set True to stop after the exchange (see resume())
        self.auto_refill = True    # False: the caller runs refill() between steps
        self._paused = None
        self.merged = {}

    # ------------------------------------------------------------------ data
    def _admit(self, rid: int) -> None:
        iid = self.home[rid]
        inst = self.instances[iid]
        assert inst.kv.alloc(rid, self.tokens[rid])
        slot = self.slots[iid].get(rid)
        assert inst.pool.grow([(slot, 0, self.L, -(-self.tokens[rid] // self.shape.block_tokens))])

    def _fill_weights(self) -> None:
        """bf16 randn x 0.02 per layer, seed 1000 + layer: identical replicas,
        so a restored layer is checkable bit for bit."""
        torch = self.torch
        n = self.shape.layer_weight_bytes // 2
        for l in range(self.L):
            for iid, pool in self.pools.items():
                g = torch.Generator(device=f"cuda:{pool.rt.device}").manual_seed(1000 + l)
                slab = pool.weight_bytes(l)
                slab[2 * n:].zero_()  # 2 MiB rounding tail
                w = slab[:2 * n].view(torch.bfloat16)
                w.copy_((torch.randn(n, device=w.device, generator=g) * 0.02).to(torch.bfloat16))
        torch.cuda.synchronize()

    def burst_for(self, seed: int) -> dict:
        """A queued ShareGPT-shaped burst per replica (traceio.synth_burst
        lengths) whose KV outgrows the replica's free pool by at least a
        quarter of one parameter copy: instance -> prompt lengths."""
        kvbpt = self.model.kv_bytes_per_token
        trace = synth_burst(10_000.0, 8.0, 32.0, 0.0, 10_000.0, 1660, 373, seed=seed)
        out, k = {}, 0
        for iid, inst in sorted(self.instances.items()):
            need = inst.kv.free_tokens + self.model.param_bytes // 4 // kvbpt
            lens = []
            while sum(lens) < need:
                lens.append(trace[k % len(trace)].input_len)
                k += 1
            out[iid] = lens
        return out

    def home_first_pages(self):
        """Device int32 [residents]: each long-lived resident's first layer-0
        page on its home pool after the cycle (the step's result, read back
        by bench.py's end-to-end leg); -1 for transient residents."""
        torch = self.torch
        order = sorted(self.tokens)
        out = torch.full((len(order),), -1, dtype=torch.int32, device="cuda")
        per_pool: dict[int, tuple[list[int], list[int]]] = {}
        for k, rid in enumerate(order):
            if rid in self.transient:
                continue
            iid = self.home[rid]
            pos, cell = per_pool.setdefault(iid, ([], []))
            pos.append(k)
            cell.append(self.slots[iid].of[rid] * self.L * self._maxp(iid))  # layer 0, page 0
        for iid, (pos, cell) in per_pool.items():
            bt = self._bt_view(iid).reshape(-1)
            # index vectors through pinned memory, copied asynchronously: a
            # pageable H2D copy would block the host until the stream (queued
            # behind the whole cycle) drained
            dev = lambda xs: torch.tensor(xs, dtype=torch.int64).pin_memory().to(  # noqa: E731
                "cuda", non_blocking=True)
            out[dev(pos)] = bt[dev(cell)]
        return out

    def _maxp(self, iid) -> int:
        return self.pools[iid].rt.max_pages_per_seq

    def _bt_view(self, iid):
        torch = self.torch
        inf = self.pools[iid].info()
        bt = runtime.device_bytes(inf.block_table,
                                  inf.max_slots * self.L * inf.max_pages_per_seq * 4)
        return bt.view(torch.int32).view(inf.max_slots, self.L, inf.max_pages_per_seq)

    def weight_checksums(self) -> dict:
        """(iid, layer) -> position-sensitive 64-bit hash of the layer's whole
        slab (runtime.hash_segments: every word's position enters the hash,
        so a permuted or misplaced 16-byte vector changes it)."""
        out = {}
        for iid, pool in self.pools.items():
            with self.torch.cuda.device(pool.rt.device):
                h = runtime.hash_segments(pool.weight_ptr(0), self.model.bytes_per_layer,
                                          self.L).cpu().tolist()
            out.update({(iid, l): h[l] for l in range(self.L)})
        return out

    def kv_checksums(self) -> dict:
        """Long-lived residents: position-sensitive 64-bit hash of every
        (layer, page) of their KV on their home instance, in block-table
        order (a page moved to the wrong slot, or bytes moved inside a page,
        change the vector)."""
        torch = self.torch
        out = {}
        for iid, pool in self.pools.items():
            bt = self._bt_view(iid)
            rids, idx = [], []
            for rid, home in sorted(self.home.items()):
                if home != iid or rid in self.transient:
                    continue
                npg = -(-self.tokens[rid] // self.shape.block_tokens)
                rids.append((rid, npg * self.L))
                idx.append(bt[self.slots[iid].of[rid], :, :npg].reshape(-1))
            if not idx:
                continue
            pages = torch.cat(idx).to(torch.int64)
            h = runtime.hash_segments(pool.info().kv_base, pool.page_bytes, pages.numel(),
                                      index=pages).cpu()
            o = 0
            for rid, n in rids:
                out[rid] = h[o:o + n]
                o += n
        return out

    # ------------------------------------------------------------------ cycle
    def step(self, burst: dict | None = None, on_enqueued=None,
             light: bool = False) -> CycleReport:
        """One overload cycle.  burst: instance -> prompt lengths of the
        requests queued on it (the step's input; plan_drop sizes the merge
        from their KV demand).  Default: a queue that outgrows every
        replica's free KV by a quarter of one parameter copy.
        on_enqueued(): called once the cycle's last device operation is
        queued (before the host-side accounting, which waits on events), on
        a stream ordered after it -- e.g. the read-back of the step's result.
        light: skip the per-launch kernel timing (hundreds of event
        elapsed-time reads after the device finishes); payload and phase
        times are still reported."""
        torch = self.torch
        rep = CycleReport()
        st = self.te.bulk
        ev = {k: torch.cuda.Event(enable_timing=True) for k in
              ("t0", "drop", "exch", "drain", "restore", "cons")}
        kvbpt = self.model.kv_bytes_per_token
        L = self.L
        ev["t0"].record(st)
        h0 = time.perf_counter()
        rep.param_launches = self.te.stats.param_launches  # baseline; a delta at the end
        # ---- plan (engine.py:616-648): a queued burst that outgrows every
        # replica's free KV by a quarter of one parameter copy
        groups = [Group(i, [i], {i: (0, L)}) for i in sorted(self.instances)]
        demand = 0
        for i, inst in sorted(self.instances.items()):
            free = inst.kv.free_tokens * kvbpt
            pending = (sum(burst[i]) if burst is not None
                       else (free + self.model.param_bytes // 4) // kvbpt)
            demand += compute_demand(pending, free, kvbpt)
        plan = plan_drop(groups, demand, self.model)
        assert plan.merges and not plan.fallback, plan.to_text()
        orig_map = {rid: {h: (0, L)} for rid, h in self.home.items()}
        # ---- merge: drops, then re-share (engine.py:751-830)
        live = {g.gid: g for g in groups}
        for m in plan.merges:
            live.pop(m.gid_a)
            live.pop(m.gid_b)
            new = Group(m.gid, list(m.members), dict(m.stage_layer_map))
            new.validate_coverage(L)
            for iid in m.members:
                held = self.instances[iid].table.held_ranges()
                drops, fetches = member_moves(held, m.stage_layer_map[iid])
                assert not fetches  # equal-depth merges are in-place drops
                for lo, hi in drops:
                    memory.drop_layers(self.instances[iid], (lo, hi), new)
                    rep.remap_ns += self.pools[iid].last_remap_ns
            live[m.gid] = new
        ev["drop"].record(st)
        h_drop = time.perf_counter()
        final = {iid: g for g in live.values() for iid in g.member_instances}
        # ---- exchange per original-map cohort (engine.py:690-726); the
        # device work is queued first, the host-only re-share follows
        tid = 0
        for g in sorted(live.values(), key=lambda g: g.gid):
            cohorts: dict[tuple, list[int]] = {}
            for rid in sorted(self.tokens):
                if final[self.home[rid]] is g:
                    cohorts.setdefault(tuple(sorted(orig_map[rid].items())), []).append(rid)
            for key in sorted(cohorts):
                old_map = dict(key)
                # planned and submitted in batches of residents: the first
                # copies start while the host plans the rest (the flows, and
                # so the bytes, are those of one plan_exchange over the cohort;
                # only the round-robin order differs)
                rids = cohorts[key]
                b0, size = 0, self.exchange_batch
                while b0 < len(rids):
                    toks = {rid: self.tokens[rid] for rid in rids[b0:b0 + size]}
                    b0 += size
                    size *= 2  # first copies early, then fewer, larger batches
                    tasks = plan_exchange(toks, old_map, g.stage_layer_map, L, kvbpt,
                                          self.kv_chunk, tid_start=tid)
                    tid += len(tasks)
                    self.te.register_exchange(tasks, old_map, g.stage_layer_map, toks)
                    self.te.submit_many(tasks)
                    rep.n_tasks += len(tasks)
        # no host wait: source releases queue behind the copies
        self.te.finish_flow_sources(ordered=True)
        # re-share (engine.py:823-830): token accounting per member stage
        for rid, tok in self.tokens.items():
            g = final[self.home[rid]]
            for iid in g.member_instances:
                self.instances[iid].kv.free(rid)
            for iid in g.member_instances:
                lo, hi = g.stage_layer_map[iid]
                share = memory.stage_share(tok, lo, hi, L)
                if share:
                    assert self.instances[iid].kv.alloc(rid, share)
        ev["exch"].record(st)
        rep.host_ms = {"drop": (h_drop - h0) * 1e3,
                       "exchange": (time.perf_counter() - h_drop) * 1e3}
        rep.tid_marks = [tid]
        self.merged = live
        if self.pause_merged:
            self._paused = (rep, live, ev, tid)
            return rep
        return self._finish(rep, live, ev, tid, on_enqueued, light)

    def merged_decode_layout(self):
        """instance -> ((lo, hi), [(rid, slot, ctx)]) of the merged state."""
        out = {}
        for g in self.merged.values():
            for iid in g.member_instances:
                res = [(rid, self.slots[iid].of[rid], self.tokens[rid])
                       for rid in sorted(self.tokens) if self.home[rid] in g.member_instances]
                out[iid] = (g.stage_layer_map[iid], res)
        return out

    def resume(self) -> CycleReport:
        rep, live, ev, tid = self._paused
        self._paused = None
        self.pause_merged = False
        return self._finish(rep, live, ev, tid)

    def _finish(self, rep: CycleReport, live: dict, ev: dict, tid: int,
                on_enqueued=None, light: bool = False) -> CycleReport:
        torch = self.torch
        st = self.te.bulk
        L = self.L
        kvbpt = self.model.kv_bytes_per_token
        # ---- drain: transient residents finish (engine.py:_finish -> group_free)
        gone: dict[int, list[int]] = {}
        for rid in sorted(self.transient):
            for iid, inst in self.instances.items():
                inst.kv.free(rid)
                slot = self.slots[iid].of.get(rid)
                if slot is not None:
                    gone.setdefault(iid, []).append(slot)
                    self.slots[iid].drop(rid)
        for iid, slots in gone.items():
            self.pools[iid].release(slots, 0, L, stream=st)
        ev["drain"].record(st)
        h1 = time.perf_counter()
        restored = []
        # ---- restore (engine.py:1093-1157): reserve + compaction + remap, pulls
        for g in sorted(live.values(), key=lambda g: g.gid):
            missing, holders = {}, {}
            for iid in g.member_instances:
                holders[iid] = self.instances[iid].table.held_ranges()
                _, need = member_moves(holders[iid], (0, L))
                if need:
                    missing[iid] = need
            for iid in sorted(missing):
                for rng in missing[iid]:
                    memory.restore_layers(self.instances[iid], rng, -1, tid=0, stream=st)
                    rep.remap_ns += self.pools[iid].last_remap_ns
                    restored.append(iid)
            # one plan per range index: a member of a PP-4 group can miss two
            # disjoint ranges, and plan_restore_transfers takes one range per
            # target (the reference's engine.py:1127 keeps only the last one)
            tasks = []
            for k in range(max(len(r) for r in missing.values()) if missing else 0):
                flat = {iid: rngs[k] for iid, rngs in missing.items() if len(rngs) > k}
                tasks += plan_restore_transfers(flat, holders, self.model.bytes_per_layer,
                                                self.param_chunk, tid_start=tid + len(tasks))
            tid += len(tasks)
            self.te.register_restore(tasks, self.model.bytes_per_layer)
            self.te.submit_many(tasks)  # one pull launch per contiguous run
            rep.n_tasks += len(tasks)
            # bookkeeping flips now; the pulls are ordered on the bulk stream
            # before anything that reads the restored layers
            for iid, rngs in missing.items():
                for rng in rngs:
                    memory.complete_restore(self.instances[iid], rng)
        ev["restore"].record(st)
        h2 = time.perf_counter()
        rep.tid_marks.append(tid)
        # ---- dissolve + consolidation (engine.py:1159-1254)
        cons_tasks = []
        for rid in sorted(self.tokens):
            if rid in self.transient:
                continue
            home = self.home[rid]
            g = next(g for g in live.values() if home in g.member_instances)
            for iid in g.member_instances:
                if iid == home:
                    continue
                lo, hi = g.stage_layer_map[iid]
                left = share_bytes(self.tokens[rid], lo, hi, L, kvbpt)
                chunks = []
                while left > 0:
                    take = min(self.kv_chunk, left)
                    left -= take
                    chunks.append(TransferTask(tid, TaskKind.KVCACHE_CHUNK, iid, home, take,
                                               rid=rid))
                    tid += 1
                self.te.register_chunked_kv(chunks, (lo, hi), {rid: self.tokens[rid]})
                cons_tasks += chunks
        self.te.submit_many(cons_tasks)
        rep.n_tasks += len(cons_tasks)
        self.te.finish_flow_sources(ordered=True)
        for rid, tok in self.tokens.items():
            if rid in self.transient:
                continue
            home = self.home[rid]
            for iid, inst in self.instances.items():
                if iid != home:
                    inst.kv.free(rid)
                    self.slots[iid].drop(rid)
            inst = self.instances[home]
            extra = tok - inst.kv.allocated_tokens.get(rid, 0)
            if extra:
                assert inst.kv.alloc(rid, extra)
        ev["cons"].record(st)
        h3 = time.perf_counter()
        if on_enqueued is not None:
            cur = torch.cuda.current_stream()
            cur.wait_event(ev["cons"])
            on_enqueued()
        rep.host_ms.update({"restore": (h2 - h1) * 1e3, "consolidate": (h3 - h2) * 1e3})
        # ---- accounting, after the fact (nothing above waited on the GPU;
        # polling the completions while the device runs measured 0.1 ms
        # slower per step than this one blocking drain)
        done = self.te.drain()
        x_end, r_end = rep.tid_marks
        for p in done:
            k = p.task.tid
            if k < x_end:
                rep.bytes_kv_exchange += p.bytes_moved
                rep.payload_kv_exchange += p.task.size_bytes
            elif k < r_end:
                rep.bytes_param += p.bytes_moved
                rep.payload_param += p.task.size_bytes
            else:
                rep.bytes_kv_consolidate += p.bytes_moved
                rep.payload_kv_consolidate += p.task.size_bytes
        for kind, a, b, nbytes in ([] if light else self.te.kernel_spans):
            if kind == "kv":
                rep.kv_copy_ms += a.elapsed_time(b)
                rep.kv_copy_bytes += nbytes
                rep.kv_copy_launches += 1
            else:
                rep.param_copy_ms += a.elapsed_time(b)
                rep.param_copy_bytes += nbytes
        self.te.kernel_spans.clear()
        if not light:
            rep.kv_kernel_ms += _span_ms([p for p in done
                                          if p.task.kind is TaskKind.KVCACHE_CHUNK])
            rep.param_kernel_ms += _span_ms([p for p in done
                                             if p.task.kind is TaskKind.PARAM_SHARD])
        rep.pages_compacted = sum(self.pools[iid].last_moved_pages for iid in restored)
        rep.param_launches = self.te.stats.param_launches - rep.param_launches
        rep.bytes_compaction = rep.pages_compacted * self.shape.page_bytes
        # ---- refill: the next burst re-admits the transient residents
        if self.auto_refill:
            self.refill()
        ev["cons"].synchronize()
        parts = {"drop": ev["t0"].elapsed_time(ev["drop"]),
                 "exchange": ev["drop"].elapsed_time(ev["exch"]),
                 "restore": ev["drain"].elapsed_time(ev["restore"]),
                 "consolidate": ev["restore"].elapsed_time(ev["cons"])}
        parts["total"] = sum(parts.values())
        parts["drain_untimed"] = ev["exch"].elapsed_time(ev["drain"])
        rep.ms = parts
        return rep

    def close(self) -> None:
        self.torch.cuda.synchronize()
        for pool in self.pools.values():
            pool.close()

    def refill(self) -> None:
        torch = self.torch
        for rid in sorted(self.transient):
            self._admit(rid)
        for iid, pool in self.pools.items():
            bt = self._bt_view(iid)
            rows = []
            for rid in sorted(self.transient):
                if self.home[rid] == iid:
                    npg = -(-self.tokens[rid] // self.shape.block_tokens)
                    rows.append(bt[self.slots[iid].of[rid], :, :npg].reshape(-1))
            if rows:
                kv = pool.kv_bytes().view(torch.int32).view(-1, pool.page_bytes // 4)
                pages = torch.cat(rows).long()
                kv.index_fill_(0, pages, 0x5A5A5A5A)
        torch.cuda.synchronize()
