"""One parameter-centric overload cycle on real device pools.

drop -> KV exchange -> restore -> consolidate, driven through the same
public calls the reference's engine makes (pkg/src/dropsim/engine.py):

  plan     compute_demand + plan_drop               engine.py:616-648
  drop     member_moves + memory.drop_layers         engine.py:751-807
  re-share stage_share allocations                   engine.py:823-830
  exchange plan_exchange per original-map cohort     engine.py:690-726
  restore  memory.restore_layers + plan_restore_transfers +
           complete_restore                          engine.py:1093-1157
  dissolve consolidation of peer KV back home        engine.py:1159-1254

Every byte movement runs on the GPU through transfer.TransferEngine; the
cycle returns the instances to their boot layout, so it can be repeated.
Used by bench.py (the headline drop/restore GB/s) and by the GPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import memory, runtime
from .core import Group, ModelShape
from .exchange import TaskKind, TransferTask, plan_exchange, plan_restore_transfers, share_bytes
from .planner import compute_demand, member_moves, plan_drop
from .traceio import synth_burst
from .transfer import SlotTable, TransferEngine


@dataclass
class CycleReport:
    bytes_kv_exchange: int = 0
    bytes_param: int = 0
    bytes_kv_consolidate: int = 0
    bytes_compaction: int = 0
    pages_compacted: int = 0
    remap_ns: int = 0
    n_tasks: int = 0
    ms: dict = field(default_factory=dict)
    param_kernel_ms: float = 0.0   # device time of the parameter-pull launches

    @property
    def bytes_moved(self) -> int:
        return (self.bytes_kv_exchange + self.bytes_param + self.bytes_kv_consolidate
                + self.bytes_compaction)


class OverloadCycle:
    """N instances (replicas) on the devices of `runtimes` (one per instance,
    several instances may share a GPU), each filled to `fill` of its KV
    budget with ShareGPT-shaped residents."""

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
        self._fill_weights()
        # residents: ShareGPT-shaped lengths, dealt round-robin until full
        trace = synth_burst(10_000.0, 4.0, 16.0, 0.0, 10_000.0, input_mean, 373, seed=seed)
        self.tokens: dict[int, int] = {}
        self.home: dict[int, int] = {}
        B = shape.block_tokens
        full = {i: False for i in self.instances}
        rid = 0
        for rec in trace:
            if all(full.values()):
                break
            iid = rid % len(self.instances)
            rid += 1
            if full[iid]:
                continue
            inst = self.instances[iid]
            cap = inst.kv.capacity_tokens
            if inst.kv.used_tokens + rec.input_len > fill * cap:
                full[iid] = True
                continue
            assert inst.kv.alloc(rid, rec.input_len)
            slot = self.slots[iid].get(rid)
            assert inst.pool.grow([(slot, 0, self.L, -(-rec.input_len // B))])
            self.tokens[rid] = rec.input_len
            self.home[rid] = iid
        torch.cuda.synchronize()
        # synthetic KV content: deterministic random bytes over every mapped page
        for iid, pool in self.pools.items():
            g = torch.Generator(device=f"cuda:{pool.rt.device}").manual_seed(77 + iid)
            kv = pool.kv_bytes()
            kv.view(torch.int32).copy_(torch.randint(-2**31, 2**31 - 1, (kv.numel() // 4,),
                                                     dtype=torch.int32, device=kv.device,
                                                     generator=g))
        torch.cuda.synchronize()
        self.pause_merged = False  # set True to stop after the exchange (see resume())
        self._paused = None

    # ------------------------------------------------------------------ data
    def _fill_weights(self) -> None:
        """bf16 randn x 0.02 per layer, seed 1000 + layer: identical replicas,
        so a restored layer is checkable bit for bit."""
        torch = self.torch
        n = self.shape.layer_weight_bytes // 2
        for l in range(self.L):
            for iid, pool in self.pools.items():
                g = torch.Generator(device=f"cuda:{pool.rt.device}").manual_seed(1000 + l)
                w = pool.weight_bytes(l)[:2 * n].view(torch.bfloat16)
                w.copy_((torch.randn(n, device=w.device, generator=g) * 0.02).to(torch.bfloat16))
        torch.cuda.synchronize()

    def weight_checksums(self) -> dict:
        torch = self.torch
        out = {}
        for iid, pool in self.pools.items():
            for l in range(self.L):
                w = pool.weight_bytes(l).view(torch.int32)
                out[(iid, l)] = int(w.to(torch.int64).sum().item())
        return out

    def kv_checksums(self) -> dict:
        """Per resident: per (layer, page index) int32-sum of the page bytes
        on its home instance, in block-table order."""
        torch = self.torch
        out = {}
        for iid, pool in self.pools.items():
            inf = pool.info()
            bt = runtime.device_bytes(inf.block_table,
                                      inf.max_slots * self.L * inf.max_pages_per_seq * 4)
            bt = bt.view(torch.int32).view(inf.max_slots, self.L, inf.max_pages_per_seq)
            kv = pool.kv_bytes().view(torch.int32).view(-1, pool.page_bytes // 4)
            for rid, home in self.home.items():
                if home != iid:
                    continue
                slot = self.slots[iid].of[rid]
                npg = -(-self.tokens[rid] // self.shape.block_tokens)
                pages = bt[slot, :, :npg].reshape(-1).long()
                out[rid] = kv.index_select(0, pages).to(torch.int64).sum(dim=1).cpu()
        return out

    # ------------------------------------------------------------------ cycle
    def step(self) -> CycleReport:
        torch = self.torch
        rep = CycleReport()
        st = self.te.bulk
        ev = {k: torch.cuda.Event(enable_timing=True) for k in
              ("t0", "drop", "exch", "restore", "cons")}
        kvbpt = self.model.kv_bytes_per_token
        L = self.L
        ev["t0"].record(st)
        # ---- plan (engine.py:616-648)
        groups = [Group(i, [i], {i: (0, L)}) for i in sorted(self.instances)]
        # a queued burst that outgrows every replica's free KV by a quarter of
        # one parameter copy: the planner answers with one merge per pair
        demand = 0
        for i, inst in sorted(self.instances.items()):
            free = inst.kv.free_tokens * kvbpt
            pending = (free + self.model.param_bytes // 4) // kvbpt
            demand += compute_demand(pending, free, kvbpt)
        plan = plan_drop(groups, demand, self.model)
        assert plan.merges and not plan.fallback, plan.to_text()
        orig_map = {rid: {h: (0, L)} for rid, h in self.home.items()}
        # ---- merge: drops, then re-share (engine.py:751-830)
        live = {g.gid: g for g in groups}
        for m in plan.merges:
            ga, gb = live.pop(m.gid_a), live.pop(m.gid_b)
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
        final = {iid: g for g in live.values() for iid in g.member_instances}
        for rid, tok in self.tokens.items():
            g = final[self.home[rid]]
            for iid in g.member_instances:
                self.instances[iid].kv.free(rid)
            for iid in g.member_instances:
                lo, hi = g.stage_layer_map[iid]
                share = memory.stage_share(tok, lo, hi, L)
                if share:
                    assert self.instances[iid].kv.alloc(rid, share)
        # ---- exchange per original-map cohort (engine.py:690-726)
        tid = 0
        for g in sorted(live.values(), key=lambda g: g.gid):
            cohorts: dict[tuple, list[int]] = {}
            for rid in sorted(self.tokens):
                if final[self.home[rid]] is g:
                    cohorts.setdefault(tuple(sorted(orig_map[rid].items())), []).append(rid)
            for key in sorted(cohorts):
                old_map = dict(key)
                toks = {rid: self.tokens[rid] for rid in cohorts[key]}
                tasks = plan_exchange(toks, old_map, g.stage_layer_map, L, kvbpt, self.kv_chunk,
                                      tid_start=tid)
                tid += len(tasks)
                self.te.register_exchange(tasks, old_map, g.stage_layer_map, toks)
                for t in tasks:
                    self.te.submit(t)
                rep.n_tasks += len(tasks)
        done = self.te.drain()
        rep.bytes_kv_exchange = sum(p.bytes_moved for p in done)
        self.te.finish_flow_sources()
        ev["exch"].record(st)
        self.merged = live
        return self._restore_and_dissolve(rep, live, ev, tid)

    def merged_decode_layout(self):
        """(instance -> (layers, [(rid, slot, ctx)])) of the merged state, for
        the decode measurement that runs between exchange and restore."""
        out = {}
        for g in self.merged.values():
            for iid in g.member_instances:
                res = [(rid, self.slots[iid].of[rid], self.tokens[rid])
                       for rid in sorted(self.tokens) if self.home[rid] in g.member_instances]
                out[iid] = (g.stage_layer_map[iid], res)
        return out

    def _restore_and_dissolve(self, rep: CycleReport, live: dict, ev: dict,
                              tid: int) -> CycleReport:
        torch = self.torch
        st = self.te.bulk
        L = self.L
        kvbpt = self.model.kv_bytes_per_token
        if self.pause_merged:
            self._paused = (rep, live, ev, tid)
            return rep
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
                    memory.restore_layers(self.instances[iid], rng, -1, tid=0)
                    rep.remap_ns += self.pools[iid].last_remap_ns
                    rep.pages_compacted += self.pools[iid].last_moved_pages
            flat = {iid: rng for iid, rngs in missing.items() for rng in rngs}
            tasks = plan_restore_transfers(flat, holders, self.model.bytes_per_layer,
                                           self.param_chunk, tid_start=tid)
            tid += len(tasks)
            self.te.register_restore(tasks, self.model.bytes_per_layer)
            for t in tasks:
                self.te.submit(t)
            rep.n_tasks += len(tasks)
            done = self.te.drain()
            rep.bytes_param += sum(p.bytes_moved for p in done)
            rep.param_kernel_ms += sum(p.start_event.elapsed_time(p.event) for p in done
                                       if p.start_event is not None)
            for iid, rngs in missing.items():
                for rng in rngs:
                    memory.complete_restore(self.instances[iid], rng)
        rep.bytes_compaction = rep.pages_compacted * self.shape.page_bytes * 2  # read + write
        ev["restore"].record(st)
        # ---- dissolve + consolidation (engine.py:1159-1254)
        cons_tasks = []
        for rid in sorted(self.tokens):
            home = self.home[rid]
            g = next(g for g in live.values() if home in g.member_instances)
            for iid in g.member_instances:
                if iid == home:
                    continue
                lo, hi = g.stage_layer_map[iid]
                nbytes = share_bytes(self.tokens[rid], lo, hi, L, kvbpt)
                left = nbytes
                chunks = []
                while left > 0:
                    take = min(self.kv_chunk, left)
                    left -= take
                    chunks.append(TransferTask(tid, TaskKind.KVCACHE_CHUNK, iid, home, take,
                                               rid=rid))
                    tid += 1
                self.te.register_chunked_kv(chunks, (lo, hi), {rid: self.tokens[rid]})
                cons_tasks += chunks
        for t in cons_tasks:
            self.te.submit(t)
        rep.n_tasks += len(cons_tasks)
        done = self.te.drain()
        rep.bytes_kv_consolidate = sum(p.bytes_moved for p in done)
        self.te.finish_flow_sources()
        for rid, tok in self.tokens.items():
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
        ev["cons"].synchronize()
        rep.ms = {"drop": ev["t0"].elapsed_time(ev["drop"]),
                  "exchange": ev["drop"].elapsed_time(ev["exch"]),
                  "restore": ev["exch"].elapsed_time(ev["restore"]),
                  "consolidate": ev["restore"].elapsed_time(ev["cons"]),
                  "total": ev["t0"].elapsed_time(ev["cons"])}
        return rep

    def resume(self) -> CycleReport:
        rep, live, ev, tid = self._paused
        self._paused = None
        self.pause_merged = False
        return self._restore_and_dissolve(rep, live, ev, tid)
