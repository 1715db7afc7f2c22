"""The overload cycle across processes: one replica per GPU, PP-2 groups
spanning two GPUs, KV exchange and parameter restore pulled over NVLink.

BASELINE.json configs[2] ("Llama-3-8B bf16, 8 replicas on 8xB200 dropped to
4 PP-2 groups, KV exchange + param restore at burst end").  Rank r owns
instance r; plan_drop (pkg/src/dropsim/planner.py:70-114) pairs gids
(0,1), (2,3), ... so every merged group spans two GPUs.

Every rank runs the reference's control plane for ALL instances -- the
same memory.* / KVAllocator / plan_exchange / plan_restore_transfers calls
in the same order, so the host state (segment tables, token accounting,
block-table slots) is identical everywhere -- and executes on its GPU only
what its own instance does:
  * drops, restores (compaction) and block-table growth of its own pool;
  * every task whose DESTINATION is its instance, pulling from the source's
    pool through a PeerPool view (dist.share_pools): the copy kernels read
    the peer's pages / slabs over NVLink and write local HBM;
  * the release of its own source pages once the peer's pulls landed.
Cross-rank ordering is explicit: after each phase whose pulls read a peer's
memory, every rank synchronizes its transfer stream and the ranks meet at a
barrier before a source releases (exchange, consolidation) or compacts
(restore) pages a peer may still read.  Timing: CUDA events on each rank's
transfer stream (they include the barrier waits), max over ranks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import memory
from .core import Group, ModelShape
from .cycle import _span_ms
from .dist import max_over_ranks, share_pools, sum_over_ranks
from .exchange import HOST, TaskKind, TransferTask, plan_exchange, plan_restore_transfers, share_bytes
from .planner import compute_demand, member_moves, plan_drop
from .traceio import synth_burst
from .transfer import SlotTable, TransferEngine


@dataclass
class DistReport:
    bytes_pulled: int = 0          # payload this rank pulled (all phases)
    bytes_pulled_peer: int = 0     # ... of it from another rank's GPU (NVLink)
    bytes_kv_exchange: int = 0
    bytes_param: int = 0
    bytes_kv_consolidate: int = 0
    bytes_compaction: int = 0
    kv_kernel_ms: float = 0.0
    param_kernel_ms: float = 0.0
    payload_bytes: int = 0         # sum of this rank's TransferTask.size_bytes
    copy_kernel_ms: float = 0.0    # the copy launches alone (kernel_spans)
    copy_kernel_bytes: int = 0
    ms: dict = field(default_factory=dict)


class DistCycle:
    def __init__(self, rt, shape: ModelShape, kv_budget_bytes: int, fill: float = 0.9,
                 seed: int = 3, kv_chunk_bytes: int = 64 << 20,
                 param_chunk_bytes: int = 256 << 20, input_mean: int = 1660,
                 key: str = "cycle", pp: int = 2):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.me = self.rank
        self.shape = shape
        self.model = shape.spec()
        self.L = self.model.num_layers
        if pp not in (2, 4) or dist.get_world_size() % pp:
            raise ValueError(f"pp must be 2 or 4 and divide the world size, got {pp}")
        self.pp = pp
        self.kv_chunk = kv_chunk_bytes
        self.param_chunk = param_chunk_bytes
        self.device = rt.device
        hbm = self.model.param_bytes + kv_budget_bytes
        self.instances = {}
        for iid in range(self.world):
            local = iid == self.me
            self.instances[iid] = memory.build_instance(
                iid, self.model, hbm, 900_000_000_000,
                device=rt if local else None, shape=shape if local else None)
        self.pool = self.instances[self.me].pool
        self.slots = {iid: SlotTable(rt.max_slots) for iid in self.instances}
        trace = synth_burst(10_000.0, 4.0, 16.0, 0.0, 10_000.0, input_mean, 373, seed=seed)
        self.tokens: dict[int, int] = {}
        self.home: dict[int, int] = {}
        full = {i: False for i in self.instances}
        rid = 0
        for rec in trace:
            if all(full.values()):
                break
            iid = rid % self.world
            rid += 1
            if full[iid]:
                continue
            inst = self.instances[iid]
            if inst.kv.used_tokens + rec.input_len > fill * inst.kv.capacity_tokens:
                full[iid] = True
                continue
            self.tokens[rid] = rec.input_len
            self.home[rid] = iid
            self._admit(rid)
        # every other resident of each home is transient (finishes in the drain)
        self.transient = set()
        for iid in self.instances:
            self.transient |= set(sorted(r for r, h in self.home.items() if h == iid)[1::2])
        g = torch.Generator(device=f"cuda:{self.device}").manual_seed(77 + self.me)
        head = self.pool.info().extent_pages * self.pool.page_bytes
        kv = self.pool.kv_bytes()[:head].view(torch.int32)
        kv.copy_(torch.randint(-2**31, 2**31 - 1, (kv.numel(),), dtype=torch.int32,
                               device=kv.device, generator=g))
        n = self.shape.layer_weight_bytes // 2
        for l in range(self.L):
            gl = torch.Generator(device=f"cuda:{self.device}").manual_seed(1000 + l)
            slab = self.pool.weight_bytes(l)
            slab[2 * n:].zero_()
            w = slab[:2 * n].view(torch.bfloat16)
            w.copy_((torch.randn(n, device=w.device, generator=gl) * 0.02).to(torch.bfloat16))
        torch.cuda.synchronize(self.device)
        self.views = share_pools(rt, {self.me: self.pool}, self.model, shape,
                                 key=f"{key}-{self._job_key()}")
        self.pools = {self.me: self.pool, **self.views}
        self.te = TransferEngine(self.pools, self.slots, timing=True)
        self.rt = rt
        self.head_pages = self.pool.info().extent_pages  # slab l's alias starts here
        # tests: overwrite dropped slabs, so a restore that skipped a layer
        # cannot pass the weight checksums by leaving the old bytes in place
        self.poison_drops = False
        self.last_groups: dict = {}
        self.on_merged = None  # callback(live groups, instance -> group) in the merged state
        self._sync_views()

    @staticmethod
    def _job_key() -> str:
        import os
        return os.environ.get("MASTER_PORT", "0")

    # ---------------------------------------------------------------- helpers
    def _poison(self, lo: int, hi: int) -> None:
        sp = self.model.bytes_per_layer // self.shape.page_bytes
        a = (self.head_pages + lo * sp) * self.shape.page_bytes
        b = (self.head_pages + hi * sp) * self.shape.page_bytes
        with self.torch.cuda.stream(self.te.bulk):  # ordered before the exchange grows / copies
            self.pool.kv_bytes()[a:b].fill_(0x7F)

    def _admit(self, rid: int) -> None:
        iid = self.home[rid]
        inst = self.instances[iid]
        assert inst.kv.alloc(rid, self.tokens[rid])
        slot = self.slots[iid].get(rid)
        if iid == self.me:
            assert self.pool.grow([(slot, 0, self.L, -(-self.tokens[rid] // self.shape.block_tokens))])

    def _sync_views(self) -> None:
        """Phase boundary: this rank's device work is done, every rank is
        here, and the views reflect the owners' page counts / layer states."""
        self.torch.cuda.synchronize(self.device)
        self.dist.barrier()
        for iid, v in self.views.items():
            v.refresh(self.instances[iid].table.layers_held())

    def _submit_local(self, tasks: list[TransferTask]) -> None:
        """Mirror the slot assignment of every destination (the owners do the
        same get() calls in the same order), then run the tasks whose
        destination is this rank; drop the bookkeeping of the others."""
        for t in tasks:
            if t.kind is TaskKind.KVCACHE_CHUNK:
                key, _ = self.te.chunk_of[t.tid]
                fl = self.te.flows[key]
                self.slots[fl.dst].get(fl.rid)
        mine = [t for t in tasks if t.dst == self.me]
        for t in tasks:
            if t.dst != self.me:
                self.te.chunk_of.pop(t.tid, None)
                self.te.param_off.pop(t.tid, None)
        if mine:
            self.te.submit_many(mine)

    def _release_sources(self) -> None:
        """After the barrier: free this rank's source pages of every flow
        (all flows' chunks were submitted by their destinations and have
        landed -- every rank synchronized before the barrier)."""
        batches: dict[tuple[int, int], list[int]] = {}
        for key, fl in list(self.te.flows.items()):
            if fl.src == self.me:
                slot = self.slots[fl.src].of.get(fl.rid)
                if slot is not None:
                    batches.setdefault(fl.layers, []).append(slot)
            del self.te.flows[key]
        for (lo, hi), slots in batches.items():
            self.pool.release(slots, lo, hi, stream=self.te.bulk)

    # ------------------------------------------------------------------ checks
    def weight_checksums(self) -> list[int]:
        """Position-sensitive 64-bit hash of every layer slab (kb_hash_segments)."""
        from .runtime import hash_segments
        with self.torch.cuda.device(self.device):
            return hash_segments(self.pool.weight_ptr(0), self.model.bytes_per_layer,
                                 self.L).cpu().tolist()

    def kv_checksums(self) -> dict:
        """This rank's long-lived home residents: position-sensitive hash of
        every (layer, page), in block-table order."""
        torch = self.torch
        inf = self.pool.info()
        from .runtime import device_bytes, hash_segments
        bt = device_bytes(inf.block_table, inf.max_slots * self.L * inf.max_pages_per_seq * 4)
        bt = bt.view(torch.int32).view(inf.max_slots, self.L, inf.max_pages_per_seq)
        rids, idx = [], []
        for rid, home in sorted(self.home.items()):
            if home != self.me or rid in self.transient:
                continue
            npg = -(-self.tokens[rid] // self.shape.block_tokens)
            rids.append((rid, npg * self.L))
            idx.append(bt[self.slots[self.me].of[rid], :, :npg].reshape(-1))
        out = {}
        if idx:
            pages = torch.cat(idx).to(torch.int64)
            h = hash_segments(inf.kv_base, self.pool.page_bytes, pages.numel(), index=pages).cpu()
            o = 0
            for rid, n in rids:
                out[rid] = h[o:o + n]
                o += n
        return out

    # ------------------------------------------------------------------- cycle
    def step(self) -> DistReport:
        torch = self.torch
        rep = DistReport()
        st = self.te.bulk
        L = self.L
        kvbpt = self.model.kv_bytes_per_token
        ev = {k: torch.cuda.Event(enable_timing=True) for k in
              ("t0", "exch", "drain", "restore", "cons")}
        self.dist.barrier()
        ev["t0"].record(st)
        # ---- plan: every replica's queued burst outgrows its free KV by just
        # under (pp-1)/pp of a parameter copy, so plan_drop merges the
        # replicas into PP-pp groups (configs[2]: PP-2; configs[3]: PP-4)
        groups = [Group(i, [i], {i: (0, L)}) for i in sorted(self.instances)]
        demand = 0
        excess = self.model.param_bytes * (self.pp - 1) // self.pp - kvbpt
        for i, inst in sorted(self.instances.items()):
            free = inst.kv.free_tokens * kvbpt
            pending = (free + excess) // kvbpt
            demand += compute_demand(pending, free, kvbpt)
        plan = plan_drop(groups, demand, self.model)
        assert plan.merges and not plan.fallback, plan.to_text()
        orig_map = {rid: {h: (0, L)} for rid, h in self.home.items()}
        live = {g.gid: g for g in groups}
        for m in plan.merges:
            live.pop(m.gid_a)
            live.pop(m.gid_b)
            new = Group(m.gid, list(m.members), dict(m.stage_layer_map))
            new.validate_coverage(L)
            for iid in m.members:
                drops, fetches = member_moves(self.instances[iid].table.held_ranges(),
                                              m.stage_layer_map[iid])
                assert not fetches
                for lo, hi in drops:
                    memory.drop_layers(self.instances[iid], (lo, hi), new)
                    if self.poison_drops and iid == self.me:
                        self._poison(lo, hi)
            live[m.gid] = new
        final = {iid: g for g in live.values() for iid in g.member_instances}
        self.last_groups = dict(live)
        # ---- exchange (engine.py:690-726): pulls into this rank's pool
        tid = 0
        all_tasks = []
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
                all_tasks += tasks
        self._submit_local(all_tasks)
        self._sync_views()            # every pull landed
        self._release_sources()       # now the sources may free
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
        x_end = tid
        if self.on_merged is not None:  # untimed: runs between the exch and drain events
            self.on_merged(live, final)
        # ---- drain (untimed): the transient residents finish
        gone = []
        for rid in sorted(self.transient):
            for iid, inst in self.instances.items():
                inst.kv.free(rid)
                slot = self.slots[iid].drop(rid)
                if slot is not None and iid == self.me:
                    gone.append(slot)
        self.pool.release(gone, 0, L, stream=st)
        self._sync_views()
        ev["drain"].record(st)
        # ---- restore (engine.py:1093-1157): compaction here, pulls from holders
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
                    if iid == self.me:  # each compaction's size (waits for it)
                        rep.bytes_compaction += self.pool.last_moved_pages * self.shape.page_bytes
            # one plan per range index: a member of a PP-4 group can miss two
            # disjoint ranges, and plan_restore_transfers takes one range per
            # target (the reference's engine.py:1127 keeps only the last one)
            tasks = []
            for k in range(max(len(r) for r in missing.values()) if missing else 0):
                flat = {iid: rngs[k] for iid, rngs in missing.items() if len(rngs) > k}
                tasks += plan_restore_transfers(flat, holders, self.model.bytes_per_layer,
                                                self.param_chunk, tid_start=tid + len(tasks))
            assert all(t.src != HOST for t in tasks)
            tid += len(tasks)
            self.te.register_restore(tasks, self.model.bytes_per_layer)
            self._submit_local(tasks)
            for iid, rngs in missing.items():
                for rng in rngs:
                    memory.complete_restore(self.instances[iid], rng)
        r_end = tid
        self._sync_views()  # compactions done before a peer reads our block tables
        ev["restore"].record(st)
        # ---- dissolve + consolidation (engine.py:1159-1254)
        cons = []
        for rid in sorted(self.tokens):
            if rid in self.transient:
                continue
            home = self.home[rid]
            g = final[home]
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
                cons += chunks
        self._submit_local(cons)
        self._sync_views()
        self._release_sources()
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
        # ---- accounting
        done = self.te.drain()
        for p in done:
            k = p.task.tid
            if k < x_end:
                rep.bytes_kv_exchange += p.bytes_moved
            elif k < r_end:
                rep.bytes_param += p.bytes_moved
            else:
                rep.bytes_kv_consolidate += p.bytes_moved
            rep.bytes_pulled += p.bytes_moved
            rep.payload_bytes += p.task.size_bytes
            if p.task.src != self.me:
                rep.bytes_pulled_peer += p.bytes_moved
        for _, a, b, nbytes in self.te.kernel_spans:
            rep.copy_kernel_ms += a.elapsed_time(b)
            rep.copy_kernel_bytes += nbytes
        self.te.kernel_spans.clear()
        rep.kv_kernel_ms = _span_ms([p for p in done if p.task.kind is TaskKind.KVCACHE_CHUNK])
        rep.param_kernel_ms = _span_ms([p for p in done if p.task.kind is TaskKind.PARAM_SHARD])
        ev["cons"].synchronize()
        parts = {"exchange": ev["t0"].elapsed_time(ev["exch"]),
                 "restore": ev["drain"].elapsed_time(ev["restore"]),
                 "consolidate": ev["restore"].elapsed_time(ev["cons"])}
        parts["total"] = sum(parts.values())
        parts["drain_untimed"] = ev["exch"].elapsed_time(ev["drain"])
        rep.ms = parts
        self.refill()
        return rep

    # --------------------------------------------------- pipelined group decode
    def pipeline_decode(self, final: dict, iters: int = 3, microbatches: int = 2) -> dict:
        """One decode token for every resident of this rank's merged PP-2
        group, executed as a real pipeline across the two ranks: the stage-0
        rank runs its layers (cuBLAS GEMMs + this repo's kv_append and
        tcgen05 paged decode over its pool) per microbatch and hands the
        activation rows to the stage-1 rank through an ActChannel (the
        copy kernel storing into the peer's HBM), which runs the remaining
        layers.  Returns timing (CUDA events, max over ranks is the caller's)
        and the transport checksums."""
        import torch
        from .dist import ActChannel
        from .runtime import hash_tensor
        from .serving import StageRunner
        g = final[self.me]
        members = list(g.member_instances)
        if len(members) != 2:
            raise ValueError("pipeline_decode expects PP-2 groups")
        stage = members.index(self.me)
        lo, hi = g.stage_layer_map[self.me]
        res = sorted(r for r in self.tokens if self.home[r] in members)
        mbs = [res[k::microbatches] for k in range(microbatches)]
        H = self.shape.hidden
        dev = f"cuda:{self.device}"
        runner = StageRunner(self.pool, self.shape, max_seqs=max(len(m) for m in mbs))
        chan = ActChannel(self.rt, members[0], members[1],
                          slot_bytes=max(len(m) for m in mbs) * H * 2, slots=2,
                          key=f"pipe{g.gid}")

        def batch(mb):
            i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
            sl = [self.slots[self.me].of[r] for r in mb]
            ctx = [self.tokens[r] for r in mb]
            return {"n": len(mb), "slots": i32(sl), "pos": i32([c - 1 for c in ctx]),
                    "np": 0, "nd": len(mb), "n_prefill_rows": 0,
                    "d_rows": torch.arange(len(mb), dtype=torch.int64, device=dev),
                    "d_slots": i32(sl), "d_ctx": i32(ctx), "d_max": max(ctx)}
        batches = [batch(mb) for mb in mbs]
        gen = torch.Generator(device=dev).manual_seed(99)
        inputs = [(torch.randn((len(mb), H), device=dev, generator=gen) * 0.5).to(torch.bfloat16)
                  for mb in mbs]
        sums = []

        def one_pass(record):
            for k, b in enumerate(batches):
                if stage == 0:
                    x = runner.run(lo, hi, inputs[k], b)
                    chan.send(x.contiguous())
                    if record:
                        sums.append(hash_tensor(x.contiguous())[0])
                else:
                    raw = chan.recv(b["n"] * H * 2)
                    x = raw.view(torch.bfloat16).view(b["n"], H).clone()
                    chan.done()
                    if record:
                        sums.append(hash_tensor(x)[0])
                    runner.run(lo, hi, x, b)
        one_pass(True)  # warm-up (cuBLAS handles, lazy attributes) + checksums
        torch.cuda.synchronize(self.device)
        self.dist.barrier()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            one_pass(False)
        e.record()
        e.synchronize()
        ms = a.elapsed_time(e) / iters
        chan.close()
        return {"ms_per_token_step": ms, "tokens_per_step": len(res), "stage": stage,
                "handoff_bytes_per_step": len(res) * H * 2,
                "checksums": [int(x.item()) for x in sums], "group": g.gid}

    def refill(self) -> None:
        torch = self.torch
        for rid in sorted(self.transient):
            self._admit(rid)
        inf = self.pool.info()
        from .runtime import device_bytes
        bt = device_bytes(inf.block_table, inf.max_slots * self.L * inf.max_pages_per_seq * 4)
        bt = bt.view(torch.int32).view(inf.max_slots, self.L, inf.max_pages_per_seq)
        rows = []
        for rid in sorted(self.transient):
            if self.home[rid] == self.me:
                npg = -(-self.tokens[rid] // self.shape.block_tokens)
                rows.append(bt[self.slots[self.me].of[rid], :, :npg].reshape(-1))
        if rows:
            kv = self.pool.kv_bytes().view(torch.int32).view(-1, self.pool.page_bytes // 4)
            kv.index_fill_(0, torch.cat(rows).long(), 0x5A5A5A5A)
        self._sync_views()

    def close(self) -> None:
        self.torch.cuda.synchronize(self.device)
        self.dist.barrier()
        for v in self.views.values():
            v.close()
        self.dist.barrier()
        self.pool.close()


def run(rt, shape, kv_budget_bytes: int, steps: int, warmup: int, pipeline: bool = False,
        **kw) -> dict:
    """pipeline: also time the merged PP-2 groups decoding as cross-rank
    pipelines (pp=2 only)."""
    """Warm-up + timed steps; whole-job numbers (sum of bytes over ranks,
    max of step time over ranks) and the parity verdict."""
    import torch.distributed as dist
    poison = kw.pop("poison_drops", False)
    cyc = DistCycle(rt, shape, kv_budget_bytes, **kw)
    cyc.poison_drops = poison
    dev = f"cuda:{rt.device}" if dist.get_backend() == "nccl" else None
    w0 = cyc.weight_checksums()
    k0 = cyc.kv_checksums()
    for _ in range(warmup):
        cyc.step()
    reps = [cyc.step() for _ in range(steps)]
    ms = sum(r.ms["total"] for r in reps)
    w_ok = cyc.weight_checksums() == w0
    k1 = cyc.kv_checksums()
    kv_ok = set(k0) == set(k1) and all(bool((k0[r] == k1[r]).all()) for r in k0)
    pipe = None
    if pipeline and cyc.pp == 2:
        # after the parity checks (the decode appends K/V): one more cycle,
        # pipelined group decode in its merged state
        got = {}
        cyc.on_merged = lambda live, final: got.update(cyc.pipeline_decode(final))
        cyc.step()
        cyc.on_merged = None
        objs = [None] * dist.get_world_size()
        dist.all_gather_object(objs, got)
        by_group: dict = {}
        for o in objs:
            by_group.setdefault(o["group"], {})[o["stage"]] = o
        ok = all(len(v) == 2 and v[0]["checksums"] == v[1]["checksums"]
                 for v in by_group.values())
        ms_max = max(o["ms_per_token_step"] for o in objs)
        toks = sum(v[0]["tokens_per_step"] for v in by_group.values())
        pipe = {"tokens_per_s": toks / (ms_max / 1e3), "ms_per_token_step": ms_max,
                "handoff_bytes_per_step": sum(v[0]["handoff_bytes_per_step"]
                                              for v in by_group.values()),
                "groups": len(by_group), "handoff_bit_exact": ok}
    out = {
        "ms_total_max": max_over_ranks(ms, device=dev),
        # headline bytes: the reference's payload (TransferTask.size_bytes);
        # page-granular device bytes and the compaction separately
        "bytes_total": sum_over_ranks(sum(r.payload_bytes for r in reps), device=dev),
        "bytes_device": sum_over_ranks(sum(r.bytes_pulled for r in reps), device=dev),
        "bytes_compaction": sum_over_ranks(sum(r.bytes_compaction for r in reps), device=dev),
        "bytes_peer": sum_over_ranks(sum(r.bytes_pulled_peer for r in reps),
                                     device=dev),
        "peer_kernel_ms_max": max_over_ranks(sum(r.kv_kernel_ms + r.param_kernel_ms for r in reps),
                                             device=dev),
        # the copy launches alone, max over ranks, and the bytes they moved
        # (all ranks): the NVLink roofline's kernel time
        "copy_kernel_ms_max": max_over_ranks(sum(r.copy_kernel_ms for r in reps), device=dev),
        "copy_kernel_bytes": sum_over_ranks(sum(r.copy_kernel_bytes for r in reps), device=dev),
        "parity_fail": sum_over_ranks(0.0 if (w_ok and kv_ok) else 1.0,
                                      device=dev),
        "residents_local": len(k0),
        "peers_on_same_gpu": any(v.owner_device == rt.device for v in cyc.views.values()),
        "group_sizes": sorted(len(g.member_instances) for g in cyc.last_groups.values()),
        "last": reps[-1],
        "pipeline": pipe,
    }
    cyc.close()
    return out
