"""Pipeline-group serving engine: overload -> drop -> exchange -> restore.

Mirror of the reference's `dropsim.engine` (pkg/src/dropsim/engine.py) --
Engine(cfg, trace, policy, seed).run() -> SimResult and run_sim -- with the
same scheduling decisions, event order and event-log format, so in model
mode (cost-model stage times, link-model transfers) it reproduces the
reference's logs byte for byte (tests/test_engine.py against
tests/golden/engine_logs.json).

With `cfg.device.shape` set, every instance is a real device pool
(memory.build_instance(device=...)): drops / restores become device page
remaps and compactions, and `transfer_hook` (if given) executes every
TransferTask on the GPU through transfer.TransferEngine while the event
clock keeps the reference's timing model.  Section references below are to
the reference engine.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Callable, Optional

from . import memory
from .config import SimConfig
from .core import Chunk, Group, Microbatch, Request, RequestState, s_to_us
from .costmodel import batch_cost
from .exchange import (HOST, LinkModel, Network, TaskKind, TransferTask, finish_link,
                       plan_exchange, plan_restore_transfers, schedule_link, share_bytes)
from .formulation import attach_decode, lookahead_formulation, token_count_chunking
from .planner import DropPlan, compute_demand, member_moves, plan_drop
from .traceio import TraceRecord


class EventQueue:
    """(time_us, seq, fn) min-heap; seq breaks ties in push order (engine.py:48-66)."""

    def __init__(self) -> None:
        self._h: list = []
        self._n = 0

    def push(self, t: int, fn: Callable[[], None]) -> None:
        heapq.heappush(self._h, (t, self._n, fn))
        self._n += 1

    def pop(self):
        return heapq.heappop(self._h)

    def peek_time(self) -> int:
        return self._h[0][0]

    def __len__(self) -> int:
        return len(self._h)


@dataclass
class RoundState:
    no: int
    mbs: list
    members: list
    times: list          # [stage][mb] us
    act_ready: list      # [stage][mb] arrival us or None
    next_k: list
    free_at: list
    final_done: int = 0


@dataclass
class GroupRun:
    group: Group
    queue: list = field(default_factory=list)
    active: set = field(default_factory=set)
    admit_order: list = field(default_factory=list)
    ready_at_us: int = 0
    in_round: bool = False
    pause: bool = False
    no_admit: bool = False
    round_no: int = 0
    restoring: bool = False
    params_restored: bool = False
    rstate: Optional[RoundState] = None


@dataclass
class MonitorState:
    tick_us: int
    restore_threshold: float
    overload_seen_ticks: int = 0
    above_autoscale_since: Optional[int] = None
    autoscale_logged: bool = False


@dataclass
class SimResult:
    requests: dict
    log_lines: list
    end_us: int
    drop_events: int
    evictions: int
    fallbacks: int


class Engine:
    def __init__(self, cfg: SimConfig, trace: list[TraceRecord], policy: Optional[str] = None,
                 seed: int = 0, runtimes: Optional[dict] = None,
                 transfer_hook: Optional[Callable[[TransferTask], None]] = None):
        self.cfg = cfg
        self.policy = policy or cfg.policy.kind
        self.seed = seed
        self.model = cfg.model
        self.coeffs = cfg.cost
        self.trace = trace
        self.now = 0
        self.evq = EventQueue()
        self.log_lines: list[str] = []
        self.requests: dict[int, Request] = {}
        self.transfer_hook = transfer_hook
        L = self.model.num_layers
        cl = cfg.cluster
        shape = getattr(cfg.device, "shape", None)
        self.instances = {}
        for i in range(cl.instances):
            dev = None
            if shape is not None:
                if runtimes is None:
                    raise ValueError("device mode needs runtimes (device id -> Runtime)")
                devs = cfg.device.devices
                dev = runtimes[devs[i % len(devs)]]
            self.instances[i] = memory.build_instance(i, self.model, cl.hbm_bytes,
                                                      cl.nic_bandwidth, cl.map_latency_us,
                                                      device=dev, shape=shape)
        self.groups: dict[int, GroupRun] = {}
        self.group_of: dict[int, int] = {}
        k = cl.initial_group_size
        for lead in range(0, cl.instances, k):
            members = list(range(lead, lead + k))
            cuts = [j * L // k for j in range(k + 1)]
            smap = {members[j]: (cuts[j], cuts[j + 1]) for j in range(k)}
            g = Group(gid=lead, member_instances=members, stage_layer_map=smap)
            g.validate_coverage(L)
            self.groups[lead] = GroupRun(group=g)
            for iid in members:
                self.group_of[iid] = lead
                lo, hi = smap[iid]
                if lo > 0:
                    memory.drop_layers(self.instances[iid], (0, lo), g)
                if hi < L:
                    memory.drop_layers(self.instances[iid], (hi, L), g)
        self.network = Network({i: inst.nic_bandwidth for i, inst in self.instances.items()},
                               cl.host_bandwidth, cl.link_base_latency_us)
        self.total_alloc: dict[int, int] = {}
        self.pending_prefill: dict[int, int] = {}
        self.prefilled_in_round: dict[int, int] = {}
        self.resume_state: dict[int, RequestState] = {}
        self.move_outstanding: dict[int, int] = {}
        self.consolidating: dict[int, dict] = {}
        self.swapped_out: list[int] = []
        self.swap_inflight: set[int] = set()
        self.admit_seq: dict[int, int] = {}
        self._admit_counter = 0
        self.round_counter = 0
        self._tid = 0
        self._task_cb: dict[int, Callable] = {}
        self.transition_tasks = 0
        self.deferred_drops: dict[int, list] = {}
        self.fetch_gate: dict[int, int] = {}
        self._restore_left: dict[int, dict] = {}
        self._restore_ranges: dict[int, dict] = {}
        self.monitor = MonitorState(cfg.policy.monitor_tick_us, cfg.policy.restore_threshold)
        self.overload_flag = False
        self.policy_pending = False
        self.drop_events = 0
        self.evictions = 0
        self.fallbacks = 0
        last = trace[-1].arrival_us if trace else 0
        self.horizon_us = last + s_to_us(cfg.report.drain_s)

    # ------------------------------------------------------------ event log
    def log(self, kind: str, **fields) -> None:
        """"<now> <KIND> k=v ..." (engine.py:189-193)."""
        self.log_lines.append(" ".join([str(self.now), kind] +
                                       [f"{k}={v}" for k, v in fields.items()]))

    # ------------------------------------------------ token-unit accounting
    def _share_delta(self, group: Group, iid: int, t0: int, delta: int) -> int:
        lo, hi = group.stage_layer_map[iid]
        L = self.model.num_layers
        return memory.stage_share(t0 + delta, lo, hi, L) - memory.stage_share(t0, lo, hi, L)

    def group_can_alloc(self, grun: GroupRun, rid: int, delta: int) -> bool:
        """Every member can take its stage share of `delta` more tokens (engine.py:205-212)."""
        t0 = self.total_alloc.get(rid, 0)
        g = grun.group
        return all(self._share_delta(g, iid, t0, delta) <= self.instances[iid].kv.free_tokens
                   for iid in g.member_instances)

    def group_alloc(self, grun: GroupRun, rid: int, delta: int) -> bool:
        if not self.group_can_alloc(grun, rid, delta):
            return False
        t0 = self.total_alloc.get(rid, 0)
        for iid in grun.group.member_instances:
            inc = self._share_delta(grun.group, iid, t0, delta)
            if inc:
                assert self.instances[iid].kv.alloc(rid, inc)
        self.total_alloc[rid] = t0 + delta
        return True

    def group_free(self, grun: GroupRun, rid: int) -> None:
        for iid in grun.group.member_instances:
            self.instances[iid].kv.free(rid)
        self.total_alloc.pop(rid, None)

    def group_free_tokens(self, grun: GroupRun) -> int:
        """Largest admissible request in tokens (engine.py:236-244)."""
        L = self.model.num_layers
        caps = [self.instances[iid].kv.free_tokens * L // (hi - lo)
                for iid, (lo, hi) in ((i, grun.group.stage_layer_map[i])
                                      for i in grun.group.member_instances)]
        return min(caps) if caps else 0

    def _live_instances(self):
        return [inst for inst in self.instances.values() if not inst.failed]

    def free_kv_bytes(self) -> int:
        return sum(i.kv.free_tokens * self.model.kv_bytes_per_token for i in self._live_instances())

    def base_kv_bytes(self) -> int:
        return sum(i.hbm_bytes - self.model.param_bytes for i in self._live_instances())

    def used_kv_bytes(self) -> int:
        return sum(i.kv.used_tokens * self.model.kv_bytes_per_token for i in self._live_instances())

    # ------------------------------------------------------------- dispatch
    def dispatch(self, req: Request) -> int:
        """Group with most free tokens, ties by lowest lead (engine.py:258-271)."""
        best = min(((-self.group_free_tokens(gr), gr.group.member_instances[0], gid)
                    for gid, gr in self.groups.items()), key=lambda t: (t[0], t[1]))
        gid = best[2]
        grun = self.groups[gid]
        req.home_instance = grun.group.member_instances[0]
        grun.queue.append(req.rid)
        self.log("DISPATCH", req=req.rid, inst=req.home_instance, group=gid)
        return req.home_instance

    # ------------------------------------------------------------ transfers
    def _next_tid(self) -> int:
        self._tid += 1
        return self._tid

    def enqueue_task(self, task: TransferTask, cb: Callable) -> None:
        link = self.network.link(task.src, task.dst)
        link.enqueue(task, self.now)
        self._task_cb[task.tid] = cb
        self._pump(link)

    def _pump(self, link: LinkModel) -> None:
        got = schedule_link(link, self.now)
        if got is None:
            return
        task, start, done = got
        if self.transfer_hook is not None:
            self.transfer_hook(task)
        self.evq.push(done, lambda: self._xfer_done(link, task, start, done))

    def _xfer_done(self, link: LinkModel, task: TransferTask, start: int, done: int) -> None:
        finish_link(link, task)
        self.log("XFER", task=task.kind.value, src=task.src, dst=task.dst,
                 bytes=task.size_bytes, start=start,
                 rid=task.rid if task.rid is not None else -1)
        cb = self._task_cb.pop(task.tid, None)
        if cb is not None:
            cb(task, done)
        self._pump(link)

    # --------------------------------------------------------------- rounds
    def _formulate(self, grun: GroupRun, items: list[Chunk]) -> list[Microbatch]:
        mode = self.cfg.policy.formulation
        look = (self.policy == "kunserve" and grun.group.size >= 2) if mode == "auto" \
            else mode == "lookahead"
        if look:
            return lookahead_formulation(items, self.coeffs, self.cfg.policy.min_batch_tokens)
        return token_count_chunking(items, self.cfg.policy.token_budget)

    def kick(self, gid: int) -> None:
        grun = self.groups.get(gid)
        if grun is None or grun.in_round or grun.pause or self.fetch_gate.get(gid, 0) > 0:
            return
        if grun.ready_at_us > self.now:  # remap gate
            self.evq.push(grun.ready_at_us, lambda: self.kick(gid))
            return
        self._form_round(grun)

    def _decode_chunks(self, grun: GroupRun) -> list[Chunk]:
        out, blocked = [], 0
        for rid in sorted(grun.active):
            req = self.requests[rid]
            if req.state is not RequestState.DECODING:
                continue
            if self.group_alloc(grun, rid, 1):
                out.append(Chunk(rid, 1, req.context_len, decode=True))
            else:
                blocked += 1
        if blocked:
            self.overload_flag = True
            self.log("OOM", group=grun.group.gid, blocked=blocked)
        return out

    def _admit_queue(self, grun: GroupRun) -> None:
        gid = grun.group.gid
        while grun.queue:
            rid = grun.queue[0]
            req = self.requests[rid]
            need = req.input_len + req.tokens_decoded
            if not self.group_alloc(grun, rid, need):
                self.overload_flag = True
                self.log("OOM", group=gid, head=rid, need=need)
                return
            grun.queue.pop(0)
            grun.active.add(rid)
            grun.admit_order.append(rid)
            self._admit_counter += 1
            self.admit_seq[rid] = self._admit_counter
            req.set_state(RequestState.PREFILLING)
            self.pending_prefill[rid] = need
            self.prefilled_in_round[rid] = 0
            self.log("ADMIT", req=rid, group=gid, tokens=need)

    def _form_round(self, grun: GroupRun) -> None:
        """Snapshot decoders + admissible queue, formulate, start stage 0
        (engine.py:331-408)."""
        gid = grun.group.gid
        decode = self._decode_chunks(grun)
        if self.policy == "swap":
            self._try_swap_in(grun)
        if not grun.no_admit:
            self._admit_queue(grun)
        items = []
        for rid in grun.admit_order:
            if rid not in grun.active:
                continue
            req = self.requests[rid]
            if req.state is RequestState.PREFILLING:
                left = self.pending_prefill[rid] - req.tokens_prefilled
                if left > 0:
                    items.append(Chunk(rid, left, req.tokens_prefilled))
        mbs = self._formulate(grun, items) if items else []
        mbs = attach_decode(mbs, decode)
        if not mbs:
            return
        grun.in_round = True
        self.round_counter += 1
        grun.round_no = self.round_counter
        members = grun.group.member_instances
        L = self.model.num_layers
        spans = [grun.group.stage_layer_map[i][1] - grun.group.stage_layer_map[i][0]
                 for i in members]
        times = self._stage_times(grun, mbs, spans)
        act_ready = [[self.now if s == 0 else None for _ in mbs] for s in range(len(members))]
        grun.rstate = RoundState(grun.round_no, mbs, members, times, act_ready,
                                 [0] * len(members), [self.now] * len(members))
        self.log("ROUND", group=gid, rnd=grun.round_no, n_mb=len(mbs), prefill=len(items),
                 decode=len(decode))
        self._try_start_stage(gid, 0)

    def _stage_times(self, grun: GroupRun, mbs: list[Microbatch], spans: list[int]) -> list:
        """[stage][mb] execution us: the cost model scaled by each stage's
        layer share (engine.py:389-397).  serving.DeviceEngine measures them."""
        L = self.model.num_layers
        costs = [batch_cost(mb.chunks, self.coeffs) for mb in mbs]
        return [[max(1, int(round(c * 1_000_000 * span / L))) for c in costs] for span in spans]

    # device hooks (no-ops in model mode; serving.DeviceEngine implements them)
    def _on_exchange_planned(self, tasks, old_map, new_map, tokens) -> None:
        pass

    def _on_params_planned(self, tasks, fetch: bool, **restore) -> None:
        pass

    def _on_consolidation_planned(self, rid: int, peer: int, home: int, layers, tasks) -> None:
        pass

    def _on_consolidated(self, rid: int, peers) -> None:
        pass

    def _try_start_stage(self, gid: int, s: int) -> None:
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None:
            return
        rs = grun.rstate
        while rs.next_k[s] < len(rs.mbs):
            k = rs.next_k[s]
            ready = rs.act_ready[s][k]
            if ready is None:
                return
            start = max(rs.free_at[s], ready)
            end = start + rs.times[s][k]
            rs.free_at[s] = end
            rs.next_k[s] += 1
            self.evq.push(end, lambda k=k, s=s, start=start, end=end:
                          self._stage_done(gid, rs.no, k, s, start, end))

    def _stage_done(self, gid: int, rnd: int, k: int, s: int, start: int, end: int) -> None:
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None or grun.rstate.no != rnd:
            return  # stale: the group changed under this round
        rs = grun.rstate
        self.log("STAGE", group=gid, rnd=rnd, stage=s, mb=k, start=start, end=end)
        if s < len(rs.members) - 1:
            nbytes = max(1, rs.mbs[k].token_count * self.model.hidden_bytes_per_token)
            task = TransferTask(self._next_tid(), TaskKind.ACTIVATION, rs.members[s],
                                rs.members[s + 1], nbytes)
            self.enqueue_task(task, lambda t, done, k=k, s=s:
                              self._act_arrived(gid, rnd, k, s + 1, done))
        else:
            self._complete_microbatch(grun, rs.mbs[k], end)
            rs.final_done += 1
            if rs.final_done == len(rs.mbs):
                self._end_round(grun, end)
                return
        self._try_start_stage(gid, s)

    def _act_arrived(self, gid: int, rnd: int, k: int, s: int, when: int) -> None:
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None or grun.rstate.no != rnd:
            return
        grun.rstate.act_ready[s][k] = when
        self._try_start_stage(gid, s)

    def _complete_microbatch(self, grun: GroupRun, mb: Microbatch, when: int) -> None:
        saved, self.now = self.now, when
        for ch in mb.chunks:
            req = self.requests[ch.rid]
            if req.state is RequestState.QUEUED:
                # evicted while the round was in flight (the fallback's
                # recompute relief does not wait for round ends,
                # engine.py:663-668): its chunk's work is discarded.  The
                # reference would count a token, or raise KeyError on
                # pending_prefill; the wall-clock engine, whose rounds run
                # on the device while the monitor ticks, reaches this.
                continue
            if ch.decode:
                req.record_token(when)
                self.log("TOKEN", req=ch.rid, n=req.tokens_decoded)
                if req.done:
                    self._finish(grun, req)
                continue
            req.tokens_prefilled += ch.token_count
            if req.tokens_prefilled < self.pending_prefill[ch.rid]:
                continue
            # prefill done; a re-prefill after eviction folds decoded context back
            req.tokens_prefilled = req.input_len
            req.set_state(RequestState.DECODING)
            if req.first_token_us is None:
                req.record_token(when)
                self.log("FIRST_TOKEN", req=ch.rid, ttft_us=when - req.arrival_us)
                if req.done:
                    self._finish(grun, req)
        self.now = saved

    def _finish(self, grun: GroupRun, req: Request) -> None:
        req.set_state(RequestState.FINISHED)
        grun.active.discard(req.rid)
        self.group_free(grun, req.rid)
        self.pending_prefill.pop(req.rid, None)
        self.log("FINISH", req=req.rid)

    def _end_round(self, grun: GroupRun, when: int) -> None:
        gid = grun.group.gid
        grun.in_round = False
        grun.rstate = None
        self.log("ROUND_END", group=gid, rnd=grun.round_no)
        if self.policy_pending:
            self._policy_step()
        if grun.params_restored and gid in self.groups and self._dissolve(grun):
            return
        self.kick(gid)

    def _arrive(self, rec: TraceRecord, rid: int) -> None:
        req = Request(rid=rid, arrival_us=rec.arrival_us, input_len=rec.input_len,
                      output_len=rec.output_len)
        self.requests[rid] = req
        self.log("ARRIVE", req=rid, inp=rec.input_len, out=rec.output_len)
        self.dispatch(req)
        self.kick(self.group_of[req.home_instance])

    # -------------------------------------------------------------- monitor
    def _occupancy_bp(self) -> int:
        base = self.base_kv_bytes()
        return (self.used_kv_bytes() * 10_000) // base if base else 0

    def _head_blocked(self, grun: GroupRun) -> bool:
        if not grun.queue:
            return False
        req = self.requests[grun.queue[0]]
        return not self.group_can_alloc(grun, req.rid, req.input_len + req.tokens_decoded)

    def _tick(self) -> None:
        """Monitor (engine.py:520-567): overload = blocked decode or blocked
        queue head, debounced over two ticks."""
        queued = sum(len(g.queue) for g in self.groups.values())
        stalled = sum(1 for r in self.requests.values() if r.state is RequestState.STALLED)
        self.log("OCC", bp=self._occupancy_bp(), queued=queued, stalled=stalled)
        if not self.overload_flag:
            for grun in self.groups.values():
                if self._blocked_decode(grun) or self._head_blocked(grun):
                    self.overload_flag = True
                    break
        m = self.monitor
        m.overload_seen_ticks = m.overload_seen_ticks + 1 if self.overload_flag else 0
        self.overload_flag = False
        if m.overload_seen_ticks >= 2 and not self.policy_pending:
            self.policy_pending = True
        if self.policy_pending:
            self._policy_step()
        if self.policy == "kunserve":
            self._restore_check()
            for gid in sorted(self.groups):
                grun = self.groups.get(gid)
                if grun is not None and grun.params_restored and not grun.in_round \
                        and grun.group.size > 1:
                    self._dissolve(grun)
            self._consolidation_retry()
            self._autoscale_check()
        if self.policy == "swap":
            for gid in sorted(self.groups):
                self.kick(gid)
        nxt = self.now + m.tick_us
        if nxt <= self.horizon_us:
            self.evq.push(nxt, self._tick)

    def _autoscale_check(self) -> None:
        m = self.monitor
        dropped = any(g.group.size > 1 for g in self.groups.values())
        if dropped and self._occupancy_bp() / 10_000 >= self.cfg.policy.autoscale_occupancy:
            if m.above_autoscale_since is None:
                m.above_autoscale_since = self.now
            if not m.autoscale_logged and \
                    self.now - m.above_autoscale_since >= s_to_us(self.cfg.policy.autoscale_window_s):
                self.log("AUTOSCALE", occ_bp=self._occupancy_bp())
                m.autoscale_logged = True
        else:
            m.above_autoscale_since = None

    # -------------------------------------------------------- policy actions
    def _group_pending_tokens(self, grun: GroupRun) -> int:
        n = sum(self.requests[r].input_len + self.requests[r].tokens_decoded for r in grun.queue)
        for rid in sorted(grun.active):
            if self.requests[rid].state is RequestState.DECODING and \
                    not self.group_can_alloc(grun, rid, 1):
                n += 1
        return n

    def _group_free_bytes(self, grun: GroupRun) -> int:
        return sum(self.instances[i].kv.free_tokens for i in grun.group.member_instances) \
            * self.model.kv_bytes_per_token

    def _blocked_decode(self, grun: GroupRun) -> bool:
        return any(self.requests[rid].state is RequestState.DECODING
                   and not self.group_can_alloc(grun, rid, 1) for rid in sorted(grun.active))

    def _policy_step(self) -> None:
        if not self.policy_pending:
            return
        if self.policy == "kunserve":
            self._kunserve_step()
        else:
            self._baseline_step()

    def _kunserve_step(self) -> None:
        """Plan and apply drops (engine.py:608-648)."""
        if self.transition_tasks > 0:
            return
        kvbpt = self.model.kv_bytes_per_token
        demand = sum(compute_demand(self._group_pending_tokens(gr), self._group_free_bytes(gr),
                                    kvbpt) for _, gr in sorted(self.groups.items()))
        if demand == 0:
            self.policy_pending = False
            for g in self.groups.values():
                g.pause = False
            return
        plan = plan_drop([g.group for g in self.groups.values()], demand, self.model)
        self.log("OVERLOAD", demand=demand)
        if not plan.merges:
            self.fallbacks += 1
            self.log("PLAN", merges=0, freed=0, fallback=1)
            self.log("AUTOSCALE", occ_bp=self._occupancy_bp())
            for gid in sorted(self.groups):  # recompute-style relief
                self._act_recompute(self.groups[gid])
                self.kick(gid)
            self.policy_pending = False
            return
        busy = [g for st in plan.merges for g in (st.gid_a, st.gid_b)
                if g in self.groups and self.groups[g].in_round]
        if busy:
            for g in busy:
                self.groups[g].pause = True
            return  # retried at round ends
        self._apply_plan(plan)
        self.policy_pending = False

    def _redispatch_queues(self) -> None:
        waiting = []
        for gid in sorted(self.groups):
            waiting.extend(self.groups[gid].queue)
            self.groups[gid].queue = []
        waiting.sort(key=lambda rid: (self.requests[rid].arrival_us, rid))
        for rid in waiting:
            self.dispatch(self.requests[rid])
        for gid in sorted(self.groups):
            self.kick(gid)

    def _apply_plan(self, plan: DropPlan) -> None:
        """Merges, re-dispatch, one exchange per original-map cohort (engine.py:670-727)."""
        self.log("PLAN", merges=len(plan.merges), freed=plan.freed_bytes,
                 fallback=int(plan.fallback))
        orig: dict[int, dict] = {}
        for st in plan.merges:
            for gid in (st.gid_a, st.gid_b):
                grun = self.groups.get(gid)
                if grun is not None:
                    for rid in grun.active:
                        orig.setdefault(rid, dict(grun.group.stage_layer_map))
        for st in plan.merges:
            self._merge_groups(st)
        self.drop_events += len(plan.merges)
        self._redispatch_queues()
        chunk = self._exchange_chunk_bytes()
        L, kvbpt = self.model.num_layers, self.model.kv_bytes_per_token
        for gid in sorted(self.groups):
            grun = self.groups[gid]
            if grun.group.size < 2:
                continue
            cohorts: dict[tuple, list[int]] = {}
            for rid in sorted(grun.active):
                if rid in orig:
                    cohorts.setdefault(tuple(sorted(orig[rid].items())), []).append(rid)
            for key in sorted(cohorts):
                toks = {rid: self.requests[rid].context_len for rid in cohorts[key]
                        if self.requests[rid].context_len > 0}
                if not toks:
                    continue
                tasks = plan_exchange(toks, dict(key), grun.group.stage_layer_map, L, kvbpt,
                                      chunk, tid_start=self._tid + 1)
                self._tid += len(tasks)
                self._on_exchange_planned(tasks, dict(key), grun.group.stage_layer_map, toks)
                if tasks:
                    self.log("EXCHANGE", group=gid, tasks=len(tasks),
                             bytes=sum(t.size_bytes for t in tasks))
                for rid in sorted({t.rid for t in tasks}):
                    req = self.requests[rid]
                    self.resume_state[rid] = req.state
                    req.set_state(RequestState.STALLED)
                    self.move_outstanding[rid] = sum(1 for t in tasks if t.rid == rid)
                    self.log("STALL", req=rid)
                for t in tasks:
                    self.transition_tasks += 1
                    self.enqueue_task(t, self._exchange_chunk_done)
            self.kick(gid)

    def _exchange_chunk_bytes(self) -> int:
        """~one stage execution of link time, >= 1 MB (engine.py:729-734)."""
        est = batch_cost([Chunk(0, self.cfg.policy.token_budget, 0)], self.coeffs)
        stages = max((g.group.size for g in self.groups.values()), default=1)
        bw = min(inst.nic_bandwidth for inst in self.instances.values())
        return max(1_000_000, int(est / max(1, stages) * bw))

    def _exchange_chunk_done(self, task: TransferTask, when: int) -> None:
        self.transition_tasks -= 1
        rid = task.rid
        left = self.move_outstanding.get(rid, 0) - 1
        self.move_outstanding[rid] = left
        if left:
            return
        del self.move_outstanding[rid]
        req = self.requests[rid]
        if req.state is RequestState.STALLED:
            req.set_state(self.resume_state.pop(rid, RequestState.DECODING))
            self.log("RESUME", req=rid)
        gid = self.group_of.get(req.home_instance)
        if gid is not None:
            self.kick(gid)

    def _merge_groups(self, st) -> None:
        """Fetch-before-drop, deferred drops, remap gate, re-share (engine.py:751-836)."""
        ga, gb = self.groups.pop(st.gid_a), self.groups.pop(st.gid_b)
        new = Group(gid=st.gid, member_instances=list(st.members),
                    stage_layer_map=dict(st.stage_layer_map))
        new.validate_coverage(self.model.num_layers)
        residents = [(ga, rid) for rid in sorted(ga.active)] + \
                    [(gb, rid) for rid in sorted(gb.active)]
        held = {iid: self.instances[iid].table.held_ranges() for iid in st.members}
        moves = {iid: member_moves(held[iid], st.stage_layer_map[iid]) for iid in st.members}
        fetches = {iid: mv[1] for iid, mv in moves.items() if mv[1]}
        protected: set = set()
        fetch_tasks: list[TransferTask] = []
        if fetches:
            fetch_tasks = plan_restore_transfers(
                {iid: rng for iid, rngs in fetches.items() for rng in rngs}, held,
                self.model.bytes_per_layer, self._exchange_chunk_bytes(),
                tid_start=self._tid + 1)
            self._tid += len(fetch_tasks)
            self._on_params_planned(fetch_tasks, fetch=True)
            for t in fetch_tasks:
                if t.src != HOST and t.layers:
                    protected.update((t.src, l) for l in range(*t.layers))
        max_delay = 0
        for iid in st.members:
            drops = moves[iid][0]
            freed, blocks = 0, 0
            for lo, hi in drops:
                for layer in range(lo, hi):
                    if (iid, layer) in protected:  # last live copy: drop after the fetch
                        self.deferred_drops.setdefault(iid, []).append((layer, layer + 1, st.gid))
                        continue
                    freed += memory.drop_layers(self.instances[iid], (layer, layer + 1), new)
                    blocks += 1
            if blocks:
                delay = self.instances[iid].table.map_latency_us * blocks
                max_delay = max(max_delay, delay)
                self.log("DROP", inst=iid, blocks=blocks, freed=freed)
                self.log("REMAP", inst=iid, blocks=blocks, delay_us=delay)
        merged = GroupRun(group=new)
        merged.ready_at_us = max(ga.ready_at_us, gb.ready_at_us, self.now + max_delay)
        merged.queue = sorted(ga.queue + gb.queue,
                              key=lambda rid: (self.requests[rid].arrival_us, rid))
        merged.active = ga.active | gb.active
        merged.admit_order = [rid for rid in sorted(ga.admit_order + gb.admit_order,
                                                    key=lambda rid: self.admit_seq[rid])
                              if rid in merged.active]
        self.groups[st.gid] = merged
        for iid in st.members:
            self.group_of[iid] = st.gid
        self.log("GROUP", gid=st.gid, members=",".join(map(str, st.members)),
                 stages=",".join(f"{iid}:{lo}:{hi}" for iid, (lo, hi) in
                                 sorted(st.stage_layer_map.items())))
        L = self.model.num_layers
        for grun, rid in residents:  # capacity grew, so the new shares fit
            total = self.total_alloc.get(rid, 0)
            for iid in grun.group.member_instances:
                self.instances[iid].kv.free(rid)
            for iid in sorted(new.member_instances):
                lo, hi = new.stage_layer_map[iid]
                share = memory.stage_share(total, lo, hi, L)
                if share:
                    assert self.instances[iid].kv.alloc(rid, share)
        for t in fetch_tasks:
            self.fetch_gate[st.gid] = self.fetch_gate.get(st.gid, 0) + 1
            self.transition_tasks += 1
            self.enqueue_task(t, lambda task, when, gid=st.gid: self._fetch_done(gid, task, when))

    def _fetch_done(self, gid: int, task: TransferTask, when: int) -> None:
        self.transition_tasks -= 1
        self.fetch_gate[gid] = self.fetch_gate.get(gid, 1) - 1
        if task.layers and task.src != HOST:
            keep = []
            for lo, hi, owner in self.deferred_drops.get(task.src, []):
                if task.layers[0] <= lo and hi <= task.layers[1]:
                    grun = self.groups.get(owner)
                    freed = memory.drop_layers(self.instances[task.src], (lo, hi),
                                               grun.group if grun else None)
                    self.log("DROP", inst=task.src, blocks=hi - lo, freed=freed)
                else:
                    keep.append((lo, hi, owner))
            if keep:
                self.deferred_drops[task.src] = keep
            else:
                self.deferred_drops.pop(task.src, None)
        if self.fetch_gate.get(gid, 0) == 0:
            self.fetch_gate.pop(gid, None)
            self.kick(gid)

    # ------------------------------------------------------------ baselines
    def _baseline_step(self) -> None:
        act = {"recompute": self._act_recompute, "swap": self._act_swap,
               "migrate": self._act_migrate}[self.policy]
        for gid in sorted(self.groups):
            grun = self.groups[gid]
            if not self._blocked_decode(grun):
                continue
            if grun.in_round:
                grun.pause = True
                continue
            act(grun)
            grun.pause = False
            self.kick(gid)
        if not any(g.pause for g in self.groups.values()):
            self.policy_pending = False

    def _victims_newest_first(self, grun: GroupRun) -> list[int]:
        live = (RequestState.DECODING, RequestState.PREFILLING)
        return sorted((rid for rid in grun.active if self.requests[rid].state in live),
                      key=lambda rid: -self.admit_seq[rid])

    def _evict_one(self, grun: GroupRun, rid: int) -> None:
        req = self.requests[rid]
        self.group_free(grun, rid)
        grun.active.discard(rid)
        grun.admit_order.remove(rid)
        req.set_state(RequestState.DROPPED)
        req.set_state(RequestState.QUEUED)
        req.tokens_prefilled = 0
        self.pending_prefill.pop(rid, None)
        grun.queue.insert(0, rid)
        self.evictions += 1
        self.log("EVICT", req=rid, group=grun.group.gid)

    def _act_recompute(self, grun: GroupRun) -> None:
        while self._blocked_decode(grun):
            victims = self._victims_newest_first(grun)
            if not victims:
                return
            self._evict_one(grun, victims[0])

    def _act_swap(self, grun: GroupRun) -> None:
        iid = grun.group.member_instances[0]
        if not self._blocked_decode(grun):
            return
        victims = [r for r in self._victims_newest_first(grun) if r not in self.swap_inflight]
        if not victims:
            return
        rid = victims[0]
        req = self.requests[rid]
        self.resume_state[rid] = req.state
        req.set_state(RequestState.STALLED)
        self.swap_inflight.add(rid)
        nbytes = self.total_alloc.get(rid, 0) * self.model.kv_bytes_per_token
        task = TransferTask(self._next_tid(), TaskKind.KVCACHE_CHUNK, iid, HOST, nbytes, rid=rid)
        self.evictions += 1
        self.log("SWAP_OUT", req=rid, bytes=nbytes)
        self.enqueue_task(task, lambda t, when, g=grun.group.gid: self._swap_out_done(g, t, when))

    def _swap_out_done(self, gid: int, task: TransferTask, when: int) -> None:
        grun = self.groups.get(gid)
        if grun is None:
            return
        rid = task.rid
        self.group_free(grun, rid)
        grun.active.discard(rid)
        if rid in grun.admit_order:
            grun.admit_order.remove(rid)
        self.swap_inflight.discard(rid)
        self.swapped_out.append(rid)
        self.kick(gid)

    def _try_swap_in(self, grun: GroupRun) -> None:
        iid = grun.group.member_instances[0]
        while self.swapped_out:
            rid = self.swapped_out[0]
            req = self.requests[rid]
            need = req.context_len
            if rid in self.swap_inflight or not self.group_can_alloc(
                    grun, rid, need + self.cfg.policy.swap_headroom_tokens):
                return
            self.swapped_out.pop(0)
            self.swap_inflight.add(rid)
            assert self.group_alloc(grun, rid, need)
            nbytes = need * self.model.kv_bytes_per_token
            task = TransferTask(self._next_tid(), TaskKind.KVCACHE_CHUNK, HOST, iid, nbytes, rid=rid)
            self.log("SWAP_IN", req=rid, bytes=nbytes)
            self.enqueue_task(task, lambda t, when, g=grun.group.gid: self._swap_in_done(g, t, when))

    def _swap_in_done(self, gid: int, task: TransferTask, when: int) -> None:
        grun = self.groups.get(gid)
        if grun is None:
            return
        rid = task.rid
        self.swap_inflight.discard(rid)
        grun.active.add(rid)
        grun.admit_order.append(rid)
        self._admit_counter += 1
        self.admit_seq[rid] = self._admit_counter
        self.requests[rid].set_state(self.resume_state.pop(rid, RequestState.DECODING))
        self.log("RESUME", req=rid)
        self.kick(gid)

    def _act_migrate(self, grun: GroupRun) -> None:
        while self._blocked_decode(grun):
            victims = [r for r in self._victims_newest_first(grun)
                       if r not in self.move_outstanding]
            if not victims:
                return
            rid = victims[0]
            req = self.requests[rid]
            need = self.total_alloc.get(rid, 0)
            dest = None
            for _, gid in sorted(((-self.group_free_tokens(g), g.group.gid)
                                  for g in self.groups.values() if g is not grun)):
                if self.group_free_tokens(self.groups[gid]) >= need:
                    dest = self.groups[gid]
                    break
            if dest is None:
                self.log("MIGRATE_NOOP", group=grun.group.gid)
                self._evict_one(grun, rid)
                continue
            src_iid = grun.group.member_instances[0]
            dst_iid = dest.group.member_instances[0]
            saved = self.total_alloc.pop(rid)
            assert self.group_alloc(dest, rid, saved)
            self.resume_state[rid] = req.state
            req.set_state(RequestState.STALLED)
            grun.active.discard(rid)
            grun.admit_order.remove(rid)
            nbytes = req.context_len * self.model.kv_bytes_per_token
            task = TransferTask(self._next_tid(), TaskKind.KVCACHE_CHUNK, src_iid, dst_iid,
                                max(1, nbytes), rid=rid)
            self.log("MIGRATE", req=rid, src=src_iid, dst=dst_iid, bytes=nbytes)
            self.move_outstanding[rid] = 1
            self.enqueue_task(task, lambda t, when, g=grun.group.gid, d=dest.group.gid, n=saved:
                              self._migrate_done(g, d, t, n, when))
            return  # one move per step; the next tick re-evaluates

    def _migrate_done(self, src_gid: int, dst_gid: int, task: TransferTask, tokens: int,
                      when: int) -> None:
        rid = task.rid
        src, dst = self.groups.get(src_gid), self.groups.get(dst_gid)
        if src is not None:
            self.instances[src.group.member_instances[0]].kv.free(rid)
        self.move_outstanding.pop(rid, None)
        req = self.requests[rid]
        if dst is not None:
            dst.active.add(rid)
            dst.admit_order.append(rid)
            self._admit_counter += 1
            self.admit_seq[rid] = self._admit_counter
            req.home_instance = dst.group.member_instances[0]
        req.set_state(self.resume_state.pop(rid, RequestState.DECODING))
        self.log("RESUME", req=rid)
        if src is not None:
            self.kick(src_gid)
        if dst is not None:
            self.kick(dst_gid)

    # ------------------------------------------------------------- restore
    def _restore_check(self) -> None:
        """Below restore_threshold occupancy, restore merged groups (engine.py:1051-1066)."""
        if self.transition_tasks > 0:
            return
        merged = [g for g in self.groups.values() if g.group.size > 1]
        if not merged:
            return
        if self.used_kv_bytes() / self.base_kv_bytes() >= self.monitor.restore_threshold:
            return
        chunk = self._exchange_chunk_bytes()
        for grun in merged:
            if not grun.restoring and self._plan_homes(grun) is not None:
                self._start_restore(grun, chunk)

    def _plan_homes(self, grun: GroupRun) -> Optional[dict]:
        """First-fit decreasing homes for the dissolve (engine.py:1068-1091)."""
        kvbpt = self.model.kv_bytes_per_token
        room = {iid: (self.instances[iid].hbm_bytes - self.model.param_bytes) // kvbpt
                for iid in grun.group.member_instances}
        needs = sorted(((self.total_alloc.get(rid, 0) + self.requests[rid].output_len
                         - self.requests[rid].tokens_decoded, rid) for rid in sorted(grun.active)),
                       key=lambda t: (-t[0], t[1]))
        homes = {}
        for need, rid in needs:
            iid = max(sorted(room), key=lambda i: (room[i], -i))
            if room[iid] < need:
                return None
            room[iid] -= need
            homes[rid] = iid
        return homes

    def _start_restore(self, grun: GroupRun, chunk: int) -> None:
        gid = grun.group.gid
        L = self.model.num_layers
        missing, holders = {}, {}
        for iid in grun.group.member_instances:
            holders[iid] = self.instances[iid].table.held_ranges()
            need = member_moves(holders[iid], (0, L))[1]
            if need:
                missing[iid] = need
        if not missing:
            grun.restoring = grun.params_restored = True
            return
        # reserve on every member first; any refusal retries the group next tick
        tickets = []
        try:
            for iid in sorted(missing):
                for rng in missing[iid]:
                    memory.restore_layers(self.instances[iid], rng, HOST, tid=self._next_tid())
                    tickets.append((iid, rng))
        except ValueError:
            for iid, rng in tickets:
                self.instances[iid].kv.release_reservation((rng[1] - rng[0]) *
                                                           self.model.bytes_per_layer)
                pool = self.instances[iid].pool
                if pool is not None:  # hand the vacated slabs back to the KV pool
                    pool.restore_complete(*rng)
                    pool.drop_layers(*rng)
            return
        grun.restoring = True
        self.log("RESTORE", group=gid, members=",".join(map(str, sorted(missing))))
        flat = {iid: rng for iid, rngs in missing.items() for rng in rngs}
        tasks = plan_restore_transfers(flat, holders, self.model.bytes_per_layer, chunk,
                                       tid_start=self._tid + 1)
        self._tid += len(tasks)
        self._on_params_planned(tasks, fetch=False, missing=missing, holders=holders, chunk=chunk)
        left: dict[int, int] = {}
        for t in tasks:
            left[t.dst] = left.get(t.dst, 0) + 1
        self._restore_left[gid] = left
        self._restore_ranges[gid] = missing
        for t in tasks:
            self.transition_tasks += 1
            self.enqueue_task(t, lambda task, when, g=gid: self._restore_chunk_done(g, task, when))

    def _restore_chunk_done(self, gid: int, task: TransferTask, when: int) -> None:
        self.transition_tasks -= 1
        left = self._restore_left[gid]
        left[task.dst] -= 1
        if left[task.dst] == 0:
            for rng in self._restore_ranges[gid][task.dst]:
                memory.complete_restore(self.instances[task.dst], rng)
            self.log("RESTORE_DONE", inst=task.dst)
        grun = self.groups.get(gid)
        if grun is None:
            return
        if all(v == 0 for v in left.values()):
            grun.params_restored = True
            if not grun.in_round:
                self._dissolve(grun)

    def _dissolve(self, grun: GroupRun) -> bool:
        """Back to singleton groups; split residents consolidate home (engine.py:1159-1209)."""
        gid = grun.group.gid
        old = dict(grun.group.stage_layer_map)
        members = list(grun.group.member_instances)
        residents, queued = sorted(grun.active), list(grun.queue)
        homes = self._plan_homes(grun)
        if homes is None:
            return False
        del self.groups[gid]
        L = self.model.num_layers
        for iid in members:
            self.groups[iid] = GroupRun(group=Group(gid=iid, member_instances=[iid],
                                                    stage_layer_map={iid: (0, L)}))
            self.group_of[iid] = iid
        self.log("DISSOLVE", gid=gid, members=",".join(map(str, members)))
        for rid in residents:
            req = self.requests[rid]
            home = homes[rid]
            req.home_instance = home
            self.groups[home].active.add(rid)
            self.groups[home].admit_order.append(rid)
            peers = {iid: share_bytes(req.context_len, *old[iid], L, self.model.kv_bytes_per_token)
                     for iid in members
                     if iid != home and self.instances[iid].kv.allocated_tokens.get(rid, 0) > 0}
            if not peers:
                continue
            if req.state is not RequestState.STALLED:
                self.resume_state[rid] = req.state
                req.set_state(RequestState.STALLED)
                self.log("STALL", req=rid)
            self.consolidating[rid] = {"home": home, "peers": peers, "started": False,
                                       "layers": {iid: old[iid] for iid in peers}}
        self._consolidation_retry()
        for rid in queued:
            self.dispatch(self.requests[rid])
        for iid in members:
            self.kick(iid)
        return True

    def _consolidation_retry(self) -> None:
        chunk = self._exchange_chunk_bytes()
        for rid in sorted(self.consolidating):
            st = self.consolidating[rid]
            if st["started"]:
                continue
            inst = self.instances[st["home"]]
            extra = self.total_alloc.get(rid, 0) - inst.kv.allocated_tokens.get(rid, 0)
            if extra > inst.kv.free_tokens:
                continue
            if extra:
                assert inst.kv.alloc(rid, extra)
            st["started"] = True
            st["left"] = 0
            for iid in sorted(st["peers"]):
                left = st["peers"][iid]
                tasks = []
                while left > 0:
                    take = min(chunk, left)
                    left -= take
                    tasks.append(TransferTask(self._next_tid(), TaskKind.KVCACHE_CHUNK, iid,
                                              st["home"], take, rid=rid))
                self._on_consolidation_planned(rid, iid, st["home"], st["layers"][iid], tasks)
                for task in tasks:
                    st["left"] += 1
                    self.transition_tasks += 1
                    self.enqueue_task(task, lambda t, when, r=rid:
                                      self._consolidate_chunk_done(r, t, when))

    def _consolidate_chunk_done(self, rid: int, task: TransferTask, when: int) -> None:
        self.transition_tasks -= 1
        st = self.consolidating[rid]
        st["left"] -= 1
        if st["left"] > 0:
            return
        self._on_consolidated(rid, sorted(st["peers"]))
        for iid in sorted(st["peers"]):
            self.instances[iid].kv.free(rid)
        del self.consolidating[rid]
        self.requests[rid].set_state(self.resume_state.pop(rid, RequestState.DECODING))
        self.log("RESUME", req=rid)
        self.kick(self.group_of[st["home"]])

    # ------------------------------------------------------------- failures
    def schedule_failure(self, iid: int, at_us: int) -> None:
        """Inject the failure of instance `iid` at `at_us` (see fail_instance)."""
        self.evq.push(at_us, lambda: self._try_fail(iid))

    def _try_fail(self, iid: int) -> None:
        # a drop / exchange / restore in flight finishes first (its tasks
        # name the instance); the failure lands at the next monitor tick
        if self.transition_tasks > 0:
            self.evq.push(self.now + self.monitor.tick_us, lambda: self._try_fail(iid))
            return
        self.fail_instance(iid)

    def fail_instance(self, iid: int) -> None:
        """Fault injection and failure restore (B200 addition).

        The reference carries Instance.failed (core.py:188) and leaves failed
        instances out of its capacity sums (engine.py:242-254) but never sets
        it.  The paper's fault tolerance: a failed node
        disrupts the other members of its pipeline group, which are restored
        to full parameter copies -- from a surviving replica, or from the host
        copy (exchange.HOST, exchange.py:18, 224-233).  Here:
          * the instance leaves service (failed = True, no group);
          * its group's round in flight is abandoned and every resident of
            the group is evicted and re-queued (the KV slice the failed
            member held is gone: the request re-prefills, as after a
            recompute eviction, engine.py:_evict_one);
          * every surviving member becomes a singleton group, gated until it
            holds all layers again: the layers it lacks are pulled from the
            lowest-id live holder outside the failed set, else HOST
            (plan_restore_transfers; one plan per missing range, since a
            middle member of a PP-4 group misses two);
          * the evicted requests are dispatched again across live groups.
        """
        inst = self.instances[iid]
        if inst.failed:
            raise ValueError(f"instance {iid} already failed")
        inst.failed = True
        gid = self.group_of.pop(iid)
        grun = self.groups.pop(gid)
        self.log("FAIL", inst=iid, group=gid)
        grun.rstate = None
        grun.in_round = False
        for rid in sorted(grun.active):
            self._evict_one(grun, rid)
        requeue = list(grun.queue)
        L = self.model.num_layers
        survivors = [m for m in grun.group.member_instances if m != iid]
        live = [i for i in sorted(self.instances) if not self.instances[i].failed]
        holders = {i: self.instances[i].table.held_ranges() for i in live}
        missing = {}
        for m in survivors:
            self.groups[m] = GroupRun(group=Group(gid=m, member_instances=[m],
                                                  stage_layer_map={m: (0, L)}))
            self.group_of[m] = m
            need = member_moves(holders[m], (0, L))[1]
            if need:
                missing[m] = need
        for m in sorted(missing):
            for rng in missing[m]:
                memory.restore_layers(self.instances[m], rng, HOST, tid=self._next_tid())
        tasks = []
        for k in range(max((len(r) for r in missing.values()), default=0)):
            flat = {m: rngs[k] for m, rngs in missing.items() if len(rngs) > k}
            tasks += plan_restore_transfers(flat, holders, self.model.bytes_per_layer,
                                            self._exchange_chunk_bytes(),
                                            tid_start=self._tid + 1 + len(tasks))
        self._tid += len(tasks)
        if missing:
            self.log("RESTORE", group=gid, members=",".join(map(str, sorted(missing))))
        self._on_params_planned(tasks, fetch=False)
        left: dict[int, int] = {}
        for t in tasks:
            left[t.dst] = left.get(t.dst, 0) + 1
        for m in missing:
            self.fetch_gate[m] = left[m]
        self._failover = getattr(self, "_failover", {})
        self._failover.update({m: missing[m] for m in missing})
        for t in tasks:
            self.transition_tasks += 1
            self.enqueue_task(t, lambda task, when: self._failover_chunk_done(task, when))
        for rid in requeue:
            self.dispatch(self.requests[rid])
        for g in sorted(self.groups):
            self.kick(g)

    def _failover_chunk_done(self, task: TransferTask, when: int) -> None:
        self.transition_tasks -= 1
        m = task.dst
        self.fetch_gate[m] -= 1
        if self.fetch_gate[m] == 0:
            del self.fetch_gate[m]
            for rng in self._failover.pop(m):
                memory.complete_restore(self.instances[m], rng)
            self.log("RESTORE_DONE", inst=m)
            self.kick(m)

    # ------------------------------------------------------------------ run
    def run(self) -> SimResult:
        self.log("CONFIG", policy=self.policy, seed=self.seed, instances=len(self.instances),
                 layers=self.model.num_layers)
        for rid, rec in enumerate(self.trace):
            self.evq.push(rec.arrival_us, lambda rec=rec, rid=rid: self._arrive(rec, rid))
        self.evq.push(self.monitor.tick_us, self._tick)
        while len(self.evq) and self.evq.peek_time() <= self.horizon_us:
            t, _, fn = self.evq.pop()
            self.now = max(self.now, t)
            fn()
        done = sum(r.state is RequestState.FINISHED for r in self.requests.values())
        queued = sum(r.state is RequestState.QUEUED for r in self.requests.values())
        self.log("END", finished=done, queued=queued)
        return SimResult(self.requests, self.log_lines, self.now, self.drop_events,
                         self.evictions, self.fallbacks)


def run_sim(cfg: SimConfig, trace: list[TraceRecord], policy: Optional[str] = None,
            seed: int = 0) -> SimResult:
    return Engine(cfg, trace, policy=policy, seed=seed).run()
