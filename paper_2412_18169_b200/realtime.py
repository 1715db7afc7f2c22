"""Wall-clock serving: the reference's scheduler running in real time on B200.

serving.DeviceEngine executes every stage on the device but keeps the
reference's discrete-event clock: stage durations are measured one by one,
then fed to the simulated timeline, and links stay on the link model
(exchange.py:49-101).  WallClockEngine removes the simulation:

  * time is the host's wall clock (perf_counter, us since the run started);
    arrivals fire when the wall clock reaches the trace's arrival time, the
    monitor ticks every monitor_tick_us of wall time (engine.py:520-567);
  * every pipeline stage (engine.py:410-426) is LAUNCHED on its instance's
    own CUDA stream when its input is ready and COMPLETES when the GPU says
    so: the stage's STAGE start / end and every FIRST_TOKEN / TOKEN time are
    CUDA-event timestamps on the device (converted to the run's clock
    through a reference event recorded at t = 0).  Instances sharing a GPU
    run their stages concurrently, as separate GPUs would;
  * the ACTIVATION hand-off (engine.py:428-455) is a real copy of the stage's
    output rows into the next stage's input buffer, on the transfer engine's
    high-priority stream; the next stage starts when that copy's event fires;
  * KV chunks and parameter shards start on the device as soon as the engine
    enqueues them (the low-priority bulk stream is the link: it serializes
    them in FIFO order) and their callbacks fire when their events complete
    -- no link model, no bandwidth assumption;
  * decode-only microbatches replay CUDA graphs padded to power-of-two
    batch buckets, captured before the clock starts.

Every scheduling decision is still the reference's (engine.Engine's code);
only time and execution are real.  The event log keeps the reference's
format, so metrics.collect / percentile / bubble_ratio read it unchanged.
"""

from __future__ import annotations

import gc
import heapq
import time
from typing import Optional

from . import runtime
from .core import Microbatch, RequestState
from .exchange import TaskKind
from .serving import DeviceEngine


class WallClockEngine(DeviceEngine):
    clock = "wall"

    def __init__(self, cfg, trace, policy: Optional[str] = None, seed: int = 0,
                 runtimes: Optional[dict] = None, max_seqs: Optional[int] = None,
                 graph_buckets=(1, 2, 4, 8, 16, 32, 64), precapture_depths=(1, 2),
                 poll_sleep_s: float = 20e-6):
        super().__init__(cfg, trace, policy=policy, seed=seed, runtimes=runtimes,
                         max_seqs=max_seqs)
        torch = self.torch
        self.te.timing = True             # start / end events on every transfer
        self.page_stream = self.te.meta   # grows / releases off the bulk stream
        self.compute = {iid: torch.cuda.Stream(device=self._dev_of(iid)) for iid in self.pools}
        self.poll_sleep_s = poll_sleep_s
        self.buckets = tuple(sorted(graph_buckets))
        self.inflight: list = []          # (event, callback) in launch order
        self._act_tasks: dict = {}        # (gid, rnd, k, s) -> ACTIVATION task after stage s
        self._act_key = None              # the hand-off _stage_done is about to enqueue
        self.stage_launches = 0
        # host time split of the loop (seconds): stage launches, device
        # callbacks, timed events, idle sleeps
        self.host_prof = {"launch": 0.0, "callbacks": 0.0, "events": 0.0, "idle": 0.0}
        L = self.model.num_layers
        # dummy slot per pool for padded decode rows: one page per layer
        self.dummy = {}
        for iid, pool in self.pools.items():
            st = self.slots[iid]
            slot = st._free.pop(0)        # the highest slot id, never handed out
            self.dummy[iid] = slot
            assert pool.grow([(slot, 0, L, 1)])
        # capture the padded decode graphs of every stage range a group of
        # depth d in precapture_depths can assign (plan_drop's even split,
        # planner.py:65-114), so the clock never waits for a capture
        for iid, runner in self.runners.items():
            for d in precapture_depths:
                cuts = [j * L // d for j in range(d + 1)]
                for lo, hi in zip(cuts, cuts[1:]):
                    with torch.cuda.stream(self.compute[iid]):
                        for n in self.buckets:
                            runner.capture_padded(lo, hi, n, self.dummy[iid])
        torch.cuda.synchronize()

    # ------------------------------------------------------------ clock
    def _wall_us(self) -> int:
        return int((time.perf_counter() - self._t0) * 1e6)

    def _dev_us(self, ev, dev: int) -> int:
        """Device timestamp (us on the run's clock) of a completed CUDA event
        recorded on device `dev`."""
        return int(round(self._t0_ev[dev].elapsed_time(ev) * 1000))

    # ------------------------------------------------------------ stages
    def _stage_times(self, grun, mbs, spans) -> list:
        # nothing is measured ahead: stages run when they are launched
        return [[0] * len(mbs) for _ in spans]

    def _bucket(self, n: int) -> Optional[int]:
        for b in self.buckets:
            if b >= n:
                return b
        return None

    def _to_device(self, xs, dtype, dev):
        """Index lists staged through pinned memory and copied asynchronously
        on the current (stage) stream: a pageable H2D copy would block the
        host until that stream drained."""
        t = self.torch.tensor(xs, dtype=dtype, pin_memory=True)
        return t.to(dev, non_blocking=True)

    def _try_start_stage(self, gid: int, s: int) -> None:
        """The base engine calls this for stage 0 when a round forms and for
        stage s+1 when a hand-off lands (engine.py:410-455).  Here the whole
        round is launched at once when it forms: every microbatch's stage
        chain is queued on the device with event dependencies (stage s on
        its instance's stream -> hand-off copy on the priority stream ->
        stage s+1 on the next instance's stream), so no host round trip sits
        between a stage and its successor.  The host only observes the
        completions, in causal order, and runs the reference's callbacks on
        them; the later calls are bookkeeping."""
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None:
            return
        rs = grun.rstate
        if s == 0:
            t_host = time.perf_counter()
            while rs.next_k[0] < len(rs.mbs):
                k = rs.next_k[0]
                rs.next_k[0] += 1
                self._launch_chain(gid, grun, rs, k)
            self.host_prof["launch"] += time.perf_counter() - t_host
        else:
            while rs.next_k[s] < len(rs.mbs) and rs.act_ready[s][rs.next_k[s]] is not None:
                rs.next_k[s] += 1

    def _stage_batch(self, iid: int, mb, n_pad: Optional[int]) -> dict:
        """The microbatch's index vectors for member iid, all int32 lists
        packed into ONE pinned tensor and one async H2D copy on the current
        stream (decode rows padded to n_pad with the dummy slot)."""
        torch = self.torch
        dev = self._dev_of(iid)
        of = self.slots[iid].of
        pre = [ch for ch in mb.chunks if not ch.decode]
        dec = [ch for ch in mb.chunks if ch.decode]
        slots, pos, p_slots, p_off, p_len, p_prefix, last = [], [], [], [], [], [], []
        row = 0
        for ch in pre:
            c, p = ch.token_count, ch.prefix_len
            slots += [of[ch.rid]] * c
            pos += range(p, p + c)
            p_off.append(row)
            p_slots.append(of[ch.rid])
            p_len.append(c)
            p_prefix.append(p)
            row += c
            last.append(row - 1)
        npr = row
        d_slots = [of[ch.rid] for ch in dec]
        d_ctx = [ch.prefix_len for ch in dec]
        last += range(npr, npr + len(dec))
        n = npr + len(dec)
        if n_pad is not None:
            extra = n_pad - n
            d_slots += [self.dummy[iid]] * extra
            d_ctx += [1] * extra
        slots += d_slots
        pos += [c - 1 for c in d_ctx]
        parts = [slots, pos, p_slots, p_off, p_len, p_prefix, d_slots, d_ctx, last]
        flat = torch.tensor([v for part in parts for v in part], dtype=torch.int32,
                            pin_memory=True).to(f"cuda:{dev}", non_blocking=True)
        views, at = [], 0
        for part in parts:
            views.append(flat[at:at + len(part)])
            at += len(part)
        (slots_t, pos_t, p_slots_t, p_off_t, p_len_t, p_prefix_t, d_slots_t, d_ctx_t, last_t) = views
        nd = len(d_slots)
        return {"n": n, "slots": slots_t, "pos": pos_t, "n_prefill_rows": npr, "np": len(pre),
                "p_slots": p_slots_t, "p_off": p_off_t, "p_len": p_len_t, "p_prefix": p_prefix_t,
                "p_max": max(p_len, default=0),
                "p_kv_max": max((a + b for a, b in zip(p_prefix, p_len)), default=0),
                "nd": nd, "d_slots": d_slots_t, "d_ctx": d_ctx_t,
                "d_max": max(d_ctx, default=0), "last": last_t.long(),
                "units": sum(ch.token_count * ch.prefix_len + (ch.token_count ** 2 +
                                                              ch.token_count) / 2 for ch in pre)}

    def _launch_chain(self, gid: int, grun, rs, k: int) -> None:
        torch = self.torch
        mb = rs.mbs[k]
        S = len(rs.members)
        prev = None  # (output rows, end event) of the previous stage
        for s, iid in enumerate(rs.members):
            lo, hi = grun.group.stage_layer_map[iid]
            dev = self._dev_of(iid)
            cs = self.compute[iid]
            runner = self.runners[iid]
            decode_only = all(ch.decode for ch in mb.chunks)
            n = sum(ch.token_count for ch in mb.chunks)
            n_pad = self._bucket(n) if decode_only else None
            if n_pad is not None and (lo, hi, n_pad) not in getattr(runner, "_graphs", {}):
                n_pad = None
            with torch.cuda.device(dev):
                if s > 0:
                    # the hand-off (ACTIVATION task, engine.py:428-448): stage
                    # s-1's rows into this instance's input, on the priority
                    # stream, after stage s-1 ends
                    src, e_prev = prev
                    urgent = self.te.urgent
                    with torch.cuda.stream(urgent):
                        urgent.wait_event(e_prev)
                        x = torch.empty_like(src, device=f"cuda:{dev}")
                        ca = torch.cuda.Event(enable_timing=True)
                        ce = torch.cuda.Event(enable_timing=True)
                        ca.record(urgent)
                        runtime.copy_bytes(x.data_ptr(), src.data_ptr(),
                                           src.numel() * src.element_size(), stream=urgent)
                        ce.record(urgent)
                    src.record_stream(urgent)
                    self.inflight.append((ce, lambda s=s, ca=ca, ce=ce, dev=dev:
                                          self._act_copied(gid, rs.no, k, s - 1, ca, ce, dev)))
                with torch.cuda.stream(cs):
                    b = self._stage_batch(iid, mb, n_pad)
                    if s == 0:
                        ids = torch.randint(0, self.shape.vocab, (n,), device=f"cuda:{dev}")
                        x = self.emb[dev].index_select(0, ids)
                    else:
                        cs.wait_event(ce)
                        x.record_stream(cs)
                    a = torch.cuda.Event(enable_timing=True)
                    e = torch.cuda.Event(enable_timing=True)
                    a.record(cs)
                    if n_pad is not None:
                        y = runner.run_padded_decode(lo, hi, x, dict(b, n=n_pad, nd=n_pad), n_pad)
                    else:
                        y = runner.run(lo, hi, x, b)
                    if s == S - 1 and b["last"].numel():  # sample each sequence's next token
                        (y.index_select(0, b["last"]) @ self.emb[dev].t()).argmax(dim=-1)
                    e.record(cs)
            self.stage_launches += 1
            meta = (n, b["units"], len([c for c in mb.chunks if c.decode]), hi - lo)
            self.inflight.append((e, lambda s=s, iid=iid, a=a, e=e, meta=meta:
                                  self._stage_finished(gid, rs.no, k, s, iid, a, e, meta)))
            prev = (y, e)

    def _stage_finished(self, gid, rnd, k, s, iid, a, e, meta) -> None:
        dev = self._dev_of(iid)
        start, end = self._dev_us(a, dev), self._dev_us(e, dev)
        n, units, nd, layers = meta
        self.stage_samples.append((n, units, nd, layers, max(1, end - start)))
        self.pools[iid].check_kv_range(synchronize=False)
        self._act_key = (gid, rnd, k, s)
        try:
            self._stage_done(gid, rnd, k, s, start, end)
        finally:
            self._act_key = None

    def _complete_microbatch(self, grun, mb, when) -> None:
        """A request the monitor stalled or moved while its round ran on
        the device (a KV exchange, swap-out, migration or consolidation
        planned at a tick mid-round) gets no credit for that round's chunk:
        its KV is moving, and it runs the step again after RESUME (the append
        rewrites the same position) -- in its new group if it migrated, so a
        chunk counts only while the request is still one of this group's.
        The reference's event clock never changes a request inside its own
        round; without this a stalled request whose last token lands would
        go STALLED -> FINISHED (illegal, core.py), and a migrated one would
        be finished against its old group's allocation."""
        keep = [ch for ch in mb.chunks
                if self.requests[ch.rid].state is not RequestState.STALLED
                and ch.rid in grun.active]
        if len(keep) != len(mb.chunks):
            mb = Microbatch(mb.mbid, keep)
        super()._complete_microbatch(grun, mb, when)

    def _act_copied(self, gid, rnd, k, s, ca, ce, dev) -> None:
        """The hand-off after stage s of microbatch k landed: the reference's
        _xfer_done for its ACTIVATION task (XFER line, then the callback
        that marks stage s+1's input ready)."""
        got = self._act_tasks.pop((gid, rnd, k, s), None)
        if got is None:
            return   # the round went stale before the task was enqueued
        self._task_finished(got, ca, ce, dev)

    # ------------------------------------------------------------ transfers
    def _pump(self, link) -> None:
        """Start every queued task now (priority order): the device's
        streams are the link -- activations on the high-priority stream,
        KV / parameter tasks FIFO on the bulk stream."""
        while link.pending:
            task = heapq.heappop(link.pending)[3]
            self._start_task(link, task)

    def _start_task(self, link, task) -> None:
        torch = self.torch
        if task.kind is TaskKind.ACTIVATION:
            # launched with the round's stage chain (_launch_chain); its
            # completion callback (_act_copied) finishes the task
            self._act_tasks[self._act_key] = task
            return
        self._run_task(task)   # DeviceEngine: te.submit on the bulk stream
        p = self.te.pending[-1]
        dev = self._dev_of(task.dst if task.dst >= 0 else task.src)
        self.inflight.append((p.event, lambda: self._task_finished(task, p.start_event, p.event,
                                                                    dev)))

    def _task_finished(self, task, a, e, dev: int) -> None:
        self.te.poll()   # FIFO bulk stream: every earlier transfer landed too
        start, done = self._dev_us(a, dev), self._dev_us(e, dev)
        self.log("XFER", task=task.kind.value, src=task.src, dst=task.dst,
                 bytes=task.size_bytes, start=start,
                 rid=task.rid if task.rid is not None else -1)
        cb = self._task_cb.pop(task.tid, None)
        if cb is not None:
            cb(task, done)

    def _transfers_landed(self) -> None:
        self.te.poll()

    # ------------------------------------------------------------ loop
    def _poll(self) -> bool:
        """Fire the callbacks of completed device work; True if any fired.
        Only the work in flight when the poll starts: a callback launches the
        next stage, and if that one completed before the scan reached it the
        scan would go on firing a fast model's decode chain for a whole
        request, starving the arrivals and monitor ticks due meanwhile."""
        fired = False
        i = 0
        n = len(self.inflight)
        t0 = time.perf_counter()
        while i < n:
            ev, fn = self.inflight[i]
            if ev.query():
                self.inflight.pop(i)
                n -= 1
                self.now = max(self.now, self._wall_us())
                fn()
                fired = True
            else:
                i += 1
        if fired:
            self.host_prof["callbacks"] += time.perf_counter() - t0
        return fired

    def _settled(self) -> bool:
        if self.inflight or self._arrivals_left:
            return False
        if any(r.state is not RequestState.FINISHED for r in self.requests.values()):
            return False
        if self.policy == "kunserve":
            return (self.transition_tasks == 0 and not self.consolidating and
                    all(g.group.size == 1 for g in self.groups.values()))
        return True

    def run(self):
        torch = self.torch
        self.log("CONFIG", policy=self.policy, seed=self.seed, instances=len(self.instances),
                 layers=self.model.num_layers)
        self._arrivals_left = len(self.trace)

        def arrive(rec, rid):
            self._arrivals_left -= 1
            self._arrive(rec, rid)
        for rid, rec in enumerate(self.trace):
            self.evq.push(rec.arrival_us, lambda rec=rec, rid=rid: arrive(rec, rid))
        self.evq.push(self.monitor.tick_us, self._tick)
        torch.cuda.synchronize()
        # t = 0: one reference event per device, host and device aligned
        self._t0_ev = {}
        for d in sorted({self._dev_of(i) for i in self.pools}):
            with torch.cuda.device(d):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                ev.synchronize()
                self._t0_ev[d] = ev
        self._t0 = time.perf_counter()
        gc.collect()
        gc.disable()
        try:
            while True:
                fired = self._poll()
                w = self._wall_us()
                if len(self.evq) and self.evq.peek_time() <= w:
                    t, _, fn = self.evq.pop()
                    self.now = max(self.now, t)
                    t1 = time.perf_counter()
                    fn()
                    self.host_prof["events"] += time.perf_counter() - t1
                    continue
                if w > self.horizon_us or self._settled():
                    break
                if not fired:
                    nxt = self.evq.peek_time() - w if len(self.evq) else 1000
                    t1 = time.perf_counter()
                    time.sleep(min(max(nxt, 0) / 1e6, self.poll_sleep_s))
                    self.host_prof["idle"] += time.perf_counter() - t1
        finally:
            gc.enable()
        torch.cuda.synchronize()
        self.now = max(self.now, self._wall_us())
        done = sum(r.state is RequestState.FINISHED for r in self.requests.values())
        queued = sum(r.state is RequestState.QUEUED for r in self.requests.values())
        self.log("END", finished=done, queued=queued)
        from .engine import SimResult
        return SimResult(self.requests, self.log_lines, self.now, self.drop_events,
                         self.evictions, self.fallbacks)
