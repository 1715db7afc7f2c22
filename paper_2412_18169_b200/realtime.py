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
from .core import RequestState
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
        self.stage_out: dict = {}         # (gid, rnd, k, s) -> output rows of stage s
        self.act_in: dict = {}            # (gid, rnd, k, s) -> input rows of stage s
        self._act_key = None              # the hand-off _stage_done is about to enqueue
        self._xfer_ev: dict = {}          # tid -> pending device transfer
        self.stage_launches = 0
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
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None:
            return
        rs = grun.rstate
        while rs.next_k[s] < len(rs.mbs):
            k = rs.next_k[s]
            if rs.act_ready[s][k] is None:
                return
            rs.next_k[s] += 1
            self._launch_stage(gid, grun, rs, s, k)

    def _launch_stage(self, gid: int, grun, rs, s: int, k: int) -> None:
        torch = self.torch
        iid = rs.members[s]
        lo, hi = grun.group.stage_layer_map[iid]
        dev = self._dev_of(iid)
        cs = self.compute[iid]
        runner = self.runners[iid]
        last = s == len(rs.members) - 1
        with torch.cuda.device(dev), torch.cuda.stream(cs):
            b = self._batch(iid, rs.mbs[k])
            if s == 0:
                ids = torch.randint(0, self.shape.vocab, (b["n"],), device=f"cuda:{dev}")
                x = self.emb[dev].index_select(0, ids)
            else:
                x = self.act_in.pop((gid, rs.no, k, s))
                x.record_stream(cs)
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record(cs)
            n_pad = self._bucket(b["n"]) if b["np"] == 0 else None
            if n_pad is not None and (lo, hi, n_pad) not in getattr(runner, "_graphs", {}):
                n_pad = None
            if n_pad is not None:
                y = runner.run_padded_decode(lo, hi, x, runner.padded_batch(b, n_pad,
                                                                            self.dummy[iid]),
                                             n_pad)
            else:
                y = runner.run(lo, hi, x, b)
            if last and b["last"].numel():  # sample the next token of each sequence
                (y.index_select(0, b["last"]) @ self.emb[dev].t()).argmax(dim=-1)
            e.record(cs)
        self.stage_launches += 1
        if not last:
            self.stage_out[(gid, rs.no, k, s)] = y
        meta = (b["n"], b["units"], b["nd"], hi - lo)
        self.inflight.append((e, lambda: self._stage_finished(gid, rs.no, k, s, iid, a, e, meta)))

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
            self.stage_out.pop((gid, rnd, k, s), None)

    def _act_arrived(self, gid: int, rnd: int, k: int, s: int, when: int) -> None:
        grun = self.groups.get(gid)
        if grun is None or grun.rstate is None or grun.rstate.no != rnd:
            self.act_in.pop((gid, rnd, k, s), None)   # the round went stale
            return
        super()._act_arrived(gid, rnd, k, s, when)

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
            gid, rnd, k, s = self._act_key
            src = self.stage_out.pop((gid, rnd, k, s))
            dst_dev = self._dev_of(task.dst)
            urgent = self.te.urgent
            with torch.cuda.device(dst_dev), torch.cuda.stream(urgent):
                dst = torch.empty_like(src, device=f"cuda:{dst_dev}")
                a = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                a.record(urgent)
                runtime.copy_bytes(dst.data_ptr(), src.data_ptr(),
                                   src.numel() * src.element_size(), stream=urgent)
                e.record(urgent)
            src.record_stream(urgent)
            self.act_in[(gid, rnd, k, s + 1)] = dst
            self.inflight.append((e, lambda: self._task_finished(task, a, e, dst_dev)))
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
        """Fire the callbacks of completed device work; True if any fired."""
        fired = False
        i = 0
        while i < len(self.inflight):
            ev, fn = self.inflight[i]
            if ev.query():
                self.inflight.pop(i)
                self.now = max(self.now, self._wall_us())
                fn()
                fired = True
            else:
                i += 1
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
                    fn()
                    continue
                if w > self.horizon_us or self._settled():
                    break
                if not fired:
                    nxt = self.evq.peek_time() - w if len(self.evq) else 1000
                    time.sleep(min(max(nxt, 0) / 1e6, self.poll_sleep_s))
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
