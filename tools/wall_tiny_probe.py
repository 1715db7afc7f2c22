"""Where does the wall-clock engine's host loop spend its time on the tiny
model (tests/test_device_engine.py's kunserve-wall scenario)?  Prints the
event-kind counts, the OCC lines, and the slowest host calls (event
handlers and device-completion callbacks) with their wall time."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2412_18169_b200 import build  # noqa: E402

build.build()
from paper_2412_18169_b200.core import SHAPES  # noqa: E402
from paper_2412_18169_b200.metrics import parse_line  # noqa: E402
from paper_2412_18169_b200.realtime import WallClockEngine  # noqa: E402
from paper_2412_18169_b200.serving import device_config  # noqa: E402
from paper_2412_18169_b200.traceio import TraceRecord  # noqa: E402

slow = []
popped = []


class Probe(WallClockEngine):
    def _poll(self):
        fired = False
        i = 0
        while i < len(self.inflight):
            ev, fn = self.inflight[i]
            if ev.query():
                self.inflight.pop(i)
                self.now = max(self.now, self._wall_us())
                t = time.perf_counter()
                fn()
                d = time.perf_counter() - t
                if d > 0.005:
                    slow.append((round(d * 1e3, 1), "cb", getattr(fn, "__qualname__", str(fn)),
                                 self._wall_us()))
                fired = True
            else:
                i += 1
        return fired


def main():
    shape = SHAPES["tiny"]
    cfg = device_config(shape, instances=2, kv_bytes=1 << 20)
    cfg.policy.kind = sys.argv[1] if len(sys.argv) > 1 else "kunserve"
    cfg.policy.min_batch_tokens = 256
    cfg.policy.monitor_tick_us = 20_000
    trace = [TraceRecord(2000 * i, 250, 600) for i in range(32)]
    t0 = time.perf_counter()
    eng = Probe(cfg, trace)
    print("init_s", round(time.perf_counter() - t0, 2), flush=True)
    pop = eng.evq.pop

    def timed_pop():
        t, seq, fn = pop()
        if len(popped) < 400:
            popped.append((t, eng._wall_us(), getattr(fn, "__qualname__", str(fn))[-40:]))

        def wrapped(fn=fn):
            a = time.perf_counter()
            fn()
            d = time.perf_counter() - a
            if d > 0.005:
                slow.append((round(d * 1e3, 1), "ev", getattr(fn, "__qualname__", str(fn)),
                             eng._wall_us()))
        return t, seq, wrapped
    eng.evq.pop = timed_pop
    t0 = time.perf_counter()
    res = eng.run()
    print("run_s", round(time.perf_counter() - t0, 2))
    kinds = {}
    for line in res.log_lines:
        k = parse_line(line)[1]
        kinds[k] = kinds.get(k, 0) + 1
    print(json.dumps(kinds))
    print("host_prof", json.dumps({k: round(v, 3) for k, v in eng.host_prof.items()}))
    occ = [l for l in res.log_lines if " OCC " in l]
    print("OCC", len(occ), occ[:12])
    for s in sorted(slow, reverse=True)[:25]:
        print("slow", s)
    print("popped (t, wall, fn) first 60:", popped[:60])
    print("popped 200-260:", popped[200:260])
    first = [l for l in res.log_lines if any(k in l for k in ("ADMIT", "FIRST_TOKEN", "FINISH"))]
    print("timeline", first[:10], first[-5:])


if __name__ == "__main__":
    main()
