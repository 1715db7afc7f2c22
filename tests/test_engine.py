"""Engine (pipeline-group scheduler) vs the reference's own event logs.

tests/golden/engine_logs.json holds complete run_sim logs produced by the
unmodified reference (tests/golden/make_golden.py); this engine must emit the
same lines, byte for byte, and end in the same memory state.  Plus the
reference's engine tests restated (pkg/tests/test_engine.py).
"""

import random

import pytest

from conftest import load_golden
from paper_2412_18169_b200.config import SimConfig
from paper_2412_18169_b200.engine import Engine, run_sim
from paper_2412_18169_b200.metrics import collect, parse_line, percentile
from paper_2412_18169_b200.traceio import TraceRecord, synth_burst


def cfg_for(run):
    cfg = SimConfig()
    cfg.cluster.instances = run["cluster"]["instances"]
    cfg.cluster.hbm_bytes = run["cluster"]["hbm_bytes"]
    cfg.policy.kind = run["policy"]
    return cfg


def state_of(inst):
    t, kv = inst.table, inst.kv
    return {"extent": t.kvcache_virtual_extent, "capacity": kv.capacity_tokens,
            "used": kv.used_tokens, "free": kv.free_tokens, "reserved": kv.reserved_bytes,
            "held": t.layers_held(), "held_ranges": [list(r) for r in t.held_ranges()],
            "alloc": {str(k): v for k, v in sorted(kv.allocated_tokens.items())}}


@pytest.mark.parametrize("name", ["single_request", "drop_cycle_2x", "two_burst", "fallback_1x",
                                  "burst_short", "unequal_merge"])
def test_engine_log_matches_reference_byte_for_byte(name):
    run = next(r for r in load_golden("engine_logs.json") if r["name"] == name)
    trace = [TraceRecord(*r) for r in run["trace"]]
    eng = Engine(cfg_for(run), trace, policy=run["policy"], seed=0)
    res = eng.run()
    for i, (got, want) in enumerate(zip(res.log_lines, run["log"])):
        assert got == want, f"line {i}: {got!r} != {want!r}"
    assert len(res.log_lines) == len(run["log"])
    assert (res.end_us, res.drop_events, res.evictions, res.fallbacks) == \
        (run["end_us"], run["drop_events"], run["evictions"], run["fallbacks"])
    assert {str(i): state_of(inst) for i, inst in eng.instances.items()} == run["final"]


def small_cfg(instances=2, hbm=16_800_000_000):
    cfg = SimConfig()
    cfg.cluster.instances = instances
    cfg.cluster.hbm_bytes = hbm
    return cfg


def events(lines, kind):
    return [(t, f) for t, k, f in map(parse_line, lines) if k == kind]


def test_single_request_timeline():
    res = run_sim(SimConfig(), [TraceRecord(0, 100, 3)], policy="kunserve")
    assert events(res.log_lines, "FIRST_TOKEN") == [(9913, {"req": "0", "ttft_us": "9913"})]
    assert [(t, f["n"]) for t, f in events(res.log_lines, "TOKEN")] == \
        [(9913 + 9603, "2"), (9913 + 2 * 9603, "3")]


def test_kunserve_cycle_counts_and_clean_end():
    trace = [TraceRecord(0, 2500, 50) for _ in range(4)]
    eng = Engine(small_cfg(), trace, policy="kunserve")
    res = eng.run()
    count = lambda k: len(events(res.log_lines, k))  # noqa: E731
    assert (count("PLAN"), count("DROP"), count("REMAP"), count("EXCHANGE"), count("STALL"),
            count("RESUME"), count("RESTORE_DONE"), count("DISSOLVE")) == (1, 2, 2, 2, 2, 2, 2, 1)
    for inst in eng.instances.values():
        assert inst.table.layers_held() == list(range(8))
        assert inst.kv.allocated_tokens == {} and inst.kv.reserved_bytes == 0
    assert eng.transition_tasks == 0 and res.evictions == 0


def test_lifecycle_invariants_random_traces():
    for pol in ("kunserve", "recompute", "swap", "migrate"):
        rng = random.Random(hash(pol) % 97)
        t, trace = 0, []
        for _ in range(10):
            t += rng.randrange(0, 300_000)
            trace.append(TraceRecord(t, rng.randrange(300, 3200), rng.randrange(1, 30)))
        eng = Engine(small_cfg(), trace, policy=pol)
        res = eng.run()
        assert len(events(res.log_lines, "FINISH")) == len(trace)
        times = [parse_line(l)[0] for l in res.log_lines]
        assert times == sorted(times)
        if pol == "kunserve":
            assert res.evictions == 0


def test_p99_ttft_ordering_on_reference_burst():
    """Acceptance criterion 4 of the reference (tests/test_acceptance.py:146-163)."""
    trace = synth_burst(30.0, 2.0, 12.0, 8.0, 20.0, 600, 120, seed=3)
    rows = {}
    for pol in ("kunserve", "recompute", "swap", "migrate"):
        cfg = small_cfg(instances=4)
        cfg.policy.kind = pol
        st = collect(run_sim(cfg, trace).log_lines)
        assert st.finished() == len(trace)
        rows[pol] = percentile(st.ttfts(), 99)
    best_baseline = min(rows[p] for p in ("recompute", "swap", "migrate"))
    assert best_baseline / rows["kunserve"] >= 5.0
