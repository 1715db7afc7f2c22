"""Failure injection and failure restore in model mode (engine.Engine).

The reference keeps Instance.failed (core.py:188) and leaves failed
instances out of its capacity sums (engine.py:242-254) but never sets it;
the paper restores the pipeline-group members a failure disrupts from a
surviving replica or the host copy (exchange.HOST,
exchange.py:18, 224-233).  Engine.fail_instance implements that; the GPU
variant (tests/test_device_scenarios.py) byte-checks the restored slabs.
"""

from paper_2412_18169_b200.config import SimConfig
from paper_2412_18169_b200.engine import Engine
from paper_2412_18169_b200.exchange import HOST
from paper_2412_18169_b200.metrics import collect, parse_line
from paper_2412_18169_b200.traceio import TraceRecord


def run(instances, fail_at=50_000, fail=1):
    cfg = SimConfig()
    cfg.cluster.instances = instances
    cfg.cluster.hbm_bytes = 40_000_000_000
    cfg.cluster.initial_group_size = 2          # start as PP-2 groups
    trace = [TraceRecord(1000 * i, 2500, 50) for i in range(6)]
    eng = Engine(cfg, trace, seed=0)
    eng.schedule_failure(fail, fail_at)
    return eng, eng.run()


def test_failure_restores_survivor_from_host_when_no_replica_lives():
    eng, res = run(2)
    lines = [parse_line(l) for l in res.log_lines]
    fail_t = next(t for t, k, f in lines if k == "FAIL")
    pulls = [f for t, k, f in lines if k == "XFER" and f["task"] == "param_shard" and t > fail_t]
    assert pulls and all(int(f["src"]) == HOST and f["dst"] == "0" for f in pulls)
    assert sum(int(f["bytes"]) for f in pulls) == 4 * eng.model.bytes_per_layer
    assert eng.instances[1].failed and 1 not in eng.group_of
    assert eng.instances[0].table.layers_held() == list(range(8))
    # every request is served by the survivor; none by the failed instance
    st = collect(res.log_lines)
    assert st.finished() == 6
    assert all(int(f["inst"]) == 0 for t, k, f in lines if k == "DISPATCH" and t >= fail_t)
    assert eng.groups[0].group.member_instances == [0]
    done_t = next(t for t, k, f in lines if k == "RESTORE_DONE" and f["inst"] == "0")
    assert all(t >= done_t for t, k, f in lines if k == "STAGE" and t > fail_t)


def test_failure_restores_from_the_lowest_live_holder():
    eng, res = run(4)
    lines = [parse_line(l) for l in res.log_lines]
    fail_t = next(t for t, k, f in lines if k == "FAIL")
    pulls = [f for t, k, f in lines if k == "XFER" and f["task"] == "param_shard"
             and f["dst"] == "0" and t > fail_t]
    # layers 4..8 live on instance 3 (group {2, 3} holds 2:(0,4), 3:(4,8))
    assert pulls and {f["src"] for f in pulls} == {"3"}
    assert collect(res.log_lines).finished() == 6
    assert all(not i.failed for k, i in eng.instances.items() if k != 1)
