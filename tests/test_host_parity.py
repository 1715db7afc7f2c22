"""Host control plane vs golden fixtures produced by the reference itself.

Fixtures: tests/golden/*.json, written by tests/golden/make_golden.py from
the unmodified reference (pkg/src/dropsim).  Every record replays the same
calls on this package and must match value for value, error text for error
text.
"""

import pytest

from paper_2412_18169_b200 import memory
from paper_2412_18169_b200.core import Group, ModelSpec
from paper_2412_18169_b200.exchange import (HOST, LinkModel, TaskKind, TransferTask,
                                            finish_link, plan_exchange,
                                            plan_restore_transfers, schedule_link,
                                            share_bytes)
from paper_2412_18169_b200.planner import compute_demand, member_moves, plan_drop

from conftest import load_golden

MODELS = {
    "small": dict(num_layers=8, bytes_per_layer=2_000_000_000, kv_bytes_per_token=200_000),
    "tiny": dict(num_layers=2, bytes_per_layer=2_097_152, kv_bytes_per_token=1_024,
                 hidden_bytes_per_token=512),
    "llama3_8b": dict(num_layers=32, bytes_per_layer=438_304_768,
                      kv_bytes_per_token=131_072, hidden_bytes_per_token=8_192),
    "qwen25_14b": dict(num_layers=48, bytes_per_layer=551_550_976,
                       kv_bytes_per_token=196_608, hidden_bytes_per_token=10_240),
}


def state_of(inst):
    t, kv = inst.table, inst.kv
    return {"extent": t.kvcache_virtual_extent, "capacity": kv.capacity_tokens,
            "used": kv.used_tokens, "free": kv.free_tokens,
            "reserved": kv.reserved_bytes, "held": t.layers_held(),
            "held_ranges": [list(r) for r in t.held_ranges()],
            "alloc": {str(k): v for k, v in sorted(kv.allocated_tokens.items())}}


def replay_memory_op(inst, op):
    kind = op["op"]
    if kind == "drop":
        return memory.drop_layers(inst, tuple(op["range"]))
    if kind == "drop_group":
        L = inst.table.model.num_layers
        cut = op["stage"][1]
        g = Group(gid=0, member_instances=[0, 1], stage_layer_map={0: (0, cut), 1: (cut, L)})
        return memory.drop_layers(inst, tuple(op["range"]), g)
    if kind == "restore":
        t = memory.restore_layers(inst, tuple(op["range"]), source=1, tid=9)
        return [t.tid, t.kind.value, t.src, t.dst, t.size_bytes, list(t.layers)]
    if kind == "complete":
        return memory.complete_restore(inst, tuple(op["range"]))
    if kind == "alloc":
        return inst.kv.alloc(op["rid"], op["n"])
    if kind == "free":
        return inst.kv.free(op["rid"])
    if kind == "shrink":
        return inst.kv.shrink(op["rid"], op["n"])
    if kind == "reserve":
        return inst.kv.reserve(op["n"])
    if kind == "release":
        return inst.kv.release_reservation(op["n"])
    raise AssertionError(kind)


def test_memory_op_sequences_match_reference():
    data = load_golden("memory_ops.json")
    n = 0
    for seq in data["sequences"]:
        model = ModelSpec(**MODELS[seq["model"]])
        inst = memory.build_instance(0, model, seq["hbm"], 25_000_000_000)
        assert state_of(inst) == seq["init"]
        for op in seq["ops"]:
            try:
                ret = replay_memory_op(inst, op)
                assert "err" not in op, (op, ret)
                assert ret == op["ret"], op
            except ValueError as exc:
                assert op.get("err") == str(exc), (op, str(exc))
            assert state_of(inst) == op["state"], op
            n += 1
    assert n >= 1000
    for rec in data["build_errors"]:
        with pytest.raises(ValueError) as ei:
            memory.build_instance(3, ModelSpec(**MODELS[rec["model"]]), rec["hbm"], 1)
        assert str(ei.value) == rec["err"]


def test_stage_share_matches_reference():
    for n, lo, hi, L, want in load_golden("stage_share.json"):
        assert memory.stage_share(n, lo, hi, L) == want


def test_compute_demand_matches_reference():
    for p, f, k, want in load_golden("planner.json")["demand"]:
        assert compute_demand(p, f, k) == want


def test_plan_drop_matches_reference():
    plans = load_golden("planner.json")["plans"]
    assert len(plans) >= 100
    for rec in plans:
        model = ModelSpec(**MODELS[rec["model"]])
        groups = [Group(gid=g["gid"], member_instances=g["members"],
                        stage_layer_map={int(k): tuple(v) for k, v in g["map"].items()})
                  for g in rec["groups"]]
        plan = plan_drop(groups, rec["demand"], model)
        assert plan.to_text() == rec["text"]
        assert plan.heap_ops == rec["heap_ops"]
        assert plan.fallback == rec["fallback"]
        assert plan.freed_bytes == rec["freed"]
        for m, gm in zip(plan.merges, rec["merges"]):
            assert (m.gid_a, m.gid_b, m.gid, list(m.members), m.freed_bytes) == \
                (gm["gid_a"], gm["gid_b"], gm["gid"], gm["members"], gm["freed"])
            assert {str(k): list(v) for k, v in m.stage_layer_map.items()} == gm["map"]


def test_member_moves_matches_reference():
    for rec in load_golden("planner.json")["member_moves"]:
        d, f = member_moves([tuple(h) for h in rec["held"]], tuple(rec["target"]))
        assert [list(x) for x in d] == rec["drops"]
        assert [list(x) for x in f] == rec["fetches"]


def task_json(t):
    return [t.tid, t.kind.value, t.src, t.dst, t.size_bytes, t.rid,
            list(t.layers) if t.layers else None, t.last_for_rid]


def test_share_bytes_matches_reference():
    for tok, lo, hi, L, kv, want in load_golden("exchange.json")["share_bytes"]:
        assert share_bytes(tok, lo, hi, L, kv) == want


def test_plan_exchange_matches_reference():
    for rec in load_golden("exchange.json")["plan_exchange"]:
        tasks = plan_exchange({int(k): v for k, v in rec["reqs"].items()},
                              {int(k): tuple(v) for k, v in rec["old"].items()},
                              {int(k): tuple(v) for k, v in rec["new"].items()},
                              rec["L"], rec["kv"], rec["chunk"], tid_start=rec["tid0"])
        assert [task_json(t) for t in tasks] == rec["tasks"]


def test_plan_restore_matches_reference():
    for rec in load_golden("exchange.json")["plan_restore"]:
        tasks = plan_restore_transfers(
            {int(k): tuple(v) for k, v in rec["missing"].items()},
            {int(k): [tuple(r) for r in v] for k, v in rec["holders"].items()},
            rec["bpl"], rec["chunk"], tid_start=3)
        assert [task_json(t) for t in tasks] == rec["tasks"]


def test_link_schedules_match_reference():
    import heapq
    for rec in load_golden("exchange.json")["links"]:
        link = LinkModel(0, 1, rec["bw"], rec["lat"])
        evq = []
        for t, tid, kind, size in rec["enqueue"]:
            heapq.heappush(evq, (t, tid, "enq", TransferTask(tid, TaskKind(kind), 0, 1, size)))
        seq, starts = 1000, []
        while evq:
            now, _, what, task = heapq.heappop(evq)
            if what == "enq":
                link.enqueue(task, now)
            else:
                finish_link(link, task)
            got = schedule_link(link, now)
            if got:
                nxt, start, done = got
                starts.append([nxt.tid, start, done])
                heapq.heappush(evq, (done, seq, "fin", nxt))
                seq += 1
        assert starts == rec["starts"]


# --- the reference's own known-answer tests, restated against this package ---

def test_known_answers_memory(small_model):
    inst = memory.build_instance(0, small_model, 24_000_000_000, 25_000_000_000)
    assert inst.table.kvcache_virtual_extent == 8_000_000_000
    assert inst.kv.capacity_tokens == 40_000
    assert memory.drop_layers(inst, (4, 8)) == 8_000_000_000
    assert inst.kv.capacity_tokens == 80_000
    snapshot = None
    inst2 = memory.build_instance(0, small_model, 24_000_000_000, 25_000_000_000)
    snapshot = [(b.size, b.owner, b.layer) for b in inst2.table.blocks]
    memory.drop_layers(inst2, (4, 8))
    t = memory.restore_layers(inst2, (4, 8), source=1, tid=7)
    assert (t.size_bytes, t.layers) == (8_000_000_000, (4, 8))
    memory.complete_restore(inst2, (4, 8))
    assert [(b.size, b.owner, b.layer) for b in inst2.table.blocks] == snapshot
    assert memory.stage_share(1001, 0, 4, 8) == 501


def test_known_answers_exchange_and_planner(small_model):
    assert compute_demand(5000, 80_000_000, 200_000) == 920_000_000
    assert share_bytes(1, 3, 8, 8, 100_001) == 62_501
    tasks = plan_exchange({7: 960}, {0: (0, 8)}, {0: (0, 4), 1: (4, 8)}, 8, 200_000, 40_000_000)
    assert [(t.src, t.dst, t.size_bytes) for t in tasks] == [
        (0, 1, 40_000_000), (0, 1, 40_000_000), (0, 1, 16_000_000)]
    tasks = plan_restore_transfers({2: (0, 8)}, {1: [(0, 4)], 2: [(4, 8)]}, 2_000_000_000, 10**12)
    assert [(t.src, t.dst, t.layers) for t in tasks] == [(1, 2, (0, 4)), (HOST, 2, (4, 8))]
    groups = [Group(0, [0, 1], {0: (0, 4), 1: (4, 8)}), Group(1, [2, 3], {2: (0, 4), 3: (4, 8)})]
    m = plan_drop(groups, 1, small_model).merges[0]
    assert m.members == (0, 2, 1, 3)
    assert m.stage_layer_map == {0: (0, 2), 2: (2, 4), 1: (4, 6), 3: (6, 8)}
