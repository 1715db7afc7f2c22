"""Generate golden fixtures by running the UNMODIFIED reference (dropsim).

Runs only in the build container, where /root/reference exists; the JSON it
writes is committed under tests/golden/ so the GPU box (which has no
/root/reference) can check parity against it.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is a list of (inputs, outputs) records produced by calling the
reference's public functions:
  memory_ops.json    build_instance / drop_layers / restore_layers /
                     complete_restore / KVAllocator op sequences
                     (pkg/src/dropsim/memory.py:70-222)
  planner.json       compute_demand / plan_drop / member_moves
                     (pkg/src/dropsim/planner.py:22-141)
  exchange.json      share_bytes / plan_exchange / plan_restore_transfers /
                     LinkModel schedules (pkg/src/dropsim/exchange.py:49-249)
  stage_share.json   stage_share (pkg/src/dropsim/memory.py:215-222)
  engine_logs.json   run_sim event logs (pkg/src/dropsim/engine.py:1258-1285)
"""

from __future__ import annotations

import heapq
import json
import os
import random
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from dropsim import memory  # noqa: E402
from dropsim.config import SimConfig  # noqa: E402
from dropsim.core import Group, ModelSpec  # noqa: E402
from dropsim.engine import Engine  # noqa: E402
from dropsim.exchange import (LinkModel, TaskKind, TransferTask,  # noqa: E402
                              finish_link, plan_exchange,
                              plan_restore_transfers, schedule_link,
                              share_bytes)
from dropsim.planner import compute_demand, member_moves, plan_drop  # noqa: E402
from dropsim.traceio import TraceRecord, synth_burst  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# Models the fixtures are generated on: the reference's own test model, the
# tiny config-1 model, and the two BASELINE models at 2 MiB slab rounding.
MODELS = {
    "small": dict(num_layers=8, bytes_per_layer=2_000_000_000,
                  kv_bytes_per_token=200_000),
    "tiny": dict(num_layers=2, bytes_per_layer=2_097_152,
                 kv_bytes_per_token=1_024, hidden_bytes_per_token=512),
    "llama3_8b": dict(num_layers=32, bytes_per_layer=438_304_768,
                      kv_bytes_per_token=131_072,
                      hidden_bytes_per_token=8_192),
    "qwen25_14b": dict(num_layers=48, bytes_per_layer=551_550_976,
                       kv_bytes_per_token=196_608,
                       hidden_bytes_per_token=10_240),
}


def state_of(inst):
    t, kv = inst.table, inst.kv
    return {
        "extent": t.kvcache_virtual_extent,
        "capacity": kv.capacity_tokens,
        "used": kv.used_tokens,
        "free": kv.free_tokens,
        "reserved": kv.reserved_bytes,
        "held": t.layers_held(),
        "held_ranges": [list(r) for r in t.held_ranges()],
        "alloc": {str(k): v for k, v in sorted(kv.allocated_tokens.items())},
    }


def gen_memory_ops():
    cases = []
    rng = random.Random(2412)
    for name, mkw in MODELS.items():
        model = ModelSpec(**mkw)
        L = model.num_layers
        for seq_no in range(6):
            hbm = model.param_bytes + rng.choice(
                [model.kv_bytes_per_token * rng.randrange(1, 400),
                 model.bytes_per_layer * rng.randrange(1, 4),
                 4 * 1024 * 1024])
            ops = []
            inst = memory.build_instance(0, model, hbm, 25_000_000_000)
            rec = {"model": name, "hbm": hbm, "init": state_of(inst), "ops": ops}
            for _ in range(60):
                kind = rng.choice(["drop", "drop", "restore", "complete",
                                   "alloc", "alloc", "alloc", "free", "shrink",
                                   "reserve", "release", "drop_group"])
                op = {"op": kind}
                try:
                    if kind in ("drop", "restore", "complete", "drop_group"):
                        lo = rng.randrange(0, L)
                        hi = rng.randrange(lo + 1, L + 1) if rng.random() < 0.9 else lo
                        op["range"] = [lo, hi]
                        if kind == "drop":
                            op["ret"] = memory.drop_layers(inst, (lo, hi))
                        elif kind == "drop_group":
                            cut = rng.randrange(1, L) if L > 1 else 1
                            smap = {0: (0, cut), 1: (cut, L)}
                            op["stage"] = [0, cut]
                            g = Group(gid=0, member_instances=[0, 1],
                                      stage_layer_map=smap)
                            op["ret"] = memory.drop_layers(inst, (lo, hi), g)
                        elif kind == "restore":
                            t = memory.restore_layers(inst, (lo, hi), source=1, tid=9)
                            op["ret"] = [t.tid, t.kind.value, t.src, t.dst,
                                         t.size_bytes, list(t.layers)]
                        else:
                            memory.complete_restore(inst, (lo, hi))
                            op["ret"] = None
                    elif kind == "alloc":
                        rid = rng.randrange(6)
                        n = rng.randrange(0, max(2, inst.kv.capacity_tokens // 3 + 2))
                        op["rid"], op["n"] = rid, n
                        op["ret"] = inst.kv.alloc(rid, n)
                    elif kind == "free":
                        rid = rng.randrange(6)
                        op["rid"] = rid
                        op["ret"] = inst.kv.free(rid)
                    elif kind == "shrink":
                        rid = rng.randrange(6)
                        cur = inst.kv.allocated_tokens.get(rid, 0)
                        n = rng.randrange(0, cur + 3)
                        op["rid"], op["n"] = rid, n
                        inst.kv.shrink(rid, n)
                        op["ret"] = None
                    elif kind == "reserve":
                        n = rng.randrange(0, model.bytes_per_layer * 2)
                        op["n"] = n
                        op["ret"] = inst.kv.reserve(n)
                    elif kind == "release":
                        n = rng.randrange(0, max(1, inst.kv.reserved_bytes + 2))
                        op["n"] = n
                        inst.kv.release_reservation(n)
                        op["ret"] = None
                except ValueError as exc:
                    op["err"] = str(exc)
                op["state"] = state_of(inst)
                ops.append(op)
            cases.append(rec)
    # undersized HBM refusal
    errs = []
    for name, mkw in MODELS.items():
        model = ModelSpec(**mkw)
        try:
            memory.build_instance(3, model, model.param_bytes, 1)
            errs.append({"model": name, "hbm": model.param_bytes, "err": None})
        except ValueError as exc:
            errs.append({"model": name, "hbm": model.param_bytes, "err": str(exc)})
    return {"sequences": cases, "build_errors": errs}


def gen_stage_share():
    rng = random.Random(7)
    out = []
    for _ in range(400):
        L = rng.choice([1, 2, 8, 32, 48])
        lo = rng.randrange(0, L)
        hi = rng.randrange(lo, L + 1)
        n = rng.randrange(0, 40_000)
        out.append([n, lo, hi, L, memory.stage_share(n, lo, hi, L)])
    return out


def group_to_json(g):
    return {"gid": g.gid, "members": list(g.member_instances),
            "map": {str(k): list(v) for k, v in g.stage_layer_map.items()}}


def gen_planner():
    rng = random.Random(99)
    demand_cases = []
    for _ in range(200):
        p = rng.randrange(0, 100_000)
        f = rng.randrange(0, 10**10)
        k = rng.choice([1, 1024, 131_072, 196_608, 200_000])
        demand_cases.append([p, f, k, compute_demand(p, f, k)])
    plans = []
    for name in ("small", "tiny", "llama3_8b", "qwen25_14b"):
        model = ModelSpec(**MODELS[name])
        L = model.num_layers
        for _ in range(40):
            # random partition of up to 8 instances into groups of 1,2,4 (even splits)
            n_inst = rng.randrange(1, 9)
            groups = []
            iid = 0
            while iid < n_inst:
                size = rng.choice([1, 1, 2, 4])
                size = min(size, n_inst - iid)
                while L % size and size > 1:
                    size -= 1
                members = list(range(iid, iid + size))
                bounds = [k * L // size for k in range(size + 1)]
                smap = {members[k]: (bounds[k], bounds[k + 1]) for k in range(size)}
                groups.append(Group(gid=iid, member_instances=members,
                                    stage_layer_map=smap))
                iid += size
            demand = rng.randrange(0, (n_inst + 1) * model.param_bytes)
            plan = plan_drop(groups, demand, model)
            plans.append({
                "model": name, "groups": [group_to_json(g) for g in groups],
                "demand": demand, "text": plan.to_text(),
                "heap_ops": plan.heap_ops, "fallback": plan.fallback,
                "freed": plan.freed_bytes,
                "merges": [{"gid_a": m.gid_a, "gid_b": m.gid_b, "gid": m.gid,
                            "members": list(m.members),
                            "map": {str(k): list(v) for k, v in m.stage_layer_map.items()},
                            "freed": m.freed_bytes} for m in plan.merges]})
    moves = []
    for _ in range(200):
        L = rng.choice([8, 32])
        held = []
        cur = 0
        while cur < L:
            a = rng.randrange(cur, L + 1)
            b = rng.randrange(a, L + 1)
            if b > a:
                held.append((a, b))
            cur = b + 1
        tlo = rng.randrange(0, L)
        thi = rng.randrange(tlo + 1, L + 1)
        d, f = member_moves(held, (tlo, thi))
        moves.append({"held": [list(h) for h in held], "target": [tlo, thi],
                      "drops": [list(x) for x in d], "fetches": [list(x) for x in f]})
    return {"demand": demand_cases, "plans": plans, "member_moves": moves}


def task_to_json(t):
    return [t.tid, t.kind.value, t.src, t.dst, t.size_bytes,
            t.rid, list(t.layers) if t.layers else None, t.last_for_rid]


def gen_exchange():
    rng = random.Random(5)
    shares = []
    for _ in range(300):
        L = rng.choice([2, 8, 32, 48])
        lo = rng.randrange(0, L)
        hi = rng.randrange(lo, L + 1)
        tok = rng.randrange(0, 9000)
        kv = rng.choice([1, 7, 1024, 131_072, 196_608, 200_000, 100_001])
        shares.append([tok, lo, hi, L, kv, share_bytes(tok, lo, hi, L, kv)])
    exch = []
    for _ in range(80):
        L = rng.choice([2, 8, 32, 48])
        kv = rng.choice([1024, 131_072, 196_608])
        sizes_old = rng.choice([1, 2])
        sizes_new = sizes_old * 2
        base = rng.randrange(0, 4) * 2
        def even(members):
            m = len(members)
            b = [k * L // m for k in range(m + 1)]
            return {members[k]: (b[k], b[k + 1]) for k in range(m)}
        old_members = list(range(base, base + sizes_old))
        new_members = sorted(old_members + [base + 10 + k for k in range(sizes_old)])
        old_map = even(old_members)
        new_map = even(new_members)
        reqs = {rng.randrange(0, 500): rng.randrange(1, 6000)
                for _ in range(rng.randrange(1, 8))}
        total = sum(reqs.values()) * kv
        floor = max(1, total // 400)  # keep task lists small
        chunk = max(floor, rng.choice([1, 1_000_000, 64 * 1024 * 1024, 10**12,
                                       rng.randrange(1, 50_000_000)]))
        tid0 = rng.randrange(0, 100)
        tasks = plan_exchange(reqs, old_map, new_map, L, kv, chunk, tid_start=tid0)
        exch.append({"reqs": {str(k): v for k, v in reqs.items()},
                     "old": {str(k): list(v) for k, v in old_map.items()},
                     "new": {str(k): list(v) for k, v in new_map.items()},
                     "L": L, "kv": kv, "chunk": chunk, "tid0": tid0,
                     "tasks": [task_to_json(t) for t in tasks]})
    restores = []
    for _ in range(80):
        L = rng.choice([8, 32, 48])
        n = rng.randrange(2, 6)
        holders = {}
        for i in range(n):
            lo = rng.randrange(0, L)
            hi = rng.randrange(lo, L + 1)
            holders[i] = [(lo, hi)] if hi > lo else []
        missing = {}
        for i in rng.sample(range(n), rng.randrange(1, n + 1)):
            lo = rng.randrange(0, L)
            hi = rng.randrange(lo + 1, L + 1)
            missing[i] = (lo, hi)
        bpl = rng.choice([2_097_152, 438_304_768, 551_550_976])
        chunk = max(bpl // 8, rng.choice([bpl, 256 * 1024 * 1024, 10**13,
                                          rng.randrange(1, 3 * bpl)]))
        tasks = plan_restore_transfers(missing, holders, bpl, chunk, tid_start=3)
        restores.append({"missing": {str(k): list(v) for k, v in missing.items()},
                         "holders": {str(k): [list(r) for r in v] for k, v in holders.items()},
                         "bpl": bpl, "chunk": chunk,
                         "tasks": [task_to_json(t) for t in tasks]})
    # link schedules (same driver shape as the reference acceptance test 6)
    links = []
    for _ in range(60):
        link = LinkModel(0, 1, rng.randrange(1, 41) * 1_000_000_000,
                         rng.randrange(0, 101))
        max_chunk = rng.randrange(1, 65) * 1_000_000
        chunk_time = link.transfer_time_us(max_chunk)
        evq, t, enq = [], 0, []
        for tid in range(rng.randrange(3, 26)):
            t += rng.randrange(0, 2 * chunk_time)
            kind = rng.choice([TaskKind.ACTIVATION, TaskKind.KVCACHE_CHUNK,
                               TaskKind.KVCACHE_CHUNK, TaskKind.PARAM_SHARD])
            size = rng.randrange(1, max_chunk + 1)
            enq.append([t, tid, kind.value, size])
            heapq.heappush(evq, (t, tid, "enq",
                                 TransferTask(tid, kind, 0, 1, size)))
        seq = 1000
        starts = []
        while evq:
            now, _, what, task = heapq.heappop(evq)
            if what == "enq":
                link.enqueue(task, now)
            else:
                finish_link(link, task)
            started = schedule_link(link, now)
            if started:
                nxt, start, done = started
                starts.append([nxt.tid, start, done])
                heapq.heappush(evq, (done, seq, "fin", nxt))
                seq += 1
        links.append({"bw": link.bandwidth, "lat": link.base_latency_us,
                      "enqueue": enq, "starts": starts})
    return {"share_bytes": shares, "plan_exchange": exch,
            "plan_restore": restores, "links": links}


def desk_cfg(policy, instances=4, hbm=16_800_000_000):
    cfg = SimConfig()
    cfg.cluster.instances = instances
    cfg.cluster.hbm_bytes = hbm
    cfg.policy.kind = policy
    return cfg


def gen_engine_logs():
    runs = []
    scenarios = [
        ("single_request", lambda: SimConfig(), [TraceRecord(0, 100, 3)], "kunserve"),
        ("drop_cycle_2x", lambda: desk_cfg("kunserve", 2),
         [TraceRecord(0, 2500, 50) for _ in range(4)], "kunserve"),
        ("two_burst", lambda: desk_cfg("kunserve"),
         [TraceRecord(1000 * i, 2500, 50) for i in range(8)]
         + [TraceRecord(20_000_000 + 1000 * i, 2500, 50) for i in range(8)],
         "kunserve"),
        ("fallback_1x", lambda: desk_cfg("kunserve", 1),
         [TraceRecord(0, 1900, 150), TraceRecord(0, 1900, 150)], "kunserve"),
        ("burst_short", lambda: desk_cfg("kunserve"),
         synth_burst(12.0, 2.0, 12.0, 3.0, 8.0, 600, 120, seed=3), "kunserve"),
        ("unequal_merge", lambda: desk_cfg("kunserve", 3),
         [TraceRecord(1000 * i, 2500, 40) for i in range(7)], "kunserve"),
    ]
    for name, mk, trace, pol in scenarios:
        cfg = mk()
        eng = Engine(cfg, trace, policy=pol, seed=0)
        res = eng.run()
        runs.append({
            "name": name, "policy": pol,
            "cluster": {"instances": cfg.cluster.instances,
                        "hbm_bytes": cfg.cluster.hbm_bytes},
            "trace": [[r.arrival_us, r.input_len, r.output_len] for r in trace],
            "log": res.log_lines, "end_us": res.end_us,
            "drop_events": res.drop_events, "evictions": res.evictions,
            "fallbacks": res.fallbacks,
            "final": {str(i): state_of(inst) for i, inst in eng.instances.items()},
        })
    return runs


def main():
    fixtures = {
        "memory_ops.json": gen_memory_ops(),
        "stage_share.json": gen_stage_share(),
        "planner.json": gen_planner(),
        "exchange.json": gen_exchange(),
        "engine_logs.json": gen_engine_logs(),
    }
    for fname, data in fixtures.items():
        path = os.path.join(OUT, fname)
        with open(path, "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(f"{fname}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
