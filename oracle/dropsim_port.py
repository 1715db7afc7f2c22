"""ORACLE -- plain restatement of the reference's control-plane algorithms.
TEST INFRASTRUCTURE / CPU BASELINE ONLY (tests/, smoke(), bench.py's
cpu_baseline and --impl reference legs).

Each function restates one reference function (file:line under
/root/reference/pkg/src/dropsim/) as directly as possible; tests/test_oracle.py
pins every one of them against tests/golden/*.json, which
tests/golden/make_golden.py produced by running the reference itself.
"""

from __future__ import annotations

import heapq

HOST = -1  # exchange.py:18


def stage_share(n, lo, hi, L):                     # memory.py:215-222
    return -((-n * (hi - lo)) // L)


def compute_demand(pending, free, kvbpt):          # planner.py:22-32
    if pending < 0 or free < 0:
        raise ValueError("demand inputs must be >= 0")
    return max(0, pending * kvbpt - free)


def plan_drop(groups, demand, L, param_bytes):     # planner.py:65-114
    """groups: list of (gid, {iid: (lo, hi)}) with members in pipeline order.
    Returns (merges, freed, fallback, heap_ops); merges are
    (gid_a, gid_b, gid, members, {iid: (lo, hi)})."""
    if demand < 0:
        raise ValueError("demand must be >= 0")
    if demand == 0:
        return [], 0, False, 0
    heap = [(len(m), gid) for gid, m in groups]
    heapq.heapify(heap)
    ops = len(heap)
    live = {gid: [(m[i][0], i, m[i][1]) for i in m] for gid, m in groups}
    merges, freed = [], 0
    while freed < demand and len(heap) >= 2:
        _, a = heapq.heappop(heap)
        _, b = heapq.heappop(heap)
        ops += 2
        mem = sorted(live.pop(a) + live.pop(b))
        k = len(mem)
        bounds = [j * L // k for j in range(k + 1)]
        smap = {mem[j][1]: (bounds[j], bounds[j + 1]) for j in range(k)}
        gid = min(a, b)
        merges.append((a, b, gid, tuple(x[1] for x in mem), smap))
        freed += param_bytes
        live[gid] = [(smap[x[1]][0], x[1], smap[x[1]][1]) for x in mem]
        heapq.heappush(heap, (k, gid))
        ops += 1
    return merges, freed, freed < demand, ops


def _ranges(layers):
    out = []
    for l in sorted(layers):
        if out and out[-1][1] == l:
            out[-1] = (out[-1][0], l + 1)
        else:
            out.append((l, l + 1))
    return out


def member_moves(held, target):                    # planner.py:117-141
    h = {l for a, b in held for l in range(a, b)}
    t = set(range(target[0], target[1]))
    return _ranges(h - t), _ranges(t - h)


def share_bytes(tokens, lo, hi, L, kvbpt):         # exchange.py:125-137
    total = tokens * kvbpt
    return total * hi // L - total * lo // L


def plan_exchange(req_tokens, old_map, new_map, L, kvbpt, chunk, tid0=0):  # exchange.py:146-205
    """-> list of [tid, src, dst, bytes, rid, last_for_rid]."""
    if chunk < 1:
        raise ValueError("chunk_bytes must be >= 1")
    flows = []
    tid = tid0
    for rid in sorted(req_tokens):
        for s in sorted(old_map):
            for d in sorted(new_map):
                if s == d:
                    continue
                lo = max(old_map[s][0], new_map[d][0])
                hi = min(old_map[s][1], new_map[d][1])
                if hi <= lo:
                    continue
                b = share_bytes(req_tokens[rid], lo, hi, L, kvbpt)
                if b <= 0:
                    continue
                ch = []
                while b > 0:
                    take = min(chunk, b)
                    ch.append([tid, s, d, take, rid, False])
                    tid += 1
                    b -= take
                flows.append(ch)
    out = []
    i = 0
    while any(i < len(f) for f in flows):
        for f in flows:
            if i < len(f):
                out.append(f[i])
        i += 1
    last = {}
    for t in out:
        last[t[4]] = t
    for t in last.values():
        t[5] = True
    return out


def plan_restore_transfers(missing, holders, bpl, chunk, tid0=0):  # exchange.py:208-249
    """-> list of [tid, src, dst, bytes, (lo, hi)]."""
    out = []
    tid = tid0
    for tgt in sorted(missing):
        lo, hi = missing[tgt]
        src = {}
        for l in range(lo, hi):
            src[l] = HOST
            for h in sorted(holders):
                if h != tgt and any(a <= l < b for a, b in holders[h]):
                    src[l] = h
                    break
        a = lo
        while a < hi:
            b = a
            while b < hi and src[b] == src[a]:
                b += 1
            left = (b - a) * bpl
            while left > 0:
                take = min(chunk, left)
                out.append([tid, src[a], tgt, take, (a, b)])
                tid += 1
                left -= take
            a = b
    return out
