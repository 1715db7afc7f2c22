"""The CPU oracle (oracle/) against brute force and the reference's outputs."""

import random

import numpy as np

from conftest import load_golden
from oracle import dropsim_port as ds
from oracle.attention import bf16_to_f32, check_close, decode_ref, f32_to_bf16, prefill_ref
from oracle.kvpool import (RESERVED, OraclePool, bf16_bits_to_f16_bits, copy_pages, gather_kv,
                           kv_append)


def make_pool(track=False):
    # tiny model: 2 layers, 2 MiB slabs (64 pages of 32 KiB), 96 head pages
    return OraclePool(num_layers=2, slab_bytes=2 << 20, page_bytes=32768, head_pages=96,
                      max_slots=8, max_pages_per_seq=256, track_bytes=track)


def test_grow_takes_lowest_free_pages_in_request_order():
    p = make_pool()
    assert p.grow([(0, 0, 2, 3), (1, 1, 2, 2)])
    assert p.bt[(0, 0)] == [0, 1, 2] and p.bt[(0, 1)] == [3, 4, 5] and p.bt[(1, 1)] == [6, 7]
    p.release([0], 0, 1)
    assert p.grow([(2, 0, 1, 4)])
    assert p.bt[(2, 0)] == [0, 1, 2, 8]
    assert p.owner[8] == p.cell(2, 0, 3)


def test_held_slabs_are_reserved_and_refuse_growth():
    p = make_pool()
    assert p.owner_array()[96] == RESERVED and p.bitmap()[96]
    assert not p.grow([(0, 0, 2, 49)])  # 98 pages > 96 head pages
    assert p.live_pages == 0 and not p.bt


def test_drop_opens_the_layer_slab():
    p = make_pool()
    p.drop(1, 2)                           # slab of layer 1 = pages 160..223
    assert p.usable_pages == 96 + 64
    assert p.grow([(0, 0, 1, 100)])
    assert p.bt[(0, 0)][95:] == [95, 160, 161, 162, 163]


def test_restore_compacts_the_slab_into_lowest_free():
    p = make_pool()
    p.drop(0, 2)
    assert p.grow([(0, 0, 1, 120)])        # 0..95, 96..119 (layer 0's slab)
    assert p.grow([(1, 0, 1, 10)])         # 120..129
    p.release([0], 0, 1)
    moved = p.restore(0, 1)                # vacate 96..159: live 120..129
    assert moved == 10 and p.bt[(1, 0)] == list(range(10))
    assert p.reserved[96:160].all()


def test_restore_refuses_when_live_pages_cannot_fit():
    p = make_pool()
    p.drop(1, 2)
    assert p.grow([(0, 0, 1, 150)])
    assert p.restore(1, 2) == -1
    assert not p.reserved[160:].any()


def test_random_ops_keep_invariants():
    rng = random.Random(5)
    p = make_pool()
    dropped = set()
    for _ in range(600):
        op = rng.random()
        if op < 0.5:
            slot = rng.randrange(8)
            lo = rng.randrange(2)
            hi = rng.randrange(lo + 1, 3)
            if all(p.npages(slot, l) + 4 <= 256 for l in range(lo, hi)):
                p.grow([(slot, lo, hi, rng.randrange(1, 4))])
        elif op < 0.8:
            p.release([rng.randrange(8)], 0, 2)
        elif op < 0.9:
            l = rng.randrange(2)
            if l not in dropped:
                p.drop(l, l + 1)
                dropped.add(l)
        elif dropped:
            l = rng.choice(sorted(dropped))
            if p.restore(l, l + 1) >= 0:
                dropped.discard(l)
        live = set(np.flatnonzero(p.live).tolist())
        in_tables = [pg for row in p.bt.values() for pg in row]
        assert sorted(in_tables) == sorted(live)            # no leak, no double use
        assert not (p.live & p.reserved).any()              # never on live weights
        for pg in live:
            sl, idx = divmod(p.owner[pg], p.max_pages_per_seq)
            slot, layer = divmod(sl, p.num_layers)
            assert p.bt[(slot, layer)][idx] == pg


def test_copy_and_append_roundtrip_bytes():
    a, b = make_pool(True), make_pool(True)
    a.grow([(0, 0, 2, 2)])
    b.grow([(3, 0, 2, 2)])
    rng = np.random.default_rng(0)
    k = rng.integers(0, 65535, size=(100, 1, 128), dtype=np.uint16)
    v = rng.integers(0, 65535, size=(100, 1, 128), dtype=np.uint16)
    kv_append(a, 1, k, v, [0] * 100, list(range(100)), n_kv_heads=1, block_tokens=64)
    copy_pages(b, a, [(0, 3, 0, 2, 2, 0, 4)])
    k2, v2 = gather_kv(b, 3, 1, 100, 1, 64)
    assert (k2 == k).all() and (v2 == bf16_bits_to_f16_bits(v)).all()


def test_v_cache_fp16_is_exact_for_bf16_activations():
    # every bf16 value in fp16's normal range converts exactly
    x = (np.random.default_rng(2).standard_normal(4096) * 8).astype(np.float32)
    bits = f32_to_bf16(x)
    f16 = bf16_bits_to_f16_bits(bits).view(np.float16).astype(np.float32)
    assert (f16 == bf16_to_f32(bits)).all()


def test_attention_refs_agree_with_each_other():
    rng = np.random.default_rng(1)
    ctx, hq, hkv = 77, 8, 2
    q = rng.standard_normal((1, hq, 128)).astype(np.float32)
    k = rng.standard_normal((ctx, hkv, 128)).astype(np.float32)
    v = rng.standard_normal((ctx, hkv, 128)).astype(np.float32)
    d = decode_ref(q[0], k, v, 0.088)
    p = prefill_ref(q, k, v, ctx - 1, 0.088)
    assert np.allclose(d, p[0], atol=1e-5)


def test_bf16_helpers_and_tolerance():
    x = np.array([1.0, -2.5, 3.14159, 1e-3], dtype=np.float32)
    back = bf16_to_f32(f32_to_bf16(x))
    assert np.allclose(back, x, rtol=1e-2)
    assert check_close(back, back) == (0.0, 0.0)


# --- the oracle's port of the reference control plane vs the reference's outputs

def test_dropsim_port_matches_reference_goldens():
    for n, lo, hi, L, want in load_golden("stage_share.json"):
        assert ds.stage_share(n, lo, hi, L) == want
    pl = load_golden("planner.json")
    for p_, f, k, want in pl["demand"]:
        assert ds.compute_demand(p_, f, k) == want
    L_of = {"small": 8, "tiny": 2, "llama3_8b": 32, "qwen25_14b": 48}
    P_of = {"small": 16_000_000_000, "tiny": 2 * 2_097_152, "llama3_8b": 32 * 438_304_768,
            "qwen25_14b": 48 * 551_550_976}
    for rec in pl["plans"]:
        groups = [(g["gid"], {int(i): tuple(g["map"][str(i)]) for i in g["members"]})
                  for g in rec["groups"]]
        merges, freed, fb, ops = ds.plan_drop(groups, rec["demand"], L_of[rec["model"]],
                                              P_of[rec["model"]])
        assert (freed, fb, ops) == (rec["freed"], rec["fallback"], rec["heap_ops"])
        assert [(a, b, g, list(m)) for a, b, g, m, _ in merges] == \
            [(m["gid_a"], m["gid_b"], m["gid"], m["members"]) for m in rec["merges"]]
    for rec in pl["member_moves"]:
        d, f = ds.member_moves([tuple(h) for h in rec["held"]], tuple(rec["target"]))
        assert [list(x) for x in d] == rec["drops"] and [list(x) for x in f] == rec["fetches"]
    ex = load_golden("exchange.json")
    for tok, lo, hi, L, kv, want in ex["share_bytes"]:
        assert ds.share_bytes(tok, lo, hi, L, kv) == want
    for rec in ex["plan_exchange"]:
        got = ds.plan_exchange({int(k): v for k, v in rec["reqs"].items()},
                               {int(k): tuple(v) for k, v in rec["old"].items()},
                               {int(k): tuple(v) for k, v in rec["new"].items()},
                               rec["L"], rec["kv"], rec["chunk"], rec["tid0"])
        want = [[t[0], t[2], t[3], t[4], t[5], t[7]] for t in rec["tasks"]]
        assert got == want
    for rec in ex["plan_restore"]:
        got = ds.plan_restore_transfers({int(k): tuple(v) for k, v in rec["missing"].items()},
                                        {int(k): [tuple(r) for r in v]
                                         for k, v in rec["holders"].items()},
                                        rec["bpl"], rec["chunk"], 3)
        want = [[t[0], t[2], t[3], t[4], tuple(t[6])] for t in rec["tasks"]]
        assert got == want
