"""The CPU oracle (oracle/) against brute force and the reference's counters."""

import random

import numpy as np

from oracle.attention import bf16_to_f32, check_close, decode_ref, f32_to_bf16, prefill_ref
from oracle.kvpool import OraclePool, copy_pages, gather_kv, kv_append


def make_pool(track=False):
    # tiny model: 2 layers, 2 MiB slabs, 32 KiB pages (64 tokens x 512 B)
    return OraclePool(num_layers=2, slab_bytes=2 << 20, page_bytes=32768, head_pages=96,
                      max_slots=8, max_pages_per_seq=64, track_bytes=track)


def test_grow_takes_lowest_free_pages_in_request_order():
    p = make_pool()
    assert p.grow([(0, 0, 2, 3), (1, 1, 2, 2)])
    assert p.bt[(0, 0)] == [0, 1, 2] and p.bt[(0, 1)] == [3, 4, 5] and p.bt[(1, 1)] == [6, 7]
    p.release([0], 0, 1)
    assert p.grow([(2, 0, 1, 4)])
    assert p.bt[(2, 0)] == [0, 1, 2, 8]
    assert p.owner[8] == p.cell(2, 0, 3)


def test_grow_refuses_without_changes():
    p = make_pool()
    assert not p.grow([(0, 0, 2, 49)])  # 98 pages > 96
    assert p.live_pages == 0 and not p.bt


def test_restore_compacts_tail_into_lowest_free():
    p = make_pool()
    p.drop(1)
    assert p.extent == 96 + 64
    assert p.grow([(0, 0, 1, 120)])        # spills into the dropped slab
    p.release([0], 0, 1)
    assert p.grow([(1, 0, 2, 50)])         # 100 pages: 0..99
    p.release([1], 0, 1)                   # frees 0..49
    moved = p.restore(1)                   # tail = pages 96..159
    assert moved == 4                      # live 96..99 move to 0..3
    assert p.bt[(1, 1)][-4:] == [0, 1, 2, 3]
    assert p.extent == 96


def test_restore_refuses_when_live_pages_cannot_fit():
    p = make_pool()
    p.drop(1)
    assert p.grow([(0, 0, 1, 150)])
    assert p.restore(1) == -1
    assert p.extent == 160


def test_random_ops_keep_invariants():
    rng = random.Random(5)
    p = make_pool()
    for _ in range(500):
        op = rng.random()
        if op < 0.5:
            slot = rng.randrange(8)
            lo = rng.randrange(2)
            hi = rng.randrange(lo + 1, 3)
            if all(p.npages(slot, l) + 4 <= 64 for l in range(lo, hi)):
                p.grow([(slot, lo, hi, rng.randrange(1, 4))])
        elif op < 0.8:
            p.release([rng.randrange(8)], 0, 2)
        elif op < 0.9 and p.extent < p.max_pages:
            p.drop(1)
        elif p.extent > 96:
            p.restore(1)
        live = set(np.flatnonzero(p.live).tolist())
        in_tables = [pg for row in p.bt.values() for pg in row]
        assert sorted(in_tables) == sorted(live)          # no leak, no double use
        assert all(pg < p.extent for pg in live)
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
    assert (k2 == k).all() and (v2 == v).all()


def test_attention_refs_agree_with_each_other():
    rng = np.random.default_rng(1)
    ctx, hq, hkv = 77, 8, 2
    q = rng.standard_normal((1, hq, 128)).astype(np.float32)
    k = rng.standard_normal((ctx, hkv, 128)).astype(np.float32)
    v = rng.standard_normal((ctx, hkv, 128)).astype(np.float32)
    # decoding the last token == last row of a prefill over the whole context
    d = decode_ref(q[0], k, v, 0.088)
    p = prefill_ref(q, k, v, ctx - 1, 0.088)
    assert np.allclose(d, p[0], atol=1e-5)


def test_bf16_helpers_and_tolerance():
    x = np.array([1.0, -2.5, 3.14159, 1e-3], dtype=np.float32)
    back = bf16_to_f32(f32_to_bf16(x))
    assert np.allclose(back, x, rtol=1e-2)
    assert check_close(back, back) == (0.0, 0.0)
