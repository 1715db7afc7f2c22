"""GPU parity: device pool, block tables, copies and attention vs the CPU oracle.

Bit-exact for block tables, bitmaps, owners and every copied byte; attention
within BASELINE.json's bf16 tolerance (max-abs <= 2e-2, mean-rel <= 1e-3)
against the fp32 oracle rounded to bf16 (the kernels emit bf16).
"""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.attention import bf16_to_f32, check_close, decode_ref, f32_to_bf16, prefill_ref  # noqa: E402
from oracle.kvpool import OraclePool, bf16_bits_to_f16_bits  # noqa: E402

from paper_2412_18169_b200.core import SHAPES, ModelShape  # noqa: E402

TINY = SHAPES["tiny"]
MIB = 1 << 20


@pytest.fixture(scope="module")
def rt():
    from paper_2412_18169_b200 import build
    build.build()
    from paper_2412_18169_b200 import runtime
    assert torch.cuda.is_available()
    return runtime.Runtime(0, max_slots=16, max_pages_per_seq=256, slack_pages=128)


def oracle_for(pool):
    inf = pool.info()
    return OraclePool(num_layers=pool.model.num_layers, slab_bytes=pool.model.bytes_per_layer,
                      page_bytes=pool.page_bytes, head_pages=inf.extent_pages,
                      max_slots=pool.rt.max_slots, max_pages_per_seq=pool.rt.max_pages_per_seq)


def assert_same_state(pool, orc, slots):
    inf = pool.info()
    assert inf.max_pages == orc.max_pages
    assert inf.extent_pages == orc.usable_pages
    assert inf.live_pages == orc.live_pages
    assert (pool.bitmap() == orc.bitmap()).all()
    assert (pool.owners() == orc.owner_array()).all()
    for s in slots:
        for l in range(orc.num_layers):
            assert pool.block_table(s, l) == orc.bt.get((s, l), []), (s, l)


def test_pool_ops_match_oracle_bit_exact(rt):
    from paper_2412_18169_b200 import runtime
    model = TINY.spec()
    pool = rt.create_pool(0, model, model.param_bytes + MIB, TINY)
    orc = oracle_for(pool)
    rng = random.Random(17)
    slots = list(range(rt.max_slots))
    dropped = set()
    for step in range(300):
        r = rng.random()
        if r < 0.45:
            reqs, used = [], set()
            for _ in range(rng.randrange(1, 4)):
                s = rng.choice(slots)
                lo = rng.randrange(0, 2)
                hi = rng.randrange(lo + 1, 3)
                add = rng.randrange(1, 9)
                cells = {(s, l) for l in range(lo, hi)}
                if cells & used or any(orc.npages(s, l) + add > rt.max_pages_per_seq
                                       for l in range(lo, hi)):
                    continue
                used |= cells
                reqs.append((s, lo, hi, add))
            ok_dev = pool.grow(reqs)
            ok_orc = orc.grow(reqs)
            assert ok_dev == ok_orc
        elif r < 0.75:
            s = rng.sample(slots, rng.randrange(1, 4))
            lo = rng.randrange(0, 2)
            hi = rng.randrange(lo + 1, 3)
            pool.release(s, lo, hi)
            orc.release(s, lo, hi)
        elif r < 0.87:
            l = rng.randrange(2)
            if l not in dropped:
                pool.drop_layers(l, l + 1)
                orc.drop(l, l + 1)
                dropped.add(l)
        elif dropped:
            l = rng.choice(sorted(dropped))
            want = orc.restore(l, l + 1)
            if want < 0:
                with pytest.raises(runtime.Refused):
                    pool.restore_begin(l, l + 1)
            else:
                pool.restore_begin(l, l + 1)
                assert pool.last_moved_pages == want
                pool.restore_complete(l, l + 1)
                dropped.discard(l)
        assert_same_state(pool, orc, slots)
    pool.close()


def device_gather(pool, slot, layer, ctx, hkv, B):
    kv = pool.kv_bytes().cpu().numpy()
    pb = pool.page_bytes
    rows = pool.block_table(slot, layer)
    k = np.zeros((ctx, hkv, 128), dtype=np.uint16)
    v = np.zeros_like(k)
    for t in range(ctx):
        base = rows[t // B] * pb
        for h in range(hkv):
            off = base + (h * B + t % B) * 256
            k[t, h] = kv[off:off + 256].view(np.uint16)
            v[t, h] = kv[off + pb // 2:off + pb // 2 + 256].view(np.uint16)
    return k, v


def rand_bf16(shape, gen, scale=1.0):
    return (torch.randn(shape, generator=gen) * scale).to(torch.bfloat16)


def append(pool, layer, k, v, slot, start):
    from paper_2412_18169_b200 import runtime
    n = k.shape[0]
    slots = torch.full((n,), slot, dtype=torch.int32, device="cuda")
    pos = torch.arange(start, start + n, dtype=torch.int32, device="cuda")
    runtime.kv_append(pool, layer, k.cuda(), v.cuda(), slots, pos)


def test_append_exchange_compaction_bytes(rt):
    from paper_2412_18169_b200 import runtime
    model = TINY.spec()
    a = rt.create_pool(0, model, model.param_bytes + MIB, TINY)
    b = rt.create_pool(1, model, model.param_bytes + MIB, TINY)
    gen = torch.Generator().manual_seed(3)
    ctx = 300
    pages = (ctx + 63) // 64
    # filler request so the request of interest spills into a dropped slab
    a.drop_layers(1, 2)
    assert a.grow([(5, 0, 1, 190)])
    assert a.grow([(2, 0, 1, pages)])
    k = rand_bf16((ctx, 1, 128), gen)
    v = rand_bf16((ctx, 1, 128), gen)
    append(a, 0, k, v, 2, 0)
    torch.cuda.synchronize()
    kk, vv = device_gather(a, 2, 0, ctx, 1, 64)
    assert (kk == k.view(torch.int16).numpy().view(np.uint16)).all()
    # the V cache is fp16 (exact conversion of the bf16 activations)
    assert (vv == bf16_bits_to_f16_bits(v.view(torch.int16).numpy().view(np.uint16))).all()
    assert max(a.block_table(2, 0)) >= 256  # lives in layer 1's dropped slab (pages 256..319)
    # exchange a -> b (two chunks), byte exact
    assert b.grow([(7, 0, 1, pages)])
    runtime.copy_pages(b, a, [(2, 7, 0, 1, pages, 0, 2), (2, 7, 0, 1, pages, 2, pages)])
    torch.cuda.synchronize()
    kb_, vb_ = device_gather(b, 7, 0, ctx, 1, 64)
    assert (kb_ == kk).all() and (vb_ == vv).all()
    # restore on a: the filler leaves, compaction moves request 2's tail pages
    a.release([5], 0, 1)
    a.restore_begin(1, 2)
    assert a.last_moved_pages > 0
    a.restore_complete(1, 2)
    assert max(a.block_table(2, 0)) < 192
    kc, vc = device_gather(a, 2, 0, ctx, 1, 64)
    assert (kc == kk).all() and (vc == vv).all()
    a.close()
    b.close()


def test_cross_stream_ordering_without_host_sync(rt):
    """The pool orders its own operations on the device (kb_pool.cu
    pool_enter / pool_meta_begin): grows, appends, drops, releases and a
    compaction issued on three streams with no host synchronization give
    the same block tables and bytes as the serialized run."""
    from paper_2412_18169_b200 import runtime
    model = TINY.spec()
    a = rt.create_pool(0, model, model.param_bytes + MIB, TINY)
    b = rt.create_pool(1, model, model.param_bytes + MIB, TINY)
    orc = oracle_for(a)
    gen = torch.Generator().manual_seed(5)
    ctx = 300
    pages = (ctx + 63) // 64
    k = rand_bf16((ctx, 1, 128), gen).cuda()
    v = rand_bf16((ctx, 1, 128), gen).cuda()
    slots_t = torch.full((ctx,), 2, dtype=torch.int32, device="cuda")
    pos_t = torch.arange(ctx, dtype=torch.int32, device="cuda")
    big = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
    big2 = torch.empty_like(big)
    torch.cuda.synchronize()
    s1, s2, s3 = (torch.cuda.Stream() for _ in range(3))
    # s1 is busy for a while: everything it queues lands late
    for _ in range(4):
        runtime.copy_bytes(big2.data_ptr(), big.data_ptr(), big.numel(), stream=s1)
    a.drop_layers(1, 2)
    assert a.grow([(5, 0, 1, 190)], stream=s1)
    assert a.grow([(2, 0, 1, pages)], stream=s1)
    runtime.kv_append(a, 0, k, v, slots_t, pos_t, stream=s2)  # after the grows
    assert b.grow([(7, 0, 1, pages)], stream=s3)
    s3.wait_stream(s2)  # data -> data dependencies stay the caller's
    runtime.copy_pages(b, a, [(2, 7, 0, 1, pages, 0, pages)], stream=s3)
    a.release([5], 0, 1, stream=s1)      # after every stream's reader
    a.restore_begin(1, 2, stream=s2)     # compaction after the release
    orc.drop(1, 2)
    assert orc.grow([(5, 0, 1, 190)]) and orc.grow([(2, 0, 1, pages)])
    orc.release([5], 0, 1)
    assert orc.restore(1, 2) == a.last_moved_pages > 0
    a.restore_complete(1, 2)
    torch.cuda.synchronize()
    assert_same_state(a, orc, [2, 5])
    ka, va = device_gather(a, 2, 0, ctx, 1, 64)
    kb_, vb_ = device_gather(b, 7, 0, ctx, 1, 64)
    want_k = k.cpu().view(torch.int16).numpy().view(np.uint16)
    assert (ka == want_k).all() and (kb_ == want_k).all()
    assert (va == vb_).all()
    a.close()
    b.close()


def test_slab_restore_pull_bit_exact(rt):
    from paper_2412_18169_b200 import runtime
    model = TINY.spec()
    a = rt.create_pool(0, model, model.param_bytes + MIB, TINY)
    b = rt.create_pool(1, model, model.param_bytes + MIB, TINY)
    wa = a.weight_bytes(1)
    wa.copy_(torch.randint(0, 256, (model.bytes_per_layer,), dtype=torch.uint8, device="cuda"))
    b.drop_layers(1, 2)
    assert b.weight_ptr(1) == 0
    b.restore_begin(1, 2)
    half = model.bytes_per_layer // 2
    runtime.copy_slabs(b, a, 1, 2, 0, half)           # two chunks, like plan_restore_transfers
    runtime.copy_slabs(b, a, 1, 2, half, model.bytes_per_layer)
    b.restore_complete(1, 2)
    torch.cuda.synchronize()
    assert torch.equal(b.weight_bytes(1), a.weight_bytes(1))
    # host replica source (exchange.HOST)
    host = torch.randint(0, 256, (model.bytes_per_layer,), dtype=torch.uint8).pin_memory()
    b.drop_layers(1, 2)
    b.restore_begin(1, 2)
    runtime.copy_slabs_from_host(b, host.data_ptr(), 1, 2, 0, model.bytes_per_layer)
    torch.cuda.synchronize()
    assert torch.equal(b.weight_bytes(1).cpu(), host)
    a.close()
    b.close()


def test_swap_pages_round_trip_bit_exact(rt):
    """Swap baseline (engine.py:906-970): a request's pages to pinned host
    memory, its device pages released and re-grown elsewhere, then back --
    every byte returns."""
    from paper_2412_18169_b200 import runtime
    model = TINY.spec()
    pool = rt.create_pool(0, model, model.param_bytes + 4 * MIB, TINY)
    pb = pool.page_bytes
    assert pool.grow([(0, 0, 2, 5)])
    kv = pool.kv_bytes().view(torch.uint8).view(-1, pb)
    pages = [pool.block_table(0, l) for l in range(2)]
    want = torch.randint(0, 256, (10, pb), dtype=torch.uint8, device="cuda")
    kv[torch.tensor(pages[0] + pages[1], device="cuda")] = want
    host = torch.empty(10 * pb, dtype=torch.uint8).pin_memory()
    runtime.copy_pages_host(pool, 0, 0, 2, 5, host, True)
    pool.release([0], 0, 2)
    assert pool.grow([(1, 0, 2, 3)])   # occupy the freed pages with another slot
    assert pool.grow([(0, 0, 2, 5)])   # the request comes back on other pages
    runtime.copy_pages_host(pool, 0, 0, 2, 5, host, False)
    torch.cuda.synchronize()
    assert torch.equal(host.view(10, pb), want.cpu())
    back = [pool.block_table(0, l) for l in range(2)]
    assert back != pages
    assert torch.equal(kv[torch.tensor(back[0] + back[1], device="cuda")], want)
    pool.close()


@pytest.mark.parametrize("kv_splits", [1, 2])
def test_paged_prefill_rescale_paths(rt, kv_splits):
    """Keys whose scores jump far above the running row max, in the first
    and in the second 64-key half of later tiles: the prefill takes its
    rare rescale paths (O, l rescaled; P recomputed; for the second half
    after the first half's P.V has landed) and still matches the oracle."""
    from paper_2412_18169_b200 import runtime
    shape = ATTN_SHAPES[0]
    model = shape.spec()
    pool = rt.create_pool(0, model, model.param_bytes + 64 * MIB, shape)
    gen = torch.Generator().manual_seed(31)
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    pre, c = 640, 256
    n = pre + c
    assert pool.grow([(0, 0, 1, (n + B - 1) // B)])
    q = rand_bf16((c, hq, 128), gen)
    k = rand_bf16((n, hkv, 128), gen)
    v = rand_bf16((n, hkv, 128), gen)
    qdir = q.float().mean(dim=(0, 1))
    qdir = qdir / qdir.norm()
    for pos, gain in ((150, 40.0), (300, 80.0), (420, 120.0), (700, 160.0)):
        # 300 and 700 sit in the second half of their 128-key tiles
        k[pos, :, :] = (qdir * gain).to(torch.bfloat16)
    append(pool, 0, k, v, 0, 0)
    out = torch.zeros((c, hq, 128), dtype=torch.bfloat16, device="cuda")
    dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
    runtime.paged_prefill(pool, 0, q.cuda(), dev([0]), dev([0]), dev([c]), dev([pre]), c, out,
                          128 ** -0.5, kv_splits=kv_splits)
    torch.cuda.synchronize()
    want = prefill_ref(q.float().numpy(), k.float().numpy(), v.float().numpy(), pre, 128 ** -0.5)
    ma, mr = check_close(out.float().cpu().numpy(), bf16_to_f32(f32_to_bf16(want)))
    assert ma <= 2e-2 and mr <= 1e-3, (kv_splits, ma, mr)
    pool.close()


def test_baseline_moves_through_the_transfer_engine(rt):
    """The baselines' whole-request KV moves as the engine issues them
    (engine.py:906-1047): swap out to HOST, swap back in on other pages,
    then migrate to another instance's pool -- every byte arrives."""
    from paper_2412_18169_b200.exchange import HOST, TaskKind, TransferTask
    from paper_2412_18169_b200.transfer import SlotTable, TransferEngine
    model = TINY.spec()
    a = rt.create_pool(0, model, model.param_bytes + 4 * MIB, TINY)
    b = rt.create_pool(1, model, model.param_bytes + 4 * MIB, TINY)
    slots = {0: SlotTable(rt.max_slots), 1: SlotTable(rt.max_slots)}
    te = TransferEngine({0: a, 1: b}, slots)
    rid, tokens = 7, 5 * TINY.block_tokens - 3   # 5 pages per layer
    sa = slots[0].get(rid)
    assert a.grow([(sa, 0, 2, 5)])
    kv_a = a.kv_bytes().view(-1, a.page_bytes)
    pages = [a.block_table(sa, l) for l in range(2)]
    want = torch.randint(0, 256, (10, a.page_bytes), dtype=torch.uint8, device="cuda")
    kv_a[torch.tensor(pages[0] + pages[1], device="cuda")] = want
    # the transfer engine copies on its own streams: the bytes must have landed
    # (the engines launch transfers only after observing the writers' events)
    torch.cuda.synchronize()
    nbytes = tokens * model.kv_bytes_per_token
    out = TransferTask(1, TaskKind.KVCACHE_CHUNK, 0, HOST, nbytes, rid=rid)
    te.register_request_move(out, (0, 2), tokens)
    te.submit(out)
    te.drain()
    a.release([sa], 0, 2)
    slots[0].drop(rid)
    assert a.grow([(slots[0].get(99), 0, 2, 2)])   # the freed pages go elsewhere
    sa = slots[0].get(rid)
    assert a.grow([(sa, 0, 2, 5)])
    back = TransferTask(2, TaskKind.KVCACHE_CHUNK, HOST, 0, nbytes, rid=rid)
    te.register_request_move(back, (0, 2), tokens)
    te.submit(back)
    te.drain()
    te.release_host(rid)
    got = [a.block_table(sa, l) for l in range(2)]
    assert torch.equal(kv_a[torch.tensor(got[0] + got[1], device="cuda")], want)
    # migrate 0 -> 1 (destination pages allocated first, as group_alloc does)
    sb = slots[1].get(rid)
    assert b.grow([(sb, 0, 2, 5)])
    mig = TransferTask(3, TaskKind.KVCACHE_CHUNK, 0, 1, nbytes, rid=rid)
    te.register_request_move(mig, (0, 2), tokens)
    te.submit(mig)
    te.drain()
    kv_b = b.kv_bytes().view(-1, b.page_bytes)
    pb = [b.block_table(sb, l) for l in range(2)]
    assert torch.equal(kv_b[torch.tensor(pb[0] + pb[1], device="cuda")], want)
    assert te.host_kv == {}
    a.close()
    b.close()


def test_host_replica_restore_through_the_plan(rt):
    """exchange.HOST (exchange.py:18, 224-233): when no live instance holds a
    layer, plan_restore_transfers sources it from the host replica; the
    transfer engine pulls it from pinned host memory into the vacated slab."""
    from paper_2412_18169_b200 import memory
    from paper_2412_18169_b200.exchange import HOST, plan_restore_transfers
    from paper_2412_18169_b200.transfer import SlotTable, TransferEngine
    model = TINY.spec()
    inst = memory.build_instance(0, model, model.param_bytes + MIB, 25_000_000_000,
                                 device=rt, shape=TINY)
    host = torch.randint(0, 256, (model.param_bytes,), dtype=torch.uint8).pin_memory()
    memory.drop_layers(inst, (0, 2))
    task = memory.restore_layers(inst, (0, 2), HOST)
    tasks = plan_restore_transfers({0: (0, 2)}, {0: []}, model.bytes_per_layer, 1 << 20)
    assert tasks and all(t.src == HOST and t.dst == 0 for t in tasks)
    assert sum(t.size_bytes for t in tasks) == task.size_bytes
    te = TransferEngine({0: inst.pool}, {0: SlotTable(rt.max_slots)}, host_replica=host)
    te.register_restore(tasks, model.bytes_per_layer)
    te.submit_many(tasks)
    te.drain()
    memory.complete_restore(inst, (0, 2))
    for l in range(2):
        lo = l * model.bytes_per_layer
        assert torch.equal(inst.pool.weight_bytes(l).cpu(), host[lo:lo + model.bytes_per_layer])
    inst.pool.close()


ATTN_SHAPES = [
    ModelShape("g2", num_layers=2, hidden=256, n_q_heads=2, n_kv_heads=1, head_dim=128,
               ffn=768, vocab=1024, block_tokens=64),
    ModelShape("g4", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
               ffn=1024, vocab=1024, block_tokens=64),
    ModelShape("g5", num_layers=2, hidden=5120, n_q_heads=40, n_kv_heads=8, head_dim=128,
               ffn=1024, vocab=1024, block_tokens=64),
]


@pytest.mark.parametrize("shape", ATTN_SHAPES, ids=lambda s: s.name)
def test_paged_decode_matches_oracle(rt, shape):
    from paper_2412_18169_b200 import runtime
    model = shape.spec()
    pool = rt.create_pool(0, model, model.param_bytes + 64 * MIB, shape)
    gen = torch.Generator().manual_seed(11)
    ctxs = [1, 63, 64, 65, 127, 128, 129, 300, 1000, 2047]
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    ks, vs = [], []
    for i, c in enumerate(ctxs):
        assert pool.grow([(i, 1, 2, (c + B - 1) // B)])
        k = rand_bf16((c, hkv, 128), gen)
        v = rand_bf16((c, hkv, 128), gen)
        append(pool, 1, k, v, i, 0)
        ks.append(k)
        vs.append(v)
    q = rand_bf16((len(ctxs), hq, 128), gen)
    scale = 128 ** -0.5
    slots = torch.arange(len(ctxs), dtype=torch.int32, device="cuda")
    lens = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    out = torch.empty((len(ctxs), hq, 128), dtype=torch.bfloat16, device="cuda")
    # stream-K plan: max_splits 1 cuts only at pair borders; the KV splits
    # merge inside the attention kernel or in the combine launch
    for max_splits, combine in ((1, False), (2, False), (4, False), (4, True), (16, False),
                                (16, True)):
        ws = torch.empty(runtime.decode_workspace_bytes(len(ctxs), hq, max_splits),
                         dtype=torch.uint8, device="cuda")
        out.zero_()
        runtime.paged_decode(pool, 1, q.cuda(), slots, lens, max(ctxs), out, ws, scale,
                             max_splits=max_splits, combine=combine)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
        for i, c in enumerate(ctxs):
            want = decode_ref(q[i].float().numpy(), ks[i].float().numpy(), vs[i].float().numpy(),
                              scale)
            want = bf16_to_f32(f32_to_bf16(want))
            ma, mr = check_close(got[i], want)
            assert ma <= 2e-2 and mr <= 1e-3, (shape.name, c, max_splits, combine, ma, mr)
    pool.close()


@pytest.mark.parametrize("combine", [False, True])
@pytest.mark.parametrize("batch", ["small", "large"])
def test_paged_decode_plan_reuse_across_layers(rt, batch, combine):
    """One plan, several layer launches (KB_DECODE_REUSE_PLAN), as a decode
    step runs them.  The attention kernel merges the KV splits of the pairs
    a CTA border cuts, and its per-(sequence, kv head) counters must re-arm
    after every launch, so each layer -- and a repeat of the first -- still
    matches the oracle (combine=True: the separate combine launch merges).
    Small batch: long pairs cut into many pieces; large batch (>= 4
    (sequence, kv head) pairs per SM): many whole pairs per CTA."""
    from paper_2412_18169_b200 import runtime
    # large: Llama-3-8B heads (8 kv heads), so 80 sequences give 640 pairs
    shape = ATTN_SHAPES[0] if batch == "small" else next(x for x in ATTN_SHAPES if x.name == "g4")
    model = shape.spec()
    r = rt if batch == "small" else runtime.Runtime(0, max_slots=96, max_pages_per_seq=256,
                                                    slack_pages=128)
    pool = r.create_pool(0, model, model.param_bytes + 256 * MIB, shape)
    gen = torch.Generator().manual_seed(13)
    ctxs = [2047, 1500, 700, 129, 64, 1]
    if batch == "large":  # two long sequences (split 16 ways) among many short ones
        ctxs = [4000, 3000] + [1 + (37 * i) % 200 for i in range(78)]
        assert len(ctxs) * shape.n_kv_heads >= 4 * 148
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    kv = {}
    for i, c in enumerate(ctxs):
        assert pool.grow([(i, 0, 2, (c + B - 1) // B)])
        for l in (0, 1):
            k = rand_bf16((c, hkv, 128), gen)
            v = rand_bf16((c, hkv, 128), gen)
            append(pool, l, k, v, i, 0)
            kv[(i, l)] = (k.float().numpy(), v.float().numpy())
    q = rand_bf16((len(ctxs), hq, 128), gen)
    scale = 128 ** -0.5
    slots = torch.arange(len(ctxs), dtype=torch.int32, device="cuda")
    lens = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    ws = torch.empty(runtime.decode_workspace_bytes(len(ctxs), hq, 16), dtype=torch.uint8,
                     device="cuda")
    for n, l in enumerate((0, 1, 0, 1)):
        out = torch.empty((len(ctxs), hq, 128), dtype=torch.bfloat16, device="cuda")
        runtime.paged_decode(pool, l, q.cuda(), slots, lens, max(ctxs), out, ws, scale,
                             max_splits=16, reuse_plan=n > 0, combine=combine)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
        for i in range(len(ctxs)):
            k, v = kv[(i, l)]
            want = bf16_to_f32(f32_to_bf16(decode_ref(q[i].float().numpy(), k, v, scale)))
            ma, mr = check_close(got[i], want)
            assert ma <= 2e-2 and mr <= 1e-3, (n, l, ctxs[i], ma, mr)
    pool.close()


@pytest.mark.parametrize("kv_splits", [1, 3, 8])
@pytest.mark.parametrize("shape", ATTN_SHAPES, ids=lambda s: s.name)
def test_paged_prefill_matches_oracle(rt, shape, kv_splits):
    from paper_2412_18169_b200 import runtime
    model = shape.spec()
    pool = rt.create_pool(0, model, model.param_bytes + 64 * MIB, shape)
    gen = torch.Generator().manual_seed(12)
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    # (prefix, chunk) pairs: cold prefill, chunk after a prefix, ragged tails
    cases = [(0, 1), (0, 100), (0, 128), (0, 300), (64, 64), (200, 77), (1000, 129)]
    qs, ks, vs, offs = [], [], [], []
    off = 0
    for i, (pre, c) in enumerate(cases):
        n = pre + c
        assert pool.grow([(i, 0, 1, (n + B - 1) // B)])
        k = rand_bf16((n, hkv, 128), gen)
        v = rand_bf16((n, hkv, 128), gen)
        append(pool, 0, k, v, i, 0)
        qs.append(rand_bf16((c, hq, 128), gen))
        ks.append(k)
        vs.append(v)
        offs.append(off)
        off += c
    q = torch.cat(qs).cuda()
    out = torch.zeros_like(q)
    dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
    scale = 128 ** -0.5
    runtime.paged_prefill(pool, 0, q, dev(list(range(len(cases)))), dev(offs),
                          dev([c for _, c in cases]), dev([p for p, _ in cases]),
                          max(c for _, c in cases), out, scale, kv_splits=kv_splits)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for i, (pre, c) in enumerate(cases):
        want = prefill_ref(qs[i].float().numpy(), ks[i].float().numpy(), vs[i].float().numpy(),
                           pre, scale)
        want = bf16_to_f32(f32_to_bf16(want))
        ma, mr = check_close(got[offs[i]:offs[i] + c], want)
        assert ma <= 2e-2 and mr <= 1e-3, (shape.name, kv_splits, pre, c, ma, mr)
    pool.close()


def test_attention_at_full_context_sampled_rows():
    """BASELINE config 4's sizes: the last 2,048-token chunk of a 32k Qwen
    prompt (prefix 30,720) and decodes at 32k context, with the split counts
    the runtime picks and explicit ones.  The oracle is exact per row, so
    sampled rows (tile borders, split borders, the causal diagonal's end)
    are checked against it; every head of each sampled row."""
    from paper_2412_18169_b200 import runtime
    rt32 = runtime.Runtime(0, max_slots=4, max_pages_per_seq=520, slack_pages=64)
    shape = ATTN_SHAPES[2]  # Qwen2.5-14B heads: 40 q / 8 kv (GQA group 5)
    assert (shape.n_q_heads, shape.n_kv_heads) == (40, 8)
    model = shape.spec()
    pool = rt32.create_pool(0, model, model.param_bytes + 400 * MIB, shape)
    gen = torch.Generator().manual_seed(32)
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    n, c = 32768, 2048
    pre = n - c
    assert pool.grow([(0, 0, 1, n // B), (1, 0, 1, (n - 1 + B - 1) // B)])
    k = rand_bf16((n, hkv, 128), gen)
    v = rand_bf16((n, hkv, 128), gen)
    append(pool, 0, k, v, 0, 0)
    append(pool, 0, k[:n - 1], v[:n - 1], 1, 0)
    kf, vf = k.float().numpy(), v.float().numpy()
    scale = 128 ** -0.5
    dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
    q = rand_bf16((c, hq, 128), gen)
    rows = [0, 1, 63, 64, 127, 128, 129, 1000, 1023, 1024, 1535, 2046, 2047]
    # None: the split count the runtime picks for this geometry (the bench's)
    assert runtime.prefill_splits(1, hq, c, n) == 4
    for kv_splits in (None, 1, 4, 8):
        out = torch.zeros((c, hq, 128), dtype=torch.bfloat16, device="cuda")
        kw = {"max_kv_len": n} if kv_splits is None else {"kv_splits": kv_splits}
        runtime.paged_prefill(pool, 0, q.cuda(), dev([0]), dev([0]), dev([c]), dev([pre]), c, out,
                              scale, **kw)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
        for r in rows:
            want = prefill_ref(q[r:r + 1].float().numpy(), kf[:pre + r + 1], vf[:pre + r + 1],
                               pre + r, scale)
            ma, mr = check_close(got[r:r + 1], bf16_to_f32(f32_to_bf16(want)))
            assert ma <= 2e-2 and mr <= 1e-3, (kv_splits, r, ma, mr)
    # decode: context 32,768 and 32,767 (a ragged last page)
    qd = rand_bf16((2, hq, 128), gen)
    lens = [n, n - 1]
    for max_splits in (1, 16):
        ws = torch.empty(runtime.decode_workspace_bytes(2, hq, max_splits), dtype=torch.uint8,
                         device="cuda")
        out = torch.empty((2, hq, 128), dtype=torch.bfloat16, device="cuda")
        runtime.paged_decode(pool, 0, qd.cuda(), dev([0, 1]), dev(lens), n, out, ws, scale,
                             max_splits=max_splits)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
        for i, ctx in enumerate(lens):
            want = decode_ref(qd[i].float().numpy(), kf[:ctx], vf[:ctx], scale)
            ma, mr = check_close(got[i], bf16_to_f32(f32_to_bf16(want)))
            assert ma <= 2e-2 and mr <= 1e-3, (max_splits, ctx, ma, mr)
    pool.close()


def test_attention_empty_batches(rt):
    """No prefill chunks / no decode sequences: the calls are no-ops that
    leave the output untouched (the device engine issues them for
    decode-only and prefill-only microbatches)."""
    from paper_2412_18169_b200 import runtime
    shape = ATTN_SHAPES[0]
    model = shape.spec()
    pool = rt.create_pool(0, model, model.param_bytes + 64 * MIB, shape)
    e32 = torch.empty(0, dtype=torch.int32, device="cuda")
    q = torch.empty((0, shape.n_q_heads, 128), dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    ws = torch.empty(runtime.decode_workspace_bytes(1, shape.n_q_heads, 4), dtype=torch.uint8,
                     device="cuda")
    runtime.paged_decode(pool, 0, q, e32, e32, 0, out, ws, 1.0, max_splits=4)
    runtime.paged_prefill(pool, 0, q, e32, e32, e32, e32, 0, out, 1.0)
    torch.cuda.synchronize()
    pool.close()


def test_layer_elementwise_kernels_match_torch(rt):
    """kb_add_rmsnorm / kb_silu_mul (the device engine's stage execution)
    against a plain PyTorch fp32 reference of the same ops."""
    from paper_2412_18169_b200 import runtime
    g = torch.Generator(device="cuda").manual_seed(3)
    n, H, F = 37, 4096, 14336
    x = torch.randn((n, H), device="cuda", generator=g).to(torch.bfloat16)
    res = torch.randn((n, H), device="cuda", generator=g).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn((H,), device="cuda", generator=g)).to(torch.bfloat16)
    want_x = (x.float() + res.float()).to(torch.bfloat16)
    xf = want_x.float()
    want = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    out = torch.empty_like(x)
    runtime.add_rmsnorm(x, res, w, out)
    torch.cuda.synchronize()
    assert torch.equal(x, want_x)                      # the residual stream, in place
    assert (out.float() - want).abs().max().item() <= 3e-2 * want.abs().max().item()
    gu = torch.randn((n, 2 * F), device="cuda", generator=g).to(torch.bfloat16)
    act = torch.empty((n, F), dtype=torch.bfloat16, device="cuda")
    runtime.silu_mul(gu, act)
    torch.cuda.synchronize()
    want = torch.nn.functional.silu(gu[:, :F].float()) * gu[:, F:].float()
    err = (act.float() - want).abs() / want.abs().clamp_min(1e-2)
    assert err.mean().item() <= 1e-2
