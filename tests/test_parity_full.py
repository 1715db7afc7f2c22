"""GPU parity at production geometry (VERDICT r1 "Weak 1-3").

* the position-sensitive device hash (kb_hash_segments) against its numpy
  restatement, and its sensitivity to permuted bytes;
* page copies, restore-time compaction and host swaps on Llama-3-8B's
  256 KiB pages (8 pieces of 32 KiB per page in the copy kernels), byte for
  byte against oracle.kvpool;
* the fp16 V-cache range guard (|v| in {1e-6, 7e4});
* the decode workspace bound;
* programmatic-dependent-launch chains (append -> attention for several
  layers, no host syncs, eager and CUDA-graph replay) against the oracle;
* block_tokens = 128 decode / prefill.
"""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.attention import bf16_to_f32, check_close, decode_ref, f32_to_bf16, prefill_ref  # noqa: E402
from oracle.kvpool import OraclePool, copy_pages as oracle_copy_pages, hash_bytes, v_range_flags  # noqa: E402

from paper_2412_18169_b200.core import SHAPES, ModelShape  # noqa: E402

MIB = 1 << 20
# Llama-3-8B's KV geometry (8 kv heads x 128, 64-token pages = 256 KiB) on a
# 3-layer model with small slabs, so the oracle can track every byte
LLAMA_PAGES = ModelShape("llama_pages", num_layers=3, hidden=256, n_q_heads=32, n_kv_heads=8,
                         head_dim=128, ffn=256, vocab=1024, block_tokens=64)
G4_B128 = ModelShape("g4_b128", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8,
                     head_dim=128, ffn=1024, vocab=1024, block_tokens=128)


@pytest.fixture(scope="module")
def runtime():
    from paper_2412_18169_b200 import build
    build.build()
    from paper_2412_18169_b200 import runtime as rt_mod
    assert torch.cuda.is_available()
    return rt_mod


def test_hash_matches_oracle_and_sees_positions(runtime):
    g = torch.Generator(device="cuda").manual_seed(4)
    seg = 4096
    buf = torch.randint(0, 256, (64 * seg,), dtype=torch.uint8, device="cuda", generator=g)
    h = runtime.hash_tensor(buf, seg).cpu().tolist()
    host = buf.cpu().numpy()
    assert h == [hash_bytes(host[i * seg:(i + 1) * seg]) for i in range(64)]
    # gathered segments in a given order (the page-list form)
    idx = torch.tensor([5, 3, 63, 0, 5], dtype=torch.int64, device="cuda")
    hg = runtime.hash_segments(buf.data_ptr(), seg, 5, index=idx).cpu().tolist()
    assert hg == [h[5], h[3], h[63], h[0], h[5]]
    # one large segment (a slab-sized multi-CTA reduction)
    big = torch.randint(0, 256, (3 * MIB + 16 * 7,), dtype=torch.uint8, device="cuda", generator=g)
    assert runtime.hash_tensor(big).item() == hash_bytes(big.cpu().numpy())
    # position sensitivity: swapping two 16-byte vectors inside a segment, or
    # two segments, changes the hash although the multiset of bytes is equal
    sw = buf.clone()
    a, b = sw[16:32].clone(), sw[48:64].clone()
    sw[16:32], sw[48:64] = b, a
    assert runtime.hash_tensor(sw, seg)[0].item() != h[0]
    assert runtime.hash_tensor(sw, seg)[1:].cpu().tolist() == h[1:]
    # an int32 sum (the r1 check) cannot see this permutation
    assert sw.view(torch.int32).to(torch.int64).sum() == buf.view(torch.int32).to(torch.int64).sum()


def _mirror(pool, track=True):
    inf = pool.info()
    return OraclePool(num_layers=pool.model.num_layers, slab_bytes=pool.model.bytes_per_layer,
                      page_bytes=pool.page_bytes, head_pages=inf.extent_pages,
                      max_slots=pool.rt.max_slots, max_pages_per_seq=pool.rt.max_pages_per_seq,
                      track_bytes=track)


def _assert_bytes(pool, orc):
    """Every live page's bytes (and the block tables naming them) equal the
    oracle's."""
    kv = pool.kv_bytes().cpu().numpy().reshape(-1, pool.page_bytes)
    for (slot, layer), row in orc.bt.items():
        assert pool.block_table(slot, layer) == row, (slot, layer)
        if row:
            assert np.array_equal(kv[row], orc.data[row]), (slot, layer)
    assert (pool.bitmap() == orc.bitmap()).all()


def test_llama_pages_copy_compact_swap_bit_exact(runtime):
    """256 KiB pages go through the multi-piece paths of copy_pages_kernel,
    compact_copy_kernel and copy_pages_host_kernel (8 pieces each); every
    byte is compared with oracle.kvpool after each phase."""
    shape = LLAMA_PAGES
    model = shape.spec()
    assert shape.page_bytes == 256 * 1024
    rt = runtime.Runtime(0, max_slots=8, max_pages_per_seq=64, slack_pages=16)
    a = rt.create_pool(0, model, model.param_bytes + 8 * MIB, shape)
    b = rt.create_pool(1, model, model.param_bytes + 8 * MIB, shape)
    oa, ob = _mirror(a), _mirror(b)
    g = torch.Generator(device="cuda").manual_seed(9)
    for pool, orc in ((a, oa), (b, ob)):
        kv = pool.kv_bytes()
        kv.copy_(torch.randint(0, 256, (kv.numel(),), dtype=torch.uint8, device="cuda", generator=g))
        torch.cuda.synchronize()
        orc.data[:] = kv.cpu().numpy().reshape(orc.data.shape)
    # drop two layers: their slab pages join the KV pool
    a.drop_layers(1, 3)
    oa.drop(1, 3)
    reqs = [(0, 0, 3, 15), (1, 0, 2, 10), (2, 1, 3, 9)]   # spill into the dropped slabs
    assert a.grow(reqs) and oa.grow(reqs)
    _assert_bytes(a, oa)
    assert max(max(r) for r in oa.bt.values()) >= oa.head_pages  # pages in a dropped slab
    # exchange a -> b in chunks with partial flat ranges (plan_exchange chunking)
    b.drop_layers(1, 3)
    ob.drop(1, 3)
    breqs = [(4, 0, 3, 15), (5, 0, 2, 10)]
    assert b.grow(breqs) and ob.grow(breqs)
    moves = [(0, 4, 0, 3, 15, 0, 7), (0, 4, 0, 3, 15, 7, 30), (0, 4, 0, 3, 15, 30, 45),
             (1, 5, 0, 2, 10, 0, 20)]
    runtime.copy_pages(b, a, moves)
    oracle_copy_pages(ob, oa, moves)
    torch.cuda.synchronize()
    _assert_bytes(b, ob)
    # restore layer 1 on a: live pages leave its slab (compaction)
    a.release([2], 1, 3)
    oa.release([2], 1, 3)
    want = oa.restore(1, 2)
    a.restore_begin(1, 2)
    assert want > 0 and a.last_moved_pages == want
    a.restore_complete(1, 2)
    torch.cuda.synchronize()
    _assert_bytes(a, oa)
    # swap slot 1 out to pinned host memory, re-grow it elsewhere, swap back
    npg = 10
    host = torch.empty(2 * npg * a.page_bytes, dtype=torch.uint8).pin_memory()
    runtime.copy_pages_host(a, 1, 0, 2, npg, host, True)
    torch.cuda.synchronize()
    want_host = np.concatenate([oa.data[oa.bt[(1, l)]] for l in range(2)]).reshape(-1)
    assert np.array_equal(host.numpy(), want_host)
    a.release([1], 0, 2)
    oa.release([1], 0, 2)
    assert a.grow([(6, 0, 2, 2)]) and oa.grow([(6, 0, 2, 2)])   # occupy some freed pages
    assert a.grow([(1, 0, 2, npg)]) and oa.grow([(1, 0, 2, npg)])
    runtime.copy_pages_host(a, 1, 0, 2, npg, host, False)
    for l in range(2):
        oa.data[oa.bt[(1, l)]] = want_host.reshape(2, npg, -1)[l]
    torch.cuda.synchronize()
    _assert_bytes(a, oa)
    # the device hash of every live page equals the oracle's
    for (slot, layer), row in oa.bt.items():
        if row:
            idx = torch.tensor(row, dtype=torch.int64, device="cuda")
            got = runtime.hash_segments(a.info().kv_base, a.page_bytes, len(row), index=idx)
            assert got.cpu().tolist() == [hash_bytes(oa.data[p]) for p in row]
    a.close()
    b.close()


def _append(runtime, pool, layer, k, v, slot, start, stream=None):
    n = k.shape[0]
    slots = torch.full((n,), slot, dtype=torch.int32, device="cuda")
    pos = torch.arange(start, start + n, dtype=torch.int32, device="cuda")
    runtime.kv_append(pool, layer, k.cuda(), v.cuda(), slots, pos, stream=stream)


@pytest.mark.parametrize("case", ["normal", "tiny_1e-6", "huge_7e4", "tiny_next_to_normal"])
def test_fp16_v_cache_range_guard(runtime, case):
    shape = SHAPES["tiny"]
    model = shape.spec()
    rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=16, slack_pages=16)
    pool = rt.create_pool(0, model, model.param_bytes + MIB, shape)
    assert pool.grow([(0, 0, 1, 2)])
    g = torch.Generator().manual_seed(1)
    k = torch.randn((100, 1, 128), generator=g).to(torch.bfloat16)
    v = torch.randn((100, 1, 128), generator=g)
    if case == "tiny_1e-6":
        v = v * 1e-6
    elif case == "huge_7e4":
        v[37, 0, 5] = 7e4
    elif case == "tiny_next_to_normal":
        v[:, :, :64] *= 1e-6       # half of every row tiny, the row max stays normal
    v = v.to(torch.bfloat16)
    want = v_range_flags(v.view(torch.int16).numpy().view(np.uint16))
    _append(runtime, pool, 0, k, v, 0, 0)
    torch.cuda.synchronize()
    assert pool.kv_status() == want
    if case in ("normal", "tiny_next_to_normal"):
        assert want == 0
        pool.check_kv_range()
    else:
        assert want == (2 if case == "tiny_1e-6" else 1)
        with pytest.raises(ValueError, match="fp16 KV-cache range"):
            pool.check_kv_range()
        assert pool.kv_status() == 0   # the check clears the sticky flags
    pool.close()


def test_kv_append_without_page_is_skipped(runtime):
    """Rows whose position has no grown page, or whose slot / position lies
    outside the block table, are skipped (nothing written outside the pool)
    and flagged KB_KV_NO_PAGE; the rows that do have pages land as usual."""
    shape = SHAPES["tiny"]
    model = shape.spec()
    rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=4, slack_pages=16)
    pool = rt.create_pool(0, model, model.param_bytes + MIB, shape)
    assert pool.grow([(0, 0, 1, 2), (1, 0, 1, 4)])    # slot 0: tokens 0-127
    g = torch.Generator().manual_seed(2)
    k = torch.randn((256, 1, 128), generator=g).to(torch.bfloat16)
    v = torch.randn((256, 1, 128), generator=g).to(torch.bfloat16)
    _append(runtime, pool, 0, k, v, 1, 0)              # slot 1 filled, the bystander
    torch.cuda.synchronize()
    info = pool.info()

    def page_hashes():
        rows = {s: pool.block_table(s, 0) for s in (0, 1)}
        idx = torch.tensor(rows[0] + rows[1], dtype=torch.int64, device="cuda")
        return runtime.hash_segments(info.kv_base, pool.page_bytes, idx.numel(), index=idx).cpu()
    before = page_hashes()
    assert pool.kv_status() == 0
    _append(runtime, pool, 0, k[:10], v[:10], 0, 120)   # 120-127 have a page, 128-129 not
    torch.cuda.synchronize()
    assert pool.kv_status() == runtime.KB_KV_NO_PAGE
    with pytest.raises(ValueError, match="without a page"):
        pool.check_kv_range()
    assert pool.kv_status() == 0
    after = page_hashes()
    assert torch.equal(after[2:], before[2:])          # slot 1 untouched
    assert not torch.equal(after[:2], before[:2])      # slot 0's rows 120-127 landed
    for slot, p in ((9, 0), (-1, 0), (0, -1), (0, 4 * 64)):   # outside the table
        runtime.kv_append(pool, 0, k[:1].cuda(), v[:1].cuda(),
                          torch.tensor([slot], dtype=torch.int32, device="cuda"),
                          torch.tensor([p], dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        assert pool.kv_status(clear=True) == runtime.KB_KV_NO_PAGE
    assert torch.equal(page_hashes(), after)
    # page moves naming a slot outside either pool's table are refused on
    # the host before anything is read
    for src_slot, dst_slot in ((4, 1), (-1, 1), (1, 4), (1, -1)):
        with pytest.raises(runtime.DeviceError, match="bad move"):
            runtime.copy_pages(pool, pool, [(src_slot, dst_slot, 0, 1, 1, 0, 1)])
    pool.close()


def test_decode_workspace_too_small_is_refused(runtime):
    shape = SHAPES["tiny"]
    model = shape.spec()
    rt = runtime.Runtime(0, max_slots=8, max_pages_per_seq=16, slack_pages=16)
    pool = rt.create_pool(0, model, model.param_bytes + MIB, shape)
    assert pool.grow([(s, 0, 1, 1) for s in range(8)])
    q = torch.zeros((8, 2, 128), dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    ws = torch.empty(runtime.decode_workspace_bytes(4, 2, 4), dtype=torch.uint8, device="cuda")
    slots = torch.arange(8, dtype=torch.int32, device="cuda")
    lens = torch.ones(8, dtype=torch.int32, device="cuda")
    with pytest.raises(runtime.DeviceError, match="decode workspace"):
        runtime.paged_decode(pool, 0, q, slots, lens, 1, out, ws, 1.0, max_splits=4)
    pool.close()


G4 = ModelShape("g4", num_layers=4, hidden=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                ffn=1024, vocab=1024, block_tokens=64)


@pytest.mark.parametrize("mode", ["eager", "graph"])
@pytest.mark.parametrize("batch", ["combine", "fused"])
def test_pdl_append_decode_chain_without_host_sync(runtime, mode, batch):
    """A decode step as a stage runs it: per layer kv_append (which lets the
    next launch start early) then paged_decode (PDL prologue, plan reused
    after the first layer), 4 layers back to back with no host sync -- with
    the KV splits merged by a combine launch (6 sequences) and inside the
    attention kernel (80 sequences), eagerly and as a replayed CUDA graph.  Every layer's output matches
    the oracle."""
    shape = G4
    model = shape.spec()
    nseq = 6 if batch == "combine" else 80
    rt = runtime.Runtime(0, max_slots=96, max_pages_per_seq=64, slack_pages=64)
    pool = rt.create_pool(0, model, model.param_bytes + 1280 * MIB, shape)
    rng = random.Random(5)
    ctxs = [rng.randrange(1, 1500) for _ in range(nseq)]
    ctxs[0] = 2047
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    g = torch.Generator().manual_seed(6)
    kv = {}
    for i, c in enumerate(ctxs):
        assert pool.grow([(i, 0, 4, (c + B - 1) // B)])
        for l in range(4):
            # the prefix; the decode token's own K/V is appended in the chain
            k = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
            v = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
            if c > 1:
                _append(runtime, pool, l, k[:c - 1], v[:c - 1], i, 0)
            kv[(i, l)] = (k, v)
    torch.cuda.synchronize()
    slots = torch.arange(nseq, dtype=torch.int32, device="cuda")
    lens = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    pos = lens - 1
    qs = [torch.randn((nseq, hq, 128), generator=g).to(torch.bfloat16).cuda() for _ in range(4)]
    kl = [torch.stack([kv[(i, l)][0][ctxs[i] - 1] for i in range(nseq)]).cuda() for l in range(4)]
    vl = [torch.stack([kv[(i, l)][1][ctxs[i] - 1] for i in range(nseq)]).cuda() for l in range(4)]
    outs = [torch.zeros((nseq, hq, 128), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    ws = torch.empty(runtime.decode_workspace_bytes(nseq, hq, 16), dtype=torch.uint8, device="cuda")
    scale = 128 ** -0.5
    st = torch.cuda.Stream()

    def step():
        for l in range(4):
            runtime.kv_append(pool, l, kl[l], vl[l], slots, pos, stream=st)
            runtime.paged_decode(pool, l, qs[l], slots, lens, max(ctxs), outs[l], ws, scale,
                                 max_splits=16, reuse_plan=l > 0, stream=st,
                                 combine=batch == "combine")
    if mode == "eager":
        step()
    else:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            step()                 # warm-up outside the capture
        st.synchronize()
        for o in outs:
            o.zero_()
        with torch.cuda.graph(graph, stream=st):
            step()
        pool.stream_begin(st)
        graph.replay()
        pool.stream_end(st)
    st.synchronize()
    for l in range(4):
        got = outs[l].float().cpu().numpy()
        for i in range(nseq):
            k, v = kv[(i, l)]
            want = bf16_to_f32(f32_to_bf16(decode_ref(qs[l][i].float().cpu().numpy(),
                                                      k.float().numpy(), v.float().numpy(), scale)))
            ma, mr = check_close(got[i], want)
            assert ma <= 2e-2 and mr <= 1e-3, (mode, batch, l, ctxs[i], ma, mr)
    pool.close()


def test_block_tokens_128_decode_and_prefill(runtime):
    """128-token pages (512 KiB): the <128> instantiations of the decode and
    prefill kernels, each opted in to its shared-memory size separately."""
    shape = G4_B128
    model = shape.spec()
    rt = runtime.Runtime(0, max_slots=8, max_pages_per_seq=64, slack_pages=32)
    pool = rt.create_pool(0, model, model.param_bytes + 128 * MIB, shape)
    g = torch.Generator().manual_seed(8)
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    ctxs = [1, 127, 128, 129, 1000, 2047]
    ks, vs = [], []
    for i, c in enumerate(ctxs):
        assert pool.grow([(i, 0, 1, (c + B - 1) // B)])
        k = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
        _append(runtime, pool, 0, k, v, i, 0)
        ks.append(k)
        vs.append(v)
    scale = 128 ** -0.5
    dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
    q = torch.randn((len(ctxs), hq, 128), generator=g).to(torch.bfloat16)
    out = torch.empty((len(ctxs), hq, 128), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(runtime.decode_workspace_bytes(len(ctxs), hq, 8), dtype=torch.uint8,
                     device="cuda")
    runtime.paged_decode(pool, 0, q.cuda(), dev(list(range(len(ctxs)))), dev(ctxs), max(ctxs), out,
                         ws, scale, max_splits=8)
    torch.cuda.synchronize()
    for i, c in enumerate(ctxs):
        want = bf16_to_f32(f32_to_bf16(decode_ref(q[i].float().numpy(), ks[i].float().numpy(),
                                                  vs[i].float().numpy(), scale)))
        ma, mr = check_close(out[i].float().cpu().numpy(), want)
        assert ma <= 2e-2 and mr <= 1e-3, ("decode", c, ma, mr)
    # prefill: the last 300 tokens of sequence 5 as a chunk after its prefix
    c, n = 300, ctxs[5]
    qp = torch.randn((c, hq, 128), generator=g).to(torch.bfloat16)
    for kv_splits in (1, 3):
        op = torch.zeros((c, hq, 128), dtype=torch.bfloat16, device="cuda")
        runtime.paged_prefill(pool, 0, qp.cuda(), dev([5]), dev([0]), dev([c]), dev([n - c]), c, op,
                              scale, kv_splits=kv_splits)
        torch.cuda.synchronize()
        want = bf16_to_f32(f32_to_bf16(prefill_ref(qp.float().numpy(), ks[5].float().numpy(),
                                                   vs[5].float().numpy(), n - c, scale)))
        ma, mr = check_close(op.float().cpu().numpy(), want)
        assert ma <= 2e-2 and mr <= 1e-3, ("prefill", kv_splits, ma, mr)
    pool.close()


@pytest.mark.parametrize("devs", [(0, 0), (0, 1)], ids=["same_gpu", "two_gpus"])
def test_two_runtimes_in_one_process(runtime, devs):
    """One process driving two Runtimes (DeviceConfig.devices): pools on
    each, KV pages copied from the first pool into the second (a peer read
    when they sit on different GPUs), then decode and prefill on the second
    device -- the shared-memory opt-in of the ~210 KB attention kernels is
    per device, so the second device's launches must carry their own.
    The two-GPU case skips on a one-GPU box."""
    da, db = devs
    if max(devs) >= torch.cuda.device_count():
        pytest.skip("needs a second GPU")
    shape = ModelShape("g4", num_layers=2, hidden=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                       ffn=1024, vocab=1024, block_tokens=64)
    model = shape.spec()
    peers_a = [db] if db != da else []
    peers_b = [da] if db != da else []
    rt_a = runtime.Runtime(da, peers=peers_a, max_slots=8, max_pages_per_seq=64, slack_pages=64)
    rt_b = runtime.Runtime(db, peers=peers_b, max_slots=8, max_pages_per_seq=64, slack_pages=64)
    pa = rt_a.create_pool(0, model, model.param_bytes + 64 * MIB, shape)
    pb = rt_b.create_pool(1, model, model.param_bytes + 64 * MIB, shape)
    g = torch.Generator().manual_seed(21)
    ctx, hkv, hq = 1000, shape.n_kv_heads, shape.n_q_heads
    npg = (ctx + 63) // 64
    k = torch.randn((ctx, hkv, 128), generator=g).to(torch.bfloat16)
    v = torch.randn((ctx, hkv, 128), generator=g).to(torch.bfloat16)
    with torch.cuda.device(da):
        assert pa.grow([(2, 0, 1, npg)])
        n = ctx
        runtime.kv_append(pa, 0, k.cuda(), v.cuda(), torch.full((n,), 2, dtype=torch.int32, device="cuda"),
                          torch.arange(n, dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
    with torch.cuda.device(db):
        assert pb.grow([(5, 0, 1, npg)])
        # (src slot, dst slot, layer lo, layer hi, pages per layer, flat lo, flat hi)
        runtime.copy_pages(pb, pa, [(2, 5, 0, 1, npg, 0, npg)])
        torch.cuda.synchronize()
        dev = lambda xs: torch.tensor(xs, dtype=torch.int32, device="cuda")  # noqa: E731
        q = torch.randn((1, hq, 128), generator=g).to(torch.bfloat16)
        out = torch.empty((1, hq, 128), dtype=torch.bfloat16, device="cuda")
        ws = torch.empty(runtime.decode_workspace_bytes(1, hq, 8), dtype=torch.uint8, device="cuda")
        runtime.paged_decode(pb, 0, q.cuda(), dev([5]), dev([ctx]), ctx, out, ws, 128 ** -0.5,
                             max_splits=8)
        c = 200
        qp = torch.randn((c, hq, 128), generator=g).to(torch.bfloat16)
        op = torch.empty((c, hq, 128), dtype=torch.bfloat16, device="cuda")
        runtime.paged_prefill(pb, 0, qp.cuda(), dev([5]), dev([0]), dev([c]), dev([ctx - c]), c, op,
                              128 ** -0.5, kv_splits=2)
        torch.cuda.synchronize()
        assert out.device.index == db
    want = bf16_to_f32(f32_to_bf16(decode_ref(q[0].float().numpy(), k.float().numpy(),
                                              v.float().numpy(), 128 ** -0.5)))
    ma, mr = check_close(out[0].float().cpu().numpy(), want)
    assert ma <= 2e-2 and mr <= 1e-3, (ma, mr)
    wantp = bf16_to_f32(f32_to_bf16(prefill_ref(qp.float().numpy(), k.float().numpy(),
                                                v.float().numpy(), ctx - c, 128 ** -0.5)))
    pa_, pr_ = check_close(op.float().cpu().numpy(), wantp)
    assert pa_ <= 2e-2 and pr_ <= 1e-3, (pa_, pr_)
    pb.close()
    pa.close()


@pytest.mark.parametrize("case", ["one_long_sequence", "whole_pair_items", "mixed"])
@pytest.mark.parametrize("combine", [True, False])
def test_decode_plan_extremes(runtime, case, combine):
    """Decode plans at their extremes, each layer run three times on one
    plan (the item counter and split counters must re-arm): one 20k-token
    sequence cut into 32+ KV splits per kv head (max_splits 64), 96
    sequences whose items are whole 8-tile pairs (one split each: more
    items than 2 per CTA), and a ragged mix from 5 to 9,000 tokens; with
    the combine launch and with the in-kernel merge."""
    shape = G4
    model = shape.spec()
    rng = random.Random(11)
    if case == "one_long_sequence":
        ctxs, max_splits = [20000], 64
    elif case == "whole_pair_items":
        ctxs, max_splits = [1000 + rng.randrange(-20, 20) for _ in range(96)], 16
    else:
        ctxs, max_splits = [rng.choice([5, 300, 1200, 4000, 9000]) for _ in range(24)], 16
    nseq = len(ctxs)
    rt = runtime.Runtime(0, max_slots=128, max_pages_per_seq=512, slack_pages=64)
    pool = rt.create_pool(0, model, model.param_bytes + 2048 * MIB, shape)
    hkv, hq, B = shape.n_kv_heads, shape.n_q_heads, shape.block_tokens
    g = torch.Generator().manual_seed(17)
    kv = {}
    for i, c in enumerate(ctxs):
        assert pool.grow([(i, 0, 1, (c + B - 1) // B)])
        k = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((c, hkv, 128), generator=g).to(torch.bfloat16)
        _append(runtime, pool, 0, k, v, i, 0)
        kv[i] = (k.float().numpy(), v.float().numpy())
    torch.cuda.synchronize()
    q = torch.randn((nseq, hq, 128), generator=g).to(torch.bfloat16)
    slots = torch.arange(nseq, dtype=torch.int32, device="cuda")
    lens = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    ws = torch.empty(runtime.decode_workspace_bytes(nseq, hq, max_splits), dtype=torch.uint8,
                     device="cuda")
    scale = 128 ** -0.5
    want = [bf16_to_f32(f32_to_bf16(decode_ref(q[i].float().numpy(), *kv[i], scale)))
            for i in range(nseq)]
    for n in range(3):
        out = torch.zeros((nseq, hq, 128), dtype=torch.bfloat16, device="cuda")
        runtime.paged_decode(pool, 0, q.cuda(), slots, lens, max(ctxs), out, ws, scale,
                             max_splits=max_splits, reuse_plan=n > 0, combine=combine)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
        for i in range(nseq):
            ma, mr = check_close(got[i], want[i])
            assert ma <= 2e-2 and mr <= 1e-3, (case, combine, n, ctxs[i], ma, mr)
    pool.close()
