"""Cross-process peer views and the multi-rank overload cycle on the GPU.

Two processes share the one B200 of the test box (gloo carries the control
plane; NCCL refuses two ranks on one device): each owns one replica's pool,
exports its VMM handles, imports the other's as a read-only view and pulls
KV pages and layer slabs from it -- the exact code path that crosses NVLink
when the ranks sit on different GPUs (bench.py --gpus N).  Everything moved
must be bit-identical."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPES_L = {"llama3_8b": 32, "qwen25_14b": 48}
SLAB = {"llama3_8b": 438_304_768, "qwen25_14b": 551_550_976}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _guard(target, rank, world, port, q, *args):
    try:
        target(rank, world, port, q, *args)
    except BaseException:
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))
        raise


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_guard, args=(target, r, world, port, q, *args))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, v = q.get(timeout=600)
        assert not (isinstance(v, str) and v.startswith("ERROR")), f"rank {r}: {v}"
        res[r] = v
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _view_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.core import SHAPES
    from paper_2412_18169_b200.dist import share_pools
    _init(rank, world, port)
    try:
        shape = SHAPES["tiny"]
        model = shape.spec()
        rt = runtime.Runtime(0, max_slots=8, max_pages_per_seq=64)
        pool = rt.create_pool(rank, model, model.param_bytes + (8 << 20), shape)
        # owner-written content: layer slabs and 5 pages of slot 0, layers 0-1
        for l in range(model.num_layers):
            w = pool.weight_bytes(l).view(torch.int32)
            w.copy_(torch.arange(w.numel(), dtype=torch.int32, device="cuda") * (rank + 3) + l)
        assert pool.grow([(0, 0, 2, 5)])
        kv = pool.kv_bytes().view(torch.int32).view(-1, pool.page_bytes // 4)
        for l in range(2):
            for i, pg in enumerate(pool.block_table(0, l)):
                kv[pg].fill_(1000 * rank + 10 * l + i)
        torch.cuda.synchronize()
        views = share_pools(rt, {rank: pool}, model, shape, key=f"vt{port}")
        peer = 1 - rank
        v = views[peer]
        assert runtime.is_view(v) and not runtime.is_view(pool)
        v.refresh(range(model.num_layers))
        assert v.npages(0, 0) == 5 and v.npages(0, 1) == 5
        # the view refuses mutation (its owner performs it)
        with pytest.raises(runtime.DeviceError, match="read-only peer view"):
            runtime._check(runtime._lib.kb_drop_layers(v.h, 0, 1, None))
        # a copy cannot land in a view
        with pytest.raises(runtime.DeviceError, match="owns"):
            runtime.copy_slabs(v, pool, 0, 1, 0, 1024)
        # pull the peer's pages into slot 1 here
        assert pool.grow([(1, 0, 2, 5)])
        runtime.copy_pages(pool, v, [(0, 1, 0, 2, 5, 0, 10)])
        # pull the peer's slab of layer `rank` after dropping + vacating ours
        # (the peer keeps that layer: it restores the other one)
        mine, other = rank, 1 - rank
        pool.drop_layers(mine, mine + 1)
        pool.restore_begin(mine, mine + 1)
        runtime.copy_slabs(pool, v, mine, mine + 1, 0, model.bytes_per_layer)
        pool.restore_complete(mine, mine + 1)
        torch.cuda.synchronize()
        ok_pages = all(bool((kv[pg] == 1000 * peer + 10 * l + i).all())
                       for l in range(2) for i, pg in enumerate(pool.block_table(1, l)))
        w1 = pool.weight_bytes(mine).view(torch.int32)
        want = torch.arange(w1.numel(), dtype=torch.int32, device="cuda") * (peer + 3) + mine
        ok_slab = bool((w1 == want).all())
        # our other layer is untouched
        w0 = pool.weight_bytes(other).view(torch.int32)
        ok_own = bool((w0 == torch.arange(w0.numel(), dtype=torch.int32, device="cuda")
                       * (rank + 3) + other).all())
        dist.barrier()
        for x in views.values():
            x.close()
        dist.barrier()
        pool.close()
        q.put((rank, (ok_pages, ok_slab, ok_own)))
    finally:
        dist.destroy_process_group()


def test_peer_view_pulls_pages_and_slabs_bit_exact():
    res = _spawn(_view_worker, 2)
    assert res[0] == (True, True, True) and res[1] == (True, True, True)


def _cycle_worker(rank, world, port, q, shape_name, kv_budget, chunk, input_mean, pp=2):
    import torch.distributed as dist

    from paper_2412_18169_b200 import dist_cycle, runtime
    from paper_2412_18169_b200.core import SHAPES
    _init(rank, world, port)
    try:
        rt = runtime.Runtime(0, max_slots=512, max_pages_per_seq=1024)
        out = dist_cycle.run(rt, SHAPES[shape_name], kv_budget, steps=2, warmup=1,
                             kv_chunk_bytes=chunk, param_chunk_bytes=chunk,
                             input_mean=input_mean, key=f"ct{port}", pipeline=True, pp=pp,
                             poison_drops=True)
        last = out["last"]
        q.put((rank, {"parity_fail": out["parity_fail"], "residents": out["residents_local"],
                      "kv": last.bytes_kv_exchange, "param": last.bytes_param,
                      "cons": last.bytes_kv_consolidate, "peer": last.bytes_pulled_peer,
                      "pulled": last.bytes_pulled, "pipe": out["pipeline"],
                      "groups": out["group_sizes"]}))
    finally:
        dist.destroy_process_group()


# the KV budget stays below the dropped half of the parameters (the
# parameter-centric regime): tiny = 2 layers of 2 MiB, 4 MiB of KV
@pytest.mark.parametrize("shape_name,kv_budget,chunk,input_mean", [
    ("tiny", 4 << 20, 64 << 10, 300),
    ("llama3_8b", 4 << 30, 64 << 20, 1660),
])
def test_two_rank_cycle_bit_exact(shape_name, kv_budget, chunk, input_mean):
    """configs[2] in miniature: replica r on rank r, one PP-2 group spanning
    the ranks; exchange, restore and consolidation are pulls through peer
    views; weights and every long-lived resident's KV survive bit for bit."""
    res = _spawn(_cycle_worker, 2, shape_name, kv_budget, chunk, input_mean)
    for r in (0, 1):
        d = res[r]
        assert d["parity_fail"] == 0
        assert d["residents"] > 0
        assert d["kv"] > 0 and d["param"] > 0 and d["cons"] > 0
        assert d["peer"] == d["pulled"]   # every pull reads the other rank's pool
    # the two halves of the group move mirror-image byte counts
    assert res[0]["param"] == res[1]["param"]
    # pipelined decode of the merged group across the ranks: every
    # activation hand-off arrives bit for bit
    pipe = res[0]["pipe"]
    assert pipe["groups"] == 1 and pipe["handoff_bit_exact"]
    assert pipe["tokens_per_s"] > 0 and pipe["handoff_bytes_per_step"] > 0


@pytest.mark.parametrize("shape_name,kv_budget,chunk,input_mean", [
    ("llama3_8b", 1 << 30, 16 << 20, 1660),
    ("qwen25_14b", 2 << 30, 64 << 20, 1660),
])
def test_four_rank_pp4_cycle_bit_exact(shape_name, kv_budget, chunk, input_mean):
    """configs[3] in miniature (Qwen2.5-14B shape): four replicas on four
    ranks merge into one PP-4 group (three merges, 12 layers per member for
    Qwen); the exchange fans every resident's KV out to three peers,
    restore pulls 36 layers from three holders, consolidation fans back in
    -- all through peer views, bit for bit."""
    res = _spawn(_cycle_worker, 4, shape_name, kv_budget, chunk, input_mean, 4)
    for r in range(4):
        d = res[r]
        assert d["parity_fail"] == 0 and d["groups"] == [4]
        assert d["residents"] > 0 and d["kv"] > 0 and d["param"] > 0 and d["cons"] > 0
        assert d["peer"] == d["pulled"]
    # every member misses 3/4 of the layers and pulls all of them (a member
    # in the middle holds one range and misses two disjoint ones)
    L = SHAPES_L[shape_name]
    slab = SLAB[shape_name]
    assert all(res[r]["param"] == (L - L // 4) * slab for r in range(4))


def test_eight_rank_pp2_cycle_bit_exact():
    """configs[2] with its real replica count: eight Llama-3-8B replicas on
    eight ranks (sharing the test box's GPU) merge into four PP-2 groups;
    every group's exchange / restore / consolidation runs concurrently
    through peer views, and the merged groups decode as cross-rank
    pipelines with bit-exact activation hand-offs."""
    res = _spawn(_cycle_worker, 8, "llama3_8b", 1 << 30, 16 << 20, 1660, 2)
    for r in range(8):
        d = res[r]
        assert d["parity_fail"] == 0 and d["groups"] == [2, 2, 2, 2]
        assert d["residents"] > 0 and d["kv"] > 0 and d["param"] > 0 and d["cons"] > 0
        assert d["peer"] == d["pulled"]
        assert d["param"] == 16 * SLAB["llama3_8b"]
    pipe = res[0]["pipe"]
    assert pipe["groups"] == 4 and pipe["handoff_bit_exact"]


def _sweep_rank(rank, world, port, q):
    _init(rank, world, port)
    import torch.distributed as dist
    from paper_2412_18169_b200 import build
    build.build()
    from paper_2412_18169_b200 import runtime
    from paper_2412_18169_b200.dist import nvlink_sweep
    rt = runtime.Runtime(0)
    res = nvlink_sweep(rt, max_bytes=16 << 20, iters=2)
    dist.destroy_process_group()
    q.put((rank, res))


def test_nvlink_sweep_two_ranks_bytes_checked():
    """Config 5 across ranks (here two ranks on one GPU): 64 KiB x 2^k up to
    16 MiB pulled from the partner's CUDA-IPC-mapped buffer, every byte of
    the largest point checked against the owner's hash of its pattern."""
    res = _spawn(_sweep_rank, 2)
    for r in (0, 1):
        sizes = [s for s, _ in res[r]["sizes_gbs"]]
        assert sizes == [(64 << 10) << k for k in range(9)]
        assert res[r]["bytes_checked"] is True
