"""N>1 control plane over gloo (world size 2, CPU): every rank derives the
same drop plan from all-gathered group state and owns disjoint merges."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2412_18169_b200 import memory
    from paper_2412_18169_b200.core import Group, ModelSpec
    from paper_2412_18169_b200.dist import (RankView, gather_groups, global_plan, max_over_ranks,
                                            split_plan, sum_over_ranks)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = ModelSpec(num_layers=8, bytes_per_layer=2_000_000_000, kv_bytes_per_token=200_000)
        view = RankView(rank, world, per_rank=2)
        local = []
        for iid in view.instances:
            inst = memory.build_instance(iid, model, 24_000_000_000, 25_000_000_000)
            g = Group(gid=iid, member_instances=[iid], stage_layer_map={iid: (0, 8)})
            # an overloaded replica: 70k queued tokens vs 40k free
            local.append((g, 70_000, inst.kv.free_tokens * model.kv_bytes_per_token))
        groups = gather_groups(view, local)
        plan = global_plan(groups, model)
        mine, remote = split_plan(plan, view)
        t = max_over_ranks(1.0 + rank)
        s = sum_over_ranks(10.0)
        q.put((rank, plan.to_text(), [m.members for m in mine], [m.members for m in remote], t, s))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_plan_and_split_merges():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, text0, mine0, rem0, t0, s0), (r1, text1, mine1, rem1, t1, s1) = res
    assert text0 == text1                       # one plan everywhere
    assert "merges=2" in text0.splitlines()[0]  # 4 overloaded replicas -> 2 pairs
    assert mine0 == [(0, 1)] and mine1 == [(2, 3)]  # pairs stay on their GPU
    assert rem0 == [] and rem1 == []
    assert t0 == t1 == 2.0 and s0 == s1 == 20.0


def _fd_worker(rank, world, port, q):
    import tempfile

    import torch.distributed as dist

    from paper_2412_18169_b200.dist import exchange_fds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # two entries per rank, each a descriptor blob plus three open files
        mine, files = {}, []
        for k in range(2):
            iid = 10 * rank + k
            fds = []
            for j in range(3):
                f = tempfile.TemporaryFile()
                f.write(f"rank{rank}-entry{iid}-file{j}".encode())
                f.flush()
                files.append(f)
                fds.append(os.dup(f.fileno()))
            mine[iid] = (f"desc-{iid}".encode() * 5, fds)
        got = exchange_fds(mine, f"t{port}")
        for _, fds in mine.values():
            for fd in fds:
                os.close(fd)
        seen = {}
        for iid, (blob, fds) in sorted(got.items()):
            texts = []
            for fd in fds:
                # received fds share the sender's file offset with every
                # other receiver: positional reads only
                texts.append(os.pread(fd, 100, 0).decode())
                os.close(fd)
            seen[iid] = (blob.decode(), texts)
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_fd_exchange_passes_descriptors_between_ranks():
    """share_pools' transport: every rank receives every other rank's
    descriptor blobs and working file descriptors (SCM_RIGHTS)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        want = {}
        for peer in range(world):
            if peer == rank:
                continue
            for k in range(2):
                iid = 10 * peer + k
                want[iid] = (f"desc-{iid}" * 5, [f"rank{peer}-entry{iid}-file{j}" for j in range(3)])
        assert res[rank] == want
