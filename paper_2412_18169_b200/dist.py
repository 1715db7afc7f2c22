"""Multi-GPU control plane: one process per GPU, the plan shared by all.

The drop path shards into independent groups: plan_drop
(pkg/src/dropsim/planner.py:70-114) is deterministic, so every rank computes
the same plan from the same all-gathered group state and executes only the
merges whose members it owns -- no data-path collective.  Pairs of replicas
live on one GPU in the single-GPU configuration (rank r owns instances
k*r .. k*r+k-1); a merge that spans ranks is remote: its KV exchange and
restore run through peer views (share_pools): every rank exports its pools'
VMM handles as file descriptors, passes them to the other ranks over a
Unix socket (SCM_RIGHTS), and imports the peers' pools as read-only views
mapped in its own VA -- the copy kernels then pull pages and slabs over
NVLink (dist_cycle.DistCycle).

torch.distributed carries only metadata (object all-gathers, a max-reduce of
timings, barriers between the phases whose device work crosses ranks); it is
plumbing for the multi-process launch bench.py gets from torchrun, and the
tests run it over gloo.
"""

from __future__ import annotations

import os
import socket
import struct
import threading
from dataclasses import dataclass

from .core import Group, ModelSpec
from .planner import DropPlan, compute_demand, plan_drop


@dataclass
class RankView:
    rank: int
    world: int
    per_rank: int  # instances owned by each rank

    def owns(self, iid: int) -> bool:
        return iid // self.per_rank == self.rank

    @property
    def instances(self) -> list[int]:
        return list(range(self.rank * self.per_rank, (self.rank + 1) * self.per_rank))


def gather_groups(view: RankView, local: list[tuple[Group, int, int]]):
    """All-gather (group, pending_tokens, free_kv_bytes) of every rank's
    groups; returns them ordered by gid (the reference iterates sorted)."""
    import torch.distributed as dist
    out: list = [None] * view.world
    dist.all_gather_object(out, local)
    merged = [g for part in out for g in part]
    return sorted(merged, key=lambda t: t[0].gid)


def global_plan(groups_state, model: ModelSpec) -> DropPlan:
    """The same plan on every rank: demand summed per group in gid order
    (engine.py:621-625), then plan_drop."""
    demand = sum(compute_demand(p, f, model.kv_bytes_per_token) for _, p, f in groups_state)
    return plan_drop([g for g, _, _ in groups_state], demand, model)


def split_plan(plan: DropPlan, view: RankView):
    """(local merges, remote merges) for this rank: a merge is local when
    this rank owns every member; a merge with members on several ranks is
    remote (owned by the rank of its smallest member)."""
    local, remote = [], []
    for m in plan.merges:
        owners = {iid // view.per_rank for iid in m.members}
        if owners == {view.rank}:
            local.append(m)
        elif min(m.members) // view.per_rank == view.rank:
            remote.append(m)
    return local, remote


def max_over_ranks(x: float, device=None) -> float:
    """Max of a timing over ranks (timed regions report the slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------- fd passing

_MAX_FDS = 250  # below SCM_MAX_FD (253)


def _sock_name(key: str, rank: int) -> bytes:
    # Linux abstract namespace: nothing on the filesystem to clean up
    return f"\0kunserve-b200-{key}-{rank}".encode()


def exchange_fds(payloads: dict, key: str) -> dict:
    """All-to-all of (descriptor bytes, file descriptors) between the ranks
    of the default process group.  payloads: local id -> (bytes, [fd]);
    returns every other rank's entries as id -> (bytes, [fd]) with fds
    valid in this process (the caller owns and closes them).  File
    descriptors cannot travel through torch.distributed, so each rank serves
    its payloads on a Unix SEQPACKET socket (SCM_RIGHTS, one message per
    entry) and connects to every other rank's socket."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_SEQPACKET)
    srv.bind(_sock_name(key, rank))
    srv.listen(world)
    for k, (_, fds) in payloads.items():
        if len(fds) > _MAX_FDS:
            raise ValueError(f"entry {k}: {len(fds)} fds exceed one SCM_RIGHTS message")

    def serve():
        for _ in range(world - 1):
            conn, _ = srv.accept()
            with conn:
                conn.sendall(struct.pack("<q", len(payloads)))
                for k, (blob, fds) in sorted(payloads.items()):
                    socket.send_fds(conn, [struct.pack("<qq", k, len(fds)) + blob], fds)
                conn.recv(1)  # the peer holds its copies: done

    th = threading.Thread(target=serve, daemon=True)
    th.start()
    dist.barrier()  # every listener is up
    out = {}
    try:
        for peer in range(world):
            if peer == rank:
                continue
            with socket.socket(socket.AF_UNIX, socket.SOCK_SEQPACKET) as c:
                c.connect(_sock_name(key, peer))
                n = struct.unpack("<q", c.recv(8))[0]
                for _ in range(n):
                    msg, fds, _flags, _addr = socket.recv_fds(c, 1 << 16, _MAX_FDS)
                    k, nfd = struct.unpack("<qq", msg[:16])
                    if len(fds) != nfd:
                        raise RuntimeError(f"entry {k}: received {len(fds)} of {nfd} fds")
                    out[k] = (msg[16:], list(fds))
                c.sendall(b"x")
    finally:
        th.join(timeout=60)
        srv.close()
    dist.barrier()
    return out


def share_pools(rt, local_pools: dict, model, shape, key: str = "pools") -> dict:
    """Export this rank's pools, import every other rank's as PeerPool views
    on this rank's device.  local_pools: iid -> DevicePool.  Returns
    iid -> PeerPool for the remote instances."""
    from .runtime import PeerPool
    mine = {iid: pool.export() for iid, pool in local_pools.items()}
    try:
        theirs = exchange_fds(mine, key)
    finally:
        for _, fds in mine.values():
            for fd in fds:
                os.close(fd)
    views = {}
    for iid, (blob, fds) in sorted(theirs.items()):
        try:
            views[iid] = PeerPool(rt, iid, model, shape, blob, fds)
        finally:
            for fd in fds:
                os.close(fd)
    return views


# ------------------------------------------------------ activation hand-off

class ActChannel:
    """Stage s -> s+1 activation hand-off between two ranks of a pipeline
    group (engine.py:428-448: the ACTIVATION task of every microbatch).

    The receiver owns `slots` device buffers (CUDA IPC-exported); the sender
    maps them and writes each microbatch's rows with the repo's copy kernel
    (runtime.copy_bytes: 16-byte stores into the peer's HBM over NVLink).
    Ordering never blocks a GPU: the sender records an interprocess CUDA
    event after the copy and publishes the microbatch number in a shared
    host counter; the receiver's stream waits on that event once the
    counter shows the record happened.  The receiver acknowledges a slot the
    same way (its event after the consuming stage), so the sender reuses a
    slot only after the receiver is done with it.  Both sides poll the host
    counters with a timeout instead of ever spinning on the device.
    """

    def __init__(self, rt, sender: int, receiver: int, slot_bytes: int, slots: int = 2,
                 key: str = "act", timeout_s: float = 120.0):
        import numpy as np
        import torch
        import torch.distributed as dist
        from multiprocessing import shared_memory
        from .runtime import IpcBuffer
        self.torch = torch
        self.rank = dist.get_rank()
        self.sender, self.receiver = sender, receiver
        self.is_sender = self.rank == sender
        assert self.rank in (sender, receiver)
        self.slot_bytes = (slot_bytes + 255) // 256 * 256
        self.slots = slots
        self.timeout_s = timeout_s
        self.device = rt.device
        name = f"kbact_{os.environ.get('MASTER_PORT', '0')}_{key}_{sender}_{receiver}"
        # the receiver creates the buffer, the counters and its ack event
        info = None
        if not self.is_sender:
            self.buf = IpcBuffer.allocate(rt.device, self.slot_bytes * slots)
            self.shm = shared_memory.SharedMemory(name=name, create=True, size=64)
            self.recv_ev = torch.cuda.Event(interprocess=True)
            info = (self.buf.export(), self.recv_ev.ipc_handle())
        objs = [None] * dist.get_world_size()
        dist.all_gather_object(objs, (self.rank, info))
        theirs = dict(objs)
        if self.is_sender:
            mem_h, ev_h = theirs[receiver]
            self.buf = IpcBuffer.open(rt.device, mem_h, self.slot_bytes * slots)
            self.shm = shared_memory.SharedMemory(name=name)
            try:  # the receiver owns (and unlinks) the segment
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
            self.recv_ev = torch.cuda.Event.from_ipc_handle(self.device, ev_h)
            self.send_ev = torch.cuda.Event(interprocess=True)
            h = self.send_ev.ipc_handle()
        else:
            h = None
        dist.all_gather_object(objs, (self.rank, h))
        if not self.is_sender:
            self.send_ev = torch.cuda.Event.from_ipc_handle(self.device, dict(objs)[sender])
        self.ctr = np.ndarray((2,), dtype=np.int64, buffer=self.shm.buf)  # [sent, acked]
        if not self.is_sender:
            self.ctr[:] = -1
        dist.barrier()
        self.n = 0

    def _poll(self, idx: int, want: int) -> None:
        import time
        t0 = time.perf_counter()
        while self.ctr[idx] < want:
            if time.perf_counter() - t0 > self.timeout_s:
                raise TimeoutError(f"activation channel {self.sender}->{self.receiver}: "
                                   f"waited {self.timeout_s}s for counter {idx} >= {want}")
            time.sleep(0)

    def slot(self, n: int):
        off = (n % self.slots) * self.slot_bytes
        return self.buf.tensor()[off:off + self.slot_bytes]

    def send(self, x, stream=None) -> int:
        """Hand x (contiguous device tensor) to the receiver as microbatch
        n = the n-th send; returns n."""
        from .runtime import copy_bytes
        torch = self.torch
        st = stream or torch.cuda.current_stream()
        n = self.n
        nbytes = x.numel() * x.element_size()
        if nbytes > self.slot_bytes:
            raise ValueError(f"{nbytes} activation bytes exceed the {self.slot_bytes}-byte slot")
        if n >= self.slots:  # the receiver is done with this slot's previous use
            self._poll(1, n - self.slots)
            st.wait_event(self.recv_ev)
        copy_bytes(self.buf.ptr + (n % self.slots) * self.slot_bytes, x.data_ptr(), nbytes,
                   stream=st)
        self.send_ev.record(st)
        self.ctr[0] = n
        self.n += 1
        return n

    def recv(self, nbytes: int, stream=None):
        """uint8 view of the next microbatch's rows; call done() after the
        stage consumed it."""
        torch = self.torch
        st = stream or torch.cuda.current_stream()
        n = self.n
        self._poll(0, n)
        st.wait_event(self.send_ev)
        return self.slot(n)[:nbytes]

    def done(self, stream=None) -> None:
        torch = self.torch
        st = stream or torch.cuda.current_stream()
        self.recv_ev.record(st)
        self.ctr[1] = self.n
        self.n += 1

    def close(self) -> None:
        import torch.distributed as dist
        self.torch.cuda.synchronize(self.device)
        dist.barrier()
        self.buf.close()
        self.shm.close()
        if not self.is_sender:
            dist.barrier()
            self.shm.unlink()
        else:
            dist.barrier()


def nvlink_sweep(rt, max_bytes: int = 2 << 30, iters: int = 5) -> dict:
    """Config 5 across GPUs: every rank pulls contiguous byte ranges (64 KiB
    x 2^k up to `max_bytes`) from its partner's (rank ^ 1) device buffer
    through a CUDA-IPC mapping with the repo's copy kernel -- the transfer a
    layer restore makes -- both directions at once.  Returns
    [[bytes, GB/s per direction], ...] with the time max-reduced over ranks.
    The buffers hold a (rank, offset) pattern; every byte of the largest
    point is checked against the owner's position-sensitive hash."""
    import torch
    import torch.distributed as dist
    from .runtime import IpcBuffer, copy_bytes, hash_tensor
    rank, world = dist.get_rank(), dist.get_world_size()
    peer = rank ^ 1
    mine = IpcBuffer.allocate(rt.device, max_bytes)
    words = mine.tensor().view(torch.int32)
    words.copy_((torch.arange(words.numel(), dtype=torch.int64, device=words.device) * 2654435761
                 + rank).remainder(1 << 31).to(torch.int32))
    my_hash = int(hash_tensor(mine.tensor()).item())
    objs = [None] * world
    dist.all_gather_object(objs, mine.export())
    theirs = IpcBuffer.open(rt.device, objs[peer], max_bytes) if peer < world else None
    dst = torch.empty(max_bytes, dtype=torch.uint8, device=f"cuda:{rt.device}")
    st = torch.cuda.current_stream()
    dev = f"cuda:{rt.device}" if dist.get_backend() == "nccl" else None
    out = []
    size = 64 << 10
    while size <= max_bytes:
        torch.cuda.synchronize(rt.device)
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if theirs is not None:
            copy_bytes(dst.data_ptr(), theirs.ptr, size, stream=st)  # warm-up
            a.record(st)
            for _ in range(iters):
                copy_bytes(dst.data_ptr(), theirs.ptr, size, stream=st)
            b.record(st)
            b.synchronize()
            ms = a.elapsed_time(b) / iters
        else:
            ms = 0.0
        ms = max_over_ranks(ms, device=dev)
        out.append([size, round(size / (ms / 1e3) / 1e9, 1) if ms > 0 else None])
        size *= 2
    torch.cuda.synchronize(rt.device)
    hashes = [None] * world
    dist.all_gather_object(hashes, my_hash)
    ok = (int(hash_tensor(dst).item()) == hashes[peer]) if theirs is not None else True
    dist.barrier()
    if theirs is not None:
        theirs.close()
    dist.barrier()
    mine.close()
    return {"sizes_gbs": out, "bytes_checked": ok,
            "unit": "GB/s per direction (each rank pulls from rank ^ 1 concurrently)"}
