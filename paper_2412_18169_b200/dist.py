"""Multi-GPU control plane: one process per GPU, the plan shared by all.

The drop path shards into independent groups: plan_drop
(pkg/src/dropsim/planner.py:70-114) is deterministic, so every rank computes
the same plan from the same all-gathered group state and executes only the
merges whose members it owns -- no data-path collective.  Pairs of replicas
live on one GPU in the single-GPU configuration (rank r owns instances
k*r .. k*r+k-1); a merge that spans ranks is reported as remote (its KV
exchange needs the cross-process NVLink pool mapping, not built this round).

torch.distributed carries only metadata (object all-gathers, a max-reduce of
timings); it is plumbing for the multi-process launch bench.py gets from
torchrun, and the tests run it over gloo.
"""

from __future__ import annotations

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
