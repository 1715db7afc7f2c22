"""B200-native parameter-centric overload path (KunServe, arXiv 2412.18169).

Host modules mirror the reference simulator's API (`dropsim`): core,
memory, planner, exchange, engine.  The device data plane (VMM slab pool,
paged KV pool, page/slab copy kernels, paged attention) lives in the C-ABI
library `_kb.so` built from csrc/ and is reached through `runtime`.
"""

from .core import (Chunk, Group, Instance, Microbatch, ModelShape, ModelSpec,  # noqa: F401
                   Request, RequestState, SHAPES, tpot, ttft)
from .planner import DropPlan, compute_demand, member_moves, plan_drop  # noqa: F401

__version__ = "0.1.0"
