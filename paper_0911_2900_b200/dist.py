"""Multi-GPU plumbing: one process per GPU (torchrun), torch.distributed for the rendezvous.

The simulation itself is decomposed in the C library (strip.cu): each rank owns an
x-strip of the grid and exchanges, once per step, the walks that can touch another strip.  This
module only wires a rank's context to its transport:
  * NCCL (one process per GPU): rank 0 makes the ncclUniqueId, torch.distributed broadcasts it,
    and the library runs ncclAllGather on its own stream -- no Python in the step;
  * host (e.g. gloo on CPU tensors): a Python allgather callback, used by the tests to run two
    ranks on one GPU without their kernels waiting on each other.
`aggregate` is the benchmark's max-over-ranks time / sum-over-ranks work reduction.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def aggregate(wall_s: float, updates: float, device: torch.device | None = None) -> tuple[float, float]:
    """(max over ranks of wall_s, sum over ranks of updates); identity without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(wall_s), float(updates)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([wall_s, updates], dtype=torch.float64, device=device)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def strip_bounds(width: int, rank: int, world: int) -> tuple[int, int]:
    """Columns [lo, hi) of rank `rank` out of `world` near-equal strips (fp_strip_bounds)."""
    return rank * width // world, (rank + 1) * width // world


def gloo_allgather(group=None):
    """A host-transport allgather over torch.distributed CPU tensors (gloo)."""
    def ag(send: memoryview, recv: memoryview):
        world = dist.get_world_size(group)
        src = torch.frombuffer(bytearray(send), dtype=torch.uint8)
        out = torch.empty(world * len(send), dtype=torch.uint8)
        dist.all_gather_into_tensor(out, src, group=group)
        recv[:] = memoryview(out.numpy()).cast("B")
    return ag


def strip_rank(grid, field, roster, device: int, transport: str = "nccl", **kw):
    """This process's StripRank of the default process group (rank r owns strip r)."""
    from . import fastped as fp
    rank, world = dist.get_rank(), dist.get_world_size()
    if transport == "nccl":
        obj = [fp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return fp.StripRank(grid, field, roster, rank, world, device, nccl_id=obj[0], **kw)
    return fp.StripRank(grid, field, roster, rank, world, device, exchange=gloo_allgather(), **kw)


def gather_state(st) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """The whole roster (x, y, alive) on every rank, each agent from the rank that owns it."""
    from . import fastped as fp
    x, y, a = st.agents()
    o = st.owned()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (x.copy(), y.copy(), a.copy(), o.copy()))
    return fp.merge_strip_agents(parts)
