"""Multi-GPU plumbing of the benchmark: one process per GPU (torchrun), each rank runs its own
replica of the workload; the job's throughput is the sum of the ranks' agent
updates over the slowest rank's device time."""
from __future__ import annotations

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


# ----------------------------------------------------------------- x-strip decomposition
# SURVEY 8e / DESIGN.md 6: rank r plans the agents standing in columns [x_lo, x_hi) of the grid
# (fp_plan_strip; the others' desired cells are zeroed), one SUM all-reduce over NVLink
# completes every rank's desired-cell arrays (each agent is planned by exactly one rank), and
# the motion -- a sequential walk in one global order -- runs on every rank on identical
# inputs, so every rank holds the whole, bit-identical state and nothing migrates.

def strip_bounds(width: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous columns of rank `rank` out of `world` near-equal strips."""
    return rank * width // world, (rank + 1) * width // world


class _DeviceArray:
    """Zero-copy view of an engine-owned device array (for torch.distributed collectives)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def device_int32(ptr: int, n: int) -> torch.Tensor:
    return torch.as_tensor(_DeviceArray(ptr, n), device="cuda")


class StripStepper:
    """step()/run() of one simulation decomposed over the ranks of the default process group."""

    def __init__(self, st, rank: int | None = None, world: int | None = None):
        self.st = st
        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        self.x_lo, self.x_hi = strip_bounds(st.grid.width, self.rank, self.world)

    def combine(self):
        """SUM all-reduce of the desired-cell arrays (in place, on the engine's device memory)."""
        if self.world == 1:
            return
        dxp, dyp = self.st.desired_device()
        n = self.st.n
        if n == 0:
            return
        dx, dy = device_int32(dxp, n), device_int32(dyp, n)
        dist.all_reduce(dx, op=dist.ReduceOp.SUM)
        dist.all_reduce(dy, op=dist.ReduceOp.SUM)
        torch.cuda.current_stream().synchronize()  # the engine's stream reads them next

    def step(self, params):
        from . import fastped as fp
        self.st.plan_strip(params.k_s, params.seed, self.x_lo, self.x_hi)
        self.combine()
        out = fp.move_phase(self.st, params)
        self.st.step = self.st.step + 1
        return fp.StepStats(self.st.alive, len(out.exited), out.displacement_cells)
