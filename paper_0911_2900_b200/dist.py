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
