"""Multi-GPU execution for the bench: independent replicas, one per rank.

The E2 commit is a strictly serial replay (every decision reads the state
left by all earlier ones), so there is no data-path collective: each rank
replays its own copy of the trace on its own device and the job throughput
is all decisions over the max-over-ranks time.
"""
from __future__ import annotations

import os


def dist_env():
    return (
        int(os.environ.get("WORLD_SIZE", "1")),
        int(os.environ.get("RANK", "0")),
        int(os.environ.get("LOCAL_RANK", "0")),
    )


def max_over_ranks(values, device=None):
    """Element-wise max of per-rank floats (barrier semantics of all_reduce)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def job_throughput(world_size: int, decisions_per_rank: int, step_ms_max: float) -> float:
    return world_size * decisions_per_rank / (step_ms_max / 1000.0)
