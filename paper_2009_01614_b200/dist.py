"""Host-side multi-process plumbing for bench.py --gpus N (torchrun, one process per GPU).

north_star fixes the method to one GPU: no sharding and no collectives in the data path. N > 1
therefore runs replicas. Every rank builds the full index and answers its own
query batch, seeded per rank. The only collectives are the barrier and the max-over-ranks
timing reduction below. These helpers are backend-agnostic: nccl in the bench, and gloo with
world_size 2 on CPU in tests/test_dist_gloo.py.
"""
from __future__ import annotations

import dataclasses

QUERY_SEED_STRIDE = 7919


def rank_workload(wl, rank: int):
    """The workload rank `rank` answers: the same collection, its own query seed."""
    if rank == 0:
        return wl
    return dataclasses.replace(wl, q_seed=wl.q_seed + QUERY_SEED_STRIDE * rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. device ms of the timed region) over all ranks."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_qps(queries_per_rank: int, steps: int, world: int, max_ms: float) -> float:
    """Whole-job queries/s: every rank's queries over the slowest rank's time."""
    return queries_per_rank * steps * world / (max_ms / 1e3)
