"""Multi-GPU plumbing: env-index sharding and the rollout-statistics collectives.

Envs are independent. A batch of N global envs is therefore split into
contiguous per-rank ranges with no data-path collective:
- every rank builds the layout maxima from the global descriptor list;
- every rank keys RNG streams by the global env index, so the shards compose bitwise.

torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU tests) is used only
outside the step:
- the max-over-ranks of timings;
- a SUM all-reduce of episode statistics (a handful of scalars per rollout,
  SPEC.md:530-533, 588).
"""

from __future__ import annotations

import torch


def shard_range(num_envs: int, rank: int, world: int):
    """[lo, hi) global env indices owned by `rank` (contiguous, sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard ({rank}, {world})")
    return rank * num_envs // world, (rank + 1) * num_envs // world


STAT_FIELDS = ("episodes", "return_sum", "length_sum", "success_once", "success_at_end", "fail_once",
               "fail_at_end")


def _all_reduce(t: torch.Tensor, op, group=None) -> torch.Tensor:
    """In-place all-reduce; through host memory when the backend cannot reduce device tensors
    (gloo: the multi-rank smoke runs on one GPU and the CPU tests)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return t
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def reduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """SUM all-reduce of a statistics vector (e.g. STAT_FIELDS, float64) across ranks; a no-op
    when torch.distributed is not initialised."""
    import torch.distributed as dist

    return _all_reduce(stats, dist.ReduceOp.SUM, group)


def max_over_ranks(values: torch.Tensor, group=None) -> torch.Tensor:
    """Element-wise MAX across ranks (timings: the job is as slow as its slowest rank)."""
    import torch.distributed as dist

    return _all_reduce(values, dist.ReduceOp.MAX, group)


def describe(group=None) -> dict:
    """Communicator facts for logs: backend, world size, rank (None when not initialised)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return {"backend": None, "world_size": 1, "rank": 0}
    return {"backend": dist.get_backend(group), "world_size": dist.get_world_size(group),
            "rank": dist.get_rank(group)}


def summarize(stats: torch.Tensor) -> dict:
    """Mean episode metrics from a reduced statistics vector."""
    s = dict(zip(STAT_FIELDS, (float(x) for x in stats.tolist())))
    n = max(s["episodes"], 1.0)
    return {"episodes": int(s["episodes"]), "mean_return": s["return_sum"] / n, "mean_length": s["length_sum"] / n,
            "success_once": s["success_once"] / n, "success_at_end": s["success_at_end"] / n,
            "fail_once": s["fail_once"] / n, "fail_at_end": s["fail_at_end"] / n}
