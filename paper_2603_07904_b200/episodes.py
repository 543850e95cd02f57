"""Episode data parallelism: host-side plumbing.

Independent episodes / rollouts are the unit that shards: each rank owns a
contiguous block of episode ids, holds a full replica of the packed weights
and its own kinematic state, and runs the hot path with no collective.  The
only cross-rank traffic is the end-of-run reduction of timings (max over
ranks, CUDA-event time) and counters (bit histograms, byte totals).

Everything here is torch.distributed plumbing over whatever backend the
process group uses (NCCL on the GPU box, gloo in the CPU tests); no method
arithmetic lives here.
"""
from __future__ import annotations

from typing import Dict, Iterable, List


def shard(n_episodes: int, world: int, rank: int) -> range:
    """Contiguous block of episode ids owned by `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if n_episodes < 0:
        raise ValueError("n_episodes < 0")
    base, extra = divmod(n_episodes, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def episode_seed(e: int, seed0: int = 2000) -> int:
    """Seed of episode e's synthetic trajectory (2000 + e)."""
    return seed0 + e


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the bench's device time)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def merge_histograms(hist: Dict[int, int], keys: Iterable[int] = (2, 4, 8, 16), device=None) -> Dict[int, int]:
    """Element-wise sum of per-rank bit histograms."""
    keys = list(keys)
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return {k: int(hist.get(k, 0)) for k in keys}
    import torch
    t = torch.tensor([hist.get(k, 0) for k in keys], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return {k: int(v) for k, v in zip(keys, t.tolist())}


def gather_per_episode(rows: List[list], n_episodes: int, device=None) -> List[list]:
    """All-gather per-episode records (e.g. the bit sequence of every episode)
    so rank 0 can compare a DP run against a single-rank run; rows[i] belongs to
    episode shard(n_episodes, world, rank)[i]."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return rows
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, rows)
    merged: List[list] = []
    for part in out:
        merged.extend(part)
    if len(merged) != n_episodes:
        raise RuntimeError(f"gathered {len(merged)} episodes, expected {n_episodes}")
    return merged


def throughput(units_per_rank: float, seconds_max: float) -> float:
    """Whole-job throughput: all ranks' units / the slowest rank's time."""
    return sum_over_ranks(units_per_rank) / seconds_max
