"""Multi-GPU partitioning of the SageAttention2 forward (host logic only).

The independent unit of work is a (batch, kv-head) pair: one KV head and its H_q/H_kv query heads.
Every step of the hot path (smoothing means, per-thread quantization, Delta S, attention) stays
inside a unit, so ranks never exchange data on the hot path.  bench.py runs
weak scaling: each rank owns the same number of units, drawn from its own batch slice.
"""
import torch


def rank_units(rank, world, B, Hkv):
    """(b, h_kv) units of `rank` for a per-rank batch of B (weak scaling): batches rank*B .. rank*B+B-1."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return [(rank * B + b, h) for b in range(B) for h in range(Hkv)]


def split_units(units, rank, world):
    """Strong-scaling alternative: a contiguous, balanced split of a fixed unit list."""
    n = len(units)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return units[lo:hi]


def max_over_ranks(x, world, device=None):
    """Max of a per-rank float (e.g. the rank's CUDA-event time) across ranks."""
    if world == 1:
        return float(x)
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
