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


def gather_outputs(out, world):
    """Validation only (never on the hot path): all-gather every rank's output tensor (NCCL over
    NVLink on the GPU box, gloo in the CPU tests).  Returns the list [out_rank0, ..., out_rank{w-1}]."""
    if world == 1:
        return [out]
    import torch.distributed as dist
    parts = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(parts, out.contiguous())
    return parts


def first_unit_check(parts, recompute):
    """Rank-0 validation of a gather: for every rank r, `recompute(r)` re-runs that rank's first
    (b, h_kv) unit from its regenerated inputs and returns [group, N, d]; the gathered output of
    that unit must be bitwise identical (the path is deterministic and units are independent).
    Returns the list of ranks that mismatched."""
    bad = []
    for r, o in enumerate(parts):
        ref = recompute(r)
        if not torch.equal(o[0, : ref.shape[0]].to(ref.device), ref):
            bad.append(r)
    return bad
