"""Multi-GPU partitioning of the SageAttention2 forward (host logic only).

The independent unit of work is a (batch, kv-head) pair: one KV head and its H_q/H_kv query heads.
Every step of the hot path (smoothing means, per-thread quantization, Delta S, attention) stays
inside a unit, so ranks never exchange data on the hot path.

* strong scaling (north-star C5: a fixed B=8, H=32 batch over 1/2/4/8 GPUs): the B*H_kv units of
  the whole batch are split contiguously and evenly over the ranks (`split_units`); a rank runs its
  units as one launch of shape [n_units, H_q/H_kv, N, d] (H_kv = 1 per unit);
* weak scaling (any other config under torchrun): every rank runs the whole config on its own batch
  slice (`rank_units`).
NCCL is used only for the max-over-ranks timing reduction and, after the timed region, to gather the
outputs for validation (`gather_units`, `first_unit_check`).
"""
import torch


def all_units(B, Hkv):
    return [(b, h) for b in range(B) for h in range(Hkv)]


def split_units(units, rank, world):
    """Strong scaling: a contiguous, balanced split of a fixed unit list (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    n = len(units)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return units[lo:hi]


def rank_units(rank, world, B, Hkv):
    """Weak scaling: (b, h_kv) units of `rank` for a per-rank batch of B: batches rank*B .. rank*B+B-1."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return [(rank * B + b, h) for b in range(B) for h in range(Hkv)]


def max_over_ranks(x, world, device=None):
    """Max of a per-rank float (e.g. the rank's CUDA-event time) across ranks."""
    if world == 1:
        return float(x)
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, device=None):
    if world == 1:
        return float(x)
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_outputs(out, world):
    """Validation only (never on the hot path): all-gather every rank's equally shaped output tensor
    (NCCL over NVLink on the GPU box, gloo in the CPU tests).  Returns [out_rank0, ..., out_rank{w-1}]."""
    if world == 1:
        return [out]
    import torch.distributed as dist
    parts = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(parts, out.contiguous())
    return parts


def gather_units(out, n_units, world):
    """Validation gather for a strong split whose ranks may own different unit counts: `out` is this
    rank's [n_units, ...] output; it is zero-padded to the largest count, all-gathered, and trimmed.
    Returns the list of per-rank outputs [n_units_r, ...] in rank order."""
    if world == 1:
        return [out]
    import torch.distributed as dist
    counts = [None] * world
    dist.all_gather_object(counts, int(n_units))
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pad[:n_units] = out
    parts = gather_outputs(pad, world)
    return [p[:c] for p, c in zip(parts, counts)]


def first_unit_check(parts, recompute):
    """Rank-0 validation of a gather: for every rank r, `recompute(r)` re-runs that rank's first
    (b, h_kv) unit from its regenerated inputs and returns [group, N, d]; the gathered output of
    that unit must be bitwise identical (the path is deterministic and units are independent).
    Returns the list of ranks that mismatched."""
    bad = []
    for r, o in enumerate(parts):
        if o.shape[0] == 0:
            continue
        ref = recompute(r)
        if not torch.equal(o[0, : ref.shape[0]].to(ref.device), ref):
            bad.append(r)
    return bad
