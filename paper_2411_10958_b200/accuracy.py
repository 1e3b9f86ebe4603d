"""Accuracy of the SageAttn2 output against full-precision attention (BASELINE.json metric
"cos-sim vs FP32 attention"; the paper's three metrics).  Measurement harness only: nothing
here is on the product path (the forward pass runs in libsage2.so).

The reference is plain softmax attention, softmax(q k^T / sqrt(d)) v (causal = key <= query,
GQA head h -> kv head h / (H_q/H_kv)), evaluated in fp64 with torch on whatever device the inputs
live on, for a sample of query rows.  tests/test_accuracy_ref.py pins this reference to the oracle's
exact (quantization-off) mode, itself pinned to the textbook formula.
"""
import math

import torch


def exact_attention_rows(q, k, v, rows, causal=False):
    """O[rows] of one head in fp64.  q [N, d], k/v [N, d] (any float dtype, any device); rows: 1-D
    LongTensor of query indices.  Keys are processed in one shot per 1024-row chunk of queries."""
    d = q.shape[-1]
    out = []
    kk = k.double()
    vv = v.double()
    for r0 in range(0, rows.numel(), 1024):
        rr = rows[r0:r0 + 1024]
        s = (q[rr].double() @ kk.T) / math.sqrt(d)
        if causal:
            keys = torch.arange(k.shape[0], device=q.device)
            s = s.masked_fill(keys[None, :] > rr[:, None].to(q.device), float("-inf"))
        out.append(torch.softmax(s, dim=-1) @ vv)
    return torch.cat(out)


def metrics(o, o_ref):
    """CosSim, relative L1 and RMSE of o (quantized output) against o_ref (full precision), both
    flattened."""
    a = o.double().flatten()
    b = o_ref.double().flatten()
    cos = float((a * b).sum() / (a.norm() * b.norm()))
    rl1 = float((a - b).abs().sum() / b.abs().sum())
    rmse = float(((a - b) ** 2).mean().sqrt())
    return {"cos_sim": cos, "rel_l1": rl1, "rmse": rmse}


def sample_rows(N, full_up_to=4096):
    """Query rows compared per head: every row up to `full_up_to` tokens, else the first, a middle
    and the last (ragged) 128-row Q block."""
    if N <= full_up_to:
        return torch.arange(N)
    nT = (N + 127) // 128
    idx = []
    for i in (0, nT // 2, nT - 1):
        idx += list(range(128 * i, min(N, 128 * i + 128)))
    return torch.tensor(idx)


def evaluate(out, q, k, v, causal, heads, rows):
    """Metrics of out[b, h][rows] over the (b, h) pairs in `heads`, pooled into one vector."""
    Hq, Hkv = q.shape[1], k.shape[1]
    got, ref = [], []
    for b, h in heads:
        hk = h // (Hq // Hkv)
        ref.append(exact_attention_rows(q[b, h], k[b, hk], v[b, hk], rows.to(q.device), causal))
        got.append(out[b, h][rows.to(out.device)].double())
    return metrics(torch.cat(got), torch.cat(ref))
