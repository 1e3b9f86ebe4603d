"""Seeded synthetic Q/K/V generators (shared by the oracle side and the CUDA side).

This module holds NONE of the method's arithmetic: it only draws fp16 tensors with the shapes
and distributions of the paper's workloads (recipe in DESIGN.md "Inputs"):

* ``iid``        -- Q, K, V ~ N(0, 1), the kernel-benchmark protocol.
* ``structured`` -- Q, K ~ N(mu_c, 1) with per-channel means mu_c ~ U(-2, 2) and 4 outlier
  channels at +-20 shared by Q and K ("token-similar, channel-wise outliers", Fig. 2,
  PAPER.md:186; outliers injected as channel means per SPEC.md:406); V ~ N(0, 1) plus a channel
  bias U(8, 9) on a quarter of the channels ("ranging between 8 and 9").

Every (batch, kv-head) unit -- one KV head plus its H_q/H_kv query heads -- is drawn from its own
generator keyed by (seed, b, h_kv), so any rank can regenerate exactly its shard and a sharded run
sees bit-identical inputs to a 1-GPU run.
"""
import torch

KINDS = ("iid", "structured")


def _unit_seed(seed, b, hkv):
    return (int(seed) * 1_000_003 + int(b) * 10_007 + int(hkv) * 101 + 12345) & 0x7FFF_FFFF_FFFF


def make_unit(N, d, group, kind="iid", seed=0, b=0, hkv=0, device="cpu"):
    """One (b, h_kv) unit.  Returns q [group, N, d], k [N, d], v [N, d] (fp16 on device)."""
    if kind not in KINDS:
        raise ValueError(f"unknown input kind {kind!r}")
    g = torch.Generator(device=device)
    g.manual_seed(_unit_seed(seed, b, hkv))
    q = torch.randn((group, N, d), generator=g, device=device, dtype=torch.float32)
    k = torch.randn((N, d), generator=g, device=device, dtype=torch.float32)
    v = torch.randn((N, d), generator=g, device=device, dtype=torch.float32)
    if kind == "structured":
        mu = torch.rand((d,), generator=g, device=device) * 4.0 - 2.0
        perm = torch.randperm(d, generator=g, device=device)
        sign = torch.where(torch.rand((4,), generator=g, device=device) < 0.5, -1.0, 1.0)
        mu[perm[:4]] = 20.0 * sign
        q += mu
        k += mu
        vb = torch.zeros((d,), device=device)
        vperm = torch.randperm(d, generator=g, device=device)
        vb[vperm[: d // 4]] = 8.0 + torch.rand((d // 4,), generator=g, device=device)
        v += vb
    return q.half(), k.half(), v.half()


def make_qkv(B, Hq, Hkv, N, d, kind="iid", seed=0, device="cpu", units=None):
    """Full [B, H, N, d] fp16 tensors, or only the listed (b, h_kv) units.

    With ``units`` the returned tensors are [n_units, group, N, d] (q) and [n_units, N, d]
    (k, v), in the order given.
    """
    if Hq % Hkv:
        raise ValueError("H_q must be a multiple of H_kv")
    group = Hq // Hkv
    if units is None:
        q = torch.empty((B, Hq, N, d), dtype=torch.float16, device=device)
        k = torch.empty((B, Hkv, N, d), dtype=torch.float16, device=device)
        v = torch.empty((B, Hkv, N, d), dtype=torch.float16, device=device)
        for b in range(B):
            for h in range(Hkv):
                qu, ku, vu = make_unit(N, d, group, kind, seed, b, h, device)
                q[b, h * group:(h + 1) * group] = qu
                k[b, h] = ku
                v[b, h] = vu
        return q, k, v
    qs, ks, vs = [], [], []
    for (b, h) in units:
        qu, ku, vu = make_unit(N, d, group, kind, seed, b, h, device)
        qs.append(qu)
        ks.append(ku)
        vs.append(vu)
    return torch.stack(qs), torch.stack(ks), torch.stack(vs)
