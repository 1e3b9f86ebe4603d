"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

The whole workload runs through the product path exactly as `bench.py` runs it (sage2.prepare +
sage2.attention, default kernel, HBM-resident inputs); the CPU oracle then recomputes a sample of
whole 128-row Q blocks (first / middle / last block, incl. the ragged last block, of the first and
last (b, h_q)) one by one, and those outputs are held to the same bar as tests/test_gpu_parity.py
(elementwise max(2e-3, 1 fp16 ulp) against the paper-verbatim fp64 oracle plus the certified
ambiguity allowance of C-21, CosSim >= 0.9999).  Properties that
hold at any size are checked on the whole output:
  * every element finite;
  * |O[:, c]| <= (1 + 2^-2) max_t |V[t, c]| per channel (O is a P^-weighted mean of the rows of the
    E4M3-quantised V: V^ delta_V and P^/448 are each within one E4M3 rounding (2^-4) of V and P~,
    normalised by l = sum P~; 2^-2 leaves room for the subnormal P^ and the fp16 output rounding);
  * bitwise determinism of a second run.
"""
import numpy as np
import pytest
import torch

import oracle as orc
from oracle import OracleConfig
from paper_2411_10958_b200 import sage2, synth
from tests._gpu_helpers import kv_tile_for
from tests.test_gpu_parity import _compare_out

pytestmark = pytest.mark.gpu

# bench.py CONFIGS (name: B, H_q, H_kv, N, d, causal, kind)
FULL = {
    "c2_32k_d128": (4, 32, 32, 32768, 128, False, "iid"),
    "c2_32k_d128_causal": (4, 32, 32, 32768, 128, True, "iid"),
    "c2_32k_d64": (4, 32, 32, 32768, 64, False, "iid"),
    "c3_cogvideox": (1, 48, 48, 17776, 64, False, "structured"),
    "c4_llama_gqa": (1, 32, 8, 100000, 128, True, "iid"),
}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    orc.build()
    sage2.lib()


@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size_sampled_parity(name):
    B, Hq, Hkv, N, d, causal, kind = FULL[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0, device="cuda")
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d)
    out = torch.empty_like(q)
    sage2.prepare(q, k, v, ws, causal=causal)
    sage2.attention(out, ws, B, Hq, Hkv, N, d, causal=causal)
    out2 = torch.empty_like(q)
    sage2.prepare(q, k, v, ws, causal=causal)
    sage2.attention(out2, ws, B, Hq, Hkv, N, d, causal=causal)
    torch.cuda.synchronize()
    # properties of the whole output
    assert torch.isfinite(out).all()
    assert torch.equal(out, out2), "second run differs (determinism)"
    vmax = v.float().abs().amax(dim=2)                                  # [B, Hkv, d]
    grp = Hq // Hkv
    bound = vmax.repeat_interleave(grp, dim=1) * (1 + 2.0 ** -2) + 1e-3  # [B, Hq, d]
    omax = out.float().abs().amax(dim=2)
    assert bool((omax <= bound).all()), float((omax - bound).max())
    del out2, ws
    # sampled Q blocks against the oracle
    nT = (N + 127) // 128
    blocks = sorted({0, nT // 2, nT - 1})
    for (b, h) in [(0, 0), (B - 1, Hq - 1)]:
        hk = h // grp
        qn = q[b, hk * grp:(hk + 1) * grp].cpu().numpy()[None]
        kn = k[b, hk].cpu().numpy()[None, None]
        vn = v[b, hk].cpu().numpy()[None, None]
        units = [(0, h - hk * grp, i) for i in blocks]
        res = orc.sage2_forward_blocks(qn, kn, vn, units, OracleConfig(causal=causal, kv_tile=kv_tile_for(N, d, causal)),
                                       debug=True)
        o_gpu = out[b, hk * grp:(hk + 1) * grp].cpu().numpy().astype(np.float64)[None]
        err, cos, worst, used, rows = _compare_out(o_gpu, res, units, N)
        print(f"{name} (b={b}, h={h}) blocks {blocks}: max|err|={err:.3e} min cos={cos:.8f} max err/bar={worst:.3f} rows beyond the bar={used}/{rows}")
