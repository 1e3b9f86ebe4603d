"""GPU parity of the v14 attention kernel (csrc/attn14.cuh: one Q tile per CTA, S double-buffered in
TMEM, KV tiles alternating over two softmax pairs, the two-level promotion in a correction warpgroup)
against the paper-verbatim oracle, at the same bar as tests/test_gpu_parity.py.

The cases cover what is new in v14: an odd and an even number of KV tiles (the pair that holds the
last tile keeps the MUFU turn), a single KV tile (pair B idle: its partial sum is zero), ragged last
tiles, the 4-deep K/V ring and the 8-deep running-max ring wrapping (N = 2048: 16 KV tiles), GQA, and
the variants the kernel accepts (SageAttn2-8b, smooth V, the E4M3 carrier, head dim 64).
"""
import numpy as np
import pytest
import torch

import oracle as orc
from oracle import OracleConfig
from paper_2411_10958_b200 import sage2
from tests._gpu_helpers import to_np16
from tests.test_gpu_parity import _compare_out, _inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    orc.build()
    sage2.lib()


def _run(B, Hq, Hkv, N, d, kind, seed=0, **kw):
    q, k, v, qg, kg, vg = _inputs(B, Hq, Hkv, N, d, kind, seed=seed)
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d)
    sage2.prepare(qg, kg, vg, ws, kernel="v14", **kw)
    out = torch.full_like(qg, float("nan"))
    sage2.attention(out, ws, B, Hq, Hkv, N, d, kernel="v14", **kw)
    torch.cuda.synchronize()
    return q, k, v, qg, kg, vg, ws, out


V14_CASES = [
    # B, Hq, Hkv, N, d, kind
    (1, 2, 1, 128, 128, "structured"),     # one KV tile: pair B idle
    (1, 2, 1, 200, 128, "iid"),            # two tiles, ragged
    (1, 2, 2, 384, 128, "structured"),     # three tiles: pair A keeps the last turn
    (2, 4, 2, 1000, 128, "structured"),    # 8 tiles, ragged, GQA
    (1, 2, 1, 1100, 128, "iid"),           # 9 tiles (odd), ragged
    (1, 1, 1, 2048, 128, "structured"),    # 16 tiles: both rings wrap
    (1, 2, 1, 333, 64, "structured"),      # head dim 64
]


@pytest.mark.parametrize("B,Hq,Hkv,N,d,kind", V14_CASES)
def test_v14_output_parity(B, Hq, Hkv, N, d, kind):
    q, k, v, qg, kg, vg, ws, out = _run(B, Hq, Hkv, N, d, kind, seed=N)
    nT = (N + 127) // 128
    units = [(b, h, i) for b in range(B) for h in range(Hq) for i in range(nT)]
    if len(units) > 24:
        units = units[:: len(units) // 12] + [units[-1]]
    res = orc.sage2_forward_blocks(q.numpy(), k.numpy(), v.numpy(), units, OracleConfig(kv_tile=128), debug=True)
    err, cos, worst, used, rows = _compare_out(to_np16(out).astype(np.float64), res, units, N)
    print(f"v14 N={N} d={d}: max|err|={err:.3e} min cos={cos:.8f} max err/bar={worst:.3f} allowance rows={used}/{rows}")


@pytest.mark.parametrize("variant", ["int8", "smooth_v", "qk_e4m3"])
def test_v14_variants(variant):
    B, Hq, Hkv, N, d = 1, 2, 1, 700, 128
    kw = {variant: True}
    q, k, v, qg, kg, vg, ws, out = _run(B, Hq, Hkv, N, d, "structured", seed=5, **kw)
    units = [(0, h, i) for h in range(Hq) for i in range((N + 127) // 128)]
    cfg = OracleConfig(kv_tile=128)
    if variant == "int8":
        cfg = OracleConfig(kv_tile=128, qk_max=127, smooth_q=False)
    elif variant == "smooth_v":
        cfg = OracleConfig(kv_tile=128, smooth_v=True)
    res = orc.sage2_forward_blocks(q.numpy(), k.numpy(), v.numpy(), units, cfg, debug=True)
    _compare_out(to_np16(out).astype(np.float64), res, units, N)


def test_v14_carrier_equals_int8_lanes():
    """The E4M3 carrier yields the same integer S (C-24), so v14's output is bitwise the same."""
    B, Hq, Hkv, N, d = 1, 4, 2, 900, 128
    *_, out_i8 = _run(B, Hq, Hkv, N, d, "iid", seed=3)
    *_, out_f8 = _run(B, Hq, Hkv, N, d, "iid", seed=3, qk_e4m3=True)
    assert torch.equal(out_i8, out_f8)


def test_v14_deterministic_and_close_to_v8():
    """Bitwise deterministic; against v8 (the same b_kv, a different order of the row-sum and
    max bookkeeping) within one fp16 ulp of the output plus the P^ ambiguity of C-21."""
    B, Hq, Hkv, N, d = 2, 8, 4, 1500, 128
    q, k, v, qg, kg, vg, ws, out = _run(B, Hq, Hkv, N, d, "iid", seed=9)
    out2 = torch.empty_like(out)
    sage2.attention(out2, ws, B, Hq, Hkv, N, d, kernel="v14")
    ws8 = sage2.alloc_workspace(B, Hq, Hkv, N, d)
    sage2.prepare(qg, kg, vg, ws8, kernel="v8")
    out8 = torch.empty_like(out)
    sage2.attention(out8, ws8, B, Hq, Hkv, N, d, kernel="v8")
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    assert torch.isfinite(out.float()).all()
    diff = (out.float() - out8.float()).abs().max().item()
    assert diff <= 4e-3, diff


def test_v14_rejected_flags():
    B, Hq, Hkv, N, d = 1, 1, 1, 256, 128
    qg = torch.zeros(B, Hq, N, d, dtype=torch.float16, device="cuda")
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d, causal=True)
    with pytest.raises(Exception):
        sage2.prepare(qg, qg, qg, ws, causal=True, kernel="v14")
