"""Pins for the oracle's number formats (no GPU).

Each check compares the oracle against something other than itself: a library routine
(numpy's float16, torch's float8_e4m3fn), or a value the paper / SPEC prints
(tests/golden/paper_examples.json)."""
import json
import os

import numpy as np
import pytest
import torch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_e4m3_decode_all_codes_matches_torch(orc):
    codes = np.arange(256, dtype=np.uint8)
    mine = orc.e4m3_decode(codes)
    ref = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(mine), nan)
    assert np.array_equal(mine[~nan], ref[~nan])
    assert nan.sum() == 2                      # 0x7f and 0xff only: the "fn" variant has no inf


def test_e4m3_encode_is_inverse_of_decode(orc):
    codes = np.arange(256, dtype=np.uint8)
    vals = orc.e4m3_decode(codes)
    fin = ~np.isnan(vals)
    assert np.array_equal(orc.e4m3_encode(vals[fin]), codes[fin])


def test_e4m3_encode_rne_matches_torch_in_range(orc):
    g = np.random.default_rng(0)
    x = np.concatenate([g.standard_normal(200000) * s for s in (1e-3, 0.05, 1, 30, 200)])
    x = x[np.abs(x) < 448]
    # midpoints between adjacent codes exercise ties-to-even
    pos = np.sort(orc.e4m3_decode(np.arange(0, 127, dtype=np.uint8)))
    mids = (pos[1:] + pos[:-1]) / 2
    x = np.concatenate([x, mids, -mids])
    mine = orc.e4m3_decode(orc.e4m3_encode(x))
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(mine, ref)


def test_e4m3_paper_values(orc):
    assert orc.e4m3_decode(orc.e4m3_encode(np.array([GOLD["e4m3_max"]["value"]])))[0] == 448.0
    ex = GOLD["p_static_scale"]
    assert orc.e4m3_decode(orc.e4m3_encode(np.array([448.0 * ex["p_tilde"]])))[0] == ex["code_value"]
    sat = GOLD["e4m3_saturate"]
    for s in (1, -1):
        v = orc.e4m3_decode(orc.e4m3_encode(np.array([s * sat["x"], s * 1e30])))
        assert np.all(v == s * sat["value"])      # satfinite, never NaN (C-6)
    # 2^-10 is the tie between 0 and the smallest subnormal 2^-9 -> even (0)
    assert orc.e4m3_decode(orc.e4m3_encode(np.array([2.0 ** -10])))[0] == 0.0
    assert orc.e4m3_decode(orc.e4m3_encode(np.array([1.5 * 2.0 ** -10])))[0] == 2.0 ** -9


def test_fp16_decode_all_bit_patterns(orc):
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    mine = orc.fp16_decode(bits)
    ref = bits.view(np.float16).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(mine), nan)
    assert np.array_equal(mine[~nan], ref[~nan])


def test_fp16_round_matches_numpy(orc):
    g = np.random.default_rng(1)
    x = np.concatenate([g.standard_normal(300000) * s for s in (1e-6, 1e-3, 1, 1e3, 3e4)])
    halfs = np.arange(0, 0x7c00, dtype=np.uint16).view(np.float16).astype(np.float64)
    ties = (halfs[1:] + halfs[:-1]) / 2          # exact midpoints -> ties to even
    x = np.concatenate([x, ties, -ties, [65504.0, 65519.9, 65520.0, 1e6]])
    mine = orc.fp16_round(x)
    ref = x.astype(np.float16).astype(np.float64)
    assert np.array_equal(mine, ref)


def test_fp22_truncation_examples(orc):
    for xin, xout in GOLD["fp22"]["cases"]:
        assert orc.fp22_truncate(np.array([float(xin)], np.float32))[0] == np.float32(float(xout))


def test_fp22_truncation_bits(orc):
    g = np.random.default_rng(2)
    u = g.integers(0, 2 ** 32, size=1_000_000, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    fin = np.isfinite(x)
    y = orc.fp22_truncate(x[fin]).view(np.uint32)
    assert np.array_equal(y, u[fin] & np.uint32(0xFFFFFC00))
    # values with <= 13 mantissa bits pass through unchanged
    z = (u[fin] & np.uint32(0xFFFFFC00)).view(np.float32)
    assert np.array_equal(orc.fp22_truncate(z), z)


@pytest.mark.parametrize("name,fn", [("cos", "cos_sim"), ("rel_l1", "rel_l1"), ("rmse", "rmse")])
def test_metrics_examples(orc, name, fn):
    for a, b, want in GOLD["metrics"][name]:
        assert getattr(orc, fn)(np.array(a, float), np.array(b, float)) == pytest.approx(want, rel=1e-15)


def test_metrics_properties(orc):
    g = np.random.default_rng(3)
    o = g.standard_normal(1000)
    assert orc.cos_sim(o, o) == pytest.approx(1.0, abs=1e-15)
    assert orc.cos_sim(o, -o) == pytest.approx(-1.0, abs=1e-15)
    assert orc.cos_sim(o, 3.0 * o) == pytest.approx(1.0, abs=1e-15)
    assert orc.rel_l1(o, 2 * o) == pytest.approx(1.0, abs=1e-15)
    assert orc.rmse(2 * o, 2 * (o + 1)) == pytest.approx(2.0, abs=1e-12)


def test_accuracy_metric_definitions(orc):
    """P:895 metrics on hand-computable vectors: CosSim of parallel / orthogonal vectors, Rel-L1 =
    sum|O - O'| / sum|O|, RMSE = sqrt(mean (O - O')^2)."""
    a = np.array([1.0, 2.0, 2.0])
    assert abs(orc.cos_sim(a, 3 * a) - 1.0) < 1e-15
    assert abs(orc.cos_sim(np.array([1.0, 0.0]), np.array([0.0, 5.0]))) < 1e-15
    b = np.array([1.0, 1.0, 4.0])                      # |a - b| = (0, 1, 2)
    assert abs(orc.rel_l1(a, b) - 3.0 / 5.0) < 1e-15
    assert abs(orc.rmse(a, b) - np.sqrt(5.0 / 3.0)) < 1e-15
