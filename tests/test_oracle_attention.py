"""Pins for the oracle's attention (no GPU).

* exact mode == dense softmax attention computed independently in numpy;
* smoothing leaves exact attention invariant (row-constant shift; P:306 for V);
* special cases N=1 (O=V), S=0 (O = mean of V), causal row invariance;
* S_int == numpy int64 matmul of the codes;
* quantized path == the naive second implementation (tests/_naive.py) on tiny inputs;
* two-level == single-level when R is exact (pure re-association);
* directions the paper states: two-level beats single-level under FP22 truncation (P:289-292,
  S:469), smoothing Q+K beats smoothing K beats none on outlier data.
"""
import numpy as np
import pytest

from oracle import OracleConfig
from tests._naive import sage2_naive


def dense_attention(Q, K, V, causal):
    """softmax(QK^T / sqrt(d)) V in fp64, written as the plain definition."""
    Q, K, V = (x.astype(np.float64) for x in (Q, K, V))
    N, d = Q.shape
    S = Q @ K.T / np.sqrt(d)
    if causal:
        S = np.where(np.tril(np.ones((N, N), bool)), S, -np.inf)
    S = S - S.max(axis=1, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=1, keepdims=True)
    return P @ V


def rnd(shape, seed, scale=1.0, mean=0.0):
    g = np.random.default_rng(seed)
    return (g.standard_normal(shape) * scale + mean).astype(np.float16)


@pytest.mark.parametrize("N,d", [(1, 64), (17, 64), (128, 128), (300, 64)])
@pytest.mark.parametrize("causal", [False, True])
def test_exact_mode_equals_dense(orc, N, d, causal):
    Q, K, V = rnd((N, d), 1), rnd((N, d), 2), rnd((N, d), 3)
    ref = dense_attention(Q, K, V, causal)
    cfg = OracleConfig(quant=False, causal=causal, smooth_q=False, smooth_k=False)
    assert np.max(np.abs(orc.attn_exact_tiled(Q, K, V, cfg) - ref)) < 1e-12


@pytest.mark.parametrize("causal", [False, True])
def test_smoothing_is_softmax_invariant(orc, causal):
    N, d = 300, 64
    Q, K, V = rnd((N, d), 4, 2, 3), rnd((N, d), 5, 2, -5), rnd((N, d), 6, 1, 8)
    ref = dense_attention(Q, K, V, causal)
    for sq, sk, sv in [(1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 1)]:
        cfg = OracleConfig(quant=False, causal=causal, smooth_q=bool(sq), smooth_k=bool(sk),
                           smooth_v=bool(sv))
        assert np.max(np.abs(orc.attn_exact_tiled(Q, K, V, cfg) - ref)) < 1e-10


def test_special_cases(orc):
    d = 64
    V = rnd((1, d), 7)
    O = orc.attn_exact_tiled(rnd((1, d), 8), rnd((1, d), 9), V, OracleConfig(quant=False))
    assert np.array_equal(O, V.astype(np.float64))          # N = 1: O = V
    N = 200
    V = rnd((N, d), 10)
    O = orc.attn_exact_tiled(np.zeros((N, d), np.float16), rnd((N, d), 11), V,
                             OracleConfig(quant=False, smooth_q=False, smooth_k=False))
    assert np.max(np.abs(O - V.astype(np.float64).mean(0))) < 1e-13   # S = 0


def test_causal_row_invariance(orc):
    N, d = 256, 64
    Q, K, V = rnd((N, d), 12), rnd((N, d), 13), rnd((N, d), 14)
    cfg = OracleConfig(quant=False, causal=True, smooth_q=False, smooth_k=False)
    O1 = orc.attn_exact_tiled(Q, K, V, cfg)
    K2, V2 = K.copy(), V.copy()
    K2[100:] = rnd((N - 100, d), 15)
    V2[100:] = rnd((N - 100, d), 16)
    O2 = orc.attn_exact_tiled(Q, K2, V2, cfg)
    assert np.array_equal(O1[:100], O2[:100])


def test_s_int_is_integer_matmul(orc):
    g = np.random.default_rng(17)
    qh = g.integers(-7, 8, size=(128, 128)).astype(np.int8)
    kh = g.integers(-7, 8, size=(384, 128)).astype(np.int8)
    assert np.array_equal(orc.s_int_block(qh, kh), qh.astype(np.int64) @ kh.astype(np.int64).T)


def _oracle_head(orc, Q, K, V, cfg):
    N, d = Q.shape
    q, k, v = Q[None, None], K[None, None], V[None, None]
    units = [(0, 0, i) for i in range(-(-N // 128))]
    O = orc.sage2_forward_blocks(q, k, v, units, cfg)["O"].reshape(-1, d)[:N]
    return O


@pytest.mark.parametrize("p_fp32", [True, False])
@pytest.mark.parametrize("N,kv_tile,causal,kind", [
    (16, 128, False, "iid"), (16, 4, True, "iid"), (13, 4, False, "outlier"),
    (9, 2, True, "outlier")])
def test_quantized_path_vs_naive(orc, N, kv_tile, causal, kind, p_fp32):
    d = 64
    if kind == "iid":
        Q, K, V = rnd((N, d), 20), rnd((N, d), 21), rnd((N, d), 22)
    else:
        Q, K, V = rnd((N, d), 23, 1, 4), rnd((N, d), 24, 1, -3), rnd((N, d), 25, 2, 8)
    cfg = OracleConfig(kv_tile=kv_tile, causal=causal, p_fp32=p_fp32)
    ref = sage2_naive(Q, K, V, causal=causal, kv_tile=kv_tile, p_fp32=p_fp32)
    got = _oracle_head(orc, Q, K, V, cfg)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_quantized_path_vs_naive_two_blocks(orc):
    N, d = 150, 64                      # two Q blocks, ragged second block
    Q, K, V = rnd((N, d), 26, 1, 1), rnd((N, d), 27), rnd((N, d), 28)
    ref = sage2_naive(Q, K, V, causal=True, kv_tile=64)
    got = _oracle_head(orc, Q, K, V, OracleConfig(kv_tile=64, causal=True))
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_two_level_equals_single_level_when_exact(orc):
    N, d = 512, 64
    Q, K, V = rnd((N, d), 30), rnd((N, d), 31), rnd((N, d), 32)
    a = _oracle_head(orc, Q, K, V, OracleConfig(two_level=True, pv_mode=0))
    b = _oracle_head(orc, Q, K, V, OracleConfig(two_level=False, pv_mode=0))
    assert np.max(np.abs(a - b)) < 1e-12


def test_single_tile_is_per_tile_formula(orc):
    """b_kv >= N: no online rescaling, O = sum e4m3(448 P~) V^ dV / (448 sum P~) exactly."""
    N, d = 100, 64
    Q, K, V = rnd((N, d), 33), rnd((N, d), 34), rnd((N, d), 35)
    a = _oracle_head(orc, Q, K, V, OracleConfig(kv_tile=128))
    ref = sage2_naive(Q, K, V, kv_tile=128)
    assert np.max(np.abs(a - ref)) < 1e-12


def test_two_level_beats_single_level_under_fp22(orc):
    """Direction of P:289-292 / S:469: with an FP22 accumulator and channel-biased V, confining
    the truncation to one block (two-level) is more accurate than one running accumulator."""
    N, d = 1024, 64
    wins = 0
    for seed in range(4):
        Q, K = rnd((N, d), 40 + seed), rnd((N, d), 50 + seed)
        V = rnd((N, d), 60 + seed, 1, 8.5)
        q, k, v = Q[None, None], K[None, None], V[None, None]
        units = [(0, 0, 7)]
        ref = orc.sage2_forward_blocks(q, k, v, units, OracleConfig(pv_mode=0))["O"]
        two = orc.sage2_forward_blocks(q, k, v, units, OracleConfig(pv_mode=2, two_level=True))["O"]
        one = orc.sage2_forward_blocks(q, k, v, units, OracleConfig(pv_mode=2, two_level=False))["O"]
        wins += orc.rmse(ref, two) < orc.rmse(ref, one)
    assert wins == 4


def test_smoothing_ordering_on_outlier_data(orc):
    """Direction of Table 4: Smooth Q+K > Smooth Q > Smooth K > None on
    channel-outlier data."""
    N, d = 512, 64
    g = np.random.default_rng(70)
    mu = g.uniform(-2, 2, d)
    mu[[3, 17, 40, 55]] = [20, -20, 20, -20]
    Q = (g.standard_normal((N, d)) + mu).astype(np.float16)
    K = (g.standard_normal((N, d)) + mu).astype(np.float16)
    V = g.standard_normal((N, d)).astype(np.float16)
    ref = dense_attention(Q, K, V, False)
    cos = {}
    for name, sq, sk in [("qk", 1, 1), ("q", 1, 0), ("k", 0, 1), ("none", 0, 0)]:
        O = _oracle_head(orc, Q, K, V, OracleConfig(smooth_q=bool(sq), smooth_k=bool(sk)))
        cos[name] = orc.cos_sim(ref, O)
    assert cos["qk"] > cos["q"] > cos["k"] > cos["none"]
    assert cos["qk"] > 0.98


def test_quantized_accuracy_iid(orc):
    """SageAttn2-4b on N(0,1) inputs stays close to exact attention (sanity, not a paper number)."""
    N, d = 512, 128
    Q, K, V = rnd((N, d), 80), rnd((N, d), 81), rnd((N, d), 82)
    ref = dense_attention(Q, K, V, False)
    O = _oracle_head(orc, Q, K, V, OracleConfig())
    assert orc.cos_sim(ref, O) > 0.97          # INT4 on pure noise: measured 0.978
    O8 = _oracle_head(orc, Q, K, V, OracleConfig(qk_max=127))
    assert orc.cos_sim(ref, O8) > 0.999        # INT8 (SageAttn2-8b) is more accurate


def test_smooth_v_constant_v_is_exact(orc):
    """Smooth V with V constant over tokens: V' = V - V_m = 0, so delta_V = 0, every
    V^ code is 0 and O = V_m = the V row exactly, whatever Q, K and the quantization of P do.
    Without smoothing the same V goes through E4M3 and is only approximated."""
    N, d = 300, 64
    row = rnd((1, d), 90, 3.0, 5.0)
    V = np.repeat(row, N, axis=0)
    Q, K = rnd((N, d), 91), rnd((N, d), 92)
    for causal in (False, True):
        O = _oracle_head(orc, Q, K, V, OracleConfig(smooth_v=True, causal=causal))
        assert np.array_equal(O, np.repeat(row.astype(np.float64), N, axis=0))
    O = _oracle_head(orc, Q, K, V, OracleConfig(smooth_v=False))
    assert not np.array_equal(O, np.repeat(row.astype(np.float64), N, axis=0))


def test_smooth_v_helps_channel_biased_v(orc):
    """Direction of P:798-799 (CosSim 98.25% -> 99.75% on a CogVideoX tensor): with a large
    per-channel bias on V (U(8, 9) on a quarter of the channels), smoothing V brings the
    quantized output closer to exact attention."""
    N, d = 512, 64
    g = np.random.default_rng(93)
    Q = g.standard_normal((N, d)).astype(np.float16)
    K = g.standard_normal((N, d)).astype(np.float16)
    bias = np.zeros(d)
    bias[g.permutation(d)[: d // 4]] = g.uniform(8, 9, d // 4)
    V = (g.standard_normal((N, d)) * 0.5 + bias).astype(np.float16)
    ref = dense_attention(Q, K, V, False)
    err = {}
    for sv in (False, True):
        O = _oracle_head(orc, Q, K, V, OracleConfig(smooth_v=sv))
        err[sv] = orc.rmse(ref, O)
    assert err[True] < err[False]


@pytest.mark.parametrize("gran", [1, 2, 3])
@pytest.mark.parametrize("N,kv_tile,causal", [(16, 4, True), (13, 128, False)])
def test_granularity_vs_naive(orc, gran, N, kv_tile, causal):
    """NEXT#4 ablation granularities (1 per-block, 2 per-token, 3 per-tensor) against the naive
    implementation, whose group lists are written out independently (tests/_naive.py)."""
    d = 64
    Q, K, V = rnd((N, d), 29, 1, 2), rnd((N, d), 30, 1, -1), rnd((N, d), 31)
    ref = sage2_naive(Q, K, V, causal=causal, kv_tile=kv_tile, gran=gran)
    got = _oracle_head(orc, Q, K, V, OracleConfig(kv_tile=kv_tile, causal=causal, qk_gran=gran))
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_per_tensor_spans_blocks(orc):
    """Per-tensor granularity takes ONE delta_Q over every Q block of the head (each
    block smoothed by its own mean): a head of three blocks against the naive implementation, and
    the delta equals the largest of the three per-block deltas."""
    N, d = 300, 64
    Q, K, V = rnd((N, d), 41, 1, 2), rnd((N, d), 42, 1, -1), rnd((N, d), 43)
    Q[140:150] *= 6.0                    # the block with the outliers sets the head's scale
    ref = sage2_naive(Q, K, V, kv_tile=128, gran=3)
    got = _oracle_head(orc, Q, K, V, OracleConfig(qk_gran=3))
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    dt = orc.q_head_delta(Q, OracleConfig(qk_gran=3))
    per_block = [orc.q_block(Q[r:r + 128], OracleConfig(qk_gran=1))["dq"][0] for r in (0, 128, 256)]
    assert dt == max(per_block)
    kv = orc.kv_head(K, V, OracleConfig(qk_gran=3))
    kv1 = orc.kv_head(K, V, OracleConfig(qk_gran=1))
    assert kv["dk"][0] == max(kv1["dk"]) and not np.any(kv["dk"][1:])


def test_granularity_accuracy_ordering(orc):
    """Direction of the paper's granularity ablation: finer groups are more accurate --
    per-token >= per-thread > per-block on channel-outlier data (INT4)."""
    N, d = 512, 64
    g = np.random.default_rng(71)
    mu = g.uniform(-2, 2, d)
    mu[[5, 30]] = [15, -15]
    scale = np.exp(g.normal(0, 1.0, (N, 1)))               # token-wise magnitude spread
    Q = ((g.standard_normal((N, d)) + mu) * scale).astype(np.float16)
    K = ((g.standard_normal((N, d)) + mu) * scale[::-1]).astype(np.float16)
    V = g.standard_normal((N, d)).astype(np.float16)
    ref = dense_attention(Q, K, V, False)
    err = {gr: orc.rmse(ref, _oracle_head(orc, Q, K, V, OracleConfig(qk_gran=gr))) for gr in (0, 1, 2)}
    assert err[2] <= err[0] < err[1], err
