"""The lossless special case: pins of the oracle's quantized block loop (orc_attn_block_dbg, the
function that produces every GPU parity reference) against closed forms written from the paper.

Inputs are built so that every quantization step of Alg. 1 except the one being
tested is exact:
  * Q = q_bar_i + dQ_g * codes and K = k_bar + dK_g * codes with integer codes in [-7, 7],
    power-of-two scales that differ from group to group (P:223, P:872 groups) and codes that
    cancel in pairs inside every group, so the smoothing means are exactly q_bar_i
    and k_bar, gamma(Q) / gamma(K) are exactly dQ * codes / dK * codes and psi returns
    exactly those codes (every group holds a +-7, so delta = 7 * 2^-k / 7 exactly);
  * V = dV_c * E4M3 values with max 448 per channel, so V^ and delta_V are exact.
A wrong group map, a wrong or missing mean, a dropped Delta S, a wrong scale or tile
order then makes the result lossy and moves O far beyond the 1e-12 bar.

Two closed forms, neither sharing code with the oracle:
  * quant=False (P~ not quantized): O == softmax(Q K^T / sqrt(d)) V, the dense definition of
    P:77 (the north-star pin "quantization disabled => exact softmax attention"); smoothing K
    and Q leaves it invariant (row-constant shift);
  * quant=True: with m_j the running row max after KV tile j (Eq. 1), P~_j =
    exp(S_j - m_j) and P^_j = E4M3(448 P~_j) (torch's float8_e4m3fn cast: 448 P~ <= 448,
    no saturation involved), the two-level recurrence O_j = e^{m_{j-1}-m_j} O_{j-1} + P^_j V_j
     has the closed form O = sum_j e^{m_j - m_last} P^_j V_j, and
    l = sum_j e^{m_j - m_last} rowsum(P~_j) (reading C-13); out = O / l / 448.
"""
import numpy as np
import pytest
import torch

from oracle import OracleConfig


def _e4m3_values():
    """All finite non-negative E4M3 values (torch decode of every code byte)."""
    codes = torch.arange(0, 0x7F, dtype=torch.uint8)       # 0x7f is NaN
    return codes.view(torch.float8_e4m3fn).to(torch.float64).numpy()


def _e4m3_round(x):
    return torch.from_numpy(np.asarray(x, np.float64)).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def _paired_codes(rng, tokens, d, pairs):
    """Integer codes in [-7, 7] for `tokens` rows whose listed row pairs cancel column by column;
    rows not in any pair are 0.  Every pair gets one +-7 somewhere so each group's absmax is 7."""
    c = np.zeros((tokens, d), np.int64)
    for (a, b) in pairs:
        x = rng.integers(-7, 8, size=d)
        x[rng.integers(0, d)] = 7 * (1 if rng.random() < 0.5 else -1)
        c[a], c[b] = x, -x
    return c


def lossless_head(N, d, seed):
    """(Q, K, V) fp16 [N, d] of one head with exactly quantizable smoothed values, plus the exact
    gamma(Q), gamma(K) and the block means (float64)."""
    rng = np.random.default_rng(seed)
    # ---- K: pairs (8k+2j, 8k+2j+1) share group g_K = 4 floor(t/64) + j; one scale per group
    kpairs = [(t, t + 1) for t in range(0, N - 1, 2)]
    ck = _paired_codes(rng, N, d, kpairs)
    gk = 4 * (np.arange(N) // 64) + (np.arange(N) % 8) // 2
    dk = 2.0 ** -(4 + (gk * 7 + 3) % 3)                    # 2^-4 .. 2^-6, varies from group to group
    kbar = rng.integers(-8, 9, size=d) / 4.0                # multiples of 1/4 in [-2, 2]
    Kp = dk[:, None] * ck
    K = kbar[None, :] + Kp
    # ---- Q: per 128-token block; pairs (32w+i, 32w+i+8), (32w+i+16, 32w+i+24) share g_Q
    Q = np.zeros((N, d))
    Qp = np.zeros((N, d))
    qbars = []
    for b0 in range(0, N, 128):
        n = min(128, N - b0)
        pairs = []
        for w in range(0, 128, 32):
            for i in range(8):
                for m in (0, 16):
                    a, b = w + i + m, w + i + m + 8
                    if b < n:
                        pairs.append((a, b))
        cq = _paired_codes(rng, n, d, pairs)
        gq = 8 * (np.arange(n) // 32) + np.arange(n) % 8
        dq = 2.0 ** -(3 + (gq * 5 + 1) % 3)                 # 2^-3 .. 2^-5 per group
        qbar = rng.integers(-8, 9, size=d) / 4.0
        Qp[b0:b0 + n] = dq[:, None] * cq
        Q[b0:b0 + n] = qbar[None, :] + Qp[b0:b0 + n]
        qbars.append(qbar)
    # ---- V: dV_c * E4M3 values, each channel reaching 448 (P:278 delta_V = max|V| / 448)
    vals = _e4m3_values()
    e = rng.choice(np.concatenate([vals, -vals]), size=(N, d))
    e[rng.integers(0, N, size=d), np.arange(d)] = 448.0
    dv = 2.0 ** -(8 + np.arange(d) % 3)
    V = dv[None, :] * e
    for X in (Q, K, V):                                     # every value is exactly an fp16
        assert np.array_equal(X.astype(np.float16).astype(np.float64), X)
    return Q.astype(np.float16), K.astype(np.float16), V.astype(np.float16), Qp, Kp, qbars


def dense_softmax_attention(Q, K, V, causal):
    """softmax(Q K^T / sqrt(d)) V, fp64."""
    Q, K, V = (x.astype(np.float64) for x in (Q, K, V))
    N, d = Q.shape
    S = Q @ K.T * (1.0 / np.sqrt(d))
    if causal:
        S = np.where(np.tril(np.ones((N, N), bool)), S, -np.inf)
    P = np.exp(S - S.max(1, keepdims=True))
    return (P / P.sum(1, keepdims=True)) @ V


def closed_form_quantized_p(Qp, Kp, qbars, V, causal, kv_tile):
    """The quantized-P~ result in closed form (module docstring); S = (gamma(Q) gamma(K)^T +
    Delta S)/sqrt(d) with Delta S_i = q_bar_i gamma(K)^T."""
    N, d = Qp.shape
    V = V.astype(np.float64)
    out = np.zeros((N, d))
    for r in range(N):
        qbar = qbars[r // 128]
        s = (Kp @ Qp[r] + Kp @ qbar) * (1.0 / np.sqrt(d))
        kend = r + 1 if causal else N
        tiles = [(j0, min(j0 + kv_tile, kend)) for j0 in range(0, kend, kv_tile)]
        ms = np.maximum.accumulate([s[a:b].max() for a, b in tiles])
        num = np.zeros(d)
        l = 0.0
        for (a, b), m in zip(tiles, ms):
            p = np.exp(s[a:b] - m)
            w = np.exp(m - ms[-1])
            num += w * (_e4m3_round(448.0 * p) @ V[a:b])
            l += w * p.sum()
        out[r] = num / l / 448.0
    return out


def _oracle(orc, Q, K, V, cfg):
    N, d = Q.shape
    units = [(0, 0, i) for i in range(-(-N // 128))]
    res = orc.sage2_forward_blocks(Q[None, None], K[None, None], V[None, None], units, cfg, keep=True)
    return res["O"].reshape(-1, d)[:N], res


CASES = [(256, 64, False, 128), (300, 64, True, 128), (300, 128, False, 128), (200, 128, True, 64),
         (130, 64, False, 32)]


@pytest.mark.parametrize("N,d,causal,kv_tile", CASES)
def test_lossless_inputs_quantize_exactly(orc, N, d, causal, kv_tile):
    """The construction really is lossless for the oracle's preprocessing: codes reproduce gamma(Q),
    gamma(K) and V exactly, and the means are the constructed ones."""
    Q, K, V, Qp, Kp, qbars = lossless_head(N, d, seed=N + d)
    _, res = _oracle(orc, Q, K, V, OracleConfig(causal=causal, kv_tile=kv_tile))
    kv = res["kv"][(0, 0)]
    assert np.array_equal(kv["kprime"].astype(np.float64), Kp)
    gk = 4 * (np.arange(N) // 64) + (np.arange(N) % 8) // 2
    assert np.array_equal(kv["khat"][:N] * kv["dk"][gk][:, None].astype(np.float64), Kp)
    assert np.array_equal(orc.e4m3_decode(kv["vhat"][:N]) * kv["dv"].astype(np.float64),
                          V.astype(np.float64))
    for u, inter in enumerate(res["inter"]):
        qb = inter["qb"]
        n = min(128, N - 128 * u)
        gq = 8 * (np.arange(n) // 32) + np.arange(n) % 8
        assert np.array_equal(qb["qbar"].astype(np.float64), qbars[u])
        assert np.array_equal(qb["qhat"][:n] * qb["dq"][gq][:, None].astype(np.float64), Qp[128 * u:128 * u + n])


@pytest.mark.parametrize("N,d,causal,kv_tile", CASES)
def test_quant_off_equals_exact_softmax_attention(orc, N, d, causal, kv_tile):
    """quant=False through orc_attn_block_dbg == softmax(QK^T/sqrt(d))V, smoothing on."""
    Q, K, V, *_ = lossless_head(N, d, seed=N + d)
    got, _ = _oracle(orc, Q, K, V, OracleConfig(causal=causal, kv_tile=kv_tile, quant=False))
    ref = dense_softmax_attention(Q, K, V, causal)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("N,d,causal,kv_tile", CASES)
def test_quantized_p_equals_closed_form(orc, N, d, causal, kv_tile):
    """The default path (P~ -> E4M3) == the closed form of the two-level recurrence."""
    Q, K, V, Qp, Kp, qbars = lossless_head(N, d, seed=N + d)
    got, _ = _oracle(orc, Q, K, V, OracleConfig(causal=causal, kv_tile=kv_tile))
    ref = closed_form_quantized_p(Qp, Kp, qbars, V, causal, kv_tile)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())
    # and the P~ quantization is visible: the two closed forms differ
    assert np.max(np.abs(ref - dense_softmax_attention(Q, K, V, causal))) > 1e-6


def test_lossless_pin_detects_a_dropped_delta_s(orc):
    """Sanity of the pin itself: without Delta S (smooth_q on, the term of P:193 omitted) the closed
    form no longer matches -- i.e. the construction exercises Delta S."""
    N, d = 256, 64
    Q, K, V, Qp, Kp, qbars = lossless_head(N, d, seed=5)
    ref = closed_form_quantized_p(Qp, Kp, [np.zeros(d)] * 2, V, False, 128)
    got, _ = _oracle(orc, Q, K, V, OracleConfig())
    assert np.max(np.abs(got - ref)) > 1e-6
