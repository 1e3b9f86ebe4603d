"""A second, deliberately naive implementation of SageAttention2 (Alg. 1)
for tiny inputs, written independently of oracle/sage2_oracle.c (shares no code with it and
no code with the CUDA path).  Used only as a brute-force pin of the C oracle.

Number formats here come from libraries: numpy float32 arithmetic (IEEE), numpy float16 and
torch's float8_e4m3fn cast (on values clamped to +-448, which is what satfinite does).
Means are exact rationals (fractions.Fraction).  Everything else is fp64 Python floats.
"""
import math
from fractions import Fraction

import numpy as np
import torch


def _mean_f32(col):
    return np.float32(float(sum(Fraction(float(x)) for x in col) / len(col)))


def _e4m3(x):
    x = min(max(float(x), -448.0), 448.0)
    return float(torch.tensor([x], dtype=torch.float64).to(torch.float8_e4m3fn).to(torch.float64)[0])


def _qgroups(n_tokens):
    """Groups of the Q block as the paper lists them: tokens i, 8+i, 16+i, 24+i of every
    32-token warp tile."""
    groups = []
    for w in range(0, 128, 32):
        for i in range(8):
            groups.append([w + i + 8 * j for j in range(4) if w + i + 8 * j < n_tokens])
    return groups


def _kgroups(n_tokens, n_pad):
    """Groups of K: tokens 8k+2j and 8k+2j+1 of every 64-token block share group j."""
    groups = []
    for b in range(0, n_pad, 64):
        for j in range(4):
            toks = []
            for k in range(8):
                toks += [b + 8 * k + 2 * j, b + 8 * k + 2 * j + 1]
            groups.append([t for t in toks if t < n_tokens])
    return groups


def _qgroups_g(n_tokens, gran):
    """Q groups of a 128-token block for a granularity (NEXT#4): 0 per-thread, 1 the
    whole block, 2 one token each."""
    if gran == 1:
        return [list(range(n_tokens))]
    if gran == 2:
        return [[t] if t < n_tokens else [] for t in range(128)]
    return _qgroups(n_tokens)


def _kgroups_g(n_tokens, n_pad, gran):
    """K groups for a granularity: 0 per-thread, 1 64-token blocks, 2 tokens,
    3 the whole head (per-tensor)."""
    if gran == 3:
        return [list(range(n_tokens))]
    if gran == 1:
        return [[t for t in range(b, b + 64) if t < n_tokens] for b in range(0, n_pad, 64)]
    if gran == 2:
        return [[t] if t < n_tokens else [] for t in range(n_pad)]
    return _kgroups(n_tokens, n_pad)


def _quant_groups(X, groups, qmax, n_rows):
    codes = np.zeros((n_rows, X.shape[1]), np.int64)
    deltas = []
    for toks in groups:
        if not toks:
            deltas.append(np.float32(0))
            continue
        amax = np.float32(np.max(np.abs(X[toks])))
        delta = np.float32(amax / np.float32(qmax))
        deltas.append(delta)
        if delta == 0:
            continue
        for t in toks:
            q = (X[t] / delta).astype(np.float32)
            codes[t] = np.clip(np.rint(q), -qmax, qmax).astype(np.int64)
    return codes, deltas


def sage2_naive(Q, K, V, causal=False, kv_tile=128, qmax=7, p_fp32=False, gran=0):
    """Q, K, V: [N, d] float16 numpy (one head).  Returns O [N, d] fp64 before fp16 rounding.

    p_fp32: scores held as fp32 in base 2 (S log2 e) and 448 P~ rounded to fp32 before the
    E4M3 cast -- the kernel's precision for that decision (C-21); else fp64 with exp."""
    N, d = Q.shape
    n_pad = -(-N // 128) * 128
    Kf = K.astype(np.float32)
    kbar = np.array([_mean_f32(K[:, c].astype(np.float64)) for c in range(d)], np.float32)
    Kp = (Kf - kbar).astype(np.float32)                       # gamma(K) = K - mean(K)
    kgroups = _kgroups_g(N, n_pad, gran)
    khat, dks = _quant_groups(Kp, kgroups, qmax, N)
    dk_of = {}
    for gi, toks in enumerate(kgroups):
        for t in toks:
            dk_of[t] = dks[gi]
    Vf = V.astype(np.float32)
    dv = (np.max(np.abs(Vf), axis=0) / np.float32(448)).astype(np.float32)
    vhat = np.zeros((N, d))
    for t in range(N):
        for c in range(d):
            vhat[t, c] = 0.0 if dv[c] == 0 else _e4m3(np.float32(Vf[t, c] / dv[c]))
    O = np.zeros((N, d))
    qdelta_tensor = None
    if gran == 3:       # per-tensor: one delta_Q over every block's gamma(Q_i) of the head
        amax = np.float32(0)
        for b0 in range(0, N, 128):
            Qb = Q[b0:b0 + 128]
            qbar = np.array([_mean_f32(Qb[:, c].astype(np.float64)) for c in range(d)], np.float32)
            amax = max(amax, np.float32(np.max(np.abs((Qb.astype(np.float32) - qbar).astype(np.float32)))))
        qdelta_tensor = np.float32(amax / np.float32(qmax))
    for b0 in range(0, N, 128):
        rows = list(range(b0, min(b0 + 128, N)))
        Qb = Q[rows]
        qbar = np.array([_mean_f32(Qb[:, c].astype(np.float64)) for c in range(d)], np.float32)
        Qp = (Qb.astype(np.float32) - qbar).astype(np.float32)
        if gran == 3:
            qhat = np.zeros((len(rows), d), np.int64)
            if qdelta_tensor != 0:
                qhat = np.clip(np.rint((Qp / qdelta_tensor).astype(np.float32)), -qmax, qmax).astype(np.int64)
            dqs = [qdelta_tensor]
        else:
            qhat, dqs = _quant_groups(Qp, _qgroups_g(len(rows), gran), qmax, len(rows))
        dq_of = {}
        for gi, toks in enumerate(_qgroups_g(len(rows), 1 if gran == 3 else gran)):
            for t in toks:
                dq_of[t] = dqs[gi]
        dS = [sum(float(qbar[c]) * float(Kp[t, c]) for c in range(d)) for t in range(N)]
        for rr, r in enumerate(rows):
            m, l = -math.inf, 0.0
            o = np.zeros(d)
            last = r + 1 if causal else N
            for j0 in range(0, last, kv_tile):
                keys = [t for t in range(j0, min(j0 + kv_tile, last))]
                S = {}
                for t in keys:
                    s_int = int(sum(int(qhat[rr, c]) * int(khat[t, c]) for c in range(d)))
                    S[t] = (s_int * float(dq_of[rr]) * float(dk_of[t]) + dS[t]) / math.sqrt(d)
                    if p_fp32:
                        S[t] = float(np.float32(S[t] * math.log2(math.e)))
                m_new = max([m] + list(S.values()))
                if p_fp32:
                    alpha = 0.0 if m == -math.inf else 2.0 ** (m - m_new)
                else:
                    alpha = 0.0 if m == -math.inf else math.exp(m - m_new)
                R = np.zeros(d)
                rs = 0.0
                for t in keys:
                    if p_fp32:
                        p448 = float(np.float32(2.0 ** (S[t] - m_new + math.log2(448.0))))
                    else:
                        p448 = 448.0 * math.exp(S[t] - m_new)
                    rs += p448 / 448.0
                    R += _e4m3(p448) * vhat[t]
                l = alpha * l + rs
                o = alpha * o + R
                m = m_new
            O[r] = o / l / 448.0 * dv.astype(np.float64)
    return O
