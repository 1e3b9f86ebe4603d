"""Pins for the oracle's smoothing and per-thread quantizers (no GPU).

Anchors: the paper's worked group examples and counts, SPEC's examples
(S:114-116), the 14x rule, quantizer fixed points and round-trip
bounds, exact rational means (C-1) and torch's e4m3 cast for V."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import OracleConfig

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
NOSMOOTH = OracleConfig(smooth_q=False, smooth_k=False)


def test_group_examples_from_paper(orc):
    for members in GOLD["q_group_members"]["members_of_group_i"]:
        assert len({orc.group_q(t) for t in members}) == 1
    gk = GOLD["k_group_members"]
    assert {orc.group_k(t) for t in gk["group0"]} == {0}
    assert {orc.group_k(t) for t in gk["group3"]} == {3}
    for t, g in GOLD["spec_group_examples"]["q"]:
        assert orc.group_q(t) == g
    for t, g in GOLD["spec_group_examples"]["k"]:
        assert orc.group_k(t) == g


def test_group_counts_and_partition(orc):
    cnt = GOLD["group_counts"]
    q = [orc.group_q(t) for t in range(128)]
    k = [orc.group_k(t) for t in range(64)]
    assert len(set(q)) == cnt["q_groups_per_128"] and all(q.count(g) == 4 for g in set(q))
    assert len(set(k)) == cnt["k_groups_per_64"] and all(k.count(g) == 16 for g in set(k))
    # every token maps to exactly one group and groups never straddle blocks
    for t in range(1024):
        assert orc.group_q(t) // 32 == t // 128
        assert orc.group_k(t) // 4 == t // 64
    # the members of a Q group are the rows one mma thread holds: {i, i+8, i+16, i+24} + 32w
    for t in range(256):
        same = [u for u in range(256) if orc.group_q(u) == orc.group_q(t)]
        assert same == [32 * (t // 32) + (t % 8) + 8 * j for j in range(4)]


def _q_groups_rows(g):
    return [32 * (g // 8) + (g % 8) + 8 * j for j in range(4)]


def test_quantizer_endpoints_and_fixed_point(orc):
    g = np.random.default_rng(0)
    d = 64
    # fixed point: X = delta * codes with a +-7 in every group returns the codes
    codes = g.integers(-7, 8, size=(128, d))
    delta = 2.0 ** g.integers(-6, 3, size=32)
    for gi in range(32):
        rows = _q_groups_rows(gi)
        codes[rows[0], 0] = 7 if gi % 2 else -7
    X = np.zeros((128, d))
    for gi in range(32):
        rows = _q_groups_rows(gi)
        X[rows] = codes[rows] * delta[gi]
    r = orc.q_block(X.astype(np.float16), NOSMOOTH)
    assert np.array_equal(r["qhat"].astype(int), codes)
    assert np.allclose(r["dq"], delta, rtol=0, atol=0)
    # endpoints: [1, -1] -> [7, -7]
    X = np.zeros((4, d))
    X[0, 0], X[0, 1] = 1.0, -1.0
    r = orc.q_block(X.astype(np.float16), NOSMOOTH)
    assert r["qhat"][0, 0] == 7 and r["qhat"][0, 1] == -7
    assert r["dq"][0] == np.float32(1.0) / np.float32(7.0)


def test_fourteen_times_rule(orc):
    ex = GOLD["fourteen_times_rule"]
    d = 64
    X = np.zeros((1, d))
    X[0, 0] = ex["group_max"]                    # delta = 1
    X[0, 1] = ex["zero_below"]                   # exactly 14x smaller: tie -> even (0)
    X[0, 2] = -ex["zero_below"]
    X[0, 3] = np.nextafter(np.float16(0.5), np.float16(1))   # just above -> 1
    X[0, 4] = 1.5                                # tie -> 2 (even)
    X[0, 5] = 2.5                                # tie -> 2 (even)
    r = orc.q_block(X.astype(np.float16), NOSMOOTH)
    assert list(r["qhat"][0, :6]) == [7, 0, 0, 1, 2, 2]


def test_zero_group(orc):
    X = np.zeros((128, 64), np.float16)
    X[0, 0] = 3.0                               # only group 0 non-zero
    r = orc.q_block(X, NOSMOOTH)
    assert r["dq"][0] > 0 and np.all(r["dq"][1:] == 0)
    assert np.count_nonzero(r["qhat"]) == 1     # C-5: zero groups -> codes 0, delta 0


def test_round_trip_bound(orc):
    g = np.random.default_rng(1)
    for d in (64, 128):
        X = (g.standard_normal((128, d)) * np.exp(g.standard_normal((128, 1)))).astype(np.float16)
        r = orc.q_block(X, NOSMOOTH)
        deq = np.zeros((128, d))
        for t in range(128):
            deq[t] = r["qhat"][t] * float(r["dq"][orc.group_q(t)])
            assert np.max(np.abs(deq[t] - X[t].astype(np.float64))) <= 0.5 * r["dq"][orc.group_q(t)] * (1 + 1e-6)
        assert np.max(np.abs(r["qhat"])) == 7


def test_exact_means(orc):
    g = np.random.default_rng(2)
    N, d = 1000, 64
    K = (g.standard_normal((N, d)) * 3 + 1).astype(np.float16)
    V = g.standard_normal((N, d)).astype(np.float16)
    kv = orc.kv_head(K, V, OracleConfig())
    for c in range(d):
        exact = sum(Fraction(float(x)) for x in K[:, c].astype(np.float64)) / N
        assert kv["kbar"][c] == np.float32(float(exact))
    # K' = fp32(K) - k_bar in fp32; column means of K' ~ 0
    assert np.array_equal(kv["kprime"], K.astype(np.float32) - kv["kbar"][None, :])
    assert np.max(np.abs(kv["kprime"].astype(np.float64).mean(0))) < 1e-5
    # q_bar of a partial block uses the present tokens only (C-18)
    qb = orc.q_block(K[:77], OracleConfig())
    for c in range(0, d, 7):
        exact = sum(Fraction(float(x)) for x in K[:77, c].astype(np.float64)) / 77
        assert qb["qbar"][c] == np.float32(float(exact))


def test_smooth_k_spec_example(orc):
    ex = GOLD["smooth_k_example"]
    K = np.array(ex["K"], np.float16)
    kv = orc.kv_head(K, K, OracleConfig())
    assert np.array_equal(kv["kbar"], np.array(ex["kbar"], np.float32))
    assert np.array_equal(kv["kprime"], np.array(ex["kprime"], np.float32))


def test_k_groups_and_padding(orc):
    g = np.random.default_rng(3)
    N, d = 200, 64                                # ragged: N_pad = 256
    K = g.standard_normal((N, d)).astype(np.float16)
    kv = orc.kv_head(K, K, OracleConfig())
    assert kv["khat"].shape == (256, d) and kv["dk"].shape == (16,)
    assert np.all(kv["khat"][N:] == 0)
    for gi in range(16):
        toks = [t for t in range(N) if orc.group_k(t) == gi]
        if not toks:
            assert kv["dk"][gi] == 0
            continue
        amax = np.max(np.abs(kv["kprime"][toks]))
        assert kv["dk"][gi] == np.float32(amax) / np.float32(7)
        assert np.max(np.abs(kv["khat"][toks])) == 7


def test_v_per_channel_fp8_matches_torch(orc):
    g = np.random.default_rng(4)
    N, d = 300, 128
    V = (g.standard_normal((N, d)) * np.exp(g.standard_normal((1, d)))).astype(np.float16)
    V[:, 5] = 0                                    # an all-zero channel: delta 0, codes 0
    kv = orc.kv_head(V, V, OracleConfig())
    dv_ref = np.max(np.abs(V.astype(np.float32)), axis=0) / np.float32(448.0)
    assert np.array_equal(kv["dv"], dv_ref.astype(np.float32))
    with np.errstate(divide="ignore", invalid="ignore"):
        x = V.astype(np.float32) / dv_ref[None, :]
    x = np.nan_to_num(np.clip(x, -448, 448))
    ref = torch.from_numpy(x.astype(np.float64)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(kv["vhat"][:N], ref)
    assert np.all(kv["vhat"][N:] == 0)
    dec = orc.e4m3_decode(kv["vhat"][:N])
    assert np.max(np.abs(dec)) == 448.0          # the channel max maps to the top code


@pytest.mark.parametrize("qk_max", [7, 127])
def test_code_range(orc, qk_max):
    g = np.random.default_rng(5)
    X = (g.standard_normal((128, 64)) * 10).astype(np.float16)
    r = orc.q_block(X, OracleConfig(qk_max=qk_max))
    assert np.max(np.abs(r["qhat"].astype(int))) == qk_max


def test_granularity_group_maps(orc):
    """NEXT#4: per-block / per-token group maps partition the tokens as their definitions say."""
    assert orc.ngroups(0) == (32, 8) and orc.ngroups(1) == (1, 2) and orc.ngroups(2) == (128, 128)
    assert {orc.group_q_g(t, 1) for t in range(128)} == {0}
    assert [orc.group_k_g(t, 1) for t in (0, 63, 64, 127, 128)] == [0, 0, 1, 1, 2]
    assert [orc.group_q_g(t, 2) for t in range(128)] == list(range(128))
    assert all(orc.group_q_g(t, 0) == orc.group_q(t) for t in range(128))
    assert all(orc.group_k_g(t, 0) == orc.group_k(t) for t in range(256))


def test_per_token_codes_reach_qmax_on_every_row(orc):
    """With per-token groups every non-zero row has a code of magnitude qmax (its own absmax maps
    to +-7), unlike per-block groups where only the block's extreme reaches it."""
    g = np.random.default_rng(5)
    Qb = (g.standard_normal((128, 64)) * np.exp(g.normal(0, 1, (128, 1)))).astype(np.float16)
    tok = orc.q_block(Qb, OracleConfig(qk_gran=2))
    blk = orc.q_block(Qb, OracleConfig(qk_gran=1))
    assert np.all(np.abs(tok["qhat"]).max(axis=1) == 7)
    assert len(blk["dq"]) == 1 and np.sum(np.abs(blk["qhat"]).max(axis=1) == 7) < 128
