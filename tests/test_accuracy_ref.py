"""The accuracy harness's fp64 reference (paper_2411_10958_b200/accuracy.py, used to report CosSim /
Rel-L1 / RMSE against full-precision attention) equals the oracle's exact mode (quantization
off: softmax attention) on small inputs, and its metrics equal the oracle's metric functions."""
import numpy as np
import pytest
import torch

import oracle as orc
from oracle import OracleConfig
from paper_2411_10958_b200 import accuracy, synth


@pytest.mark.parametrize("N,d,causal,kind", [(200, 64, False, "structured"), (300, 128, True, "iid"),
                                             (129, 64, True, "structured")])
def test_reference_equals_oracle_exact(N, d, causal, kind):
    q, k, v = synth.make_qkv(1, 2, 1, N, d, kind=kind, seed=5)
    rows = torch.arange(N)
    for h in range(2):
        ref = accuracy.exact_attention_rows(q[0, h], k[0, 0], v[0, 0], rows, causal).numpy()
        ex = orc.attn_exact_tiled(q[0, h].numpy(), k[0, 0].numpy(), v[0, 0].numpy(),
                                  OracleConfig(quant=False, causal=causal))
        assert np.max(np.abs(ref - ex)) <= 1e-10 * max(1.0, np.max(np.abs(ex)))


def test_sample_rows():
    assert accuracy.sample_rows(1000).tolist() == list(range(1000))
    r = accuracy.sample_rows(100000).tolist()
    assert r[:128] == list(range(128)) and r[-1] == 99999 and len(r) == 128 + 128 + 32
    assert r[128] == 128 * ((100000 + 127) // 128 // 2)


def test_metrics_match_oracle():
    g = np.random.default_rng(0)
    a, b = g.standard_normal((64, 32)), g.standard_normal((64, 32))
    m = accuracy.metrics(torch.from_numpy(a), torch.from_numpy(b))
    assert m["cos_sim"] == pytest.approx(orc.cos_sim(b, a), abs=1e-14)
    assert m["rel_l1"] == pytest.approx(orc.rel_l1(b, a), abs=1e-14)
    assert m["rmse"] == pytest.approx(orc.rmse(b, a), abs=1e-14)
