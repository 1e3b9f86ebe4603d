"""Accuracy metrics of the paper, Appendix "Accuracy metrics".

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  All three flatten O and O' to 1 x n
vectors and are computed in fp64.  Parity unpinned against the paper's printed values: those were
measured on real model activations; the tests check the metrics' definitions and the
paper's orderings only.
"""
import numpy as np


def _flat(x):
    return np.asarray(x, dtype=np.float64).reshape(-1)


def cos_sim(o, o_prime):
    """CosSim = sum(O O') / (sqrt(sum O^2) sqrt(sum O'^2))."""
    a, b = _flat(o), _flat(o_prime)
    return float(np.dot(a, b) / (np.sqrt(np.dot(a, a)) * np.sqrt(np.dot(b, b))))


def rel_l1(o, o_prime):
    """L1 = sum|O - O'| / sum|O|."""
    a, b = _flat(o), _flat(o_prime)
    return float(np.abs(a - b).sum() / np.abs(a).sum())


def rmse(o, o_prime):
    """RMSE = sqrt((1/n) sum (O - O')^2)."""
    a, b = _flat(o), _flat(o_prime)
    return float(np.sqrt(np.mean((a - b) ** 2)))
