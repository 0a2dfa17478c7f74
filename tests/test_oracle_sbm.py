"""Pins of the oracle's Alg. 2 SBM sampler (docs/SBM_SPEC.md) against things other than
itself: numpy's log (ln_spec64), uniformity of the stream, brute-force cell sums (RangeSum), the SBM law of
Def. 5 (each cell is an edge with probability 1 - exp(-lambda_ij), independently) checked by
frequencies over many seeds, and the degenerate parameters (Omega = 0, huge Omega)."""
import math

import numpy as np
import pytest
from scipy import stats

import oracle


def test_ln_spec64_vs_numpy():
    rng = np.random.default_rng(0)
    us = np.concatenate([rng.random(20000), np.exp(-rng.random(2000) * 36), [1.0, 0.5, 2.0 ** -53]])
    us = us[us > 0]
    for u in us:
        got, ref = oracle.ln_spec64(u), math.log(u)
        assert abs(got - ref) <= 2 * np.spacing(abs(ref)) + 1e-300


def test_uniform_stream():
    u = np.array([oracle.sbm_uniform(7, p, k, d) for p in range(3) for k in range(5) for d in range(400)])
    assert u.min() > 0 and u.max() <= 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-3
    assert len(np.unique(u)) == u.size


def _cells(tr, ts):
    if ts is None:
        n = len(tr)
        return [tr[a] * tr[b] for a in range(n) for b in range(a + 1, n)]
    return [tr[a] * ts[b] for a in range(len(tr)) for b in range(len(ts))]


@pytest.mark.parametrize("diag", [False, True])
def test_range_sum_brute_force(diag):
    rng = np.random.default_rng(1 + diag)
    for _ in range(30):
        tr = rng.uniform(0.1, 3.0, int(rng.integers(2, 9)))
        ts = None if diag else rng.uniform(0.1, 3.0, int(rng.integers(1, 9)))
        om = float(rng.uniform(0.01, 2.0))
        cells = om * np.array(_cells(tr, ts))
        T = cells.size
        for _ in range(20):
            x = int(rng.integers(0, T))
            y = int(rng.integers(x, T))
            ref = cells[x:y + 1].sum()
            assert abs(oracle.sbm_range_sum(tr, ts, om, x, y) - ref) <= 1e-12 * max(1.0, ref)


def _params(n, K, seed):
    rng = np.random.default_rng(seed)
    c = rng.integers(0, K, n).astype(np.int32)
    th = rng.uniform(0.3, 1.5, n)
    A = rng.uniform(0.05, 0.6, (K, K))
    om = (A + A.T) / 2 + np.eye(K) * 0.4
    return c, th, om


@pytest.mark.parametrize("q", [4, 20])
def test_edge_law(q):
    """Every node pair is an edge with probability 1 - exp(-theta_i theta_j Omega_{c_i c_j}) (Def. 5)."""
    n, K, S = 14, 3, 3000
    c, th, om = _params(n, K, 5)
    freq = np.zeros((n, n))
    for seed in range(S):
        src, dst = oracle.sbm_sample(c, th, om, seed, q=q)
        assert np.all(src != dst)
        key = np.minimum(src, dst) * n + np.maximum(src, dst)
        assert np.unique(key).size == key.size                     # simple graph
        freq[np.minimum(src, dst), np.maximum(src, dst)] += 1
    iu = np.triu_indices(n, 1)
    lam = th[iu[0]] * th[iu[1]] * om[c[iu[0]], c[iu[1]]]
    p = 1 - np.exp(-lam)
    f = freq[iu] / S
    z = (f - p) / np.sqrt(p * (1 - p) / S)
    assert np.max(np.abs(z)) < 4.5
    assert abs(stats.chisquare(freq[iu], p * S * (freq[iu].sum() / (p * S).sum())).pvalue) > 1e-4


def test_degenerate():
    c, th, om = _params(50, 4, 2)
    src, dst = oracle.sbm_sample(c, th, np.zeros_like(om), 3)
    assert src.size == 0
    src, dst = oracle.sbm_sample(c, th, om * 1e4, 3, q=6)    # every cell has an event
    assert src.size == 50 * 49 // 2
    src2, dst2 = oracle.sbm_sample(c, th, om * 1e4, 4, q=6)
    assert np.array_equal(src, src2) and np.array_equal(dst, dst2)   # the cell order does not depend on draws


def test_errors():
    c, th, om = _params(10, 2, 0)
    bad = om.copy()
    bad[0, 1] += 0.1
    for args in ((c, th, bad), (c, -th, om), (np.full(10, 5, np.int32), th, om)):
        with pytest.raises(oracle.OracleError):
            oracle.sbm_sample(*args, 1)
    with pytest.raises(oracle.OracleError):
        oracle.sbm_sample(c, th, om, 1, q=3)
