"""Pins of the oracle's Alg. 1 (hierarchical model selection) and its deterministic 2-means
(docs/SELECT_SPEC.md) against things other than itself: hand-derived examples (tests/golden/select_examples.json),
scikit-learn's Lloyd iteration started from the same centres, networkx modularity (the global split test is
"splitting U lowers Mod(G)"), the oracle's LMod (Eq. 7, pinned in test_oracle_graph_ops.py) for
the literal local rule, permutation equivariance and planted-partition recovery.
"""
import json
import os

import networkx as nx
import numpy as np
import pytest
from sklearn.cluster import KMeans
from sklearn.metrics import adjusted_rand_score

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "select_examples.json")))


def _graph(case):
    src, dst = [], []
    for cl in case["cliques"]:
        for a in range(len(cl)):
            for b in range(a + 1, len(cl)):
                src.append(cl[a]); dst.append(cl[b])
    for u, v in case["extra_edges"]:
        src.append(u); dst.append(v)
    return oracle.build_csr(case["n"], np.array(src, np.int32), np.array(dst, np.int32))


def _Z(case):
    Z = np.zeros((case["n"], 2), np.float32)
    for vec, nodes in case["Z_groups"]:
        Z[nodes] = vec
    return Z


@pytest.mark.parametrize("case", GOLD["kmeans2"], ids=lambda c: c["cite"][:40])
def test_kmeans2_golden(case):
    Z = np.array(case["Z"], np.float32)
    side, it = oracle.kmeans2(Z, np.arange(len(Z)))
    assert side.tolist() == case["side"] and it == case["iterations"]


@pytest.mark.parametrize("case", GOLD["model_select"], ids=lambda c: c["cite"][:40])
@pytest.mark.parametrize("rule", ["global", "local"])
def test_model_select_golden(case, rule):
    labels, K, st = oracle.model_select(_graph(case), _Z(case), rule=rule)
    assert K == case["K"] and labels.tolist() == case["labels"] and st["blocks"] == K


def _blobs(rng, n, L, k=3, spread=0.25):
    c = rng.normal(size=(k, L))
    X = c[rng.integers(0, k, n)] + spread * rng.normal(size=(n, L))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return X.astype(np.float32)


def _seeds(Z, U):
    """SELECT_SPEC §3.1 seeding restated with numpy (the Lloyd part below is sklearn's, not ours)."""
    X = Z[U].astype(np.float64)
    mean = X.mean(axis=0)
    a = U[np.argmax(((X - mean) ** 2).sum(1))]
    b = U[np.argmax(((X - Z[a].astype(np.float64)) ** 2).sum(1))]
    return a, b


@pytest.mark.parametrize("seed", range(6))
def test_kmeans2_matches_sklearn_lloyd(seed):
    """From the same two starting centres, sklearn's strict-convergence Lloyd (tol=0) reaches the same split."""
    rng = np.random.default_rng(seed)
    n, L = int(rng.integers(50, 400)), int(rng.choice([4, 8, 32]))
    Z = _blobs(rng, n, L, k=int(rng.integers(2, 5)))
    U = np.sort(rng.choice(n, size=int(n * 0.8), replace=False)).astype(np.int32)
    side, it = oracle.kmeans2(Z, U, max_iter=300)
    a, b = _seeds(Z, U)
    km = KMeans(n_clusters=2, init=np.stack([Z[a], Z[b]]).astype(np.float64), n_init=1, max_iter=300, tol=0.0,
                algorithm="lloyd").fit(Z[U].astype(np.float64))
    assert np.array_equal(side, km.labels_.astype(np.uint8))
    assert 1 <= it <= 300


def test_kmeans2_fixed_point_of_lloyd():
    """A converged result is a Lloyd fixed point: each member is nearer its own side's mean."""
    rng = np.random.default_rng(7)
    Z = _blobs(rng, 300, 16, k=4)
    U = np.arange(300, dtype=np.int32)
    side, it = oracle.kmeans2(Z, U)
    X = Z.astype(np.float64)
    mu = [X[side == c].mean(0) for c in (0, 1)]
    d = np.stack([((X - m) ** 2).sum(1) for m in mu], 1)
    assert it < 100 and np.array_equal(side, (d[:, 1] < d[:, 0]).astype(np.uint8))


def _nx(g):
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    for i in range(g.n):
        for j in g.col[g.row_ptr[i]:g.row_ptr[i + 1]]:
            if i < j:
                G.add_edge(i, int(j))
    return G


@pytest.mark.parametrize("seed", range(4))
def test_split_test_global_is_modularity_decrease(seed):
    """Global rule: U stops iff splitting it into (U_1, U_2) lowers the modularity of G (Eq. 3, networkx)."""
    rng = np.random.default_rng(100 + seed)
    gr = synth.random_edges(120, 700, seed)
    g = oracle.build_csr(120, gr[0], gr[1])
    G = _nx(g)
    for _ in range(25):
        U = np.sort(rng.choice(120, size=int(rng.integers(20, 100)), replace=False)).astype(np.int32)
        side = rng.integers(0, 2, U.size).astype(np.uint8)
        U1, U2, rest = set(U[side == 0].tolist()), set(U[side == 1].tolist()), set(range(120)) - set(U.tolist())
        before = nx.community.modularity(G, [set(U.tolist()), rest] if rest else [set(U.tolist())])
        after = nx.community.modularity(G, [U1, U2, rest] if rest else [U1, U2])
        if abs(before - after) < 1e-12 or min(len(U1), len(U2)) <= 5:
            continue
        assert oracle.split_stops(g, U, side, rule="global") == (before > after)


@pytest.mark.parametrize("seed", range(4))
def test_split_test_local_is_lmod_comparison(seed):
    """Local rule (PAPER.md:167 literal): U stops iff LMod(U; G) > LMod(U_1, U_2; G) (Eq. 7)."""
    rng = np.random.default_rng(200 + seed)
    src, dst = synth.random_edges(150, 900, seed)
    g = oracle.build_csr(150, src, dst)
    for _ in range(25):
        U = np.sort(rng.choice(150, size=int(rng.integers(20, 120)), replace=False)).astype(np.int64)
        side = rng.integers(0, 2, U.size).astype(np.uint8)
        if min((side == 0).sum(), (side == 1).sum()) <= 5:
            continue
        m1 = oracle.local_modularity(g, U, np.zeros(U.size, np.int32), 1)
        m2 = oracle.local_modularity(g, U, side.astype(np.int32), 2)
        if abs(m1 - m2) < 1e-12:
            continue
        assert oracle.split_stops(g, U.astype(np.int32), side, rule="local") == (m1 > m2)


def _embed(g, cfg, variant):
    c = synth.CONFIGS[cfg]
    return oracle.gcn(g, list(c.dims), 0, oracle.project(g, variant, c.r, 0))[-1].astype(np.float32)


def test_permutation_equivariance():
    """Relabelling the nodes relabels the partition (no decision depends on node order except exact ties)."""
    gr = synth.generate("C1", 1)
    g = oracle.build_csr(gr.n, gr.src, gr.dst)
    Z = _embed(g, "C1", "mod")
    lab, K, _ = oracle.model_select(g, Z)
    perm = np.random.default_rng(3).permutation(gr.n).astype(np.int32)   # new id of node i = perm[i]
    g2 = oracle.build_csr(gr.n, perm[gr.src], perm[gr.dst])
    Z2 = np.empty_like(Z)
    Z2[perm] = Z
    lab2, K2, _ = oracle.model_select(g2, Z2)
    assert K2 == K and adjusted_rand_score(lab, lab2[perm]) == 1.0


def test_planted_recovery_c1():
    """On C1 DC-SBM graphs the Mod embedding + Alg. 1 recovers the planted blocks (ARI, K near the truth),
    and the partition's modularity approaches the planted partition's (PAPER.md:299-340 direction)."""
    aris, ks = [], []
    for seed in range(3):
        gr = synth.generate("C1", seed)
        g = oracle.build_csr(gr.n, gr.src, gr.dst)
        lab, K, st = oracle.model_select(g, _embed(g, "C1", "mod"))
        aris.append(adjusted_rand_score(gr.labels, lab))
        ks.append(K)
        assert oracle.modularity(g, lab, K) >= 0.8 * oracle.modularity(g, gr.labels, int(gr.labels.max()) + 1)
        assert np.array_equal(np.unique(lab), np.arange(K))
        first = [int(np.flatnonzero(lab == b)[0]) for b in range(K)]
        assert first == sorted(first)                  # canonical labels: ordered by smallest member
    assert np.mean(aris) >= 0.75 and all(6 <= k <= 25 for k in ks)


def test_local_rule_oversplits():
    """Reading #28's evidence: the literal local rule keeps splitting true blocks (K far above the truth)."""
    gr = synth.generate("C1", 0)
    g = oracle.build_csr(gr.n, gr.src, gr.dst)
    Z = _embed(g, "C1", "mod")
    _, Kg, _ = oracle.model_select(g, Z, rule="global")
    _, Kl, _ = oracle.model_select(g, Z, rule="local")
    assert Kl > 3 * Kg


def test_errors():
    g = oracle.build_csr(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32))
    Z = np.zeros((3, 4), np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.model_select(g, Z, eps=-1)
    with pytest.raises(oracle.OracleError):
        oracle.model_select(g, Z, max_iter=0)
    Z[1, 2] = 1.5
    with pytest.raises(oracle.OracleError):
        oracle.model_select(g, Z)
    Z[1, 2] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.model_select(g, Z)
    lab, K, _ = oracle.model_select(oracle.build_csr(0, np.zeros(0, np.int32), np.zeros(0, np.int32)),
                                    np.zeros((0, 4), np.float32))
    assert K == 0 and lab.size == 0
