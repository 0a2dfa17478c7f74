"""Pins of the oracle's CSR build, operators, projection, GCN and scoring against things OTHER than
itself: scipy/networkx routines, dense brute force built from networkx matrices, closed forms of
the paper's equations, SPEC.md / hand-derived worked examples (tests/golden/spec_examples.json),
and planted-partition recovery.

Paper passages: PAPER.md:56 (graph), :117 (M), :100 + :123 (Q, Q~), :129 (Eq. 5), :139-147 (Eq. 6 +
l2 normalisation), :70-73 (Eq. 1), :74-82 (Eq. 2), :88-100 (Eq. 3/4), :161-168 (Eq. 7).
"""
import json
import os

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
OPS = {"ncut": oracle.NCUT, "mod": oracle.MOD, "mod_reduced": oracle.MOD_REDUCED, "prop": oracle.PROP}


def _edges(e):
    e = np.asarray(e, np.int32).reshape(-1, 2)
    return e[:, 0].copy(), e[:, 1].copy()


def _scipy_csr(n, src, dst):
    keep = src != dst
    a = sp.coo_matrix((np.ones(keep.sum()), (src[keep], dst[keep])), shape=(n, n))
    a = (a + a.T).tocsr()
    a.sum_duplicates()
    a.data[:] = 1.0
    a.sort_indices()
    return a


def _nx_graph(g: oracle.CSR):
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    for i in range(g.n):
        for p in range(g.row_ptr[i], g.row_ptr[i + 1]):
            G.add_edge(i, int(g.col[p]))
    return G


GRAPHS = [
    ("random_small", lambda: (40, *synth.random_edges(40, 120, seed=1))),
    ("random_isolated", lambda: (60, *synth.random_edges(45, 80, seed=2))),   # nodes 45..59 isolated
    ("dcsbm_c1", lambda: (lambda g: (g.n, g.src, g.dst))(synth.generate("C1", 0))),
]


# ------------------------------------------------------------------ CSR
@pytest.mark.parametrize("name,make", GRAPHS)
def test_csr_matches_scipy_canonical(name, make):
    n, src, dst = make()
    g = oracle.build_csr(n, src, dst)
    ref = _scipy_csr(n, src, dst)
    np.testing.assert_array_equal(g.row_ptr, ref.indptr.astype(np.int64))
    np.testing.assert_array_equal(g.col, ref.indices.astype(np.int32))
    assert g.deg.sum() == g.nnz and g.nnz % 2 == 0          # Σ deg = 2|E|


@pytest.mark.parametrize("case", GOLD["csr"], ids=lambda c: c["cite"][:30])
def test_csr_spec_examples(case):
    src, dst = _edges(case["edges"])
    g = oracle.build_csr(case["n"], src, dst)
    assert g.row_ptr.tolist() == case["row_ptr"]
    assert g.col.tolist() == case["col"]
    assert g.deg.tolist() == case["deg"]


def test_csr_edge_cases_and_errors():
    g = oracle.build_csr(0, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert g.row_ptr.tolist() == [0] and g.nnz == 0
    g = oracle.build_csr(5, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert g.row_ptr.tolist() == [0] * 6
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_csr(3, np.array([0, 3], np.int32), np.array([1, 1], np.int32))
    assert e.value.code == 3                                # node id out of range = DATA
    with pytest.raises(oracle.OracleError):
        oracle.build_csr(3, np.array([-1], np.int32), np.array([1], np.int32))


# ------------------------------------------------------------------ operators
def _dense_ops(g: oracle.CSR):
    """Operators built independently from networkx (not from the oracle's formulas)."""
    G = _nx_graph(g)
    n = g.n
    A = nx.to_numpy_array(G, nodelist=range(n))
    d = A.sum(1)
    nz = d > 0
    Lsym = nx.normalized_laplacian_matrix(G, nodelist=range(n)).toarray()
    M = np.eye(n) - Lsym                     # M = D^-1/2 A D^-1/2 = I - L (Eq. 2)
    M[~nz, :] = 0.0                           # networkx puts 1 on the diagonal of isolated rows
    M[:, ~nz] = 0.0
    out = {"ncut": M, "adj": A}
    if d.sum() > 0:
        Q = nx.modularity_matrix(G, nodelist=range(n))   # Q_ij = A_ij - d_i d_j / 2e (Eq. 4)
        out["mod"] = np.asarray(Q)
        out["mod_reduced"] = np.where(A != 0, out["mod"], 0.0)   # Q~
    Ah = A + np.eye(n)
    dh = Ah.sum(1)
    out["prop"] = Ah / np.sqrt(np.outer(dh, dh))             # D^-1/2 (A+I) D^-1/2 (Eq. 6)
    return out


@pytest.mark.parametrize("name,make", GRAPHS)
@pytest.mark.parametrize("op", ["ncut", "mod", "mod_reduced", "prop"])
def test_apply_equals_dense_networkx_operator(name, make, op):
    n, src, dst = make()
    g = oracle.build_csr(n, src, dst)
    D = _dense_ops(g)
    X = np.random.default_rng(5).standard_normal((n, 7))
    got = oracle.apply(g, OPS[op], X)
    ref = D[op] @ X
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("case", GOLD["operator_entries"], ids=lambda c: c["cite"][:30])
def test_operator_spec_entries(case):
    src, dst = _edges(case["edges"]) if case["edges"] else (np.zeros(0, np.int32), np.zeros(0, np.int32))
    g = oracle.build_csr(case["n"], src, dst)
    # column j of X_op = X_op @ e_j
    for i, j, val in case["entries"]:
        e = np.zeros(case["n"])
        e[j] = 1.0
        assert abs(oracle.apply(g, OPS[case["op"]], e)[i] - val) < 1e-15


@pytest.mark.parametrize("name,make", GRAPHS)
def test_operator_closed_forms(name, make):
    n, src, dst = make()
    g = oracle.build_csr(n, src, dst)
    d = g.deg.astype(np.float64)
    nz = d > 0
    # M d^1/2 = d^1/2 on non-isolated rows (the top eigenvector of M, Eq. 2's L = I - M)
    Md = oracle.apply(g, oracle.NCUT, np.sqrt(d))
    np.testing.assert_allclose(Md[nz], np.sqrt(d)[nz], rtol=1e-13)
    assert np.all(Md[~nz] == 0.0)
    # P dhat^1/2 = dhat^1/2 (Eq. 6); SPEC.md:192's "row sums <= 1" is false and is NOT tested
    dh = np.sqrt(d + 1.0)
    np.testing.assert_allclose(oracle.apply(g, oracle.PROP, dh), dh, rtol=1e-13)
    # Q 1 = 0 (rows of the modularity matrix sum to zero, Eq. 4)
    assert np.max(np.abs(oracle.apply(g, oracle.MOD, np.ones(n)))) < 1e-12 * max(1.0, d.max())
    # D^-1 A 1 = 1 on non-isolated rows: D^-1/2 M D^1/2 1 = 1
    DinvA1 = oracle.apply(g, oracle.NCUT, np.sqrt(d))[nz] / np.sqrt(d[nz])
    np.testing.assert_allclose(DinvA1, 1.0, rtol=1e-13)


def test_mod_requires_edges():
    g = oracle.build_csr(4, np.zeros(0, np.int32), np.zeros(0, np.int32))
    for op in (oracle.MOD, oracle.MOD_REDUCED):
        with pytest.raises(oracle.OracleError) as e:
            oracle.apply(g, op, np.ones(4))
        assert e.value.code == 3                     # SPEC.md:125 degenerate input
    np.testing.assert_array_equal(oracle.apply(g, oracle.NCUT, np.ones(4)), 0.0)   # isolated -> zero rows


# ------------------------------------------------------------------ projection (Eq. 5)
@pytest.mark.parametrize("name,make", GRAPHS)
@pytest.mark.parametrize("variant", ["ncut", "mod", "mod_reduced"])
def test_project_is_dense_X_times_theta(name, make, variant):
    n, src, dst = make()
    g = oracle.build_csr(n, src, dst)
    r = 12
    Y = oracle.project(g, variant, r, seed=9)
    Th = oracle.theta(n, r, seed=9).astype(np.float64)
    ref = _dense_ops(g)[variant] @ Th
    assert np.max(np.abs(Y - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())


def test_projection_jl_distance_preservation():
    # N=64 random sparse X, L=32: ratio in [0.5, 1.5] for >= 95% of 100 sampled pairs
    n, src, dst = 64, *synth.random_edges(64, 300, seed=4)
    g = oracle.build_csr(n, src, dst)
    Mx = _dense_ops(g)["ncut"]
    Y = oracle.project(g, "ncut", 32, seed=1)
    rng = np.random.default_rng(0)
    ok = 0
    for _ in range(100):
        i, j = rng.choice(n, 2, replace=False)
        dx = np.linalg.norm(Mx[i] - Mx[j])
        if dx == 0:
            ok += 1
            continue
        ratio = np.linalg.norm(Y[i] - Y[j]) / dx
        ok += 0.5 <= ratio <= 1.5
    assert ok >= 95


# ------------------------------------------------------------------ GCN (Eq. 6 + l2 norm)
@pytest.mark.parametrize("name,make", GRAPHS)
def test_gcn_equals_dense_brute_force(name, make):
    n, src, dst = make()
    g = oracle.build_csr(n, src, dst)
    dims = [12, 9, 5]
    Y = oracle.project(g, "ncut", 12, seed=2)
    Zs = oracle.gcn(g, dims, seed=2, Y=Y)
    P = _dense_ops(g)["prop"]
    Z = Y
    for k in (1, 2):
        W = oracle.weights(k, dims[k - 1], dims[k], seed=2).astype(np.float64)
        H = np.tanh(P @ Z @ W)
        nrm = np.linalg.norm(H, axis=1, keepdims=True)
        Z = np.where(nrm > 0, H / np.where(nrm > 0, nrm, 1.0), 0.0)
        np.testing.assert_allclose(Zs[k - 1], Z, rtol=0, atol=1e-12)


def test_gcn_unit_rows_and_zero_rows():
    n, src, dst = 60, *synth.random_edges(45, 80, seed=2)
    g = oracle.build_csr(n, src, dst)
    Y = oracle.project(g, "ncut", 16, seed=0)
    Z = oracle.gcn(g, [16, 16, 8], seed=0, Y=Y)[-1]
    norms = np.linalg.norm(Z, axis=1)
    iso = g.deg == 0
    assert np.all(np.abs(norms[~iso] - 1.0) < 1e-12)
    assert np.all(Z[iso] == 0.0)                            # isolated: Y row 0 -> Z row 0 (reading #9/#10)


def test_gcn_permutation_equivariance():
    n, src, dst = 50, *synth.random_edges(50, 200, seed=8)
    g = oracle.build_csr(n, src, dst)
    Y = np.random.default_rng(0).standard_normal((n, 10))
    Z = oracle.gcn(g, [10, 8, 6], seed=4, Y=Y)[-1]
    pi = np.random.default_rng(1).permutation(n).astype(np.int32)
    g2 = oracle.build_csr(n, pi[src], pi[dst])
    Y2 = np.empty_like(Y)
    Y2[pi] = Y
    Z2 = oracle.gcn(g2, [10, 8, 6], seed=4, Y=Y2)[-1]
    np.testing.assert_allclose(Z2[pi], Z, atol=1e-12)


@pytest.mark.parametrize("variant", ["ncut", "mod", "mod_reduced"])
def test_embed_rows_identical_to_full(variant):
    gr = synth.generate("C1", 1)
    g = oracle.build_csr(gr.n, gr.src, gr.dst)
    dims = [16, 12, 8]
    Y = oracle.project(g, variant, 16, seed=5)
    Zs = oracle.gcn(g, dims, seed=5, Y=Y)
    rows = synth.sample_rows(gr.n, 25, seed=0)
    Yr, Zr = oracle.embed_rows(g, variant, 16, dims, 5, rows)
    np.testing.assert_array_equal(Yr, Y[rows])
    for k in range(2):
        np.testing.assert_array_equal(Zr[k], Zs[k][rows])


def test_embed_rows_identical_to_full_ragged_and_chunked():
    """Odd sketch width (generator quads cut at r) and n > 65536 (MOD's g streamed over several chunks)."""
    n = 70_001
    src, dst = synth.random_edges(n, 150_000, seed=9)
    g = oracle.build_csr(n, src, dst)
    dims = [10, 6]
    rows = np.concatenate([synth.sample_rows(n, 20, seed=1), [n - 1, 65_535, 65_536]])
    for variant in ("ncut", "mod"):
        Y = oracle.project(g, variant, 10, seed=2)
        Z = oracle.gcn(g, dims, seed=2, Y=Y)
        Yr, Zr = oracle.embed_rows(g, variant, 10, dims, 2, rows)
        np.testing.assert_array_equal(Yr, Y[rows])
        np.testing.assert_array_equal(Zr[0], Z[0][rows])


def test_thread_count_invariance():
    """the row loops may run under OpenMP because each output row is summed sequentially by one
    thread. Pin: one thread and all threads give bit-identical CSR, projections, GCN layers and sampled rows."""
    gr = synth.generate("C2", 0)
    dims = [16, 12, 8]
    rows = synth.sample_rows(gr.n, 30, seed=3)
    out = []
    try:
        for k in (1, 0):
            oracle.set_threads(k)
            g = oracle.build_csr(gr.n, gr.src, gr.dst)
            res = [g.row_ptr, g.col]
            for v in ("ncut", "mod", "mod_reduced"):
                Y = oracle.project(g, v, 16, seed=1)
                res += [Y] + oracle.gcn(g, dims, seed=1, Y=Y)
            Yr, Zr = oracle.embed_rows(g, "mod", 16, dims, 1, rows)
            res += [Yr] + Zr
            out.append(res)
    finally:
        oracle.set_threads(0)
    assert oracle.get_threads() >= 1
    for a, b in zip(*out):
        assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_planted_partition_recovery():
    """The pipeline recovers the planted blocks of C1-shaped DC-SBM graphs, and the GNN stage is what
    makes it work (paper Table II: ARI 0.9994 at N=1E3 with its own Alg. 1 and wider layers; Table IV:
    "w/o Emb" loses quality). Here KMeans with the true K is applied to Z and to Y. Statistical pin:
    mean ARI(Z) >= 0.75 and every seed >= 0.6 per variant; mean ARI(Z) - mean ARI(Y) >= 0.4."""
    from sklearn.cluster import KMeans
    from sklearn.metrics import adjusted_rand_score
    az = {v: [] for v in ("ncut", "mod", "mod_reduced")}
    ay = {v: [] for v in az}
    for seed in range(5):
        gr = synth.generate("C1", seed)
        g = oracle.build_csr(gr.n, gr.src, gr.dst)
        K = int(gr.labels.max()) + 1
        for v in az:
            Y = oracle.project(g, v, 64, seed=seed)
            Z = oracle.gcn(g, [64, 64, 32], seed=seed, Y=Y)[-1]
            az[v].append(adjusted_rand_score(gr.labels, KMeans(K, n_init=10, random_state=0).fit_predict(Z)))
            ay[v].append(adjusted_rand_score(gr.labels, KMeans(K, n_init=10, random_state=0).fit_predict(Y)))
    for v in az:
        assert np.mean(az[v]) >= 0.75 and min(az[v]) >= 0.6, (v, az[v])
        assert np.mean(az[v]) - np.mean(ay[v]) >= 0.4, (v, az[v], ay[v])


# ------------------------------------------------------------------ scoring (Eq. 1, 3, 7)
def _bruteforce_modularity(A, assign):
    two_e = A.sum()
    d = A.sum(1)
    q = 0.0
    n = len(assign)
    for i in range(n):
        for j in range(n):
            if assign[i] == assign[j]:
                q += A[i, j] - d[i] * d[j] / two_e
    return q / two_e


@pytest.mark.parametrize("seed", range(4))
def test_modularity_vs_networkx_and_bruteforce(seed):
    n, src, dst = 30, *synth.random_edges(30, 90, seed=seed)
    g = oracle.build_csr(n, src, dst)
    k = 4
    assign = np.random.default_rng(seed).integers(0, k, n).astype(np.int32)
    q = oracle.modularity(g, assign, k)
    G = _nx_graph(g)
    comms = [set(np.flatnonzero(assign == c).tolist()) for c in range(k)]
    comms = [c for c in comms if c]
    assert abs(q - nx.community.modularity(G, comms)) < 1e-12
    A = nx.to_numpy_array(G, nodelist=range(n))
    assert abs(q - _bruteforce_modularity(A, assign)) < 1e-12
    # Eq. 4 trace form: tr(H^T Q H) / 2e with the 0/1 indicator H
    H = np.eye(k)[assign]
    QH = oracle.apply(g, oracle.MOD, H)
    assert abs(np.trace(H.T @ QH) / g.nnz - q) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_ncut_trace_identity(seed):
    n, src, dst = 30, *synth.random_edges(30, 90, seed=10 + seed)
    g = oracle.build_csr(n, src, dst)
    k = 3
    assign = np.random.default_rng(seed).integers(0, k, n).astype(np.int32)
    nc = oracle.ncut(g, assign, k)
    # Eq. 2: H_ir = sqrt(deg_i / vol_r) for i in C_r; tr(H^T L H) = 2 NCut with L = I - M
    d = g.deg.astype(np.float64)
    vol = np.bincount(assign, weights=d, minlength=k)
    H = np.zeros((n, k))
    for i in range(n):
        if vol[assign[i]] > 0:
            H[i, assign[i]] = np.sqrt(d[i] / vol[assign[i]])
    LH = H - oracle.apply(g, oracle.NCUT, H)
    assert abs(np.trace(H.T @ LH) - 2.0 * nc) < 1e-12
    # and the direct definition with networkx cut/volume (Eq. 1)
    G = _nx_graph(g)
    ref = 0.5 * sum(nx.cut_size(G, set(np.flatnonzero(assign == c))) / nx.volume(G, set(np.flatnonzero(assign == c)))
                    for c in range(k) if vol[c] > 0)
    assert abs(nc - ref) < 1e-12


@pytest.mark.parametrize("case", GOLD["scores"], ids=lambda c: c["cite"][:30])
def test_scores_spec_examples(case):
    src, dst = _edges(case["edges"])
    g = oracle.build_csr(case["n"], src, dst)
    a = np.asarray(case["assign"], np.int32)
    if "modularity" in case:
        assert abs(oracle.modularity(g, a, case["k"]) - case["modularity"]) < 1e-15
    if "ncut" in case:
        assert abs(oracle.ncut(g, a, case["k"]) - case["ncut"]) < 1e-15
    if "lmod" in case:
        assert abs(oracle.local_modularity(g, np.arange(case["n"]), a, case["k"]) - case["lmod"]) < 1e-15


@pytest.mark.parametrize("seed", range(4))
def test_local_modularity(seed):
    n, src, dst = 40, *synth.random_edges(40, 150, seed=20 + seed)
    g = oracle.build_csr(n, src, dst)
    rng = np.random.default_rng(seed)
    assign = rng.integers(0, 3, n).astype(np.int32)
    # LMod(U = V) == Newman modularity (Eq. 7 vs Eq. 3)
    assert abs(oracle.local_modularity(g, np.arange(n), assign, 3) - oracle.modularity(g, assign, 3)) < 1e-12
    # subset U: brute force from Def. 6 with FULL-graph degrees
    U = np.sort(rng.choice(n, 25, replace=False))
    b = rng.integers(0, 2, U.size).astype(np.int32)
    G = _nx_graph(g)
    A = nx.to_numpy_array(G, nodelist=range(n))
    d = A.sum(1)
    mbar = np.array([d[U[b == c]].sum() for c in range(2)])
    m = np.array([A[np.ix_(U[b == c], U[b == c])].sum() / 2 for c in range(2)])
    e = mbar.sum() / 2
    ref = float(np.sum(m / e - (mbar / (2 * e)) ** 2))
    assert abs(oracle.local_modularity(g, U, b, 2) - ref) < 1e-12


@pytest.mark.parametrize("dims", [(64, 64, 32), (32, 48, 16, 8)])
def test_gcn_np_matches_c_oracle(dims):
    """The numpy-matmul GCN used for Table I widths equals the C oracle's loops (same steps, fp64)."""
    gr = synth.generate("C1", 2)
    g = oracle.build_csr(gr.n, gr.src, gr.dst)
    Y = oracle.project(g, "mod", dims[0], 0)
    ref = oracle.gcn(g, dims, 0, Y)
    got = oracle.gcn_np(g, dims, 0, Y)
    for a, b in zip(got, ref):
        assert np.max(np.abs(a - b)) <= 1e-12
