"""GPU parity of NEXT-1 (Alg. 1 hierarchical model selection; docs/SELECT_SPEC.md) through the
C-ABI (raftgp_model_select) against the oracle's depth-first recursion.

Bar: the partition is an integer result decided by floating point, and both sides take every decision on
bit-identical numbers (SELECT_SPEC §2), so labels must match EXACTLY (canonical labels, SELECT_SPEC §5), as
must the block / split counts and the tree depth. The Z fed to both sides comes from the oracle's embedding
(never from the CUDA path). Cases: the hand-derived golden examples, C1-C3 embeddings (both variants, both
LMod readings), random clustered rows at every supported width with Lloyd caps that stop mid-iteration,
duplicate rows (argmax ties), isolated nodes (zero rows), eps = 0 and large eps, empty graphs, errors.
"""
import json
import os

import numpy as np
import pytest
import torch
from sklearn.metrics import adjusted_rand_score

import oracle
import synth

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "select_examples.json")))


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def _gpu_graph(rg, ctx, n, src, dst):
    return rg.raftgp_build_csr(ctx, n, torch.from_numpy(np.ascontiguousarray(src, np.int32)),
                               torch.from_numpy(np.ascontiguousarray(dst, np.int32)))


def _both(rg, ctx, n, src, dst, Z, **kw):
    go = oracle.build_csr(n, src, dst)
    ref, K, st = oracle.model_select(go, Z, **kw)
    g = _gpu_graph(rg, ctx, n, src, dst)
    lab, Kg, stg = rg.raftgp_model_select(g, torch.from_numpy(np.ascontiguousarray(Z)).cuda(), **kw)
    return ref, K, st, lab.cpu().numpy(), Kg, stg


def _check(ref, K, st, lab, Kg, stg):
    assert Kg == K
    assert np.array_equal(lab, ref), f"{(lab != ref).sum()} labels differ"
    assert stg["blocks"] == st["blocks"] and stg["splits"] == st["splits"] and stg["levels"] == st["depth"]


def _clique_case(case):
    src, dst = [], []
    for cl in case["cliques"]:
        for a in range(len(cl)):
            for b in range(a + 1, len(cl)):
                src.append(cl[a]); dst.append(cl[b])
    for u, v in case["extra_edges"]:
        src.append(u); dst.append(v)
    Z = np.zeros((case["n"], 8), np.float32)
    for vec, nodes in case["Z_groups"]:
        Z[nodes, :2] = vec
    return case["n"], np.array(src, np.int32), np.array(dst, np.int32), Z


@pytest.mark.parametrize("case", GOLD["model_select"], ids=lambda c: c["cite"][:40])
@pytest.mark.parametrize("rule", ["global", "local"])
def test_golden(rg, ctx, case, rule):
    n, src, dst, Z = _clique_case(case)
    ref, K, st, lab, Kg, stg = _both(rg, ctx, n, src, dst, Z, rule=rule)
    assert Kg == case["K"] and lab.tolist() == case["labels"]
    _check(ref, K, st, lab, Kg, stg)


def _oracle_Z(g, cfg, variant, seed=0):
    c = synth.CONFIGS[cfg]
    return oracle.gcn(g, list(c.dims), seed, oracle.project(g, variant, c.r, seed))[-1].astype(np.float32)


@pytest.mark.parametrize("cfg,gseed", [("C1", 0), ("C1", 1), ("C1", 2), ("C2", 0), ("C3", 0)])
@pytest.mark.parametrize("variant", ["ncut", "mod"])
def test_parity_sbm(rg, ctx, cfg, gseed, variant):
    if cfg == "C3" and variant == "ncut":
        pytest.skip("one C3 variant is enough (oracle time)")
    gr = synth.generate(cfg, gseed)
    go = oracle.build_csr(gr.n, gr.src, gr.dst)
    Z = _oracle_Z(go, cfg, variant)
    for rule in (["global", "local"] if cfg == "C1" else ["global"]):
        _check(*_both(rg, ctx, gr.n, gr.src, gr.dst, Z, rule=rule))


def _blob_Z(rng, n, L, k, spread, zero_rows=0, dup_rows=0):
    c = rng.normal(size=(k, L))
    X = c[rng.integers(0, k, n)] + spread * rng.normal(size=(n, L))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    if dup_rows:
        idx = rng.choice(n, size=dup_rows, replace=False)
        X[idx] = X[idx[0]]
    if zero_rows:
        X[rng.choice(n, size=zero_rows, replace=False)] = 0.0
    return X.astype(np.float32)


@pytest.mark.parametrize("L", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("max_iter,eps", [(100, 5), (1, 5), (2, 0), (3, 40)])
def test_parity_random(rg, ctx, L, max_iter, eps):
    rng = np.random.default_rng(L * 7 + max_iter)
    n = 3000 + L
    src, dst = synth.random_edges(n, 12 * n, seed=L + eps)
    Z = _blob_Z(rng, n, L, k=12, spread=0.6, zero_rows=37, dup_rows=25)
    _check(*_both(rg, ctx, n, src, dst, Z, eps=eps, max_iter=max_iter))


def test_isolated_and_tiny(rg, ctx):
    # two dense groups, a tail of isolated nodes (zero rows), and a graph smaller than 2 eps
    rng = np.random.default_rng(1)
    n = 400
    src = rng.integers(0, 150, 3000).astype(np.int32)
    dst = rng.integers(0, 150, 3000).astype(np.int32)
    Z = _blob_Z(rng, n, 16, k=3, spread=0.3)
    Z[150:] = 0.0
    _check(*_both(rg, ctx, n, src, dst, Z))
    _check(*_both(rg, ctx, 7, np.array([0, 1, 2], np.int32), np.array([1, 2, 3], np.int32), Z[:7]))
    # no edges at all: T = 0 -> one block
    ref, K, st, lab, Kg, stg = _both(rg, ctx, 50, np.zeros(0, np.int32), np.zeros(0, np.int32), Z[:50])
    _check(ref, K, st, lab, Kg, stg)
    assert Kg == 1


def test_empty_graph(rg, ctx):
    g = _gpu_graph(rg, ctx, 0, np.zeros(0, np.int32), np.zeros(0, np.int32))
    lab, K, st = rg.raftgp_model_select(g, torch.zeros((0, 8), dtype=torch.float32, device="cuda"))
    assert K == 0 and lab.numel() == 0


def test_errors(rg, ctx):
    src, dst = synth.random_edges(100, 400, seed=1)
    g = _gpu_graph(rg, ctx, 100, src, dst)
    Z = torch.zeros((100, 16), dtype=torch.float32, device="cuda")
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_model_select(g, torch.zeros((100, 12), dtype=torch.float32, device="cuda"))
    assert e.value.code == rg.RAFTGP_ERR_PARAM
    for kw in (dict(eps=-1), dict(max_iter=0), dict(rule=7)):
        with pytest.raises(rg.RaftGPError) as e:
            rg.raftgp_model_select(g, Z, **kw)
        assert e.value.code == rg.RAFTGP_ERR_PARAM
    Zb = Z.clone()
    Zb[17, 3] = 1.25
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_model_select(g, Zb)
    assert e.value.code == rg.RAFTGP_ERR_DATA
    Zb[17, 3] = float("nan")
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_model_select(g, Zb)
    assert e.value.code == rg.RAFTGP_ERR_DATA
    part = rg.raftgp_build_csr(ctx, 100, torch.from_numpy(src), torch.from_numpy(dst), 0, 50)
    part.set_degrees(torch.from_numpy(np.diff(oracle.build_csr(100, src, dst).row_ptr).astype(np.int32)).cuda())
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_model_select(part, Z)
    assert e.value.code == rg.RAFTGP_ERR_PARAM


def test_end_to_end_quality(rg, ctx):
    """GPU embed -> GPU Alg. 1 recovers the planted C1 blocks about as well as oracle embed -> oracle Alg. 1."""
    aris = []
    for seed in range(3):
        gr = synth.generate("C1", seed)
        g = _gpu_graph(rg, ctx, gr.n, gr.src, gr.dst)
        _, Z = rg.raftgp_embed(g, "mod", (64, 64, 32), 0, want_Y=False)
        lab, K, _ = rg.raftgp_model_select(g, Z)
        aris.append(adjusted_rand_score(gr.labels, lab.cpu().numpy()))
    assert np.mean(aris) >= 0.75


@pytest.mark.parametrize("max_iter", [1, 2, 3, 100])
def test_parity_small_sweep(rg, ctx, max_iter):
    """Many small graphs with ragged sizes (partial 32-row batches in every pass) and early Lloyd caps."""
    for seed in range(24):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(30, 400))
        src, dst = synth.random_edges(n, 6 * n, seed=seed)
        Z = _blob_Z(rng, n, 8, k=4, spread=0.7)
        _check(*_both(rg, ctx, n, src, dst, Z, max_iter=max_iter))


def test_lloyd_cap_diagnostic(rg, ctx):
    """stats capped_segments / capped_rows: the segments whose Lloyd iterations the max_iter cap stopped before
    convergence. With max_iter = 1 every Lloyd run is stopped by the cap (the root segment alone holds all n rows);
    a larger cap leaves fewer (or as many) capped segments; the partition still equals the oracle's either way."""
    gr = synth.generate("C1", 3)
    go = oracle.build_csr(gr.n, gr.src, gr.dst)
    Z = oracle.gcn(go, [64, 64, 32], 3, oracle.project(go, "ncut", 64, 3))[-1].astype(np.float32)
    res = {}
    for cap in (1, 100):
        ref, K, st, lab, Kg, stg = _both(rg, ctx, gr.n, gr.src, gr.dst, Z, max_iter=cap)
        _check(ref, K, st, lab, Kg, stg)
        res[cap] = stg
    assert res[1]["capped_segments"] >= 1 and res[1]["capped_rows"] >= gr.n
    assert 0 <= res[100]["capped_segments"] <= res[1]["capped_segments"] + res[100]["splits"]
    assert 0 <= res[100]["capped_rows"] <= res[100]["lloyd_rows"] + gr.n
