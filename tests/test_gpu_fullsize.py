"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C4 (N = 5e6, nnz ~ 2e8, r = 128, dims 128->128->64, the bench workload):
  * the whole CSR (row_ptr, col_idx, degrees) bit-exact against the oracle's sort-based build;
  * Theta bit-exact on sampled rows (incl. the ragged tail of the grid);
  * Y, Z^(1) and Z of the fused raftgp_embed (bench path) on sampled rows against the oracle's
    receptive-field computation (identical arithmetic to its full pipeline), 1e-4 relative Frobenius;
  * run-to-run determinism (bitwise).
C3 (N = 2e5, r = 128, dims 128->128->64->32): every output matrix in full against the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-4


def rel_fro(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    return raftgp


@pytest.fixture(scope="module")
def c4(rg):
    ctx = rg.Context(0)
    gr = synth.generate("C4", 0)
    g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    return ctx, gr, g, ref


def test_c4_csr_bit_exact(c4):
    ctx, gr, g, ref = c4
    rp, col, deg = g.export()
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(col, ref.col)
    assert np.array_equal(deg, ref.deg)
    assert g.info()["two_e"] == ref.nnz


def test_c4_theta_rows_bit_exact(rg, c4):
    ctx, gr, g, ref = c4
    th = rg.raftgp_sketch(ctx, 0, 0, 0, gr.n, 128, 128)
    rows = np.concatenate([synth.sample_rows(gr.n, 2000, 3), np.arange(gr.n - 64, gr.n)])
    got = th[torch.from_numpy(rows).cuda()].cpu().numpy()
    exp = np.concatenate([oracle.theta(1, 128, 0, row_begin=int(i)) for i in rows])
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("variant", ["ncut", "mod"])
def test_c4_embed_sampled_rows(rg, c4, variant):
    ctx, gr, g, ref = c4
    cfg = synth.CONFIGS["C4"]
    dims = list(cfg.dims)
    Y, Z, Zk = rg.raftgp_embed(g, variant, dims, 0, intermediates=True)
    rows = synth.sample_rows(gr.n, 8, 11)
    Yo, Zo = oracle.embed_rows(ref, variant, cfg.r, dims, 0, rows)
    idx = torch.from_numpy(rows).cuda()
    assert rel_fro(Y[idx].cpu().numpy(), Yo) <= TOL
    assert rel_fro(Zk[0][idx].cpu().numpy(), Zo[0]) <= TOL
    assert rel_fro(Z[idx].cpu().numpy(), Zo[1]) <= TOL
    # properties at every row: unit norm except isolated rows (zero)
    nrm = torch.linalg.vector_norm(Z, dim=1).cpu().numpy()
    iso = ref.deg == 0
    assert np.all(np.abs(nrm[~iso] - 1.0) < 1e-5) and np.all(nrm[iso] == 0.0)
    # determinism (bitwise) of the whole bench path
    _, Z2 = rg.raftgp_embed(g, variant, dims, 0, want_Y=False)
    assert torch.equal(Z, Z2)


@pytest.mark.parametrize("variant", ["ncut", "mod", "mod_reduced"])
def test_c3_full_parity(rg, variant):
    ctx = rg.Context(0)
    gr = synth.generate("C3", 0)
    cfg = synth.CONFIGS["C3"]
    g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    rp, col, _ = g.export()
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(col, ref.col)
    Y, Z, Zk = rg.raftgp_embed(g, variant, cfg.dims, 0, intermediates=True)
    Yo = oracle.project(ref, variant, cfg.r, 0)
    Zo = oracle.gcn(ref, cfg.dims, 0, Yo)
    assert rel_fro(Y.cpu().numpy(), Yo) <= TOL
    for k in range(len(cfg.dims) - 2):
        assert rel_fro(Zk[k].cpu().numpy(), Zo[k]) <= TOL
    assert rel_fro(Z.cpu().numpy(), Zo[-1]) <= TOL
