"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C4 (N = 5e6, nnz ~ 2e8, r = 128, dims 128->128->64, the bench workload):
  * the whole CSR (row_ptr, col_idx, degrees) bit-exact against the oracle's sort-based build;
  * Theta bit-exact on sampled rows (incl. the ragged tail of the grid);
  * Theta' = Theta W^(1) of the tcgen05 kernel at C4's tile count (~264 tiles per CTA, every CTA's last tiles);
  * raftgp_build_embed(ncut + mod) -- THE call bench.py times (Theta' on the side stream during the CSR build,
    DUAL feature hop, paired last GCN hop) -- both Z matrices in FULL against the oracle's full pipeline
    (Eq. 5 + Eq. 6 + l2), 1e-4 relative Frobenius, plus row-wise checks on the 16 largest
    hubs, the isolated rows, 128-row tile boundaries and the last rows;
  * raftgp_embed (Y and Z^(1) materialised) in full, and bitwise run-to-run determinism.
C3 (N = 2e5, r = 128, dims 128->128->64->32): every output matrix in full against the oracle.
C5 (N = 5e7, ~1.94e9 CSR entries): raftgp_build_embed on sampled rows against the oracle's
    receptive-field computation (oracle.embed_rows; MOD's g from one streaming pass over Theta).
Table I widths 4096->2048->1024->512->256 at N = 2E5 (the C3 graph, bench's table1 leg):
    both Z matrices in full against oracle.project + oracle.gcn_np.
Streaming at C4 (bench's streaming leg): the exact stream bit-identical to a fresh embed of the merged graph, the
    delta-mode stream within fp32 re-association error of it.
The oracle runs with all host cores (OpenMP over rows; bit-identical to one thread, see oracle.c header).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-4
ROW_TOL = 2e-4     # per-row l2 error of a unit-norm Z row (rows of tiny |H| amplify fp32 rounding)


def rel_fro(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)


def row_err(got, ref):
    return np.sqrt(((np.asarray(got, np.float64) - ref) ** 2).sum(axis=1))


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    return raftgp


@pytest.fixture(scope="module")
def c4(rg):
    ctx = rg.Context(0)
    gr = synth.generate("C4", 0)
    src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
    g = rg.raftgp_build_csr(ctx, gr.n, src, dst)
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    return ctx, gr, g, ref, src, dst


@pytest.fixture(scope="module")
def c4_oracle(c4):
    """Full oracle pipeline at C4 for both variants: {v: (Y, Z^(1), Z)} (fp64, ~25 GB of host memory)."""
    _, _, _, ref, _, _ = c4
    cfg = synth.CONFIGS["C4"]
    out = {}
    for v in ("ncut", "mod"):
        Y = oracle.project(ref, v, cfg.r, 0)
        Z1, Z = oracle.gcn(ref, list(cfg.dims), 0, Y)
        out[v] = (Y, Z1, Z)
    return out


def special_rows(ref, n):
    """Rows the sampled tests used to miss: the 16 largest hubs, isolated rows, 128-row tile boundaries
    (first/last row of sampled tiles) and the last rows of the matrix (ragged last tile)."""
    deg = np.diff(ref.row_ptr)
    hubs = np.argsort(deg, kind="stable")[-16:]
    iso = np.flatnonzero(deg == 0)[:64]
    tiles = synth.sample_rows((n + 127) // 128, 256, 5)
    bounds = np.concatenate([tiles * 128, np.minimum(tiles * 128 + 127, n - 1)])
    last = np.arange(max(0, n - 200), n)
    return np.unique(np.concatenate([hubs, iso, bounds, last])).astype(np.int64)


def test_c4_csr_bit_exact(c4):
    ctx, gr, g, ref, _, _ = c4
    rp, col, deg = g.export()
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(col, ref.col)
    assert np.array_equal(deg, ref.deg)
    assert g.info()["two_e"] == ref.nnz


def test_c4_theta_rows_bit_exact(rg, c4):
    ctx, gr, g, ref, _, _ = c4
    th = rg.raftgp_sketch(ctx, 0, 0, 0, gr.n, 128, 128)
    rows = np.concatenate([synth.sample_rows(gr.n, 2000, 3), np.arange(gr.n - 64, gr.n)])
    got = th[torch.from_numpy(rows).cuda()].cpu().numpy()
    exp = np.concatenate([oracle.theta(1, 128, 0, row_begin=int(i)) for i in rows])
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_c4_sketch_transform_all_tiles(rg, c4):
    """Theta' = Theta W^(1) (tcgen05, persistent over 128-row tiles: CTA b takes tiles b, b + grid, ...) at C4's
    39,063 tiles -- the mbarrier phases of ~264 tiles per CTA. Checked on the last 2 x 148 tiles (every CTA's
    final tiles, incl. the ragged one), every 97th tile's boundary rows and 3000 random rows, against the
    oracle's Theta rows times W^(1) in fp64."""
    ctx, gr, g, ref, _, _ = c4
    n = gr.n
    W = rg.raftgp_weights(ctx, 0, 1, 128, 128)
    Tp = rg.raftgp_sketch_transform(ctx, 0, n, W)
    ntiles = (n + 127) // 128
    late = np.arange(max(0, ntiles - 296), ntiles)
    every = np.arange(0, ntiles, 97)
    rows = np.concatenate([late * 128, np.minimum(late * 128 + 127, n - 1), late * 128 + 64,
                           every * 128, np.minimum(every * 128 + 127, n - 1),
                           synth.sample_rows(n, 3000, 21), [n - 1]])
    rows = np.unique(rows[rows < n]).astype(np.int64)
    got = Tp[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    th = np.concatenate([oracle.theta(1, 128, 0, row_begin=int(i)) for i in rows]).astype(np.float64)
    exp = th @ oracle.weights(1, 128, 128, 0).astype(np.float64)
    assert rel_fro(got, exp) < 5e-6
    assert np.max(np.abs(got - exp)) < 1e-5 * max(1.0, np.abs(exp).max())


def test_c4_build_embed_full(rg, c4, c4_oracle):
    """The exact call bench.py times: raftgp_build_embed(ctx, C4 edges on the device, [ncut, mod], 128-128-64,
    seed 0) on torch's current stream; both Z in full vs the oracle, row-wise checks, determinism."""
    ctx, gr, g, ref, src, dst = c4
    dims = list(synth.CONFIGS["C4"].dims)
    Z, g2 = rg.raftgp_build_embed(ctx, gr.n, src, dst, ["ncut", "mod"], dims, 0, keep_graph=True)
    torch.cuda.synchronize()
    assert g2.info()["two_e"] == ref.nnz
    rows = special_rows(ref, gr.n)
    deg = np.diff(ref.row_ptr)
    for v in ("ncut", "mod"):
        Zo = c4_oracle[v][2]
        z = Z[v].cpu().numpy()
        e = rel_fro(z, Zo)
        assert e <= TOL, f"{v}: relative Frobenius error {e:.3e}"
        re_ = row_err(z[rows], Zo[rows])
        assert re_.max() <= ROW_TOL, f"{v}: worst special row {rows[np.argmax(re_)]} error {re_.max():.3e}"
        iso = deg == 0
        assert np.all(z[iso] == 0.0)
        nrm = np.linalg.norm(z[~iso].astype(np.float64), axis=1)
        assert np.all(np.abs(nrm - 1.0) < 1e-5)
    Zb, _ = rg.raftgp_build_embed(ctx, gr.n, src, dst, ["ncut", "mod"], dims, 0)
    for v in ("ncut", "mod"):
        assert torch.equal(Z[v], Zb[v])
    g2.close()


@pytest.mark.parametrize("variant", ["ncut", "mod"])
def test_c4_embed_full(rg, c4, c4_oracle, variant):
    """raftgp_embed (Y and Z^(1) materialised, FFMA W-epilogue): Y, Z^(1), Z in full."""
    ctx, gr, g, ref, _, _ = c4
    dims = list(synth.CONFIGS["C4"].dims)
    Y, Z, Zk = rg.raftgp_embed(g, variant, dims, 0, intermediates=True)
    Yo, Z1o, Zo = c4_oracle[variant]
    assert rel_fro(Y.cpu().numpy(), Yo) <= TOL
    assert rel_fro(Zk[0].cpu().numpy(), Z1o) <= TOL
    assert rel_fro(Z.cpu().numpy(), Zo) <= TOL
    rows = special_rows(ref, gr.n)
    assert row_err(Z.cpu().numpy()[rows], Zo[rows]).max() <= ROW_TOL
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


# ------------------------------------------------------------------ C5: the largest config, sampled rows
@pytest.fixture(scope="module")
def c5(rg):
    """C5 on one GPU through the bench's call, then everything but the host data released (the GPU holds
    ~128 GB of workspace at C5)."""
    ctx = rg.Context(0)
    gr = synth.generate("C5", 0)
    dims = list(synth.CONFIGS["C5"].dims)
    src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
    Z, g = rg.raftgp_build_embed(ctx, gr.n, src, dst, ["ncut", "mod"], dims, 0, keep_graph=True)
    info = g.info()
    del src, dst
    g.close()
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    rows = np.unique(np.concatenate([synth.sample_rows(gr.n, 12, 33), [gr.n - 1],
                                     np.flatnonzero(np.diff(ref.row_ptr) == 0)[:2],
                                     [((gr.n + 127) // 128 - 1) * 128]])).astype(np.int64)
    Zs = {v: Z[v][torch.from_numpy(rows).cuda()].cpu().numpy() for v in Z}
    del Z
    ctx.trim()
    ctx.close()
    torch.cuda.empty_cache()
    return gr, ref, info, rows, Zs


def test_c5_csr_size(c5):
    """C5's 1.94e9 CSR entries (2.0e9 raw entries before dedup): 2e, and hence the last row offset, match the
    oracle. (Both stay below 2^31; row_ptr is int64 regardless.)"""
    gr, ref, info, rows, Zs = c5
    assert info["two_e"] == ref.nnz and ref.nnz > 1.9e9


@pytest.mark.parametrize("variant", ["ncut", "mod"])
def test_c5_build_embed_sampled_rows(c5, variant):
    gr, ref, info, rows, Zs = c5
    cfg = synth.CONFIGS["C5"]
    _, Zo = oracle.embed_rows(ref, variant, cfg.r, list(cfg.dims), 0, rows)
    z = Zs[variant]
    assert rel_fro(z, Zo[-1]) <= TOL
    assert row_err(z, Zo[-1]).max() <= ROW_TOL
    iso = np.diff(ref.row_ptr)[rows] == 0
    assert np.all(z[iso] == 0.0)


# ------------------------------------------------------------------ Table I widths at N = 2E5 (NEXT-2)
def test_table1_widths_2e5(rg):
    """bench.py's table1 leg in full: C3 graph (N = 2E5) with 4096->2048->1024->512->256,
    ncut + mod through raftgp_embed_multi (tcgen05 3xTF32 GEMMs, wide hops), both Z vs oracle.gcn_np."""
    ctx = rg.Context(0)
    gr = synth.generate("C3", 0)
    dims = (4096, 2048, 1024, 512, 256)
    g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
    _, Z = rg.raftgp_embed_multi(g, ["ncut", "mod"], dims, 0)
    Zh = {v: Z[v].cpu().numpy() for v in Z}
    del Z
    g.close()
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    for v in ("ncut", "mod"):
        Zo = oracle.gcn_np(ref, dims, 0, oracle.project(ref, v, dims[0], 0))[-1]
        e = rel_fro(Zh[v], Zo)
        assert e <= TOL, f"{v}: relative Frobenius error {e:.3e}"
        assert row_err(Zh[v], Zo).max() <= ROW_TOL


# ------------------------------------------------------------------ NEXT-4 streaming at C4 (bench's streaming leg)
def test_c4_stream_exact_and_delta(rg, c4):
    """Streams at the bench's size: after 10-edge batches and a 1000-edge batch the exact stream's Z equals
    raftgp_embed_multi(ncut) on the merged graph BIT FOR BIT, and the delta-mode stream (every GCN hop from stored
    sums + changed rows) stays within fp32 re-association error of it (reading #32)."""
    ctx, gr, _, _, src, dst = c4
    dims = list(synth.CONFIGS["C4"].dims)
    rng = np.random.default_rng(41)
    ex = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, src, dst), dims, 0)
    de = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, src, dst), dims, 0)
    de.set_mode("delta")
    s_all, d_all = src, dst
    for B in (10, 10, 1000):
        es = torch.from_numpy(rng.integers(0, gr.n, B).astype(np.int32)).cuda()
        ed = torch.from_numpy(rng.integers(0, gr.n, B).astype(np.int32)).cuda()
        st_e = ex.add_edges(es, ed)
        st_d = de.add_edges(es, ed)
        assert st_e["changed"] == st_d["changed"] and st_e["affected"][:-1] == st_d["affected"][:-1]
        s_all, d_all = torch.cat([s_all, es]), torch.cat([d_all, ed])
        Ze, Zd = ex.embedding(), de.embedding()
        assert (Zd - Ze).abs().max().item() <= 5e-6
        assert ((Zd - Ze).norm() / Ze.norm()).item() <= 2e-6
    g2 = rg.raftgp_build_csr(ctx, gr.n, s_all, d_all)
    _, Z = rg.raftgp_embed_multi(g2, ["ncut"], dims, 0)
    assert torch.equal(ex.embedding(), Z["ncut"])
    assert ex.graph().info()["nnz_local"] == g2.info()["nnz_local"]
    ex.close()
    de.close()
    g2.close()
