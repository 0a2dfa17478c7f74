"""GPU parity of NEXT-2 — the paper's Table I layer widths (L up to 4096, GNN stacks
4096 -> 2048 -> 1024 -> 512 -> 256) — through the C-ABI against the oracle.

* raftgp_gemm_tf32x3 (tcgen05, 3xTF32 split) against numpy's fp64 matmul: relative Frobenius error <= 2e-5
  (fp32-accurate; plain TF32 would be ~1e-3).
* raftgp_embed_multi at Table I widths (Theta W^(1) on the tensor cores, wide hops, GEMM transforms) against
  oracle.project + oracle.gcn_np: <= 1e-4 relative Frobenius per embedding matrix (north_star bar), for every
  variant, on graphs with ragged row tiles, isolated nodes, and narrow <-> wide transitions in both directions.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def rel_fro(got, ref):
    ref = np.asarray(ref, np.float64)
    return np.linalg.norm(np.asarray(got, np.float64) - ref) / max(np.linalg.norm(ref), 1e-300)


@pytest.mark.parametrize("M,K,N", [(1, 8, 1), (128, 32, 32), (300, 64, 100), (77, 40, 300), (1000, 256, 128),
                                   (513, 1024, 512), (2000, 4096, 2048), (129, 2048, 64)])
@pytest.mark.parametrize("scaled", [False, True])
def test_gemm(rg, ctx, M, K, N, scaled):
    rng = np.random.default_rng(M + K + N)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
    s = rng.uniform(0.2, 1.5, M).astype(np.float32) if scaled else None
    C = rg.raftgp_gemm_tf32x3(ctx, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(),
                              None if s is None else torch.from_numpy(s).cuda())
    ref = A.astype(np.float64) @ B.astype(np.float64)
    if s is not None:
        ref *= s[:, None]
    assert rel_fro(C.cpu().numpy(), ref) <= 2e-5


def _graph(kind, n=None):
    if kind == "c1":
        gr = synth.generate("C1", 0)
        return gr.n, gr.src, gr.dst
    if kind == "c2_small":
        gr = synth.generate("C2", 1, n=n)
        return gr.n, gr.src, gr.dst
    src, dst = synth.random_edges(n - 37, 14 * n, seed=n)   # 37 isolated nodes at the end, ragged tiles
    return n, src, dst


CASES = [
    ("c1", None, (256, 128, 64)),                        # Table I, N = 1E3
    ("c2_small", 2500, (1024, 512, 256, 128)),           # Table I, N = 5E3 widths
    ("c2_small", 1200, (4096, 2048, 1024, 512, 256)),    # Table I, N >= 1E4 widths
    ("rand", 1500, (128, 256, 128)),                     # narrow -> wide -> narrow
    ("rand", 1501, (256, 128, 256, 32)),                 # wide -> narrow -> wide -> narrow
    ("rand", 900, (512, 512, 64)),
]


@pytest.mark.parametrize("kind,n,dims", CASES, ids=[f"{c[0]}-{c[1]}-{'x'.join(map(str, c[2]))}" for c in CASES])
def test_embed_table1_widths(rg, ctx, kind, n, dims):
    n, src, dst = _graph(kind, n)
    go = oracle.build_csr(n, src, dst)
    g = rg.raftgp_build_csr(ctx, n, torch.from_numpy(src), torch.from_numpy(dst))
    variants = ["ncut", "mod", "mod_reduced"]
    _, Z = rg.raftgp_embed_multi(g, variants, dims, 0)
    for v in variants:
        Zo = oracle.gcn_np(go, dims, 0, oracle.project(go, v, dims[0], 0))[-1]
        e = rel_fro(Z[v].cpu().numpy(), Zo)
        assert e <= TOL, f"{v}: relative Frobenius error {e:.3e}"


def test_single_variant_matches_dual(rg, ctx):
    """The dual (NCut + Mod) wide feature hop gives exactly the single-variant results."""
    n, src, dst = _graph("rand", 1100)
    g = rg.raftgp_build_csr(ctx, n, torch.from_numpy(src), torch.from_numpy(dst))
    dims = (256, 512, 256)
    _, Zd = rg.raftgp_embed_multi(g, ["ncut", "mod"], dims, 3)
    for v in ("ncut", "mod"):
        _, Zs = rg.raftgp_embed_multi(g, [v], dims, 3)
        assert torch.equal(Zs[v], Zd[v])
