"""GPU checks of NEXT-4 — streaming updates — through the C-ABI (raftgp_stream_*).

The streamed NCut embedding after adding edges must be BIT-IDENTICAL to raftgp_embed(NCUT) on a graph built
from scratch with all the edges (every row's arithmetic depends only on its neighbour list and inputs), the
recomputed sets must be exactly the (k)-hop closures of the changed nodes (checked with scipy on the host), and
the result must match the oracle within 1e-4. Edge cases: duplicates of existing edges and self-loops (no
change at all), edges to isolated nodes, empty batches, errors."""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.int32))


def _fresh_ncut(rg, ctx, n, src, dst, dims, seed):
    g = rg.raftgp_build_csr(ctx, n, _t(src), _t(dst))
    _, Z = rg.raftgp_embed_multi(g, ["ncut"], dims, seed)
    return Z["ncut"]


def _closures(n, src, dst, changed, L):
    a = sp.coo_matrix((np.ones(src.size), (src, dst)), shape=(n, n)).tocsr()
    a = ((a + a.T) > 0).astype(np.int8)
    a.setdiag(0)
    a.eliminate_zeros()
    cur = changed.copy()
    sizes = []
    for _ in range(L + 1):
        cur = cur | (a @ cur.astype(np.int8) > 0)
        sizes.append(int(cur.sum()))
    return sizes


@pytest.mark.parametrize("cfg,n,dims,batches", [("C1", None, (64, 64, 32), 3), ("C2", 20000, (64, 64, 32), 2),
                                                ("C1", None, (128, 64, 32, 32), 2)])
def test_stream_equals_full_recompute(rg, ctx, cfg, n, dims, batches):
    gr = synth.generate(cfg, 4, n=n)
    rng = np.random.default_rng(9)
    m = gr.src.size
    held = rng.choice(m, size=min(m // 50, 400), replace=False)
    keep = np.setdiff1d(np.arange(m), held)
    src0, dst0 = gr.src[keep], gr.dst[keep]
    # extra new edges between random nodes (some to nodes that were isolated in the base graph)
    extra_s = rng.integers(0, gr.n, 40).astype(np.int32)
    extra_d = rng.integers(0, gr.n, 40).astype(np.int32)
    add_s = np.concatenate([gr.src[held], extra_s])
    add_d = np.concatenate([gr.dst[held], extra_d])
    g = rg.raftgp_build_csr(ctx, gr.n, _t(src0), _t(dst0))
    stream = rg.Stream(g, dims, 5)
    Z0 = stream.embedding().clone()
    assert torch.equal(Z0, _fresh_ncut(rg, ctx, gr.n, src0, dst0, dims, 5))
    cur_s, cur_d = src0, dst0
    for part_s, part_d in zip(np.array_split(add_s, batches), np.array_split(add_d, batches)):
        deg_before = np.bincount(np.concatenate([cur_s, cur_d])[np.concatenate([cur_s != cur_d] * 2)], minlength=gr.n)
        st = stream.add_edges(_t(part_s), _t(part_d))
        cur_s = np.concatenate([cur_s, part_s])
        cur_d = np.concatenate([cur_d, part_d])
        Zs = stream.embedding()
        assert torch.equal(Zs, _fresh_ncut(rg, ctx, gr.n, cur_s, cur_d, dims, 5))
        # recomputed sets = closures of the nodes whose (simple-graph) degree changed
        go = oracle.build_csr(gr.n, cur_s, cur_d)
        gb = oracle.build_csr(gr.n, cur_s[:-part_s.size] if part_s.size else cur_s,
                              cur_d[:-part_d.size] if part_d.size else cur_d)
        changed = go.deg != gb.deg
        assert st["changed"] == int(changed.sum())
        clo = _closures(gr.n, cur_s, cur_d, changed, len(dims) - 1)
        # the last level is either the exact closure or n (the last hop ran over every row: its frontier's entries
        # covered the graph 1.5 times or more)
        assert st["affected"][:-1] == clo[:-1] and st["affected"][-1] in (clo[-1], gr.n), (st["affected"], clo)
        assert st["nnz"] == go.nnz
    Zo = oracle.gcn(go, list(dims), 5, oracle.project(go, "ncut", dims[0], 5))[-1]
    e = np.linalg.norm(Zs.cpu().numpy() - Zo) / np.linalg.norm(Zo)
    assert e <= 1e-4


def test_stream_no_change_and_empty(rg, ctx):
    gr = synth.generate("C1", 0)
    g = rg.raftgp_build_csr(ctx, gr.n, _t(gr.src), _t(gr.dst))
    stream = rg.Stream(g, (64, 64, 32), 1)
    Z0 = stream.embedding().clone()
    st = stream.add_edges(_t(gr.src[:25]), _t(gr.dst[:25]))          # all already present
    assert st["changed"] == 0 and st["affected"] == [0, 0, 0]
    st = stream.add_edges(_t(np.arange(10)), _t(np.arange(10)))        # self-loops only
    assert st["changed"] == 0
    st = stream.add_edges(_t(np.zeros(0)), _t(np.zeros(0)))            # empty batch
    assert st["changed"] == 0
    assert torch.equal(stream.embedding(), Z0)
    host = stream.add_edges(torch.tensor([0], dtype=torch.int32), torch.tensor([999], dtype=torch.int32))
    assert host["changed"] in (0, 2)


def test_stream_errors(rg, ctx):
    gr = synth.generate("C1", 0)
    g = rg.raftgp_build_csr(ctx, gr.n, _t(gr.src), _t(gr.dst))
    with pytest.raises(rg.RaftGPError) as e:
        rg.Stream(g, (64, 48, 32), 1)
    assert e.value.code == rg.RAFTGP_ERR_PARAM
    stream = rg.Stream(g, (64, 64, 32), 1)
    with pytest.raises(rg.RaftGPError) as e:
        stream.add_edges(_t([0]), _t([gr.n + 5]))
    assert e.value.code == rg.RAFTGP_ERR_DATA
    # a data error is caught before the state is touched: the stream goes on, still bit-identical
    stream.add_edges(_t([0, 7]), _t([400, 900]))
    assert torch.equal(stream.embedding(), _fresh_ncut(rg, ctx, gr.n, np.concatenate([gr.src, [0, 7]]),
                                                       np.concatenate([gr.dst, [400, 900]]), (64, 64, 32), 1))


_LAST_SCRIPT = r"""
import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import synth, scipy.sparse as sp
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
mode = os.environ['RAFTGP_STREAM_FULL_LAST']
gr = synth.generate('C2', 4, n=20000)
dims = (64, 64, 32)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32))
m = gr.src.size
keep = np.arange(m - 30)
g = rg.raftgp_build_csr(ctx, gr.n, t(gr.src[keep]), t(gr.dst[keep]))
s = rg.Stream(g, dims, 3)
st = s.add_edges(t(gr.src[m - 30:]), t(gr.dst[m - 30:]))
g2 = rg.raftgp_build_csr(ctx, gr.n, t(gr.src), t(gr.dst))
_, Z = rg.raftgp_embed_multi(g2, ['ncut'], dims, 3)
assert torch.equal(s.embedding(), Z['ncut'])
a = sp.coo_matrix((np.ones(m), (gr.src, gr.dst)), shape=(gr.n, gr.n)).tocsr()
a = ((a + a.T) > 0).astype(np.int8); a.setdiag(0); a.eliminate_zeros()
import oracle
cur = oracle.build_csr(gr.n, gr.src, gr.dst).deg != oracle.build_csr(gr.n, gr.src[keep], gr.dst[keep]).deg
sizes = []
for _ in range(len(dims)):
    cur = cur | (a @ cur.astype(np.int8) > 0)
    sizes.append(int(cur.sum()))
assert st['affected'][:-1] == sizes[:-1], (st, sizes)
assert st['affected'][-1] == (gr.n if mode == '1' else sizes[-1]), (st, sizes)
print('ok', st)
"""


@pytest.mark.parametrize("mode", ["0", "1"])
def test_stream_last_hop_listed_or_full(rg, mode):
    """The last GCN hop over the listed closure (RAFTGP_STREAM_FULL_LAST=0) or over every row with the full-graph
    kernel (=1, the default when the frontier covers the graph): both bit-identical to the full recompute."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _LAST_SCRIPT], cwd=root,
                       env=dict(os.environ, RAFTGP_STREAM_FULL_LAST=mode), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- delta mode (raftgp_stream_set_mode)
def _delta_case(rg, ctx, cfg, n, dims, batches, per_batch, seed):
    gr = synth.generate(cfg, seed, n=n)
    rng = np.random.default_rng(seed + 100)
    m = gr.src.size
    held = rng.choice(m, size=min(m // 50, batches * per_batch), replace=False)
    keep = np.setdiff1d(np.arange(m), held)
    return gr, gr.src[keep], gr.dst[keep], np.array_split(gr.src[held], batches), np.array_split(gr.dst[held], batches)


@pytest.mark.parametrize("cfg,n,dims,batches", [("C1", None, (64, 64, 32), 3), ("C2", 20000, (64, 64, 32), 2),
                                                ("C1", None, (128, 64, 32, 32), 2), ("C1", None, (64, 128), 2),
                                                ("C1", None, (32, 64, 128), 2)])
@pytest.mark.parametrize("frac", ["0", "8"])
def test_stream_delta_matches_exact(rg, ctx, cfg, n, dims, batches, frac, monkeypatch):
    """Delta mode: the last hop from the stored sums A_i plus the changed rows of T_L only. Every batch: Z within
    fp32 re-association error of the exact stream (itself bit-identical to a fresh embed), rows outside the closure
    R_{L+1} bit-identical, the rewritten-row count equal to |R_{L+1}| (row i is rewritten iff i or a neighbour is in
    R_L), and the oracle within 1e-4 at the end. frac = "0": always the delta pass; "8" (default): the full pass when
    R_L holds 1/8 of the rows or more (every row rewritten)."""
    monkeypatch.setenv("RAFTGP_STREAM_DELTA_FRAC", frac)
    gr, s0, d0, bs, bd = _delta_case(rg, ctx, cfg, n, dims, batches, 60, 6)
    ex = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, _t(s0), _t(d0)), dims, 7)
    de = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, _t(s0), _t(d0)), dims, 7)
    de.set_mode("delta")
    e0 = (de.embedding() - ex.embedding()).abs().max().item()
    assert e0 <= 2e-6, e0   # the state build's own summation order
    cur_s, cur_d = s0, d0
    L = len(dims) - 1
    for ps, pd in zip(bs, bd):
        Zprev = de.embedding().clone()
        st_e = ex.add_edges(_t(ps), _t(pd))
        st_d = de.add_edges(_t(ps), _t(pd))
        gb = oracle.build_csr(gr.n, cur_s, cur_d)
        cur_s, cur_d = np.concatenate([cur_s, ps]), np.concatenate([cur_d, pd])
        go = oracle.build_csr(gr.n, cur_s, cur_d)
        changed = go.deg != gb.deg
        clo = _closures(gr.n, cur_s, cur_d, changed, L)
        assert st_d["changed"] == st_e["changed"] == int(changed.sum())
        full_pass = frac != "0" and clo[L - 1] * int(frac) >= gr.n
        assert st_d["affected"][:-1] == clo[:-1], (st_d, clo)
        assert st_d["affected"][-1] == (gr.n if full_pass else clo[-1]), (st_d, clo)
        Ze, Zd = ex.embedding(), de.embedding()
        diff = (Zd - Ze).abs().max().item()
        rel = ((Zd - Ze).norm() / Ze.norm()).item()
        assert diff <= 5e-6 and rel <= 2e-6, (diff, rel)
        # rows outside R_{L+1} are not rewritten
        a = sp.coo_matrix((np.ones(cur_s.size), (cur_s, cur_d)), shape=(gr.n, gr.n)).tocsr()
        a = ((a + a.T) > 0).astype(np.int8)
        cl = changed.copy()
        for _ in range(L + 1):
            cl = cl | (a @ cl.astype(np.int8) > 0)
        out = torch.from_numpy(~cl).cuda()
        if not full_pass:
            assert torch.equal(Zd[out], Zprev[out])
        elif int(out.sum()) > 0:
            assert (Zd[out] - Zprev[out]).abs().max().item() <= 2e-6
    Zo = oracle.gcn(go, list(dims), 7, oracle.project(go, "ncut", dims[0], 7))[-1]
    e = np.linalg.norm(de.embedding().cpu().numpy() - Zo) / np.linalg.norm(Zo)
    assert e <= 1e-4


def test_stream_delta_drift_resync_and_exact(rg, ctx, monkeypatch):
    """40 small batches in delta mode stay within 1e-5 of a fresh embed; set_mode("delta") again resyncs (the exact
    chain, then the sums: Z bit-identical to raftgp_embed); set_mode("exact") after a delta batch recomputes Z
    bit-identically; no-op batches change nothing."""
    monkeypatch.setenv("RAFTGP_STREAM_DELTA_FRAC", "0")
    dims = (64, 64, 32)
    gr, s0, d0, bs, bd = _delta_case(rg, ctx, "C1", None, dims, 40, 5, 11)
    de = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, _t(s0), _t(d0)), dims, 2)
    de.set_mode("delta")
    Z0 = de.embedding().clone()
    for st in (de.add_edges(_t(s0[:20]), _t(d0[:20])), de.add_edges(_t(np.arange(5)), _t(np.arange(5))),
               de.add_edges(_t(np.zeros(0)), _t(np.zeros(0)))):
        assert st["changed"] == 0 and st["affected"][-1] == 0
    assert torch.equal(de.embedding(), Z0)
    cur_s, cur_d = s0, d0
    for ps, pd in zip(bs, bd):
        de.add_edges(_t(ps), _t(pd))
        cur_s, cur_d = np.concatenate([cur_s, ps]), np.concatenate([cur_d, pd])
    fresh = _fresh_ncut(rg, ctx, gr.n, cur_s, cur_d, dims, 2)
    Zd = de.embedding()
    assert ((Zd - fresh).norm() / fresh.norm()).item() <= 1e-5
    de.set_mode("delta")   # a resync: the exact chain, then the sums rebuilt
    assert torch.equal(de.embedding(), fresh)
    de.add_edges(_t([1, 4]), _t([600, 800]))
    de.set_mode("exact")
    cur_s, cur_d = np.concatenate([cur_s, [1, 4]]), np.concatenate([cur_d, [600, 800]])
    assert torch.equal(de.embedding(), _fresh_ncut(rg, ctx, gr.n, cur_s, cur_d, dims, 2))
    st = de.add_edges(_t([0, 3]), _t([500, 900]))   # exact again: bit-identical
    fresh2 = _fresh_ncut(rg, ctx, gr.n, np.concatenate([cur_s, [0, 3]]), np.concatenate([cur_d, [500, 900]]), dims, 2)
    assert torch.equal(de.embedding(), fresh2), st


def test_stream_delta_large_batch_and_errors(rg, ctx):
    """A batch above the one-CTA delta sort (> 2048 pairs: the CSR-build merge path) in delta mode, and a bad mode."""
    dims = (64, 64, 32)
    gr, s0, d0, bs, bd = _delta_case(rg, ctx, "C2", 20000, dims, 1, 3000, 12)
    ex = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, _t(s0), _t(d0)), dims, 4)
    de = rg.Stream(rg.raftgp_build_csr(ctx, gr.n, _t(s0), _t(d0)), dims, 4)
    de.set_mode("delta")
    ex.add_edges(_t(bs[0]), _t(bd[0]))
    de.add_edges(_t(bs[0]), _t(bd[0]))
    Ze = ex.embedding()
    assert ((de.embedding() - Ze).norm() / Ze.norm()).item() <= 2e-6
    with pytest.raises(rg.RaftGPError) as e:
        rg._ck(rg.load_library().raftgp_stream_set_mode(de.h, 7))
    assert e.value.code == rg.RAFTGP_ERR_PARAM
