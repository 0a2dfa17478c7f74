"""Degenerate sizes through the NEXT entry points: empty and one-node graphs at Table I widths, model selection
on one node, the SBM sampler with no nodes / one block, a stream over a one-node graph."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def _g(rg, ctx, n, src, dst):
    return rg.raftgp_build_csr(ctx, n, torch.tensor(src, dtype=torch.int32), torch.tensor(dst, dtype=torch.int32))


@pytest.mark.parametrize("n", [0, 1, 2])
def test_wide_tiny(rg, ctx, n):
    src, dst = ([0], [1]) if n == 2 else ([], [])
    g = _g(rg, ctx, n, src, dst)
    dims = (256, 512, 128)
    variants = ["ncut"] if n < 2 else ["ncut", "mod"]
    _, Z = rg.raftgp_embed_multi(g, variants, dims, 1)
    for v in variants:
        assert Z[v].shape == (n, 128)
        if n:
            go = oracle.build_csr(n, np.array(src, np.int32), np.array(dst, np.int32))
            Zo = oracle.gcn_np(go, dims, 1, oracle.project(go, v, dims[0], 1))[-1]
            assert np.allclose(Z[v].cpu().numpy(), Zo, atol=1e-5)


def test_select_one_node(rg, ctx):
    g = _g(rg, ctx, 1, [], [])
    lab, K, st = rg.raftgp_model_select(g, torch.zeros((1, 8), dtype=torch.float32, device="cuda"))
    assert K == 1 and lab.cpu().tolist() == [0]


def test_sbm_degenerate(rg, ctx):
    s, d = rg.raftgp_sbm_sample(ctx, torch.zeros(0, dtype=torch.int32, device="cuda"),
                                torch.zeros(0, dtype=torch.float64, device="cuda"),
                                torch.ones((1, 1), dtype=torch.float64, device="cuda"), 0)
    assert s.numel() == 0
    c = torch.zeros(5, dtype=torch.int32, device="cuda")
    s, d = rg.raftgp_sbm_sample(ctx, c, torch.ones(5, dtype=torch.float64, device="cuda"),
                                torch.full((1, 1), 1e4, dtype=torch.float64, device="cuda"), 0)
    assert s.numel() == 10                                         # complete graph on one block
    rs, rd = oracle.sbm_sample(np.zeros(5, np.int32), np.ones(5), np.full((1, 1), 1e4), 0)
    assert np.array_equal(s.cpu().numpy(), rs) and np.array_equal(d.cpu().numpy(), rd)


def test_stream_one_node(rg, ctx):
    g = _g(rg, ctx, 2, [], [])
    st = rg.Stream(g, (32, 32, 32), 0)
    info = st.add_edges(torch.tensor([0], dtype=torch.int32), torch.tensor([1], dtype=torch.int32))
    assert info["changed"] == 2 and info["nnz"] == 2
    g2 = _g(rg, ctx, 2, [0], [1])
    _, Z = rg.raftgp_embed_multi(g2, ["ncut"], (32, 32, 32), 0)
    assert torch.equal(st.embedding(), Z["ncut"])


def test_handles_outlive_context(rg):
    """A graph or stream destroyed after its context (as a garbage collector may order it) must still find the
    context alive: the library reference-counts it (raftgp_ctx_destroy drops only the caller's reference)."""
    c = rg.Context(0)
    src = torch.tensor([0, 1, 2, 3], dtype=torch.int32)
    dst = torch.tensor([1, 2, 3, 0], dtype=torch.int32)
    g1 = rg.raftgp_build_csr(c, 4, src, dst)
    g2 = rg.raftgp_build_csr(c, 4, src, dst)
    s = rg.Stream(g2, (32, 32, 32), 7)
    s.add_edges(torch.tensor([0], dtype=torch.int32), torch.tensor([2], dtype=torch.int32))
    c.close()
    rp, col, deg = g1.export()          # the graph is still usable: its context is alive
    assert list(deg) == [2, 2, 2, 2]
    assert s.embedding().shape == (4, 32)
    g1.close()
    s.close()
    torch.cuda.synchronize()


@pytest.mark.parametrize("n,src,dst", [(0, [], []), (1, [], []), (3, [0, 1], [1, 1]), (5, [0, 0, 3], [1, 1, 4])])
@pytest.mark.parametrize("dims", [(64, 64, 32), (48, 40, 24), (256, 128, 64)])
def test_build_embed_degenerate(rg, ctx, n, src, dst, dims):
    """raftgp_build_embed on empty / one-node / self-loop / duplicate-edge graphs, at fused (tcgen05 side-stream),
    generic and Table I-style widths: same result as the separate calls, and within 1e-4 of the oracle."""
    s, d = torch.tensor(src, dtype=torch.int32), torch.tensor(dst, dtype=torch.int32)
    Z1, _ = rg.raftgp_build_embed(ctx, n, s, d, ["ncut", "mod"] if n > 1 else ["ncut"], dims, 2)
    g = _g(rg, ctx, n, src, dst)
    variants = ["ncut", "mod"] if n > 1 else ["ncut"]
    _, Z2 = rg.raftgp_embed_multi(g, variants, dims, 2)
    for v in variants:
        assert torch.equal(Z1[v], Z2[v])
        assert Z1[v].shape == (n, dims[-1])
        if n:
            go = oracle.build_csr(n, np.array(src, np.int32), np.array(dst, np.int32))
            if v == "mod" and go.row_ptr[-1] == 0:
                continue
            Zo = oracle.gcn_np(go, dims, 2, oracle.project(go, v, dims[0], 2))[-1]
            assert np.allclose(Z1[v].cpu().numpy(), Zo, atol=1e-5)


def test_build_embed_bad_ids(rg, ctx):
    s = torch.tensor([0, 7], dtype=torch.int32)
    d = torch.tensor([1, 2], dtype=torch.int32)
    with pytest.raises(rg.RaftGPError):
        rg.raftgp_build_embed(ctx, 5, s, d, ["ncut"], (64, 64, 32), 1)
    # the context stays usable after the error
    Z, _ = rg.raftgp_build_embed(ctx, 3, torch.tensor([0], dtype=torch.int32), torch.tensor([1], dtype=torch.int32),
                                 ["ncut"], (64, 64, 32), 1)
    assert Z["ncut"].shape == (3, 32)


_WINDOW_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
cases = [synth.generate('C2', 3, n=30000), synth.generate('C1', 1)]
rng = np.random.default_rng(3)
hub_src = np.concatenate([np.zeros(5000, np.int32), rng.integers(0, 20000, 40000).astype(np.int32)])
hub_dst = np.concatenate([rng.integers(1, 20000, 5000).astype(np.int32), rng.integers(0, 20000, 40000).astype(np.int32)])
empty = np.zeros(0, np.int32)
ragged = rng.integers(0, 777, (2, 3000)).astype(np.int32)
for n, src, dst in [(c.n, c.src, c.dst) for c in cases] + [(20000, hub_src, hub_dst), (5000, empty, empty),
                                                           (777, ragged[0], ragged[1])]:
    g = rg.raftgp_build_csr(ctx, n, torch.from_numpy(src), torch.from_numpy(dst))
    rp, col, deg = g.export()
    ref = oracle.build_csr(n, src, dst)
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(col, ref.col), n
print('ok')
"""


@pytest.mark.parametrize("env", [
    {"RAFTGP_BUCKET_CAP": "300"}, {"RAFTGP_BUCKET_CAP": "2048"},
    # level 2 of the two-level partition on small graphs (at most 2 / 3 coarse buckets), alone and with windows
    {"RAFTGP_CSR_COARSE": "2"}, {"RAFTGP_CSR_COARSE": "3", "RAFTGP_BUCKET_CAP": "300"},
    # level 2 writing int2 entries (the C5 form: row-in-bucket and id bits do not fit 32 bits)
    {"RAFTGP_CSR_COARSE": "2", "RAFTGP_CSR_UNPACKED": "1"},
    {"RAFTGP_CSR_COARSE": "3", "RAFTGP_CSR_UNPACKED": "1", "RAFTGP_BUCKET_CAP": "2048"},
    # the one-level partition (shared-memory atomics), kept for A/B runs
    {"RAFTGP_CSR_TWO_LEVEL": "0"}, {"RAFTGP_CSR_TWO_LEVEL": "0", "RAFTGP_BUCKET_CAP": "2048"}])
def test_bucket_windows(rg, env):
    """Buckets larger than the shared-memory window (RAFTGP_BUCKET_CAP shrinks it) are sorted window by
    window; rows longer than a window go to the fallback kernels; both partition paths and both levels of
    the two-level one. The CSR must stay bit-exact."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _WINDOW_SCRIPT], cwd=root, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_set_order_rejects_non_permutations(rg, ctx):
    """raftgp_graph_set_order checks its array on the device: out-of-range or repeated rows are a PARAM error
    (the hop kernels index with it), a true permutation is accepted and leaves the results unchanged."""
    import synth
    gr = synth.generate("C1", 0)
    g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
    _, Z0 = rg.raftgp_embed_multi(g, ["ncut"], (64, 64, 32), 0)
    bad = [np.arange(gr.n, dtype=np.int32) + 1,                                      # out of range
           np.concatenate([[0], np.arange(gr.n - 1, dtype=np.int32)]).astype(np.int32),   # repeated 0
           -np.ones(gr.n, np.int32)]
    for b in bad:
        with pytest.raises(rg.RaftGPError) as ei:
            g.set_order(torch.from_numpy(b).cuda())
        assert ei.value.code == rg.RAFTGP_ERR_PARAM
    perm = np.random.default_rng(1).permutation(gr.n).astype(np.int32)
    g.set_order(torch.from_numpy(perm).cuda())
    _, Z1 = rg.raftgp_embed_multi(g, ["ncut"], (64, 64, 32), 0)
    assert torch.equal(Z0["ncut"], Z1["ncut"])


def test_trim_returns_memory_to_the_device(rg):
    """the context's workspace lives in its own pool; raftgp_ctx_trim hands it back to the device, so
    the free memory other allocators see recovers (the device's default pool is not modified)."""
    import synth
    c = rg.Context(0)
    gr = synth.generate("C3", 0)
    src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    Z, _ = rg.raftgp_build_embed(c, gr.n, src, dst, ["ncut", "mod"], (128, 128, 64), 0)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    released = c.trim()
    free2, _ = torch.cuda.mem_get_info()
    assert released > 0 and free1 < free0
    assert free2 >= free1 + 0.9 * released
    c.close()


_OVERLAP_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
gr = synth.generate('C2', 1, n=40000)
Z, _ = rg.raftgp_build_embed(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda(),
                             ['ncut', 'mod'], (64, 64, 32), 2)
np.save(sys.argv[1], np.concatenate([Z['ncut'].cpu().numpy(), Z['mod'].cpu().numpy()], 1))
print('ok')
"""


def test_build_embed_overlap_modes_identical(rg, tmp_path):
    """raftgp_build_embed gives the same bits whether Theta' runs beside the CSR build on half the SMs (split, the
    default), in short CTAs behind a high-priority CSR stream (prio), or before it (serial)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("split", "prio", "serial"):
        f = str(tmp_path / f"{mode}.npy")
        r = subprocess.run([sys.executable, "-c", _OVERLAP_SCRIPT, f], cwd=root,
                           env=dict(os.environ, RAFTGP_OVERLAP_MODE=mode), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
        outs[mode] = np.load(f)
    assert np.array_equal(outs["split"].view(np.uint32), outs["prio"].view(np.uint32))
    assert np.array_equal(outs["split"].view(np.uint32), outs["serial"].view(np.uint32))


_RELABEL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
out = []
rng = np.random.default_rng(7)
hub_s = np.concatenate([np.zeros(3000, np.int32), rng.integers(0, 9000, 30000).astype(np.int32)])
hub_d = np.concatenate([rng.integers(1, 9000, 3000).astype(np.int32), rng.integers(0, 9000, 30000).astype(np.int32)])
cases = [(g.n, g.src, g.dst) for g in (synth.generate('C1', 2), synth.generate('C2', 5, n=60000))]
cases += [(9000, hub_s, hub_d), (12000, hub_s, hub_d)]   # hub-heavy; the second has 3000 isolated nodes
for n, s, d in cases:
    for dims in ((64, 64, 32), (128, 128, 64), (128, 128, 64, 32)):
        Z, _ = rg.raftgp_build_embed(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(),
                                     ['ncut', 'mod'], dims, 3)
        out.append(torch.cat([Z['ncut'], Z['mod']], 1).cpu().numpy())
        g = rg.raftgp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
        _, Zs = rg.raftgp_embed_multi(g, ['ncut'], dims, 3)
        out.append(Zs['ncut'].cpu().numpy())
np.savez(sys.argv[1], *out)
print('ok')
"""


def test_slot_layout_bit_identical(rg, tmp_path):
    """The slot layout of the hop operands (RAFTGP_RELABEL=1, the default: hub rows first, non-hub gathers
    evict-first) changes only where operand rows live: every embedding is bit-identical to the node-order layout
    (both variants and NCut alone, 2- and 3-layer stacks, hub-heavy graphs and isolated nodes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"r{mode}.npz")
        r = subprocess.run([sys.executable, "-c", _RELABEL_SCRIPT, f], cwd=root,
                           env=dict(os.environ, RAFTGP_RELABEL=mode), capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
        z = np.load(f)
        res[mode] = [z[k] for k in sorted(z.files, key=lambda k: int(k.split("_")[1]))]
    assert len(res["0"]) == len(res["1"])
    for a, b in zip(res["0"], res["1"]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
