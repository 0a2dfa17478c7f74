"""The row-partitioned step INSIDE the library (paper_2312_01560_b200/csrc/dist.cu).

* loopback (P logical ranks on this GPU, raftgp_build_embed_loopback): bit-identical to one GPU for P = 1, 2, 3, 8,
  ragged and empty shards (n < P), every variant set, 2- and 3-layer stacks, and the switches of the schedule
  (Theta' regenerated per rank vs. pushed by its owner; Mod's T_1 push deferred or fused) in subprocesses;
* a one-rank NCCL communicator (raftgp_ctx_create_dist) through raftgp_build_embed: the same push pipeline with a
  real ncclComm (barrier, degree all-gather, g broadcast), bit-identical to one GPU; raftgp_barrier and
  raftgp_allgather on the context stream;
* the plain-C demo in its row-partitioned mode (world = 1), matching its single-GPU printout.
Multi-rank NCCL jobs need one GPU per rank; the gloo CPU tests (test_dist_gloo.py) and the two-process IPC test
(test_gpu_dist_push.py) cover the host-side protocol."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def _graph(kind):
    if kind == "c2":
        g = synth.generate("C2", 0)
        return g.n, g.src, g.dst
    if kind == "c1":
        g = synth.generate("C1", 2)
        return g.n, g.src, g.dst
    if kind == "tiny":   # n < P for P = 8: empty shards
        return 5, np.array([0, 1, 2, 3, 4, 0], np.int32), np.array([1, 2, 3, 4, 0, 2], np.int32)
    n = 3001   # isolated tail + duplicates / self-loops
    s, d = synth.random_edges(2900, 40000, seed=5)
    return n, s, d


CASES = [
    ("c2", ["ncut", "mod"], (64, 64, 32)),
    ("c2", ["ncut", "mod"], (128, 128, 64)),
    ("c1", ["ncut", "mod", "mod_reduced"], (64, 32, 32, 32)),
    ("rand", ["mod_reduced"], (32, 64, 32)),
    ("rand", ["mod", "ncut"], (128, 64, 128)),
    ("tiny", ["ncut", "mod"], (64, 64, 32)),
]


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("kind,variants,dims", CASES, ids=[f"{c[0]}-{'+'.join(c[1])}-{'x'.join(map(str, c[2]))}"
                                                           for c in CASES])
def test_loopback_bit_identical(rg, ctx, P, kind, variants, dims):
    n, src, dst = _graph(kind)
    s, d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    ref, _ = rg.raftgp_build_embed(ctx, n, s, d, variants, dims, 7)
    got = rg.raftgp_build_embed_loopback(ctx, P, n, s, d, variants, dims, 7)
    for v in variants:
        assert torch.equal(got[v], ref[v]), (v, P)


def test_loopback_host_edges(rg, ctx):
    n, src, dst = _graph("c1")
    ref, _ = rg.raftgp_build_embed(ctx, n, torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(),
                                   ["ncut", "mod"], (64, 64, 32), 2)
    got = rg.raftgp_build_embed_loopback(ctx, 3, n, torch.from_numpy(src), torch.from_numpy(dst), ["ncut", "mod"],
                                         (64, 64, 32), 2)
    for v in ("ncut", "mod"):
        assert torch.equal(got[v], ref[v])


def test_loopback_errors(rg, ctx):
    n, src, dst = _graph("c1")
    s, d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    for P, dims in ((0, (64, 64, 32)), (9, (64, 64, 32)), (2, (64, 48, 32))):
        with pytest.raises(rg.RaftGPError) as e:
            rg.raftgp_build_embed_loopback(ctx, P, n, s, d, ["ncut"], dims, 1)
        assert e.value.code == rg.RAFTGP_ERR_PARAM
    bad = d.clone()
    bad[3] = n + 5
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_build_embed_loopback(ctx, 2, n, s, bad, ["ncut"], (64, 64, 32), 1)
    assert e.value.code == rg.RAFTGP_ERR_DATA


_SWITCH = r"""
import sys, torch, numpy as np
sys.path.insert(0, {root!r})
import synth
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
g = synth.generate("C2", 1)
s, d = torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda()
ref, _ = rg.raftgp_build_embed(ctx, g.n, s, d, ["ncut", "mod"], (128, 128, 64), 3)
for P in (2, 5):
    got = rg.raftgp_build_embed_loopback(ctx, P, g.n, s, d, ["ncut", "mod"], (128, 128, 64), 3)
    assert all(torch.equal(got[v], ref[v]) for v in ("ncut", "mod")), P
print("ok")
"""


@pytest.mark.parametrize("env", [{"RAFTGP_DIST_THETA": "regen"}, {"RAFTGP_DIST_DEFER": "0"},
                                 {"RAFTGP_DIST_SPLIT_LAST": "0"}])
def test_loopback_schedule_switches(cuda_required, env):
    out = subprocess.run([sys.executable, "-c", _SWITCH.format(root=ROOT)], capture_output=True, text=True,
                         timeout=600, env={**os.environ, **env})
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_one_rank_nccl_context(rg, ctx):
    uid = rg.raftgp_nccl_unique_id()
    dctx = rg.Context(0, dist=(0, 1, uid))
    assert dctx.rank_world() == (0, 1) and ctx.rank_world() == (0, 1)
    gr = synth.generate("C2", 0)
    s, d = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
    ref, _ = rg.raftgp_build_embed(ctx, gr.n, s, d, ["ncut", "mod"], (128, 128, 64), 0)
    for _ in range(2):   # the second step reuses the cached operand copies
        got, gh = rg.raftgp_build_embed(dctx, gr.n, s, d, ["ncut", "mod"], (128, 128, 64), 0)
        assert gh is None
        for v in ("ncut", "mod"):
            assert torch.equal(got[v], ref[v])
    got, _ = rg.raftgp_build_embed(dctx, gr.n, torch.from_numpy(gr.src), torch.from_numpy(gr.dst), ["mod_reduced"],
                                   (64, 64, 32), 4)
    ref, _ = rg.raftgp_build_embed(ctx, gr.n, s, d, ["mod_reduced"], (64, 64, 32), 4)
    assert torch.equal(got["mod_reduced"], ref["mod_reduced"])
    # collectives on the context stream
    x = torch.arange(10, dtype=torch.int32, device="cuda")
    y = torch.zeros(10, dtype=torch.int32, device="cuda")
    dctx.allgather(x, y)
    dctx.barrier()
    dctx.sync()
    assert torch.equal(x, y)
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_build_embed(dctx, gr.n, s, d, ["ncut"], (64, 64, 32), 0, keep_graph=True)
    assert e.value.code == rg.RAFTGP_ERR_PARAM
    dctx.close()


def test_c_demo_row_partitioned_one_rank(cuda_required, tmp_path):
    from paper_2312_01560_b200 import build as b
    exe = b.build_demo()
    n = 4099
    one = subprocess.run([exe, str(n), "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    dist = subprocess.run([exe, str(n), "1", "0", "1", str(tmp_path / "uid")], capture_output=True, text=True,
                          timeout=300, cwd=ROOT)
    assert one.returncode == 0 and dist.returncode == 0, dist.stderr
    a = {l.split()[0]: l for l in one.stdout.splitlines()}
    b_ = {l.split()[0]: l for l in dist.stdout.splitlines()}
    assert b_["rank"].split()[1:] == ["0", "world", "1", "rows", "0", str(n)]
    for v in ("ncut", "mod"):
        assert a[v] == b_[v]
