"""Multi-process (world_size 2 and 3, gloo, CPU) test of the row-partitioned orchestration in
paper_2312_01560_b200/dist.py: partitioning, padding, the degree all-gather and the per-hop operand
all-gather. The local compute steps run in a small fp64 numpy engine (test-only) so this runs without a
GPU; the CUDA engine is the same pipeline with libraftgp doing the local steps (covered on the GPU by
test_gpu_parity.py::test_partitioned_equals_whole). The result must equal the oracle's whole-graph
pipeline (Eq. 5 + Eq. 6)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2312_01560_b200 import dist as rdist


class NumpyEngine:
    """fp64 local steps (rows [rb, re) only; global degrees after set_degrees)."""

    def build(self, n, src, dst, rb, re):
        full = oracle.build_csr(n, src.numpy(), dst.numpy())
        rp = full.row_ptr[rb:re + 1] - full.row_ptr[rb]
        col = full.col[full.row_ptr[rb]:full.row_ptr[re]]
        return {"n": n, "rb": rb, "re": re, "rp": rp, "col": col, "rows": re - rb}

    def local_degrees(self, h):
        return torch.from_numpy(np.diff(h["rp"]).astype(np.int32))

    def set_degrees(self, h, deg_all):
        d = deg_all.numpy().astype(np.float64)
        h["d"], h["two_e"] = d, d.sum()
        with np.errstate(divide="ignore"):
            h["s"] = np.where(d > 0, 1.0 / np.sqrt(d), 0.0)
        h["sh"] = 1.0 / np.sqrt(d + 1.0)

    def project(self, h, variant, r, seed):
        th = oracle.theta(h["n"], r, seed).astype(np.float64)
        rows = range(h["rb"], h["re"])
        Y = np.zeros((h["rows"], r))
        g = h["d"] @ th if variant == "mod" else None
        for li, i in enumerate(rows):
            nb = h["col"][h["rp"][li]:h["rp"][li + 1]]
            if variant == "ncut":
                Y[li] = h["s"][i] * (h["s"][nb] @ th[nb])
            elif variant == "mod":
                Y[li] = th[nb].sum(0) - h["d"][i] * g / h["two_e"]
            else:
                Y[li] = ((1.0 - h["d"][i] * h["d"][nb] / h["two_e"]) @ th[nb])
        return torch.from_numpy(Y)

    def weights(self, seed, k, a, b):
        return torch.from_numpy(oracle.weights(k, a, b, seed).astype(np.float64))

    def feature_transform(self, h, variants, dims, seed):
        W1 = self.weights(seed, 1, dims[0], dims[1])
        return {v: self.transform(h, self.project(h, v, dims[0], seed), W1) for v in variants}

    def transform(self, h, Z, W):
        sh = h["sh"][h["rb"]:h["re"], None]
        return torch.from_numpy(sh * (Z.numpy() @ W.numpy()))

    def hop(self, h, T_full, W_next, want_Z):
        T = T_full.numpy()
        Z = np.zeros((h["rows"], T.shape[1]))
        for li, i in enumerate(range(h["rb"], h["re"])):
            nb = h["col"][h["rp"][li]:h["rp"][li + 1]]
            z = np.tanh(h["sh"][i] * (T[i] + T[nb].sum(0)))
            nrm = np.linalg.norm(z)
            Z[li] = z / nrm if nrm > 0 else z
        Tn = None
        if W_next is not None:
            Tn = torch.from_numpy(h["sh"][h["rb"]:h["re"], None] * (Z @ W_next.numpy()))
        return (torch.from_numpy(Z) if want_Z else None), Tn

    # push mode: write this rank's rows [rb, re) into every given full copy
    def feature_transform_push(self, h, variants, dims, seed, reps):
        T = self.feature_transform(h, variants, dims, seed)
        for v in variants:
            for buf in reps[v]:
                buf[h["rb"]:h["re"]] = T[v]

    def hop_push(self, h, T_own, w, W_next, reps_next):
        _, Tn = self.hop(h, T_own, W_next, want_Z=False)
        for buf in reps_next:
            buf[h["rb"]:h["re"]] = Tn

    def hop_last(self, h, T_own, w):
        return self.hop(h, T_own, None, want_Z=True)[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, src, dst, variants, dims, seed, out, push=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pipe = rdist.rank_pipeline_push if push else rdist.rank_pipeline
        gen = pipe(NumpyEngine(), n, torch.from_numpy(src), torch.from_numpy(dst), rank, world, variants, dims, seed)
        Z = rdist.run_distributed(gen)
        out[rank] = {v: Z[v].numpy() for v in Z}
    finally:
        dist.destroy_process_group()


def _run(world, n, src, dst, variants, dims, seed, push=False):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, src, dst, variants, dims, seed, out, push), nprocs=world,
             join=True)
    return {v: np.concatenate([out[r][v] for r in range(world)], 0) for v in variants}


def test_row_partition():
    ranges, R = rdist.row_partition(10, 4)
    assert R == 3 and ranges == [(0, 3), (3, 6), (6, 9), (9, 10)]
    ranges, R = rdist.row_partition(5, 4)            # an empty last rank
    assert ranges == [(0, 2), (2, 4), (4, 5), (5, 5)]
    ranges, R = rdist.row_partition(0, 2)
    assert ranges == [(0, 0), (0, 0)] and R == 1


@pytest.mark.parametrize("push", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_row_partitioned_pipeline_matches_oracle(world, push):
    """push=True: the fused-exchange pipeline (rank_pipeline_push); on CPU the peer stores are stood in for
    by an all-gather of the row blocks at each barrier."""
    gr = synth.generate("C1", 2, n=301)               # 301 rows: ragged partition (101/101/99, 151/150)
    dims = (16, 12, 8)
    variants = ["ncut", "mod"]
    Zd = _run(world, gr.n, gr.src, gr.dst, variants, dims, 7, push)
    ref = oracle.build_csr(gr.n, gr.src, gr.dst)
    for v in variants:
        Yo = oracle.project(ref, v, dims[0], 7)
        Zo = oracle.gcn(ref, dims, 7, Yo)[-1]
        np.testing.assert_allclose(Zd[v], Zo, atol=1e-10)


@pytest.mark.parametrize("variants", ["mod_reduced", ["ncut", "mod"], ["mod", "mod_reduced", "ncut"]])
def test_loopback_equals_single_rank_numpy(variants):
    gr = synth.generate("C1", 4, n=120)
    dims = (8, 8, 6, 4)
    src, dst = torch.from_numpy(gr.src), torch.from_numpy(gr.dst)
    one = rdist.run_loopback([rdist.rank_pipeline(NumpyEngine(), gr.n, src, dst, 0, 1, variants, dims, 3)])[0]
    three = rdist.run_loopback([rdist.rank_pipeline(NumpyEngine(), gr.n, src, dst, p, 3, variants, dims, 3)
                                for p in range(3)])
    if isinstance(variants, str):
        np.testing.assert_allclose(torch.cat(three, 0).numpy(), one.numpy(), atol=1e-12)
    else:
        for v in variants:
            np.testing.assert_allclose(torch.cat([t[v] for t in three], 0).numpy(), one[v].numpy(), atol=1e-12)


@pytest.mark.parametrize("variants", ["ncut", ["ncut", "mod"], ["mod", "mod_reduced", "ncut"]])
def test_loopback_push_equals_single_rank_numpy(variants):
    """Push mode in lockstep: every logical rank writes its rows into all P copies; the copies each rank
    reads must be complete, so the result equals the one-rank pipeline."""
    gr = synth.generate("C1", 4, n=120)
    dims = (8, 8, 6, 4)
    src, dst = torch.from_numpy(gr.src), torch.from_numpy(gr.dst)
    one = rdist.run_loopback([rdist.rank_pipeline(NumpyEngine(), gr.n, src, dst, 0, 1, variants, dims, 3)])[0]
    three = rdist.run_loopback([rdist.rank_pipeline_push(NumpyEngine(), gr.n, src, dst, p, 3, variants, dims, 3)
                                for p in range(3)], dtype=torch.float64)
    if isinstance(variants, str):
        np.testing.assert_allclose(torch.cat(three, 0).numpy(), one.numpy(), atol=1e-12)
    else:
        for v in variants:
            np.testing.assert_allclose(torch.cat([t[v] for t in three], 0).numpy(), one[v].numpy(), atol=1e-12)
