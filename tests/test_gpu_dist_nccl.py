"""The distributed driver over REAL NCCL on the GPU box (one rank: the round's GPU budget is one B200). It runs
the rank pipeline of paper_2312_01560_b200/dist.py through run_distributed with a 1-rank NCCL process group —
blocking and async all_gather_into_tensor, work handles waited on the compute stream, a non-default compute
stream — and checks the result is bit-identical to the single-GPU call. Multi-rank exchange logic is covered by
the gloo tests (tests/test_dist_gloo.py) and the P-rank loopback test (tests/test_gpu_parity.py). Reference: the
same pipeline driven by the loopback driver (bit-identical), and the oracle (1e-4)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group(cuda_required):
    import torch.distributed as dist
    if dist.is_initialized():
        yield dist
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_rank_pipeline_over_nccl_matches_single_gpu(nccl_group):
    from paper_2312_01560_b200 import dist as rdist
    from paper_2312_01560_b200 import raftgp as rg
    rg.load_library()
    gr = synth.generate("C2", 3)
    dims = (64, 64, 32)
    variants = ["ncut", "mod"]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx = rg.Context(0)
        src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
        keep = {}
        gen = rdist.rank_pipeline(rdist.CudaEngine(ctx), gr.n, src, dst, 0, 1, variants, dims, 5, keep)
        Z = rdist.run_distributed(gen)
        ref = rdist.run_loopback([rdist.rank_pipeline(rdist.CudaEngine(ctx), gr.n, src, dst, 0, 1, variants, dims, 5)])[0]
    torch.cuda.synchronize()
    go = oracle.build_csr(gr.n, gr.src, gr.dst)
    for v in variants:
        assert torch.equal(Z[v], ref[v]), v
        Zo = oracle.gcn(go, list(dims), 5, oracle.project(go, v, dims[0], 5))[-1]
        assert np.linalg.norm(Z[v].cpu().numpy() - Zo) / np.linalg.norm(Zo) <= 1e-4


@pytest.mark.parametrize("push", [False, True])
def test_rank_pipeline_over_library_comm(nccl_group, push):
    """The Python-driven pipelines with the exchanges on the LIBRARY's communicator (raftgp_ctx_create_dist:
    raftgp_allgather for the degree / operand all-gathers, raftgp_barrier for the push barriers)."""
    from paper_2312_01560_b200 import dist as rdist
    from paper_2312_01560_b200 import raftgp as rg
    gr = synth.generate("C2", 3)
    dims = (64, 64, 32)
    variants = ["ncut", "mod"]
    ctx = rg.Context(0)
    lib = rg.Context(0, dist=(0, 1, rg.raftgp_nccl_unique_id()))
    src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
    pipe = rdist.rank_pipeline_push if push else rdist.rank_pipeline
    bufs = rdist.PushBuffers(lib) if push else None
    gen = pipe(rdist.CudaEngine(lib), gr.n, src, dst, 0, 1, variants, dims, 5)
    Z = rdist.run_distributed(gen, push=bufs, lib_ctx=lib)
    torch.cuda.synchronize()
    if bufs is not None:
        bufs.close()
    # reference: the same pipeline driven in loopback on a plain context (one rank)
    ref = rdist.run_loopback([pipe(rdist.CudaEngine(ctx), gr.n, src, dst, 0, 1, variants, dims, 5)],
                             device=ctx.device)[0]
    for v in variants:
        assert torch.equal(Z[v], ref[v]), v
    lib.close()
