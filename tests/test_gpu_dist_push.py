"""The fused-exchange pipeline over REAL peer memory: two processes (ranks) on one GPU, each with its own
context, map each other's operand copies through CUDA IPC (raftgp_ipc_alloc / raftgp_ipc_open via
dist.PushBuffers) and the hop kernels store their rows into both copies. gloo carries the handle exchange
and host barriers (the two ranks' kernels never wait on each other). The embeddings must be bit-identical
to the one-rank pipeline (itself within 1e-4 of the oracle, test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, src, dst, variants, dims, seed, out, noipc=False):
    if noipc:
        os.environ["RAFTGP_PUSH_NOIPC"] = "1"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_01560_b200 import dist as rdist
        from paper_2312_01560_b200 import raftgp as rg
        ctx = rg.Context(0)
        push = rdist.PushBuffers(ctx)
        for rep in range(2):   # the second step reuses the mapped copies
            gen = rdist.rank_pipeline_push(rdist.CudaEngine(ctx), n, torch.from_numpy(src).cuda(),
                                           torch.from_numpy(dst).cuda(), rank, world, variants, dims, seed)
            Z = rdist.run_distributed(gen, push=push)
            torch.cuda.synchronize()
            out[(rank, rep)] = {v: Z[v].cpu().numpy() for v in Z}
            out[("mapped", rank)] = push.mapped
        push.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("noipc", [False, True])
@pytest.mark.parametrize("world", [2])
def test_ipc_push_two_processes(cuda_required, world, noipc):
    """noipc: peer mapping made to fail on every rank -> the copies are completed by all-gathers instead."""
    import synth
    from paper_2312_01560_b200 import raftgp as rg
    gr = synth.generate("C2", 1, n=20000)
    dims = (128, 128, 64)
    variants = ["ncut", "mod"]
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), gr.n, gr.src, gr.dst, variants, dims, 5, out, noipc),
                       nprocs=world, join=True, start_method="spawn")
    from paper_2312_01560_b200 import dist as rdist
    ctx = rg.Context(0)
    Z = rdist.run_loopback([rdist.rank_pipeline(rdist.CudaEngine(ctx), gr.n, torch.from_numpy(gr.src).cuda(),
                                                torch.from_numpy(gr.dst).cuda(), 0, 1, variants, dims, 5)])[0]
    assert all(out[("mapped", r)] == (not noipc) for r in range(world))
    for rep in range(2):
        for v in variants:
            got = np.concatenate([out[(r, rep)][v] for r in range(world)], 0)
            assert np.array_equal(got, Z[v].cpu().numpy()), (rep, v)
