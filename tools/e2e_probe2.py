"""e2e D2H at C4: raftgp_build_embed steps on one compute stream; Z copied to pinned host memory per step by nothing
or by the copy engines (torch copy_ on a D2H stream); ms per step (wall, 6 steps after 3 warm-up) and the library's
per-kernel event times (their sum against the wall time shows the idle gaps)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

dev = torch.device("cuda", 0)
gr = synth.generate("C4", 0)
n = gr.n
cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ctx = rg.Context(0, stream=cs)
variants, dims = ["ncut", "mod"], (128, 128, 64)
src, dst = torch.from_numpy(gr.src).to(dev), torch.from_numpy(gr.dst).to(dev)
Zb = [{v: torch.empty((n, 64), device=dev) for v in variants} for _ in range(2)]
Hb = [{v: torch.empty((n, 64)).pin_memory() for v in variants} for _ in range(2)]


def run(steps, mode, ctas=0):
    for k in range(steps):
        b = k % 2
        with torch.cuda.stream(cs):
            rg.raftgp_build_embed(ctx, n, src, dst, variants, dims, 0, Z=Zb[b])
        if mode == "none":
            continue
        ds.wait_stream(cs)
        with torch.cuda.stream(ds):
            for v in variants:
                Hb[b][v].copy_(Zb[b][v], non_blocking=True)
    torch.cuda.synchronize()


modes = [("none", 0), ("dma", 0), ("none", 0), ("dma", 0)]
for mode, ctas in modes:
    run(3, mode, ctas)
    ctx.set_profiling(True)
    ctx.prof_reset()
    t = time.perf_counter()
    run(6, mode, ctas)
    dt = (time.perf_counter() - t) / 6
    prof = {k: round(v[0] / 6, 2) for k, v in sorted(ctx.prof_read().items(), key=lambda kv: -kv[1][0]) if v[1]}
    ctx.set_profiling(False)
    print(f"d2h={mode} ctas={ctas}: {dt * 1e3:.1f} ms/step  kernels/step {prof}", flush=True)
