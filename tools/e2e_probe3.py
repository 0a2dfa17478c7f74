"""Does a concurrent D2H DMA stretch the CSR build's host read-backs? raftgp_build_csr (C4, device edges) timed with
CUDA events on its stream and by the host clock, alone and while 2.56 GB D2H copies run on another stream."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

dev = torch.device("cuda", 0)
gr = synth.generate("C4", 0)
cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ctx = rg.Context(0, stream=cs)
src, dst = torch.from_numpy(gr.src).to(dev), torch.from_numpy(gr.dst).to(dev)
Z = torch.empty((gr.n, 128), device=dev)
H = torch.empty((gr.n, 128)).pin_memory()
for bg in (False, True, False, True):
    ws, es = [], []
    for it in range(6):
        if bg:
            with torch.cuda.stream(ds):
                for _ in range(2):
                    H.copy_(Z, non_blocking=True)
        torch.cuda.synchronize(cs) if False else cs.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        with torch.cuda.stream(cs):
            e0.record(cs)
            g = rg.raftgp_build_csr(ctx, gr.n, src, dst)
            e1.record(cs)
        cs.synchronize()
        ws.append((time.perf_counter() - t) * 1e3)
        es.append(e0.elapsed_time(e1))
        g.close()
        torch.cuda.synchronize()
    print(f"background D2H={bg}: build_csr host {sum(ws[2:]) / 4:.2f} ms, events {sum(es[2:]) / 4:.2f} ms", flush=True)
