"""Do concurrent D2H DMA copies slow the HBM-bound hops? A GCN hop over C4's 128-wide operand, event-timed alone and
while 2.56 GB D2H copies (pinned destination) run on another stream."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

dev = torch.device("cuda", 0)
gr = synth.generate("C4", 0)
cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ctx = rg.Context(0, stream=cs)
g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).to(dev), torch.from_numpy(gr.dst).to(dev))
T = torch.randn((gr.n, 128), device=dev)
Zo = torch.empty((gr.n, 128), device=dev)
Zs = torch.empty((gr.n, 64), device=dev)
H = torch.empty((gr.n, 64)).pin_memory()
for bg in (False, True, False, True, "h2d"):
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(ds):
            for _ in range(8):
                if bg == "h2d":
                    Zs.copy_(H, non_blocking=True)
                else:
                    H.copy_(Zs, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        for _ in range(4):
            rg.raftgp_gcn_hop(g, T, Zo)
        e1.record(cs)
    torch.cuda.synchronize()
    print(f"background copies={bg}: gcn hop {e0.elapsed_time(e1) / 4:.2f} ms", flush=True)
