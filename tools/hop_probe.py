"""Hop probe at C4: the dual feature hop (one Theta' gather, NCut + Mod outputs) against a plain GCN hop gathering the
same Theta' operand (same widths, one output), with the library's per-kernel events; for A/B builds of spmm.cu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

gr = synth.generate("C4", 0)
ctx = rg.Context(0)
g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
Z = torch.empty((gr.n, 128), dtype=torch.float32, device="cuda")
W = rg.raftgp_weights(ctx, 0, 1, 128, 128)
TH = rg.raftgp_sketch_transform(ctx, 0, gr.n, W)
for _ in range(2):
    rg.raftgp_feature_transform(g, ["ncut", "mod"], 128, 128, 0)
    rg.raftgp_gcn_hop(g, TH, Z)
torch.cuda.synchronize()
ctx.set_profiling(True)
ctx.prof_reset()
reps = 5
for _ in range(reps):
    rg.raftgp_feature_transform(g, ["ncut", "mod"], 128, 128, 0)
    rg.raftgp_gcn_hop(g, TH, Z)
torch.cuda.synchronize()
p = ctx.prof_read()
print({k: round(v[0] / reps, 3) for k, v in p.items() if v[1]})
