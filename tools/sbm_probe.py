"""Run raftgp_sbm_sample on the C4 DC-SBM parameters (for ncu captures of the walk kernels)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--q", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda", 0)
c, th, om = synth.sbm_params(a.config, 0)
ct, tt, ot = (torch.from_numpy(x).to(dev) for x in (c, th, om))
ctx = rg.Context(0)
for i in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, d = rg.raftgp_sbm_sample(ctx, ct, tt, ot, i, q=a.q)
    torch.cuda.synchronize()
    print(f"rep {i}: {s.numel()} edges, {1e3 * (time.perf_counter() - t0):.1f} ms")
