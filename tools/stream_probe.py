"""NEXT-4 probe: C4 graph, NCut stream (dims 128 -> 128 -> 64), batches of B random new edges; prints the
time of each raftgp_stream_add_edges and the recomputed set sizes (for ncu launch lists)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--batch", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="exact", choices=["exact", "delta"])
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
gr = synth.generate(cfg, 0)
ctx = rg.Context(0)
g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
s = rg.Stream(g, cfg.dims, 0)
if a.mode == "delta":
    torch.cuda.synchronize()
    t = time.perf_counter()
    s.set_mode("delta")
    torch.cuda.synchronize()
    print(f"set_mode(delta) (state build, full pass): {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
rng = np.random.default_rng(5)
ctx.set_profiling(True)
for i in range(a.reps):
    ctx.prof_reset()
    src = torch.from_numpy(rng.integers(0, gr.n, a.batch).astype(np.int32)).cuda()
    dst = torch.from_numpy(rng.integers(0, gr.n, a.batch).astype(np.int32)).cuda()
    torch.cuda.synchronize()
    t = time.perf_counter()
    st = s.add_edges(src, dst)
    torch.cuda.synchronize()
    print(f"{a.mode} batch {a.batch}: {1e3 * (time.perf_counter() - t):.2f} ms {st}", flush=True)
    prof = ctx.prof_read()
    print("   kernels (ms, launches):", {k: (round(v[0], 3), v[1]) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])},
          "sum %.2f ms" % sum(v[0] for v in prof.values()), flush=True)
