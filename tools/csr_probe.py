"""CSR build probe: raftgp_build_csr on a config's synthetic edge list (device-resident), timed with CUDA events
over `--reps` builds, per-kernel times from the library's profiling events, and (--hash) a digest of the exported
CSR so two partition paths (RAFTGP_CSR_TWO_LEVEL=0/1, run as two processes) can be compared bit for bit.

    python tools/csr_probe.py --config C4 --reps 5 --hash
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--hash", action="store_true")
a = ap.parse_args()

t = time.time()
gr = synth.generate(a.config, 0)
print("synth", a.config, gr.n, gr.src.size, "%.1f s" % (time.time() - t), flush=True)
ctx = rg.Context(0)
src, dst = torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda()
times = []
g = None
for rep in range(a.reps):
    if g is not None:
        g.close()
    ctx.set_profiling(True)
    ctx.prof_reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g = rg.raftgp_build_csr(ctx, gr.n, src, dst)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
prof = {k: round(v[0], 4) for k, v in sorted(ctx.prof_read().items(), key=lambda kv: -kv[1][0]) if v[1]}
info = g.info()
out = {"config": a.config, "n": gr.n, "pairs": int(gr.src.size), "nnz": info["nnz_local"],
       "two_level": os.environ.get("RAFTGP_CSR_TWO_LEVEL", "1"), "ms": [round(x, 3) for x in times],
       "ms_min": round(min(times), 3), "kernels_ms_last": prof,
       "entries_per_s": info["nnz_local"] / (min(times) * 1e-3)}
if a.hash:
    rp, col, deg = g.export()
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(rp).tobytes())
    h.update(np.ascontiguousarray(col).tobytes())
    out["csr_digest"] = h.hexdigest()
print(json.dumps(out), flush=True)
