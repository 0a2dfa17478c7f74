"""Theta' = Theta W1 kernel alone (raftgp_sketch_transform) at C4's n, event-timed (for A/B builds via RAFTGP_LIB)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_01560_b200 import raftgp as rg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
ctx = rg.Context(0)
W = rg.raftgp_weights(ctx, 0, 1, 128, 128)
out = torch.empty((n, 128), dtype=torch.float32, device="cuda")
lib = rg.load_library()
for _ in range(3):
    rg._ck(lib.raftgp_sketch_transform(ctx.h, 0, n, 128, rg._ptr(W), 128, rg._ptr(out)))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    rg._ck(lib.raftgp_sketch_transform(ctx.h, 0, n, 128, rg._ptr(W), 128, rg._ptr(out)))
e1.record()
torch.cuda.synchronize()
print("sketch_w_tc n=%d: %.3f ms" % (n, e0.elapsed_time(e1) / 10))
