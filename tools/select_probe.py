"""Probe of raftgp_model_select at a config (for ncu launch lists / captures): build, embed, select."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--variant", default="mod")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--max-iter", type=int, default=100)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2312_01560_b200 import raftgp as rg
    cfg = synth.CONFIGS[a.config]
    gr = synth.generate(cfg, 0)
    ctx = rg.Context(0)
    g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
    _, Z = rg.raftgp_embed(g, a.variant, cfg.dims, 0, want_Y=False)
    for i in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        lab, K, st = rg.raftgp_model_select(g, Z, max_iter=a.max_iter)
        torch.cuda.synchronize()
        print(f"rep {i}: {1e3 * (time.perf_counter() - t):.2f} ms K={K} {st}", flush=True)


if __name__ == "__main__":
    main()
