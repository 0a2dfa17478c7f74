"""e2e overhead probe: raftgp_build_embed steps on one stream, with/without the H2D of the edges and the D2H of
Z on their own streams (C4). Shows what the copies cost the kernels."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2312_01560_b200 import raftgp as rg
dev = torch.device('cuda', 0)
gr = synth.generate(synth.CONFIGS['C4'], 0)
n, m = gr.n, gr.src.size
src_h = torch.from_numpy(gr.src).pin_memory(); dst_h = torch.from_numpy(gr.dst).pin_memory()
cs, hs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ctx = rg.Context(0, stream=cs)
variants, dims = ['ncut', 'mod'], (128, 128, 64)
Din = [(src_h.to(dev), dst_h.to(dev)) for _ in range(2)]
Zb = [{v: torch.empty((n, 64), device=dev) for v in variants} for _ in range(2)]
Hb = [{v: torch.empty((n, 64)).pin_memory() for v in variants} for _ in range(2)]
def run(steps, do_h2d, do_d2h):
    for k in range(steps):
        b = k % 2
        if do_h2d:
            hs.wait_stream(cs)
            with torch.cuda.stream(hs):
                Din[b][0].copy_(src_h, non_blocking=True); Din[b][1].copy_(dst_h, non_blocking=True)
            cs.wait_stream(hs)
        with torch.cuda.stream(cs):
            rg.raftgp_build_embed(ctx, n, Din[b][0], Din[b][1], variants, dims, 0, Z=Zb[b])
        if do_d2h:
            ds.wait_stream(cs)
            with torch.cuda.stream(ds):
                for v in variants: Hb[b][v].copy_(Zb[b][v], non_blocking=True)
    torch.cuda.synchronize()
for h2d, d2h in [(False, False), (False, True), (True, False), (True, True)]:
    run(3, h2d, d2h)
    t = time.perf_counter(); run(6, h2d, d2h); dt = (time.perf_counter() - t) / 6
    print(f"h2d={h2d} d2h={d2h}: {dt*1e3:.1f} ms/step", flush=True)
