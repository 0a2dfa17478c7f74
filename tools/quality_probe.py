"""Separability of the planted blocks in the embeddings at a config (diagnostic for the Alg. 1 quality
numbers): cosine similarity of random same-block vs different-block node pairs, and the accuracy of
assigning every node to the nearest planted-block centroid (an upper-bound-style probe of what a clustering
of Z could recover). Torch on the GPU, evaluation only."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2312_01560_b200 import raftgp as rg
    ctx = rg.Context(0)
    out = {}
    for name in a.configs.split(","):
        cfg = synth.CONFIGS[name]
        gr = synth.generate(cfg, 0)
        g = rg.raftgp_build_csr(ctx, gr.n, torch.from_numpy(gr.src).cuda(), torch.from_numpy(gr.dst).cuda())
        _, Z = rg.raftgp_embed_multi(g, ["ncut", "mod"], cfg.dims, 0)
        lab = torch.from_numpy(gr.labels.astype("int64")).cuda()
        K = int(lab.max()) + 1
        gen = torch.Generator(device="cuda").manual_seed(1)
        res = {"n": gr.n, "K": K, "dims": list(cfg.dims)}
        for v, z in Z.items():
            i = torch.randint(0, gr.n, (200000,), device="cuda", generator=gen)
            j = torch.randint(0, gr.n, (200000,), device="cuda", generator=gen)
            cos = (z[i] * z[j]).sum(1)
            same = lab[i] == lab[j]
            # same-block pairs drawn directly: a random partner from the same block
            order = torch.argsort(lab)
            starts = torch.searchsorted(lab[order], torch.arange(K + 1, device="cuda"))
            cnt = (starts[1:] - starts[:-1])[lab[i]]
            off = (torch.rand(i.shape[0], device="cuda", generator=gen) * cnt).long()
            jj = order[starts[lab[i]] + off]
            cos_same = (z[i] * z[jj]).sum(1)
            cen = torch.zeros(K, z.shape[1], device="cuda").index_add_(0, lab, z)
            cen = cen / cen.norm(dim=1, keepdim=True).clamp_min(1e-12)
            acc = 0
            for b0 in range(0, gr.n, 1 << 20):
                zz = z[b0:b0 + (1 << 20)]
                acc += int(((zz @ cen.T).argmax(1) == lab[b0:b0 + (1 << 20)]).sum())
            res[v] = {"cos_same_block_mean": float(cos_same.mean()), "cos_random_pair_mean": float(cos[~same].mean()),
                      "nearest_block_centroid_accuracy": acc / gr.n, "chance": 1.0 / K}
            # Alg. 1 on this embedding: how whole are the planted blocks inside its clusters?
            labs, Kf, _ = rg.raftgp_model_select(g, z)
            lf = torch.as_tensor(labs).cuda().long()
            tab = torch.zeros(K, Kf, device="cuda").index_put_((lab, lf), torch.ones_like(lab, dtype=torch.float32),
                                                               accumulate=True)
            purity = float(tab.max(1).values.sum() / gr.n)   # share of nodes in their block's majority cluster
            res[v]["alg1_blocks_found"] = int(Kf)
            res[v]["alg1_block_wholeness"] = purity
        out[name] = res
        print(name, json.dumps(res), flush=True)
        g.close()
    return out


if __name__ == "__main__":
    main()
