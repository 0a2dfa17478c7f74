#!/usr/bin/env python
"""Benchmark of the RaftGP embedding hot path (BASELINE.json metric) on 1..8 B200s.

One step = the whole hot path over one synthetic DC-SBM graph resident in HBM:
canonical CSR build + degree pass (a1, a2), Gaussian sketch (a3), feature hop (a4) and the GCN hops with
fused epilogues (a5) for BOTH feature operators (NCut M and modularity Q; north_star (i)), plus the per-hop
all-gather (a6) when N > 1. value = work units / time, units = sum over variants and hops of
(gathered rows G_h) x (gathered width w_h) ("nnz*r").

Prints ONE JSON line on rank 0. `--impl reference` times the CPU oracle instead (the reference arm for
this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "embedding nnz*r/s and achieved HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "nnz*r/s"
L2_BYTES = 126 * 2 ** 20
SAMPLE_N = 50_000      # single-thread oracle sample: the same DC-SBM recipe at 1/100 of C4's nodes
REF_SAMPLE_N = 500_000  # --impl reference: per-step sample at 1/10 of C4's nodes, all host cores


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="raftgp", choices=["raftgp", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--variants", default="ncut,mod")
    ap.add_argument("--rule", default="stated", choices=["stated", "law"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-select", action="store_true", help="skip the NEXT-1 model-selection measurement")
    ap.add_argument("--select-reps", type=int, default=3)
    ap.add_argument("--no-table1", action="store_true", help="skip the NEXT-2 Table I widths measurement")
    ap.add_argument("--table1-steps", type=int, default=3)
    ap.add_argument("--no-sbm", action="store_true", help="skip the NEXT-3 SBM sampler measurement")
    ap.add_argument("--e2e-lanes", type=int, default=3, help="contexts/streams the e2e steps rotate over (N = 1)")
    ap.add_argument("--e2e-steps", type=int, default=10,
                    help="timed e2e steps (at least --steps): the pipeline's fill and drain (the first step's H2D, the "
                         "last step's D2H) are amortised over a job of this many steps")
    ap.add_argument("--exchange", default="lib", choices=["lib", "push", "allgather"],
                    help="N > 1: lib = the row-partitioned step inside the library (raftgp_build_embed on a context "
                         "created with raftgp_ctx_create_dist; exchanges fused into the producing kernels, NCCL "
                         "barriers); push / allgather = the same step driven from Python (dist.py) with peer stores "
                         "or NCCL all-gathers pipelined across variants")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch check only (no GPU work): spawn/join the ranks, rendezvous, max-over-ranks, one JSON "
                         "line with dry_run = true. Not a measurement.")
    ap.add_argument("--e2e-api", default="build_embed", choices=["separate", "build_embed"],
                    help="e2e step: raftgp_build_csr + raftgp_embed_multi, or raftgp_build_embed")
    ap.add_argument("--no-stream", action="store_true", help="skip the NEXT-4 streaming-update measurement")
    ap.add_argument("--clock-period-ms", type=int, default=200)
    ap.add_argument("--clock-query", default=None)
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-fuse-variants", action="store_true",
                    help="one raftgp_embed per variant instead of raftgp_embed_multi (shared Theta gather)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """Clocks + throttle reasons during the timed region: ONE `nvidia-smi -lms 200` process started before
    the region and stopped after it (no fork inside the timed region)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 200, enabled: bool = True, query: str = None):
        self.index = index
        self.period_ms = period_ms
        self.enabled = enabled
        self.query = query or self.Q
        self.rows = []
        self._p = None
        self._f = None

    def __enter__(self):
        import tempfile
        self._f = tempfile.TemporaryFile(mode="w+")
        if not self.enabled:
            return self
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.query}",
                                        "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                       stdout=self._f, stderr=subprocess.DEVNULL)
            time.sleep(0.5)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        self._f.seek(0)
        for line in self._f.read().strip().splitlines():
            self.rows.append([x.strip() for x in line.split(",")])
        self._f.close()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def work_units(nnz, n, r, dims, nvar):
    """sum_h G_h * w_h per step: feature hop gathers nnz rows of width r; GCN hop k gathers nnz + n rows
    of width dims[k] (GEMM-first: the operand of hop k is T_k = s^ (.) Z^(k-1) W^(k), dims[k] wide)."""
    u = nnz * r
    for k in range(1, len(dims)):
        u += (nnz + n) * dims[k]
    return nvar * u


def algorithmic_bytes(nnz, n, r, dims, nvar, kernel, fused_pair=False):
    """SURVEY.md §8(d) gather model per launch, summed over one step's launches of that kernel:
    B_h = 8(N+1) + 4 nnz + 4 w_h G_h + 4 w'_h N + 4 N. With fused_pair the NCUT and MOD feature hops share
    one launch (one gather of Theta, two written T1 blocks), and so do their last GCN hops (one read of the
    CSR and of s_hat, both 64-wide operands gathered side by side)."""
    L = len(dims) - 1
    if kernel == "feature_hop":
        if fused_pair:
            b = 8 * (n + 1) + 4 * nnz + 4 * r * nnz + 2 * 4 * dims[1] * n + 4 * n
            return b + (nvar - 2) * (b - 4 * dims[1] * n), nvar - 1
        b = 8 * (n + 1) + 4 * nnz + 4 * r * nnz + 4 * dims[1] * n + 4 * n
        return nvar * b, nvar
    if kernel == "gcn_hop":
        b = 0
        for k in range(1, L + 1):
            w_out = dims[k + 1] if k < L else dims[L]
            b += 8 * (n + 1) + 4 * nnz + 4 * dims[k] * (nnz + n) + 4 * w_out * n + 4 * n
        if fused_pair and nvar >= 2 and L >= 2 and dims[L] in (32, 64):   # gcn_pair_supported (spmm.cu)
            shared = 8 * (n + 1) + 4 * nnz + 4 * n
            return nvar * b - shared, nvar * L - 1
        return nvar * b, nvar * L
    return None, None


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_spawn(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks with torch.distributed.run on this node (one per
    GPU, rendezvous on 127.0.0.1) running this same command line; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, RAFTGP_BENCH_SPAWNED="1")
    return subprocess.call(cmd, env=env)


def sketch_ok(cfg) -> bool:
    return cfg.r in (32, 64, 128) and cfg.dims[1] in (32, 64, 128)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info():
    info = {"cores": os.cpu_count()}
    try:
        info["cpu"] = [l.split(":", 1)[1].strip() for l in subprocess.run(["lscpu"], capture_output=True, text=True)
                       .stdout.splitlines() if l.startswith("Model name")][0]
    except Exception:
        pass
    try:
        info["mem_gb"] = int(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout.splitlines()[1]
                             .split()[1])
    except Exception:
        pass
    return info


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def oracle_step(gr, variants, r, dims, seed):
    import oracle
    t0 = time.perf_counter()
    g = oracle.build_csr(gr.n, gr.src, gr.dst)
    for v in variants:
        Y = oracle.project(g, v, r, seed)
        oracle.gcn(g, dims, seed, Y)
    return time.perf_counter() - t0, g.nnz


def cpu_baseline(cfg, variants, seed, rule, steps=1, n=SAMPLE_N, threads=1):
    """The oracle as it stands, timed on this host: `threads` cores (1, or 0 = all: OpenMP over output rows, bit-
    identical results) on the config's recipe at `n` nodes (None = the full config)."""
    import oracle
    import synth
    gr = synth.generate(cfg, seed, rule=rule, n=n)
    oracle.set_threads(threads)
    try:
        times, nnz = [], 0
        for _ in range(steps):
            dt, nnz = oracle_step(gr, variants, cfg.r, cfg.dims, seed)
            times.append(dt)
        cores = oracle.get_threads()
    finally:
        oracle.set_threads(0)
    units = work_units(nnz, gr.n, cfg.r, cfg.dims, len(variants))
    return units / statistics.mean(times), gr, nnz, times, cores


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import synth
    cfg = synth.CONFIGS[args.config]
    variants = args.variants.split(",")
    import oracle
    oracle.build()
    synth.build()
    gr = synth.generate(cfg, args.seed, rule=args.rule, n=REF_SAMPLE_N)
    oracle.set_threads(0)
    cores = oracle.get_threads()
    for _ in range(args.warmup):
        oracle_step(gr, variants, cfg.r, cfg.dims, args.seed)
    times, nnz = [], 0
    for _ in range(args.steps):
        dt, nnz = oracle_step(gr, variants, cfg.r, cfg.dims, args.seed)
        times.append(dt)
    units = work_units(nnz, gr.n, cfg.r, cfg.dims, len(variants))
    total = sum(times)
    value = units * args.steps / total
    sample = (f"full oracle step (CSR build + both variants' projection + GCN) on the {cfg.name} DC-SBM recipe "
              f"at N={gr.n} (nnz={nnz}), {cores} threads (OpenMP over output rows; bit-identical to 1 thread)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} recipe sample, N={gr.n}", "n": gr.n, "nnz": nnz, "r": cfg.r,
                   "dims": list(cfg.dims), "variants": variants, "rule": args.rule},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def measure_select(args, rg, ctx, gr, src_d, dst_d, variants, dims, Zbuf, barrier, peak, peak_src):
    """NEXT-1 (Alg. 1): time raftgp_model_select on the embeddings of one step. The call is
    synchronous (the host drives the tree levels), so the events bracket what a caller waits for. The Lloyd
    pass is HBM-bound: per visited row it reads segment id, side and bounds and writes the bounds (24 B); a row
    that fails the bound test also reads its node id and Z row (4L + 4 B)."""
    import torch
    from sklearn.metrics import adjusted_rand_score, normalized_mutual_info_score
    g = rg.raftgp_build_csr(ctx, gr.n, src_d, dst_d)
    rg.raftgp_embed_multi(g, variants, dims, args.seed, Z=Zbuf)
    L = dims[-1]
    out = {"call": "raftgp_model_select(eps=5, max_iter=100, rule=global)", "unit": "nodes/s", "L": L}
    for v in variants:
        lab, K, st = rg.raftgp_model_select(g, Zbuf[v])        # warm-up (allocates the workspace)
        ctx.prof_reset()
        ctx.set_profiling(True)
        barrier()
        per = []
        for _ in range(args.select_reps):   # each call timed on its own; the median is reported
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            lab, K, st = rg.raftgp_model_select(g, Zbuf[v])
            e1.record(ctx.stream)
            e1.synchronize()
            per.append(e0.elapsed_time(e1))
        barrier()
        ms = sorted(per)[len(per) // 2]
        prof = {k: (t / args.select_reps, c // args.select_reps) for k, (t, c) in ctx.prof_read().items()}
        ctx.set_profiling(False)
        labels = lab.cpu().numpy()
        lloyd_ms = prof.get("select_lloyd", (0.0, 0))[0]
        lloyd_bytes = st["lloyd_rows"] * 24 + st["rows_read"] * (4 * L + 4)
        ach = lloyd_bytes / (lloyd_ms * 1e-3) / 1e9 if lloyd_ms else None
        out[v] = {
            "ms": ms, "ms_per_call": [round(x, 3) for x in per], "timing": "median of the calls",
            "value": gr.n / (ms * 1e-3), "blocks": K, "planted_blocks": int(gr.info["k"]),
            "ari_vs_planted": float(adjusted_rand_score(gr.labels, labels)),
            "nmi_vs_planted": float(normalized_mutual_info_score(gr.labels, labels)),
            "stats": st, "kernel_ms": {k: round(t, 4) for k, (t, _) in sorted(prof.items(), key=lambda x: -x[1][0])},
            "kernel_launches": sum(c for _, c in prof.values()),
            "lloyd_roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                               "frac": (ach / peak) if ach else None, "peak_source": peak_src,
                               "bytes": lloyd_bytes,
                               "bytes_rule": "visited rows * 24 (segment, side, bounds r/w) + read rows * (4L + 4)"},
        }
    g.close()
    # end-to-end quality where the BASELINE embeddings separate the blocks (C1, C2: 11 / 44 planted blocks)
    import synth
    out["quality"] = {}
    for qcfg in ("C1", "C2"):
        c = synth.CONFIGS[qcfg]
        qg = synth.generate(c, args.seed, rule=args.rule)
        qgr = rg.raftgp_build_csr(ctx, qg.n, torch.from_numpy(qg.src).to(ctx.device),
                                  torch.from_numpy(qg.dst).to(ctx.device))
        _, qZ = rg.raftgp_embed_multi(qgr, ["mod"], c.dims, args.seed)
        qlab, qK, _ = rg.raftgp_model_select(qgr, qZ["mod"])
        qlab = qlab.cpu().numpy()
        out["quality"][qcfg] = {"variant": "mod", "blocks": qK, "planted_blocks": int(qg.info["k"]),
                                "ari_vs_planted": float(adjusted_rand_score(qg.labels, qlab)),
                                "nmi_vs_planted": float(normalized_mutual_info_score(qg.labels, qlab))}
        qgr.close()
    return out


def measure_sbm(args, rg, dev, barrier):
    """NEXT-3: Alg. 2 sampling the C4 DC-SBM (N = 5e6, K = 500, ~1e8 expected edges) with
    raftgp_sbm_sample (parameters resident on the device; the call is synchronous: count pass, scan, write
    pass). Reports edges/s, per-kernel times and the oracle's rate on C2's parameters (same algorithm, one core)."""
    import time
    import torch
    import synth
    c, th, om = synth.sbm_params("C4", args.seed, rule=args.rule)
    ct, tt, ot = (torch.from_numpy(x).to(dev) for x in (c, th, om))
    ctx = rg.Context(dev.index)
    src, dst = rg.raftgp_sbm_sample(ctx, ct, tt, ot, 0)              # warm-up, sizes the output
    cap = int(src.numel() * 1.05) + 1024
    ctx.prof_reset()
    ctx.set_profiling(True)
    barrier()
    reps = 5
    edges, per = 0, []
    for i in range(reps):   # each call timed on its own (host-side hiccups then show up as one outlier)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        s_, d_ = rg.raftgp_sbm_sample(ctx, ct, tt, ot, 1 + i, cap=cap)
        e1.record(ctx.stream)
        e1.synchronize()
        per.append(e0.elapsed_time(e1))
        edges += s_.numel()
    barrier()
    ms = sorted(per)[len(per) // 2]   # median call
    prof = {k: round(t / reps, 3) for k, (t, c_) in sorted(ctx.prof_read().items(), key=lambda x: -x[1][0])}
    ctx.set_profiling(False)
    out = {"workload": f"C4 DC-SBM parameters (N={c.size:,}, K={om.shape[0]}), q = 20", "ms": ms,
           "ms_per_call": [round(x, 3) for x in per], "timing": "median of the calls",
           "edges_per_call": edges / reps, "value": edges / reps / (ms * 1e-3), "unit": "edges/s",
           "kernel_ms": prof}
    if not args.no_cpu_baseline:
        import oracle
        oracle.build()
        c2, th2, om2 = synth.sbm_params("C2", args.seed)
        t0 = time.perf_counter()
        s2, _ = oracle.sbm_sample(c2, th2, om2, 1)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": s2.size / dt, "unit": "edges/s", "cores": 1, "kind": "oracle",
                               "sample": f"oracle.sbm_sample on C2's parameters (N={c2.size:,}, {s2.size:,} edges), "
                                         f"{dt:.2f} s, single thread"}
    return out


def measure_stream(args, rg, dev, barrier, gr, src_d, dst_d, dims):
    """NEXT-4: streaming updates on the C4 graph, NCut embedding with the bench dims: the
    time of raftgp_stream_add_edges for batches of B new random edges (one untimed batch, then the median of three,
    each with fresh edges) against a full rebuild + embed of a graph with one batch added (raftgp_build_csr +
    raftgp_embed_multi(ncut), median of two after an untimed one), in both stream modes: "exact" (Z bit-identical to the rebuild) and
    "delta" (the last hop from stored sums plus the changed rows only; equal up to fp32 rounding order)."""
    import numpy as np
    import torch
    rng = np.random.default_rng(args.seed + 17)
    out = {"workload": f"C4 graph (N={gr.n:,}), NCut, dims {list(dims)}", "batches": []}
    ctx = rg.Context(dev.index)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    def edges(B):
        return (torch.from_numpy(rng.integers(0, gr.n, B).astype(np.int32)).to(dev),
                torch.from_numpy(rng.integers(0, gr.n, B).astype(np.int32)).to(dev))

    full = {}
    for B in (10, 1000):
        es, ed = edges(B)
        s_all, d_all = torch.cat([src_d, es]), torch.cat([dst_d, ed])
        Z = {"ncut": torch.empty((gr.n, dims[-1]), dtype=torch.float32, device=dev)}
        ts = []
        for _ in range(3):   # the first (workspace growth, cold caches) untimed
            barrier()
            e0.record(ctx.stream)
            g2 = rg.raftgp_build_csr(ctx, gr.n, s_all, d_all)
            rg.raftgp_embed_multi(g2, ["ncut"], dims, args.seed, Z=Z)
            e1.record(ctx.stream)
            barrier()
            ts.append(e0.elapsed_time(e1))
            g2.close()
        full[B] = float(np.median(ts[1:]))
    # the same batches for both modes, so the delta stream's final Z can be compared with the exact one's
    batches = {B: [edges(B) for _ in range(4)] for B in (10, 1000)}
    z_exact = None
    for mode in ("exact", "delta"):
        g = rg.raftgp_build_csr(ctx, gr.n, src_d, dst_d)
        stream = rg.Stream(g, dims, args.seed)
        if mode == "delta":
            stream.set_mode("delta")
        for B in (10, 1000):
            ts, st = [], None
            for rep in range(4):
                es, ed = batches[B][rep]
                barrier()
                e0.record(ctx.stream)
                st = stream.add_edges(es, ed)
                e1.record(ctx.stream)
                barrier()
                if rep:
                    ts.append(e0.elapsed_time(e1))
            t_stream = float(np.median(ts))
            out["batches"].append({"mode": mode, "new_edges": B, "stream_ms": t_stream,
                                   "ms_per_batch": [round(t, 3) for t in ts], "full_rebuild_ms": full[B],
                                   "speedup": full[B] / t_stream, "changed_nodes": st["changed"],
                                   "recomputed_rows": st["affected"]})
        Z = stream.embedding()
        if mode == "exact":
            z_exact = Z.clone()
        else:   # after the same 8 batches: the delta stream against the exact (bit-identical to a rebuild) one
            dz = (Z - z_exact).abs()
            out["delta_vs_exact"] = {"batches": 8, "max_abs": float(dz.max().item()),
                                     "rel_frobenius": float(((Z - z_exact).norm() / z_exact.norm()).item())}
        stream.close()
    return out


TABLE1_DIMS = (4096, 2048, 1024, 512, 256)   # PAPER.md:268-273, Table I row 2E5 (and 1E4-1E5)


# SASS thread-instructions executed per generated normal by sketch_w_tc_kernel<128, 128> (Philox4x32-10, Box-Muller
# with the spec's polynomials, hi/lo split, shared-memory stores, MMA issue and drain), from ncu's
# smsp__inst_executed.sum x 32 / (n r) at C4 (profiles/r02/ncu_C4_v5.md: 1.254e9 warp-instructions, 512-thread CTAs, two quads per thread)
SKETCH_THREAD_INST_PER_NORMAL = 62.7


def measure_sketch(args, rg, ctx, n, r, l1, barrier, sm_mhz):
    """a3 as an ALU-bound kernel (normals/s and the ALU fraction): Theta' = Theta W^(1) for the
    bench's n rows on every SM (raftgp_sketch_transform), event-timed alone. peak = the issue-slot roofline: 148 SMs x
    4 warp-instructions / clock x 32 lanes / (thread-instructions per normal), at the SM clock sampled under load."""
    import torch
    W = rg.raftgp_weights(ctx, args.seed, 1, r, l1)
    out = torch.empty((n, l1), dtype=torch.float32, device=ctx.device)
    lib = rg.load_library()
    for _ in range(2):
        rg._ck(lib.raftgp_sketch_transform(ctx.h, args.seed, n, r, rg._ptr(W), l1, rg._ptr(out)))
    barrier()
    reps = 5
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(reps):
        rg._ck(lib.raftgp_sketch_transform(ctx.h, args.seed, n, r, rg._ptr(W), l1, rg._ptr(out)))
    e1.record(ctx.stream)
    barrier()
    ms = e0.elapsed_time(e1) / reps
    normals = n * r
    ach = normals / (ms * 1e-3)
    sms = torch.cuda.get_device_properties(ctx.device).multi_processor_count
    clk = (sm_mhz or 1965.0) * 1e6
    peak = sms * 4 * 32 * clk / SKETCH_THREAD_INST_PER_NORMAL
    del out
    return {"kernel": "sketch_w_tc_kernel (Theta generated on chip, tcgen05 3xTF32 Theta W1)", "ms": ms,
            "normals": normals, "bound": "alu", "achieved": ach, "unit": "normals/s", "peak": peak, "frac": ach / peak,
            "peak_rule": (f"{sms} SMs x 4 warp-instructions/clock x 32 lanes x {clk / 1e6:.0f} MHz / "
                          f"{SKETCH_THREAD_INST_PER_NORMAL} thread-instructions per normal (ncu, this kernel)"),
            "in_step": "runs on all SMs after the CSR build and the slot build (rows stored at slots chosen by degree; DESIGN.md §6)"}


def measure_table1(args, rg, dev, barrier, peak, peak_src):
    """NEXT-2: the embedding at the paper's Table I widths on the C3 DC-SBM graph (N = 2E5, the largest Table I
    size): one step = CSR build + raftgp_embed_multi(ncut, mod, dims 4096-2048-1024-512-256), inputs resident.
    Reports nnz*w/s over the gathered widths actually used (Theta W1 is formed before aggregation, so the
    feature hop gathers dims[1]), the wide-hop HBM roofline (gather-model bytes) and the tensor-core GEMM rate
    (fp32-accurate flops; each is 3 TF32 MMA flops) against the TF32 dense peak."""
    import torch
    import synth
    cfg = synth.CONFIGS["C3"]
    gr = synth.generate(cfg, args.seed, rule=args.rule)
    dims = TABLE1_DIMS
    variants = ["ncut", "mod"]
    src, dst = torch.from_numpy(gr.src).to(dev), torch.from_numpy(gr.dst).to(dev)
    ctx = rg.Context(dev.index)
    Z = {v: torch.empty((gr.n, dims[-1]), dtype=torch.float32, device=dev) for v in variants}

    def step():
        g = rg.raftgp_build_csr(ctx, gr.n, src, dst)
        rg.raftgp_embed_multi(g, variants, dims, args.seed, Z=Z)
        nnz = g.info()["nnz_local"]
        g.close()
        return nnz

    for _ in range(2):
        nnz = step()
    ctx.prof_reset()
    ctx.set_profiling(True)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(args.table1_steps):
        step()
    e1.record(ctx.stream)
    barrier()
    ms = e0.elapsed_time(e1) / args.table1_steps
    prof = {k: (t / args.table1_steps, c / args.table1_steps) for k, (t, c) in ctx.prof_read().items()}
    ctx.set_profiling(False)
    n, L = gr.n, len(dims) - 1
    units = nnz * dims[1] + len(variants) * sum((nnz + n) * dims[k] for k in range(1, L + 1))
    # wide-hop gather-model bytes per step: the dual feature hop + every GCN hop wider than 128
    hop_b = 8 * (n + 1) + 4 * nnz + 4 * dims[1] * nnz + 2 * 4 * dims[1] * n + 4 * n
    for k in range(1, L + 1):
        w = dims[k]
        if w > 128:
            out_b = 4 * w * n if k == L else 2 * 4 * w * n + 4 * n * max(1, w // 512)
            hop_b += len(variants) * (8 * (n + 1) + 4 * nnz + 4 * w * (nnz + n) + out_b + 4 * n)
    flops = 2.0 * n * dims[0] * dims[1] + len(variants) * sum(2.0 * n * dims[k] * dims[k + 1] for k in range(1, L))
    hop_ms = prof.get("wide_hop", (0.0, 0))[0]
    gemm_ms = prof.get("gemm_tf32x3", (0.0, 0))[0]
    try:
        bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        tf32_peak, tf32_src = 0.5 * bf16, "MEASURED_PEAKS.json bf16_tflops x 0.5 (nominal TF32:BF16 ratio)"
    except Exception:
        tf32_peak, tf32_src = 1125.0, "nominal 2.25 PFLOP/s bf16 x 0.5"
    hop_gbs = hop_b / (hop_ms * 1e-3) / 1e9 if hop_ms else None
    mma_tflops = 3 * flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
    return {
        "workload": f"T1-2E5: C3 DC-SBM graph (N={n:,}, nnz={nnz:,}) with Table I widths {list(dims)} "
                    f"(PAPER.md:268-273), variants ncut+mod",
        "steps": args.table1_steps, "ms_per_step": ms, "value": units / (ms * 1e-3), "unit": UNIT,
        "kernel_ms": {k: round(t, 3) for k, (t, _) in sorted(prof.items(), key=lambda x: -x[1][0])},
        "wide_hop_roofline": {"bound": "hbm", "achieved": hop_gbs, "peak": peak, "unit": "GB/s",
                              "frac": hop_gbs / peak if hop_gbs else None, "peak_source": peak_src,
                              "bytes_per_step": hop_b},
        "gemm_roofline": {"bound": "tensor", "fp32_tflops": flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None,
                          "achieved": mma_tflops, "peak": tf32_peak, "unit": "TFLOP/s (TF32 MMA, 3 per fp32 flop)",
                          "frac": mma_tflops / tf32_peak if mma_tflops else None, "peak_source": tf32_src,
                          "fp32_flops_per_step": flops},
        # context only (other hardware, the authors' own graphs, one variant per run, CSR build not included):
        # Table III's per-stage wall times at 2E5
        "paper_context": {"source": "PAPER.md:353-354 (Table III, N = 2E5)", "hardware": "2x Xeon 6130 + RTX 3090",
                          "raftgp_c_feat_s": 62.105, "raftgp_c_emb_s": 1.3236,
                          "raftgp_m_feat_s": 57.6826, "raftgp_m_emb_s": 1.5124,
                          "this_step_s_both_variants_incl_csr": ms * 1e-3},
    }


def dry_run(args):
    """Launch check: every rank joins the process group (gloo), the ranks agree on a value by max-over-ranks, rank 0
    prints one line. No kernels run, nothing is measured."""
    import torch
    import torch.distributed as tdist
    world, rank, _ = dist_env()
    if world > 1:
        tdist.init_process_group("gloo")
    t = torch.tensor([float(rank)])
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "max_rank": int(t.item()),
                          "steps": args.steps, "warmup": args.warmup, "gpus_flag": args.gpus}), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_spawn(args))
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import synth
    from paper_2312_01560_b200 import build as _build
    from paper_2312_01560_b200 import dist as rdist
    from paper_2312_01560_b200 import raftgp as rg

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as tdist
        # RAFTGP_BENCH_BACKEND=gloo + RAFTGP_BENCH_ONE_GPU=1: functional check of the N > 1 code path with all
        # ranks on one GPU (host barriers; not a measurement)
        backend = os.environ.get("RAFTGP_BENCH_BACKEND", "nccl")
        if os.environ.get("RAFTGP_BENCH_ONE_GPU") == "1":
            local = 0
            if args.exchange == "lib":   # one NCCL communicator cannot hold two ranks of one GPU
                args.exchange = "push"
        torch.cuda.set_device(local)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        _build.build()
    if world > 1:
        tdist.barrier()
    dev = torch.device("cuda", torch.cuda.current_device())
    if world > 1:
        # a non-default compute stream: NCCL's all-gathers (own streams) then overlap the hop kernels
        torch.cuda.set_stream(torch.cuda.Stream(dev))
    cfg = synth.CONFIGS[args.config]
    variants = args.variants.split(",")
    dims = tuple(cfg.dims)
    gr = synth.generate(cfg, args.seed, rule=args.rule)
    m = gr.src.size
    src_h = torch.from_numpy(gr.src).pin_memory()
    dst_h = torch.from_numpy(gr.dst).pin_memory()
    src_d, dst_d = src_h.to(dev), dst_h.to(dev)
    ctx = rg.Context(dev.index)
    lib_dist = world > 1 and args.exchange == "lib"
    dctx = None
    if lib_dist:
        # the library's own NCCL communicator (raftgp_ctx_create_dist); torch.distributed only carries the id
        uid = [rg.raftgp_nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        dctx = rg.Context(dev.index, dist=(rank, world, uid[0]))
    run_ctx = dctx if lib_dist else ctx       # the context whose stream / profile / launch count the step uses
    stream = run_ctx.stream
    ranges, _ = rdist.row_partition(gr.n, world)
    rb, re = ranges[rank]
    rows = re - rb
    assert (rb, re) == rg.local_rows(gr.n, rank, world)
    Zbuf = {v: torch.empty((max(1, rows), dims[-1]), dtype=torch.float32, device=dev)[:rows] for v in variants}

    fused_pair = (not args.no_fuse_variants) and "ncut" in variants and "mod" in variants

    def step_single(src, dst, out_host=None):
        if args.no_fuse_variants:
            g = rg.raftgp_build_csr(ctx, gr.n, src, dst)
            for v in variants:
                rg.raftgp_embed(g, v, dims, args.seed, Z=Zbuf[v], want_Y=False)
        else:   # build + embed in one call: Theta' generated on a side stream during the CSR build
            _, g = rg.raftgp_build_embed(ctx, gr.n, src, dst, variants, dims, args.seed, Z=Zbuf, keep_graph=True)
        if out_host is not None:
            for v in variants:
                out_host[v].copy_(Zbuf[v], non_blocking=True)
        nnz = g.info()["nnz_local"]
        g.close()
        return nnz

    push_bufs = rdist.PushBuffers(ctx) if (world > 1 and args.exchange == "push") else None

    def step_multi(src, dst, out_host=None):
        keep = {}
        pipe = rdist.rank_pipeline_push if push_bufs is not None else rdist.rank_pipeline
        gen = pipe(rdist.CudaEngine(ctx), gr.n, src, dst, rank, world, variants, dims, args.seed, keep)
        Z = rdist.run_distributed(gen, push=push_bufs)
        for v in variants:
            Zbuf[v].copy_(Z[v])
            if out_host is not None:
                out_host[v].copy_(Z[v], non_blocking=True)
        nnz = keep["graph"].info()["nnz_local"]
        keep["graph"].close()
        return nnz

    def step_lib(src, dst, out_host=None):
        # the row-partitioned step inside the library: one C-ABI call per rank (exchanges fused, NCCL barriers)
        rg.raftgp_build_embed(dctx, gr.n, src, dst, variants, dims, args.seed, Z=Zbuf)
        if out_host is not None:
            for v in variants:
                out_host[v].copy_(Zbuf[v], non_blocking=True)
        return None

    step = step_single if world == 1 else (step_lib if lib_dist else step_multi)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t)
        return float(t.item())

    # ---------------- warm-up
    nnz_local = 0
    for _ in range(max(3, args.warmup)):
        nnz_local = step(src_d, dst_d)
    if lib_dist:   # this rank's entries (the library call returns no graph): one local CSR build, untimed
        gl = rg.raftgp_build_csr(ctx, gr.n, src_d, dst_d, rb, re)
        nnz_local = gl.info()["nnz_local"]
        gl.close()
        ctx.trim()
    nnz = int(sum_over_ranks(nnz_local))
    # ---------------- timed region (device-resident inputs)
    run_ctx.prof_reset()
    run_ctx.set_profiling(True)
    run_ctx.launch_count(reset=True)
    barrier()
    with ClockSampler(dev.index, args.clock_period_ms, not args.no_clocks, args.clock_query) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step(src_d, dst_d)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1) / args.steps
    launches = run_ctx.launch_count()
    prof = run_ctx.prof_read()
    run_ctx.set_profiling(False)
    ms_max = max_over_ranks(ms)
    units = work_units(nnz, gr.n, cfg.r, dims, len(variants))
    value = units / (ms_max * 1e-3)

    # ---------------- roofline of the dominant kernel (of this rank's launches)
    peak, peak_src = measured_peak()
    kernel_times = {k: v[0] / args.steps for k, v in prof.items()}        # ms per step
    dom = max((k for k in prof if k in ("feature_hop", "gcn_hop")), key=lambda k: prof[k][0], default=None)
    roof = None
    hop_stats = {}
    for k in ("feature_hop", "gcn_hop"):
        if k not in prof:
            continue
        b_step, l_step = algorithmic_bytes(nnz if world == 1 else nnz_local, rows if world > 1 else gr.n, cfg.r, dims,
                                           len(variants), k, fused_pair and (world == 1 or lib_dist))
        t_step = prof[k][0] / args.steps * 1e-3
        ach = b_step / t_step / 1e9
        hop_stats[k] = {"gb_s": ach, "ms_per_step": t_step * 1e3, "launches_per_step": prof[k][1] / args.steps,
                        "bytes_per_launch": b_step / l_step}
    traffic, ncu_counters = None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tfile):
        try:
            tj = json.load(open(tfile)).get(args.config, {})
            traffic, ncu_counters = tj.get(dom), tj.get(dom + "_ncu")
            if ncu_counters is not None:
                ncu_counters = dict(ncu_counters, source=tj.get("_source"))
        except Exception:
            traffic = None
    if dom:
        ach = hop_stats[dom]["gb_s"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": peak_src, "frac_of_8TBs_nominal": ach / 8000.0, "traffic": traffic,
                "bytes_per_launch": hop_stats[dom]["bytes_per_launch"],
                "ncu": ncu_counters}   # L2 hit rate, sectors per request, DRAM % of nominal (one ncu --set full)
        if traffic:
            # the DRAM view: ncu's measured bytes per launch over this run's event-timed launch duration (the
            # gather-model bytes above count L2 hits as traffic, so frac can exceed the DRAM-side fraction)
            t_launch = hop_stats[dom]["ms_per_step"] * 1e-3 / hop_stats[dom]["launches_per_step"]
            roof["dram_gb_s"] = traffic / t_launch / 1e9
            roof["dram_frac"] = roof["dram_gb_s"] / peak

    # ---------------- N > 1: the exchange and the partition
    dist_info = None
    if world > 1:
        per_rank = [None] * world
        tdist.all_gather_object(per_rank, {"nnz_local": int(nnz_local), "rows": rows,
                                           "kernel_ms": {k: v for k, v in kernel_times.items()}})
        nl = [x["nnz_local"] for x in per_rank]
        kmax = {}
        for x in per_rank:
            for k, v in x["kernel_ms"].items():
                kmax[k] = max(kmax.get(k, 0.0), v)
        V = len(variants)
        # every operand row is stored into the P - 1 peers' copies by the kernel that produces it: Theta' (l1 wide,
        # lib path), T_1 .. T_L of every variant (dims[1..L] wide)
        per_row = (dims[1] if lib_dist else 0) + V * sum(dims[1:])
        egress = (world - 1) * rows * 4 * per_row
        producing = sum(kmax.get(k, 0.0) for k in ("sketch", "feature_hop", "gcn_hop", "push_copy"))
        dist_info = {
            "communicator": (f"library NCCL communicator of {world} ranks (raftgp_ctx_create_dist)" if lib_dist
                             else f"torch.distributed ({tdist.get_backend()}) of {world} ranks"),
            "exchange": ("fused into the producing kernels (peer stores over NVLink, CUDA IPC mappings) + stream-"
                         "ordered NCCL barriers" if args.exchange in ("lib", "push") else "NCCL all-gathers"),
            "partition": "1-D rows [p R, (p+1) R), R = ceil(n / P)",
            "nnz_local": nl, "nnz_imbalance_max_over_mean": max(nl) / (sum(nl) / len(nl)),
            "kernel_ms_per_step_max_over_ranks": {k: round(v, 4) for k, v in sorted(kmax.items(), key=lambda x: -x[1])},
            "exchange_wait_ms_per_step": kmax.get("exchange", 0.0),
            "egress_bytes_per_rank_per_step": egress,
            "egress_gb_s_during_producing_kernels": (egress / (producing * 1e-3) / 1e9) if producing else None,
            "note": ("the exchange is overlapped by construction: its stores run inside the producing kernels, so their "
                     "time is part of sketch / feature_hop / gcn_hop; exchange_wait is the time spent in NCCL barriers "
                     "and all-gathers, including waiting for the slowest rank"),
        }

    # ---------------- a3: the sketch as an ALU-bound kernel (N = 1)
    sketch_roof = None
    if world == 1 and sketch_ok(cfg):
        ctx.trim()   # the step's cached workspace back to the device (C5 holds ~128 GB of it)
        sketch_roof = measure_sketch(args, rg, ctx, min(gr.n, 5_000_000), cfg.r, dims[1], barrier,
                                     clocks.summary().get("sm_mhz"))

    # ---------------- NEXT-1: Alg. 1 model selection on this step's embeddings (whole graph, N = 1)
    select = None
    if world == 1 and not args.no_select:
        select = measure_select(args, rg, ctx, gr, src_d, dst_d, variants, dims, Zbuf, barrier, peak, peak_src)

    # ---------------- NEXT-2: Table I widths (N = 1 only)
    table1 = None
    if world == 1 and not args.no_table1:
        table1 = measure_table1(args, rg, dev, barrier, peak, peak_src)

    # ---------------- NEXT-3: Alg. 2 SBM sampler (N = 1 only)
    sbm = None
    if world == 1 and not args.no_sbm:
        sbm = measure_sbm(args, rg, dev, barrier)

    # ---------------- NEXT-4: streaming updates (N = 1 only)
    stream = None
    if world == 1 and not args.no_stream:
        stream = measure_stream(args, rg, dev, barrier, gr, src_d, dst_d, dims)

    # ---------------- e2e through the C-ABI with host buffers (H2D of edges, D2H of Z inside the timed region)
    # N = 1: three contexts on three streams, steps rotate over them, so a step's copies overlap other
    # steps' kernels (multi-buffering with the public API); every step still copies its own edges in and
    # its own Z out. N > 1: one stream, sequential.
    e2e = None
    e2e_skip = None
    e2e_steps = max(args.steps, args.e2e_steps)
    e2e_seq = world > 1
    e2e_note = None
    if not args.no_e2e:
        # each pipelined lane holds its own context (workspace) and two Z buffer sets; at C5 sizes that does
        # not fit next to the main context, so the lane count drops, and when even one lane would not fit the
        # leg runs sequential steps on the main context (the reason goes into e2e.mode)
        ctx.trim()
        torch.cuda.empty_cache()
        free_b, _ = torch.cuda.mem_get_info(dev)
        ws_b = 4 * rows * (dims[1] * (1 + len(variants)) + sum(dims[2:]) * len(variants)) + 56 * m   # Theta', T_k, CSR build
        lane_b = 2 * int(sum(rows * dims[-1] * 4 for _ in variants)) + 2 * 8 * m + ws_b   # Z x2, edges x2, workspace
        lanes_fit = int(free_b // max(1, lane_b))
        if lanes_fit < args.e2e_lanes:
            args.e2e_lanes = max(1, min(args.e2e_lanes, lanes_fit))
        if lanes_fit < 1:   # no room for a pipeline lane (C5): sequential steps on the main context instead
            e2e_seq = True
            e2e_steps = args.steps
            e2e_note = f"a pipeline lane needs ~{lane_b / 2**30:.0f} GiB, {free_b / 2**30:.0f} GiB free"
    if not args.no_e2e and e2e_skip is None:
        d2h = int(sum(rows * dims[-1] * 4 for _ in variants))
        if not e2e_seq and world == 1 and not args.no_fuse_variants and args.e2e_lanes == 1:
            # one compute stream (steps back to back, no kernel interleaving across steps) with the copies on
            # their own streams: H2D of step k+1 and D2H of step k-1 run under step k's kernels; inputs and
            # outputs double-buffered, ordered by events
            cs = torch.cuda.Stream(dev)
            hs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            c1 = rg.Context(dev.index, stream=cs)
            Din = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int32, device=dev))
                   for _ in range(2)]
            Zb = [{v: torch.empty((rows, dims[-1]), dtype=torch.float32, device=dev) for v in variants}
                  for _ in range(2)]
            Hb = [{v: torch.empty((rows, dims[-1]), dtype=torch.float32).pin_memory() for v in variants}
                  for _ in range(2)]
            in_ready = [torch.cuda.Event() for _ in range(2)]
            in_free = [torch.cuda.Event() for _ in range(2)]
            out_free = [torch.cuda.Event() for _ in range(2)]
            for b in range(2):
                in_free[b].record(cs)
                out_free[b].record(cs)

            def h2d(k):
                b = k % 2
                hs.wait_event(in_free[b])
                with torch.cuda.stream(hs):
                    Din[b][0].copy_(src_h, non_blocking=True)
                    Din[b][1].copy_(dst_h, non_blocking=True)
                    in_ready[b].record(hs)

            def run(nsteps):
                h2d(0)
                for k in range(nsteps):
                    b = k % 2
                    if k + 1 < nsteps:
                        h2d(k + 1)
                    cs.wait_event(in_ready[b])
                    cs.wait_event(out_free[b])
                    with torch.cuda.stream(cs):
                        rg.raftgp_build_embed(c1, gr.n, Din[b][0], Din[b][1], variants, dims, args.seed, Z=Zb[b])
                        in_free[b].record(cs)
                    ds.wait_stream(cs)
                    with torch.cuda.stream(ds):
                        for v in variants:
                            Hb[b][v].copy_(Zb[b][v], non_blocking=True)
                        out_free[b].record(ds)

            run(2)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            hs.wait_event(e0)
            ds.wait_event(e0)
            run(e2e_steps)
            cs.wait_stream(hs)
            cs.wait_stream(ds)
            e1.record(cs)
            torch.cuda.synchronize()
            mode = ("one compute stream (raftgp_build_embed per step) + H2D and D2H streams: step k+1's inputs and "
                    "step k-1's outputs cross PCIe under step k's kernels")
        elif not e2e_seq and world == 1 and not args.no_fuse_variants:
            lanes = []
            for _ in range(args.e2e_lanes):
                s_ = torch.cuda.Stream(dev)
                cs_ = torch.cuda.Stream(dev)          # D2H of this lane's Z, off the compute stream
                c_ = rg.Context(dev.index, stream=s_)
                # two Z buffers per lane: a step waits only for the D2H of its buffer's previous use (two
                # rounds back), recorded as an event, not for the lane's latest copy
                Zl = [{v: torch.empty((rows, dims[-1]), dtype=torch.float32, device=dev) for v in variants}
                      for _ in range(2)]
                Hl = [{v: torch.empty((rows, dims[-1]), dtype=torch.float32).pin_memory() for v in variants}
                      for _ in range(2)]
                ev = [torch.cuda.Event() for _ in range(2)]
                lanes.append((s_, c_, Zl, Hl, cs_, ev))

            def e2e_step(i):
                s_, c_, Zl, Hl, cs_, ev = lanes[i % len(lanes)]
                b = (i // len(lanes)) % 2
                with torch.cuda.stream(s_):
                    # the C-ABI gets the HOST (pinned) edge arrays (RAFTGP_HOST_PTRS): the library copies them in on
                    # its stream inside the call
                    if args.e2e_api == "build_embed":
                        s_.wait_event(ev[b])           # Zl[b] is free once its previous D2H is done
                        rg.raftgp_build_embed(c_, gr.n, src_h, dst_h, variants, dims, args.seed, Z=Zl[b])
                    else:
                        g = rg.raftgp_build_csr(c_, gr.n, src_h, dst_h)
                        s_.wait_event(ev[b])
                        rg.raftgp_embed_multi(g, variants, dims, args.seed, Z=Zl[b])
                        g.close()
                cs_.wait_stream(s_)
                with torch.cuda.stream(cs_):
                    for v in variants:
                        Hl[b][v].copy_(Zl[b][v], non_blocking=True)
                    ev[b].record(cs_)

            for i in range(len(lanes)):
                e2e_step(i)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lanes[0][0])
            for s_, *_ in lanes[1:]:
                s_.wait_event(e0)
            for i in range(e2e_steps):
                e2e_step(i)
            for s_, _, _, _, cs_, _ in lanes:
                lanes[0][0].wait_stream(s_)
                lanes[0][0].wait_stream(cs_)
            e1.record(lanes[0][0])
            torch.cuda.synchronize()
            mode = (f"pipelined: {args.e2e_lanes} contexts/streams (+ a D2H stream each), {args.e2e_api} per step with "
                    "the host edge arrays (RAFTGP_HOST_PTRS: H2D inside the C-ABI call), Z copied to pinned host "
                    "memory; step k's copies overlap other steps' kernels")
        else:
            out_host = {v: torch.empty((rows, dims[-1]), dtype=torch.float32).pin_memory() for v in variants}
            step(src_h, dst_h, out_host)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(e2e_steps):
                step(src_h, dst_h, out_host)
            e1.record(stream)
            mode = "sequential on one stream" + (f" ({e2e_note})" if e2e_note else "")
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
        e2e = {"value": units / (ems * 1e-3), "unit": UNIT, "ms_per_step": ems, "h2d_bytes_per_step": 8 * m,
               "d2h_bytes_per_step": d2h, "mode": mode, "steps": e2e_steps}

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        # the whole workload (all host cores), then the single-thread sample for comparison
        full_n = None if cfg.n <= 5_000_000 else SAMPLE_N * 10
        v, sg, snnz, times, cores = cpu_baseline(cfg, variants, args.seed, args.rule, n=full_n, threads=0)
        v1, sg1, snnz1, times1, _ = cpu_baseline(cfg, variants, args.seed, args.rule, n=SAMPLE_N, threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": (f"full oracle step (CSR build + {'/'.join(variants)} projection + GCN {list(dims)}) on the "
                          f"{cfg.name} DC-SBM recipe at N={sg.n:,} (nnz={snnz:,})"
                          f"{' = the whole bench workload' if full_n is None else ''}; {times[0]:.1f} s on {cores} "
                          f"threads (OpenMP over output rows), fp64"),
               "single_thread": {"value": v1, "unit": UNIT, "cores": 1,
                                 "sample": f"same step at N={sg1.n:,} (nnz={snnz1:,}); {times1[0]:.2f} s"},
               "host": host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: DC-SBM N={gr.n:,} K={gr.info['k']} nnz={nnz:,} r={cfg.r} "
                                   f"dims={list(dims)} variants={'+'.join(variants)}",
                       "n": gr.n, "nnz": nnz, "m_raw_pairs": m, "r": cfg.r, "dims": list(dims), "variants": variants,
                       "rule": args.rule, "fused_variant_pair": fused_pair and world == 1,
                       "parallelism": f"rowpart{world}" if world > 1 else "single",
                       "exchange": (args.exchange if world > 1 else None),
                       "launch": ("torch.distributed.run, one rank per GPU (bench.py self-spawns it for --gpus N > 1)"
                                  if world > 1 else "single process"),
                       "l2": "inputs larger than L2 (gathered operands >= 1.28 GB vs 126 MB L2); no flush"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e if e2e_skip is None else {"skipped": e2e_skip},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "kernels_ms_per_step": {k: round(v, 4) for k, v in sorted(kernel_times.items(), key=lambda x: -x[1])},
            "hops": hop_stats,
            "sketch_roofline": sketch_roof,
            "dist": dist_info,
            "model_selection": select,
            "table1_widths": table1,
            "sbm_sampler": sbm,
            "streaming": stream,
        }
        print(json.dumps(line), flush=True)
    if push_bufs is not None:
        push_bufs.close()
    if dctx is not None:
        torch.cuda.synchronize()
        dctx.close()   # collective (the cached operand copies are unmapped behind a barrier)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
