"""Row-partitioned multi-GPU orchestration of the embedding path.

One process per GPU. Rank p owns the contiguous rows [p*R, min((p+1)*R, n)) with R = ceil(n / P), so
the all-gathered (P*R)-row block indexes global rows directly. Exchange steps — the only collectives:
  1. after the CSR build: all-gather of the local degree vectors (n int32) -> every rank computes the
     global 2e, s and s^ (raftgp_graph_set_degrees);
  2. before every GCN hop: all-gather of the next operand T_k = s^ (.) (Z^(k-1) W^(k)) (n x L_k fp32).
Hop 0 needs no exchange: Theta is counter-based, so every rank regenerates the rows it gathers, and
the MOD rank-1 vector g = d^T Theta' is reduced over global fixed chunks identically on every rank.
Each row's arithmetic is a function of that row only, so the result is bit-identical for any P.
The per-hop all-gathers of two variants are software-pipelined against each other's compute.

The per-rank pipeline is a generator that yields ("gather", tensor) at each exchange point and
receives the gathered block; drivers run it over torch.distributed (NCCL on B200, gloo on CPU tests)
or, for single-GPU testing, over P shards in lockstep ("loopback"). The compute steps go through an
`engine`: `CudaEngine` calls libraftgp (the product path); tests may plug a CPU engine.

Push mode (`rank_pipeline_push`, the default on GPUs): the per-hop all-gather is fused into the producing
kernels. Every rank holds a full n-row copy of each operand T_k; the feature transform and each GCN hop
store their finished rows straight into ALL ranks' copies (peer memory over NVLink, mapped with CUDA IPC:
raftgp_feature_transform_push / raftgp_gcn_hop_push), so the exchange overlaps the hop's gathers row by
row, and one stream-ordered barrier (a 1-element all-reduce) separates producing and consuming hops.
"""
from __future__ import annotations

import os
from typing import Generator, List, Optional, Sequence

import torch

from . import raftgp as rg


def row_partition(n: int, world: int):
    """[(row_begin, row_end)] per rank and the padded block height R."""
    R = max(1, -(-n // world))
    return [(min(n, p * R), min(n, (p + 1) * R)) for p in range(world)], R


def _pad(t: torch.Tensor, R: int) -> torch.Tensor:
    if t.shape[0] == R:
        return t.contiguous()
    out = torch.zeros((R,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    out[: t.shape[0]] = t
    return out


class CudaEngine:
    """Local compute steps on one GPU through the C-ABI."""

    def __init__(self, ctx: rg.Context):
        self.ctx = ctx

    def build(self, n, src, dst, rb, re):
        return rg.raftgp_build_csr(self.ctx, n, src, dst, rb, re)

    def local_degrees(self, h):
        return h.local_degrees()

    def set_degrees(self, h, deg_all):
        h.set_degrees(deg_all)

    def feature_transform(self, h, variants, dims, seed):
        return rg.raftgp_feature_transform(h, variants, dims[0], dims[1], seed)

    def weights(self, seed, k, a, b):
        return rg.raftgp_weights(self.ctx, seed, k, a, b)

    def hop(self, h, T_full, W_next, want_Z: bool):
        rows = h.rows
        Z = torch.empty((rows, T_full.shape[1]), dtype=torch.float32, device=self.ctx.device) if want_Z else None
        _, T_next = rg.raftgp_gcn_hop(h, T_full, Z, W_next)
        return Z, T_next

    # push mode: `reps` are device pointers (IPC-mapped peers) or tensors, one per rank copy
    def feature_transform_push(self, h, variants, dims, seed, reps):
        rg.raftgp_feature_transform_push(h, variants, dims[0], dims[1], seed, reps)

    def hop_push(self, h, T_own, w, W_next, reps_next):
        rg.raftgp_gcn_hop_push(h, T_own, w, W_next, reps_next)

    def hop_last(self, h, T_own, w):
        Z = torch.empty((max(1, h.rows), w), dtype=torch.float32, device=self.ctx.device)[: h.rows]
        rg.raftgp_gcn_hop(h, T_own, Z, w=w)
        return Z


def rank_pipeline(engine, n: int, src, dst, rank: int, world: int, variants, dims: Sequence[int], seed: int,
                  keep: Optional[dict] = None) -> Generator:
    """One rank's share of the path. Yields exchange requests to its driver:
        ("gather", block)  -> the all-gathered block (blocking; used for the degree vector)
        ("start", block)   -> a handle; the all-gather runs while this rank keeps computing
        ("wait", handle)   -> the all-gathered block
    With several variants the exchanges are software-pipelined: variant A's hop-k gather is in flight
    while variant B's hop k computes and vice versa, so comm overlaps compute without changing any
    arithmetic. Returns {variant: this rank's rows of Z} (or Z itself for a single variant)."""
    single = isinstance(variants, (str, int))
    vlist = [variants] if single else list(variants)
    ranges, R = row_partition(n, world)
    rb, re = ranges[rank]
    h = engine.build(n, src, dst, rb, re)
    deg_all = yield ("gather", _pad(engine.local_degrees(h), R))
    engine.set_degrees(h, deg_all[:n].contiguous())
    L = len(dims) - 1
    T = engine.feature_transform(h, vlist, dims, seed)          # {v: T1}, local rows
    W = {k: engine.weights(seed, k, dims[k - 1], dims[k]) for k in range(2, L + 1)}
    handles = {}
    for v in vlist:
        handles[v] = yield ("start", _pad(T[v], R))
    out = {}
    for k in range(1, L + 1):
        for v in vlist:
            T_full = yield ("wait", handles[v])
            Zv, Tn = engine.hop(h, T_full[:n], W.get(k + 1), want_Z=(k == L))
            if k < L:
                handles[v] = yield ("start", _pad(Tn, R))
            else:
                out[v] = Zv
    if keep is not None:
        keep["graph"] = h
    return out[vlist[0]] if single else out


def rank_pipeline_push(engine, n: int, src, dst, rank: int, world: int, variants, dims: Sequence[int], seed: int,
                       keep: Optional[dict] = None) -> Generator:
    """One rank's share of the path with the exchange fused into the producing hops (module docstring).
    Yields to its driver:
        ("gather", block)   -> the all-gathered degree block (as in rank_pipeline)
        ("buffers", info)   -> {(variant, k): [copy of rank 0, ..., rank P-1]} full n x dims[k] copies of T_k
                               (a driver may hand out only this rank's copy: a list of length 1)
        ("barrier", [(variant, k), ...]) -> the listed copies are complete on every rank
    Same arithmetic as rank_pipeline, so the result is bit-identical to it and to P = 1."""
    single = isinstance(variants, (str, int))
    vlist = [variants] if single else list(variants)
    ranges, R = row_partition(n, world)
    rb, re = ranges[rank]
    h = engine.build(n, src, dst, rb, re)
    deg_all = yield ("gather", _pad(engine.local_degrees(h), R))
    engine.set_degrees(h, deg_all[:n].contiguous())
    L = len(dims) - 1
    spec = [(v, k, int(dims[k])) for v in vlist for k in range(1, L + 1)]
    reps = yield ("buffers", {"n": n, "spec": spec, "ranges": ranges, "R": R})

    def own(v, k):
        lst = reps[(v, k)]
        return lst[rank] if len(lst) > 1 else lst[0]

    W = {k: engine.weights(seed, k, dims[k - 1], dims[k]) for k in range(2, L + 1)}
    engine.feature_transform_push(h, vlist, dims, seed, {v: reps[(v, 1)] for v in vlist})
    yield ("barrier", [(v, 1) for v in vlist])
    out = {}
    for k in range(1, L + 1):
        produced = []
        for v in vlist:
            if k < L:
                engine.hop_push(h, own(v, k), int(dims[k]), W[k + 1], reps[(v, k + 1)])
                produced.append((v, k + 1))
            else:
                out[v] = engine.hop_last(h, own(v, k), int(dims[k]))
        if produced:
            yield ("barrier", produced)
    if keep is not None:
        keep["graph"] = h
    return out[vlist[0]] if single else out


class _Done:
    """A completed exchange (loopback / blocking drivers)."""

    def __init__(self, value):
        self.value = value

    def result(self):
        return self.value


def run_loopback(gens: List[Generator], device=None, dtype=torch.float32):
    """Advance P rank pipelines in lockstep; a gather concatenates the P blocks in rank order; push-mode
    buffers are P full copies on `device` (one per logical rank)."""
    msgs = [next(g) for g in gens]
    results: List[Optional[torch.Tensor]] = [None] * len(gens)
    while True:
        kind = msgs[0][0]
        if any(m[0] != kind for m in msgs):
            raise RuntimeError("rank pipelines went out of step")
        if kind == "wait":
            replies = [m[1].value for m in msgs]
        elif kind == "buffers":   # one full copy per logical rank, shared by all (push mode)
            info = msgs[0][1]
            bufs = {(v, k): [torch.zeros((info["n"], w), dtype=dtype, device=device) for _ in msgs]
                    for v, k, w in info["spec"]}
            replies = [bufs for _ in msgs]
        elif kind == "barrier":   # one stream, ranks in lockstep: nothing to wait for
            replies = [None for _ in msgs]
        else:
            full = torch.cat([m[1] for m in msgs], 0)
            replies = [full if kind == "gather" else _Done(full) for _ in msgs]
        nxt, done = [], 0
        for p, g in enumerate(gens):
            try:
                nxt.append(g.send(replies[p]))
            except StopIteration as stop:
                results[p] = stop.value
                nxt.append(None)
                done += 1
        if done == len(gens):
            return results
        if done:
            raise RuntimeError("rank pipelines went out of step")
        msgs = nxt


class _Pending:
    def __init__(self, work, out, parts=None):
        self.work, self.out, self.parts = work, out, parts

    def result(self):
        self.work.wait()
        return torch.cat(self.parts, 0) if self.parts is not None else self.out


class PushBuffers:
    """Per-process cache of the push-mode copies: for every (variant, k) a library-allocated n x w buffer on
    this GPU (raftgp_ipc_alloc) plus the peers' buffers mapped through CUDA IPC (raftgp_ipc_open), so steps
    after the first reuse them. Rank q's copy is at list index q."""

    def __init__(self, ctx: rg.Context, group=None):
        self.ctx, self.group, self.key, self.own, self.maps = ctx, group, None, {}, {}
        self.mapped = True   # False: some rank could not map a peer; copies are completed by all-gathers
        self.tensors = {}

    def get(self, info) -> dict:
        import torch.distributed as dist
        key = (info["n"], tuple(info["spec"]))
        if key == self.key:
            return self.maps
        self.close()
        world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        handles = {}
        for v, k, w in info["spec"]:
            buf = rg.IpcBuffer(self.ctx, max(16, info["n"] * w * 4))
            self.own[(v, k)] = buf
            handles[(v, k)] = buf.handle_bytes()
        allh = [None] * world
        dist.all_gather_object(allh, handles, group=self.group)
        opened, ok = {}, os.environ.get("RAFTGP_PUSH_NOIPC") != "1"   # test hook: force the fallback
        try:
            for vk in (handles if ok else []):
                opened[vk] = [self.own[vk].ptr if q == rank else rg.raftgp_ipc_open(self.ctx, allh[q][vk])
                              for q in range(world)]
        except rg.RaftGPError:
            ok = False
        oks = [None] * world
        dist.all_gather_object(oks, ok, group=self.group)
        self.mapped = all(oks)
        if self.mapped:
            self.maps = opened
        else:   # no peer mapping on this box: every rank keeps only its own copy (all-gathered at barriers)
            for vk, ptrs in opened.items():
                for q, p in enumerate(ptrs):
                    if q != rank and p:
                        rg.raftgp_ipc_close(self.ctx, p)
            torch.cuda.synchronize(self.ctx.device)
            dist.barrier(group=self.group)   # every mapping is gone before any rank frees its buffers
            for b in self.own.values():
                b.close()
            self.own = {}
            self.tensors = {(v, k): torch.zeros((max(1, info["n"]), w), dtype=torch.float32, device=self.ctx.device)
                            for v, k, w in info["spec"]}
            self.maps = {vk: [t.data_ptr()] for vk, t in self.tensors.items()}
        self.key = key
        dist.barrier(group=self.group)
        return self.maps

    def close(self):
        """Unmap the peers' copies, wait until every rank has done so, then free this rank's copies."""
        import torch.distributed as dist
        if self.maps and self.mapped:
            rank = dist.get_rank(self.group)
            for ptrs in self.maps.values():
                for q, p in enumerate(ptrs):
                    if q != rank:
                        rg.raftgp_ipc_close(self.ctx, p)
        if self.own and dist.is_initialized():
            torch.cuda.synchronize(self.ctx.device)
            dist.barrier(group=self.group)
        for b in self.own.values():
            b.close()
        self.key, self.own, self.maps, self.tensors, self.mapped = None, {}, {}, {}, True


def run_distributed(gen: Generator, group=None, push: Optional[PushBuffers] = None, lib_ctx: Optional[rg.Context] = None):
    """Drive one rank's pipeline over torch.distributed (NCCL on GPUs, gloo on CPU). Push-mode buffers come
    from `push` (GPU: IPC-mapped copies) or, without it, are this rank's own CPU copy only, completed at each
    barrier by an all-gather of the row blocks (the CPU stand-in for the peer stores).
    lib_ctx: a context made by raftgp_ctx_create_dist -- the device all-gathers and the push barriers then run on the
    LIBRARY's NCCL communicator, stream-ordered on lib_ctx's stream (raftgp_allgather / raftgp_barrier); torch's
    process group only carries the host-side handle exchange of the push buffers."""
    import torch.distributed as dist

    def _start(t: torch.Tensor) -> _Pending:
        world = dist.get_world_size(group)
        t = t.contiguous()
        if t.is_cuda and lib_ctx is not None:   # stream-ordered on the library's stream: usable at once
            out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            lib_ctx.allgather(t, out)
            return _Done(out)
        if t.is_cuda:
            out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            return _Pending(dist.all_gather_into_tensor(out, t, group=group, async_op=True), out)
        parts = [torch.empty_like(t) for _ in range(world)]
        return _Pending(dist.all_gather(parts, t, group=group, async_op=True), None, parts)

    cpu_copies, info = {}, None
    msg = next(gen)
    while True:
        kind, payload = msg
        if kind == "gather":
            reply = _start(payload).result()
        elif kind == "start":
            reply = _start(payload)
        elif kind == "buffers":
            info = payload
            if push is not None:
                reply = push.get(payload)
            else:
                cpu_copies = {(v, k): [torch.zeros((payload["n"], w), dtype=torch.float64)]
                              for v, k, w in payload["spec"]}
                reply = cpu_copies
        elif kind == "barrier":
            if push is not None and not push.mapped:
                # fallback without peer mappings: complete this rank's copies with all-gathers of the row blocks
                rank = dist.get_rank(group)
                rb, re = info["ranges"][rank]
                nccl = dist.get_backend(group) == "nccl"
                for vk in payload:
                    full = push.tensors[vk][: info["n"]]
                    mine = _pad(full[rb:re], info["R"])
                    blocks = _start(mine if nccl else mine.cpu()).result()   # gloo: host all-gather
                    full.copy_(blocks[: info["n"]])
            elif push is not None:
                if lib_ctx is not None:
                    lib_ctx.barrier()                    # 1-element ncclAllReduce on the library's communicator
                elif dist.get_backend(group) == "nccl":
                    flag = torch.zeros(1, dtype=torch.float32, device=push.ctx.device)
                    dist.all_reduce(flag, group=group)   # stream-ordered: every rank's producing kernels are done
                else:                                    # host barrier (tests: several processes on one GPU)
                    torch.cuda.synchronize(push.ctx.device)
                    dist.barrier(group=group)
            else:
                rank = dist.get_rank(group)
                rb, re = info["ranges"][rank]
                for vk in payload:
                    full = cpu_copies[vk][0]
                    blocks = _start(_pad(full[rb:re], info["R"])).result()
                    full.copy_(blocks[: info["n"]])
            reply = None
        else:
            reply = payload.result()
        try:
            msg = gen.send(reply)
        except StopIteration as stop:
            return stop.value


def loopback_embed(ctx: rg.Context, n: int, src, dst, world: int, variant, dims, seed: int, push: bool = False):
    """P logical ranks on ONE GPU (sequential per stage, no concurrent waiting kernels). push=True runs the
    fused-exchange pipeline: each logical rank's kernels store their rows into all P full copies."""
    eng = CudaEngine(ctx)
    pipe = rank_pipeline_push if push else rank_pipeline
    gens = [pipe(eng, n, src, dst, p, world, variant, dims, seed) for p in range(world)]
    return run_loopback(gens, device=ctx.device)
