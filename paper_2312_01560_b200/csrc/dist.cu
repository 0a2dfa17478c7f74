// dist.cu — the row-partitioned multi-GPU step INSIDE the library (SURVEY.md §8(b) multi-GPU calls, §8(e), row a6).
//
// One process and one context per GPU; the contexts of a job share an NCCL communicator (raftgp_ctx_create_dist).
// Rank p owns the rows [p R, min((p+1) R, n)), R = ceil(n / P); column ids stay global (PAPER.md:56's CSR, split by
// rows). Each row's arithmetic depends only on the row (its neighbour list, the fixed in-row order, and the
// chunked global g), so the row-partitioned result is bit-identical to one GPU.
//
// Every operand a hop gathers (Theta' = Theta W^(1), then T_k = s^ (.) (Z^(k-1) W^(k)), Eq. 5-6)
// is needed for ALL n rows on every rank. Each rank holds a full copy of each operand, and the kernel that produces
// a row stores it straight into every rank's copy (peer memory over NVLink, mapped through CUDA IPC): the
// "all-gather" is fused into the producing epilogue and overlaps its gathers. A stream-ordered 1-element NCCL
// all-reduce separates producing and consuming kernels. The exchanges of one step:
//   Theta'    each rank generates its own rows (tcgen05) and pushes them, on a side stream, WHILE the CSR build
//             runs (NVLink is otherwise idle then); with RAFTGP_DIST_THETA=regen every rank generates all rows;
//   degrees   ncclAllGather of the local degree blocks (n int32);
//   g         MOD's g = d^T Theta' over fixed global 512-row chunks: each rank sums the chunks that START in its
//             rows (reading past its end in its full Theta' copy), the partials are broadcast, every rank adds
//             all chunks in g_final's fixed order (identical to one GPU);
//   T_1       the dual feature hop pushes T_1(NCut) to every copy; T_1(Mod) goes to this rank's copy only and is
//             pushed to the peers by a copy kernel on the side stream while GCN hop 1 of NCut runs (overlap of the
//             second variant's exchange with the first variant's compute);
//   T_k       each GCN hop pushes its T_{k+1} rows (for two variants with a pairable last width, into one
//             interleaved [T_a | T_b] operand, so the last hop is one 2d-wide gather). With the deferred T_1(Mod)
//             push, NCut's last hop (its half of the pair operand) runs right after NCut's hop L-1, under that push,
//             and Mod's half after Mod's hop L-1 (RAFTGP_DIST_SPLIT_LAST=0: one paired launch at the end).
// Without peer mappings (IPC refused), every rank writes its own copy only and each barrier becomes an in-place
// ncclAllGather of the produced operands (same values).
//
// `loopback`: the same schedule with P logical ranks in one process on one GPU (P graphs on one context, P full
// copies per operand, barriers trivial on one stream): the test double of the P-GPU job (bit-identity at P = 2, 3, 8).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gauss.cuh"
#include "internal.cuh"

namespace raftgp {

namespace {

raftgp_status nccl_fail(ncclResult_t r, const char *what) {
    return fail(RAFTGP_ERR_COMM, std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
}

#define RG_NCCL(call)                                              \
    do {                                                           \
        ncclResult_t _r = (call);                                  \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);        \
    } while (0)

ncclComm_t comm_of(raftgp_ctx ctx) { return static_cast<ncclComm_t>(ctx->nccl); }

// copy rows [r0, r1) of a (rows x w) operand from src into each of the dst copies (the deferred push)
__global__ void push_rows_kernel(const float4 *__restrict__ src, int64_t i0, int64_t i1, float4 *d0, float4 *d1,
                                 float4 *d2, float4 *d3, float4 *d4, float4 *d5, float4 *d6, int nd) {
    float4 *d[7] = {d0, d1, d2, d3, d4, d5, d6};
    for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < i1; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(src + i);
        for (int q = 0; q < nd; ++q) d[q][i] = v;
    }
    __threadfence_system();
}

int theta_mode() {   // 0: each rank generates its rows and pushes them (default), 1: each rank regenerates all rows
    static const int m = [] {
        const char *e = getenv("RAFTGP_DIST_THETA");
        return (e && std::string(e) == "regen") ? 1 : 0;
    }();
    return m;
}

bool split_last_mode() {   // RAFTGP_DIST_SPLIT_LAST=0: both variants' last hops as one paired launch at the end
    static const bool d = [] {
        const char *e = getenv("RAFTGP_DIST_SPLIT_LAST");
        return !(e && e[0] == '0');
    }();
    return d;
}

bool deferred_push() {   // RAFTGP_DIST_DEFER=0: the dual feature hop pushes both variants at once
    static const bool d = [] {
        const char *e = getenv("RAFTGP_DIST_DEFER");
        return !(e && e[0] == '0');
    }();
    return d;
}

}  // namespace

// ---------------------------------------------------------------- collectives on the context stream
raftgp_status dist_barrier(raftgp_ctx ctx) {
    if (!ctx->nccl || ctx->world == 1) return RAFTGP_OK;
    LaunchScope L(ctx, K_EXCHANGE, false);
    RG_NCCL(ncclAllReduce(ctx->dist_flag, ctx->dist_flag, 1, ncclFloat, ncclSum, comm_of(ctx), ctx->stream));
    return RAFTGP_OK;
}

raftgp_status dist_allgather(raftgp_ctx ctx, const void *send, void *recv, size_t bytes_per_rank) {
    if (!ctx->nccl) return fail(RAFTGP_ERR_STATE, "not a distributed context");
    LaunchScope L(ctx, K_EXCHANGE, false);
    RG_NCCL(ncclAllGather(send, recv, bytes_per_rank, ncclChar, comm_of(ctx), ctx->stream));
    return RAFTGP_OK;
}

// ---------------------------------------------------------------- cached operand copies (NCCL contexts)
void dist_release(raftgp_ctx ctx) {
    DistBufs &d = ctx->dist;
    if (d.own.empty()) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (size_t s = 0; s < d.rep.size(); ++s)
        for (int q = 0; q < (int)d.rep[s].size(); ++q)
            if (q != ctx->rank && d.rep[s][q]) cudaIpcCloseMemHandle(d.rep[s][q]);
    // nobody may still map a copy when it is freed: every rank has closed its mappings after this barrier
    if (ctx->nccl && ctx->world > 1) {
        ncclAllReduce(ctx->dist_flag, ctx->dist_flag, 1, ncclFloat, ncclSum, comm_of(ctx), ctx->stream);
        cudaStreamSynchronize(ctx->stream);
    }
    for (float *p : d.own) cudaFree(p);
    d = DistBufs{};
}

static raftgp_status dist_buffers(raftgp_ctx ctx, int64_t rows, const std::vector<int32_t> &widths) {
    DistBufs &d = ctx->dist;
    if (d.rows == rows && d.widths == widths && !d.own.empty()) return RAFTGP_OK;
    dist_release(ctx);
    const int P = ctx->world;
    d.rows = rows;
    d.widths = widths;
    const size_t S = widths.size();
    d.own.assign(S, nullptr);
    d.rep.assign(S, std::vector<float *>(P, nullptr));
    std::vector<cudaIpcMemHandle_t> mine(S);
    for (size_t s = 0; s < S; ++s) {
        cudaError_t e = cudaMalloc(&d.own[s], sizeof(float) * (size_t)rows * widths[s]);
        if (e != cudaSuccess) {
            cudaGetLastError();
            d.own[s] = nullptr;
            dist_release(ctx);
            return cuda_fail(e, "cudaMalloc (operand copy)");
        }
        RG_CUDA(cudaIpcGetMemHandle(&mine[s], d.own[s]));
        d.rep[s][ctx->rank] = d.own[s];
    }
    // exchange the handles (host bytes through a device staging buffer and ncclAllGather)
    const size_t hb = sizeof(cudaIpcMemHandle_t) * S;
    unsigned char *dh = nullptr;
    RG_CUDA(cudaMalloc(&dh, hb * (P + 1)));
    RG_CUDA(cudaMemcpyAsync(dh + hb * P, mine.data(), hb, cudaMemcpyHostToDevice, ctx->stream));
    raftgp_status st = dist_allgather(ctx, dh + hb * P, dh, hb);
    std::vector<cudaIpcMemHandle_t> all(S * P);
    if (st == RAFTGP_OK) st = cudaMemcpyAsync(all.data(), dh, hb * P, cudaMemcpyDeviceToHost, ctx->stream) == cudaSuccess
                                  ? RAFTGP_OK : fail(RAFTGP_ERR_CUDA, "handle copy");
    cudaStreamSynchronize(ctx->stream);
    cudaFree(dh);
    if (st != RAFTGP_OK) return st;
    int ok = getenv("RAFTGP_PUSH_NOIPC") == nullptr || getenv("RAFTGP_PUSH_NOIPC")[0] != '1';
    for (int q = 0; q < P && ok; ++q) {
        if (q == ctx->rank) continue;
        for (size_t s = 0; s < S && ok; ++s) {
            void *p = nullptr;
            if (cudaIpcOpenMemHandle(&p, all[(size_t)q * S + s], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                ok = 0;
            } else {
                d.rep[s][q] = static_cast<float *>(p);
            }
        }
    }
    // every rank must agree on the mode: all-reduce (min) of the local outcome
    int *dok = nullptr;
    RG_CUDA(cudaMalloc(&dok, sizeof(int)));
    RG_CUDA(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    RG_NCCL(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm_of(ctx), ctx->stream));
    RG_CUDA(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(dok);
    d.mapped = ok != 0;
    if (!d.mapped) {   // own copies only
        for (size_t s = 0; s < S; ++s)
            for (int q = 0; q < P; ++q)
                if (q != ctx->rank && d.rep[s][q]) {
                    cudaIpcCloseMemHandle(d.rep[s][q]);
                    d.rep[s][q] = nullptr;
                }
    }
    return RAFTGP_OK;
}

// ---------------------------------------------------------------- the step
namespace {

struct Slots {   // operand slot ids
    int theta = 0;
    int T[3][8];          // T[v][k] slot, k = 1..L (variant index v in the call's list)
    int pair = -1;        // interleaved last operand of the NCut/Mod pair
};

}  // namespace

raftgp_status dist_build_embed(raftgp_ctx ctx, int P, bool loopback, int64_t n, int64_t m, const int32_t *src,
                               const int32_t *dst, int32_t nvariants, const int32_t *variants, int32_t layers,
                               const int32_t *dims, uint64_t seed, float *const *Z_dev) {
    const int32_t r = dims[0], l1 = dims[1], L = layers;
    if (!sketch_w_supported(r, l1)) return fail(RAFTGP_ERR_PARAM, "row-partitioned path: r and dims[1] in {32, 64, 128}");
    if (L > 7) return fail(RAFTGP_ERR_PARAM, "row-partitioned path: at most 7 layers");
    for (int k = 1; k <= L; ++k)
        if (!push_fusable(dims[k], 0)) return fail(RAFTGP_ERR_PARAM, "row-partitioned path: widths in {32, 64, 128}");
    if (P < 1 || P > kMaxPush) return fail(RAFTGP_ERR_PARAM, "1..8 ranks");
    int where[3] = {-1, -1, -1};
    for (int v = 0; v < nvariants; ++v) where[variants[v]] = v;
    const bool dual = where[RAFTGP_NCUT] >= 0 && where[RAFTGP_MOD] >= 0;
    const int vA = where[RAFTGP_NCUT], vB = where[RAFTGP_MOD];
    const bool pair = dual && L >= 2 && gcn_pair_supported(dims[L]);
    const int64_t R = std::max<int64_t>(1, ceil_div(n, P));
    const int64_t rows_pad = R * P;
    auto rb_of = [&](int p) { return std::min<int64_t>(n, (int64_t)p * R); };
    auto re_of = [&](int p) { return std::min<int64_t>(n, (int64_t)(p + 1) * R); };
    std::vector<int> mine;
    if (loopback) for (int p = 0; p < P; ++p) mine.push_back(p);
    else mine.push_back(ctx->rank);

    // operand slots and their copies
    Slots sl;
    std::vector<int32_t> widths{l1};
    for (int v = 0; v < nvariants; ++v)
        for (int k = 1; k <= L; ++k) {
            if (pair && k == L && (v == vA || v == vB)) {
                if (sl.pair < 0) {
                    sl.pair = (int)widths.size();
                    widths.push_back(2 * dims[L]);
                }
                sl.T[v][k] = sl.pair;
            } else {
                sl.T[v][k] = (int)widths.size();
                widths.push_back(dims[k]);
            }
        }
    std::vector<std::vector<float *>> rep(widths.size(), std::vector<float *>(P, nullptr));
    std::vector<void *> lb_blocks;   // loopback copies (pool workspace)
    bool mapped = true;
    raftgp_status st = RAFTGP_OK;
    if (loopback) {
        for (size_t s = 0; s < widths.size() && st == RAFTGP_OK; ++s)
            for (int q = 0; q < P && st == RAFTGP_OK; ++q) {
                st = dalloc_t(ctx, &rep[s][q], (size_t)rows_pad * widths[s]);
                lb_blocks.push_back(rep[s][q]);
            }
    } else {
        st = dist_buffers(ctx, rows_pad, widths);
        if (st == RAFTGP_OK) {
            mapped = ctx->dist.mapped;
            for (size_t s = 0; s < widths.size(); ++s) rep[s] = ctx->dist.rep[s];
        }
    }
    // the copies rank p writes to (all ranks' copies, or only its own without peer mappings) and the one it reads
    auto targets = [&](int s, int p, PushSpec &ps, bool second) {
        float **dstv = second ? ps.rep2 : ps.rep;
        int k = 0;
        if (mapped) {
            for (int q = 0; q < P; ++q) dstv[k++] = rep[s][q];
        } else {
            dstv[k++] = rep[s][p];
        }
        return k;
    };
    auto own = [&](int s, int p) { return rep[s][p]; };

    // barrier: stream-ordered; without peer mappings it completes the operands produced since the previous one
    auto barrier = [&](std::vector<int> slots) -> raftgp_status {
        if (loopback || P == 1) return RAFTGP_OK;
        if (mapped) return dist_barrier(ctx);
        std::sort(slots.begin(), slots.end());
        slots.erase(std::unique(slots.begin(), slots.end()), slots.end());
        for (int s : slots) {
            float *base = own(s, ctx->rank);
            const size_t cnt = (size_t)R * widths[s];
            LaunchScope LS(ctx, K_EXCHANGE, false);
            RG_NCCL(ncclAllGather(base + (size_t)ctx->rank * cnt, base, cnt, ncclFloat, comm_of(ctx), ctx->stream));
        }
        return RAFTGP_OK;
    };

    float *W1 = nullptr;
    std::vector<float *> Wk(L + 1, nullptr);
    double *gw = nullptr, *partial = nullptr;
    int32_t *deg_pad = nullptr;
    std::vector<raftgp_graph> G(P, nullptr);
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &W1, (size_t)r * l1);
    for (int k = 2; k <= L && st == RAFTGP_OK; ++k) {
        st = dalloc_t(ctx, &Wk[k], (size_t)dims[k - 1] * dims[k]);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, (uint32_t)k, 0, dims[k - 1], dims[k], dims[k - 1], Wk[k]);
    }
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, r, l1, r, W1);
    if (st == RAFTGP_OK && !ctx->side && cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess)
        st = fail(RAFTGP_ERR_CUDA, "side stream");
    if (st == RAFTGP_OK && (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                            cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess))
        st = fail(RAFTGP_ERR_CUDA, "events");

    // ---- Theta' on the side stream, overlapping the CSR build (it depends on the seed only)
    if (st == RAFTGP_OK) {
        cudaEventRecord(ev_fork, ctx->stream);
        cudaStreamWaitEvent(ctx->side, ev_fork, 0);
        cudaStream_t main = ctx->stream;
        ctx->stream = ctx->side;
        for (int p : mine) {
            if (st != RAFTGP_OK) break;
            if (theta_mode() == 1 || P == 1) {       // regenerate every row into this rank's own copy
                float *o = own(sl.theta, p);
                st = sketch_w_tc_rows(ctx, seed, 0, n, r, W1, l1, &o, 1);
            } else {
                PushSpec ps{};
                const int nt = targets(sl.theta, p, ps, false);
                st = sketch_w_tc_rows(ctx, seed, rb_of(p), re_of(p) - rb_of(p), r, W1, l1, ps.rep, nt);
            }
        }
        ctx->stream = main;
        cudaEventRecord(ev_join, ctx->side);
    }
    // ---- a1: CSR of the local rows (host-synchronous)
    for (int p : mine) {
        if (st != RAFTGP_OK) break;
        raftgp_graph g = new raftgp_graph_s();
        g->ctx = ctx;
        ctx_retain(ctx);
        G[p] = g;
        st = csr_build(ctx, n, m, src, dst, rb_of(p), re_of(p), g);
    }
    // ---- a2: global degrees (all-gather of the local blocks), s, s^, 2e
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &deg_pad, (size_t)rows_pad);
    if (st == RAFTGP_OK) {
        for (int p : mine)
            if (st == RAFTGP_OK && G[p]->nl > 0)
                st = dcopy(ctx, deg_pad + (size_t)p * R, G[p]->deg_local, sizeof(int32_t) * G[p]->nl);
        if (st == RAFTGP_OK && !loopback && P > 1)
            st = dist_allgather(ctx, deg_pad + (size_t)ctx->rank * R, deg_pad, sizeof(int32_t) * R);
        for (int p : mine) {
            if (st != RAFTGP_OK) break;
            if (n > 0) st = dcopy(ctx, G[p]->deg_all, deg_pad, sizeof(int32_t) * n);
            if (st == RAFTGP_OK) st = degrees_finalize(G[p]);
        }
    }
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v)
        if (variants[v] != RAFTGP_NCUT && G[mine[0]]->two_e == 0)
            st = fail(RAFTGP_ERR_DATA, "modularity operator needs at least one edge (2e = 0)");
    // ---- Theta' complete on every rank
    if (ev_join) cudaStreamWaitEvent(ctx->stream, ev_join, 0);
    if (st == RAFTGP_OK && theta_mode() == 0) st = barrier({sl.theta});
    // ---- g = d^T Theta' (MOD): chunks starting in each rank's rows, broadcast, summed in chunk order
    if (st == RAFTGP_OK && where[RAFTGP_MOD] >= 0) {
        const int64_t nch = g_chunks(n), CH = g_chunk_rows();
        auto c0_of = [&](int p) { return ceil_div(rb_of(p), CH); };
        auto c1_of = [&](int p) { return ceil_div(re_of(p), CH); };
        st = dalloc_t(ctx, &gw, (size_t)l1);
        if (st == RAFTGP_OK) st = dalloc_t(ctx, &partial, (size_t)std::max<int64_t>(1, nch) * l1);
        for (int p : mine)
            if (st == RAFTGP_OK)
                st = g_partials_range(G[p], own(sl.theta, p), l1, c0_of(p), c1_of(p) - c0_of(p), partial);
        if (st == RAFTGP_OK && !loopback && P > 1) {
            LaunchScope LS(ctx, K_EXCHANGE, false);
            ncclResult_t nr = ncclGroupStart();
            for (int q = 0; q < P && nr == ncclSuccess; ++q) {
                const size_t cnt = (size_t)(c1_of(q) - c0_of(q)) * l1;
                if (cnt) nr = ncclBroadcast(partial + c0_of(q) * l1, partial + c0_of(q) * l1, cnt, ncclDouble, q,
                                            comm_of(ctx), ctx->stream);
            }
            ncclResult_t ne = ncclGroupEnd();
            if (nr != ncclSuccess || ne != ncclSuccess) st = nccl_fail(nr != ncclSuccess ? nr : ne, "g broadcast");
        }
        if (st == RAFTGP_OK) st = g_final_chunks(ctx, partial, nch, l1, gw);
    }
    // ---- a4: feature hop (T_1 = s^ (.) X Theta' per variant), pushed into the copies
    const bool defer = dual && deferred_push() && mapped && P > 1;
    std::vector<int> produced;
    for (int p : mine) {
        if (st != RAFTGP_OK) break;
        const float *tw = own(sl.theta, p);
        if (dual) {
            PushSpec ps{};
            ps.row0 = rb_of(p);
            ps.nrep = targets(sl.T[vA][1], p, ps, false);
            ps.nrep2 = targets(sl.T[vB][1], p, ps, true);
            if (defer) {   // Mod's T_1 into this rank's copy only; pushed to the peers below, under NCut's hop 1
                ps.rep2[0] = rep[sl.T[vB][1]][p];
                ps.nrep2 = 1;
            }
            st = feature_hop_pre(G[p], -1, l1, tw, gw, nullptr, ps.rep2[0], &ps);
        }
        for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
            if (dual && (v == vA || v == vB)) continue;
            PushSpec ps{};
            ps.row0 = rb_of(p);
            ps.nrep = targets(sl.T[v][1], p, ps, false);
            st = feature_hop_pre(G[p], variants[v], l1, tw, gw, nullptr, nullptr, &ps);
        }
    }
    for (int v = 0; v < nvariants; ++v) produced.push_back(sl.T[v][1]);
    if (st == RAFTGP_OK && defer) {   // side stream: Mod's T_1 rows -> the peers' copies
        cudaEventRecord(ev_fork, ctx->stream);
        cudaStreamWaitEvent(ctx->side, ev_fork, 0);
        const int s = sl.T[vB][1];
        const int64_t w4 = l1 / 4;
        cudaStream_t main = ctx->stream;
        ctx->stream = ctx->side;
        for (int p : mine) {
            float4 *d[7] = {};
            int nd = 0;
            for (int q = 0; q < P; ++q)
                if (q != p) d[nd++] = reinterpret_cast<float4 *>(rep[s][q]);
            if (re_of(p) <= rb_of(p)) continue;
            LaunchScope LS(ctx, K_PUSH_COPY);
            push_rows_kernel<<<ctx->sm_count / 4 > 0 ? ctx->sm_count / 4 : 1, 256, 0, ctx->side>>>(
                reinterpret_cast<const float4 *>(rep[s][p]), rb_of(p) * w4, re_of(p) * w4, d[0], d[1], d[2], d[3], d[4],
                d[5], d[6], nd);
        }
        ctx->stream = main;
        if (cudaGetLastError() != cudaSuccess) st = fail(RAFTGP_ERR_CUDA, "push_rows_kernel launch");
        cudaEventRecord(ev_join, ctx->side);
    }
    if (st == RAFTGP_OK) st = barrier(produced);
    produced.clear();
    // ---- a5: GCN hops 1 .. L-1 (each pushes T_{k+1}), then the last hop into Z.
    // split_last: NCut's last hop (its half of the interleaved pair operand) runs right after NCut's hop L-1 and a
    // barrier, i.e. while Mod's T_1 push is still crossing NVLink; Mod's half follows its own hop L-1. Each half is the
    // paired kernel with the other half's lanes idle, so every row comes out bit-identical to the paired hop.
    const bool split_last = pair && defer && split_last_mode();
    for (int k = 1; k < L && st == RAFTGP_OK; ++k) {
        // NCut first: with the deferred push, Mod's hop 1 waits for its operand (joined below)
        std::vector<int> order;
        if (dual) order = {vA, vB};
        for (int v = 0; v < nvariants; ++v)
            if (!(dual && (v == vA || v == vB))) order.push_back(v);
        for (int v : order) {
            if (st != RAFTGP_OK) break;
            if (defer && k == 1 && v == vB) {   // Mod's T_1 must be complete everywhere: join the copy, barrier
                cudaStreamWaitEvent(ctx->stream, ev_join, 0);
                st = barrier(produced);
                produced.clear();
                if (st != RAFTGP_OK) break;
            }
            const int s_in = sl.T[v][k], s_out = sl.T[v][k + 1];
            for (int p : mine) {
                if (st != RAFTGP_OK) break;
                PushSpec ps{};
                ps.row0 = rb_of(p);
                ps.nrep = targets(s_out, p, ps, false);
                if (s_out == sl.pair) {   // interleaved [T_a | T_b]: this variant's half, row stride 2d
                    const int off = (v == vA) ? 0 : dims[k + 1];
                    for (int q = 0; q < ps.nrep; ++q) ps.rep[q] += off;
                    ps.ld = 2 * dims[k + 1];
                }
                st = gcn_hop(G[p], own(s_in, p), dims[k], nullptr, Wk[k + 1], dims[k + 1], nullptr, 0, &ps);
            }
            produced.push_back(s_out);
            if (split_last && k == L - 1 && v == vA && st == RAFTGP_OK) {   // NCut's half complete everywhere
                st = barrier(produced);
                produced.clear();
                for (int p : mine) {
                    if (st != RAFTGP_OK) break;
                    const int64_t off = loopback ? rb_of(p) : 0;
                    st = gcn_final_pair(G[p], own(sl.pair, p), dims[L], Z_dev[vA] + off * dims[L],
                                        Z_dev[vB] + off * dims[L], 1);
                }
            }
        }
        if (st == RAFTGP_OK) st = barrier(produced);
        produced.clear();
    }
    for (int p : mine) {
        if (st != RAFTGP_OK) break;
        const int64_t off = loopback ? rb_of(p) : 0;   // loopback: Z holds all n rows
        if (pair) {
            st = gcn_final_pair(G[p], own(sl.pair, p), dims[L], Z_dev[vA] + off * dims[L], Z_dev[vB] + off * dims[L],
                                split_last ? 2 : 0);
        }
        for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
            if (pair && (v == vA || v == vB)) continue;
            st = gcn_hop(G[p], own(sl.T[v][L], p), dims[L], Z_dev[v] + off * dims[L], nullptr, 0, nullptr);
        }
    }
    // ---- cleanup (the cached copies of NCCL contexts stay for the next step)
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (raftgp_graph g : G)
        if (g) raftgp_graph_destroy(g);
    dfree(ctx, W1);
    for (float *w : Wk) dfree(ctx, w);
    dfree(ctx, gw);
    dfree(ctx, partial);
    dfree(ctx, deg_pad);
    for (void *b : lb_blocks) dfree(ctx, b);
    return st;
}

}  // namespace raftgp

using namespace raftgp;

extern "C" {

raftgp_status raftgp_nccl_unique_id(void *out128) {
    if (!out128) return fail(RAFTGP_ERR_PARAM, "null output");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    RG_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_create_dist(int device, void *cuda_stream, int rank, int world, const void *id128,
                                     raftgp_ctx *out) {
    if (!out || !id128) return fail(RAFTGP_ERR_PARAM, "null argument");
    *out = nullptr;
    if (world < 1 || world > kMaxPush || rank < 0 || rank >= world) return fail(RAFTGP_ERR_PARAM, "need 0 <= rank < world <= 8");
    raftgp_ctx c = nullptr;
    RG_TRY(raftgp_ctx_create(device, cuda_stream, &c));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
        raftgp_ctx_destroy(c);
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->nccl = comm;
    c->rank = rank;
    c->world = world;
    if (cudaMalloc(&c->dist_flag, sizeof(float)) != cudaSuccess || cudaMemset(c->dist_flag, 0, sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        raftgp_ctx_destroy(c);
        return fail(RAFTGP_ERR_NOMEM, "barrier flag");
    }
    *out = c;
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_rank(raftgp_ctx ctx, int *rank, int *world) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    if (rank) *rank = ctx->rank;
    if (world) *world = ctx->world;
    return RAFTGP_OK;
}

raftgp_status raftgp_barrier(raftgp_ctx ctx) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    RG_CUDA(cudaSetDevice(ctx->device));
    return dist_barrier(ctx);
}

raftgp_status raftgp_allgather(raftgp_ctx ctx, const void *send_dev, void *recv_dev, size_t bytes_per_rank) {
    if (!ctx || (bytes_per_rank && (!send_dev || !recv_dev))) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->nccl) {   // a one-rank job: the gathered block is the block itself
        if (send_dev != recv_dev) return dcopy(ctx, recv_dev, send_dev, bytes_per_rank);
        return RAFTGP_OK;
    }
    return dist_allgather(ctx, send_dev, recv_dev, bytes_per_rank);
}

}  // extern "C"

namespace raftgp {
void dist_comm_destroy(raftgp_ctx ctx) {
    dist_release(ctx);
    if (ctx->nccl) {
        cudaStreamSynchronize(ctx->stream);
        ncclCommDestroy(comm_of(ctx));
        ctx->nccl = nullptr;
    }
    if (ctx->dist_flag) cudaFree(ctx->dist_flag);
    ctx->dist_flag = nullptr;
}
}  // namespace raftgp
