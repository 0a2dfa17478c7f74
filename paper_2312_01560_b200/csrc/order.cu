// order.cu — locality-aware processing order of the rows (a performance device; results are unchanged).
//
// The hop kernels gather one operand row per edge; with random node ids almost every gather misses L2
// (the operand is 1.3-2.6 GB at C4). The graphs of this method have community structure (it is what
// RaftGP looks for): if the rows that are processed at the same time belong to the same
// communities, most of their neighbours are shared and stay in the 126 MB L2. This file computes such an
// order cheaply, once per graph:
//   1. a few rounds of asynchronous label propagation (each row takes the most frequent label among a
//      sample of its neighbours — the first 32 in CSR order; ties go to the smallest label);
//   2. a counting sort of the rows by label.
// The hop kernels then visit rows in this order. Each row's arithmetic (its neighbour list and the fixed
// in-row summation order) does not depend on when the row is visited, so the outputs are bit-identical
// with or without the order; only the L2 hit rate changes. Label propagation here is deliberately racy
// (in-place updates): its outcome only affects speed, never values.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.cuh"

namespace raftgp {

namespace {

__device__ __forceinline__ int32_t warp_sort32_u(int32_t v, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j >= 1; j >>= 1) {
            const int32_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = ((lane & k) == 0);
            const bool lower = ((lane & j) == 0);
            v = (lower == up) ? min(v, o) : max(v, o);
        }
    }
    return v;
}

__global__ void init_labels(int32_t *__restrict__ label, int64_t nl, int64_t rb) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride)
        label[i] = static_cast<int32_t>(rb + i);
}

// One warp per row. Labels of neighbours outside [rb, re) are taken as their ids (other ranks' rows).
__global__ void label_prop(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t nl,
                           int64_t rb, int32_t *label) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nl; row += warps) {
        const int64_t beg = row_ptr[row];
        const int len = static_cast<int>(min((int64_t)32, row_ptr[row + 1] - beg));
        if (len == 0) continue;
        int32_t v = INT_MAX;
        if (lane < len) {
            const int64_t j = col[beg + lane] - rb;
            v = (j >= 0 && j < nl) ? label[j] : static_cast<int32_t>(j + rb);
        }
        v = warp_sort32_u(v, lane);
        const int32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
        const bool start = lane < len && (lane == 0 || v != prev);
        const unsigned starts = __ballot_sync(0xffffffffu, start);
        // run length of the run starting at this lane
        int runlen = 0;
        if (start) {
            const unsigned later = starts & ~((2u << lane) - 1u);
            const int next = later ? __ffs(later) - 1 : len;
            runlen = next - lane;
        }
        // best = longest run, ties -> smallest label (smallest lane, since sorted ascending)
        int key = start ? (runlen << 5) | (31 - lane) : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
        const int best_lane = 31 - (key & 31);
        const int32_t best = __shfl_sync(0xffffffffu, v, best_lane);
        if (lane == 0) label[row] = best;
    }
}

__global__ void label_hist(const int32_t *__restrict__ label, int64_t nl, int64_t rb, int64_t n,
                           int32_t *__restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
        const int64_t l = label[i];
        atomicAdd(cnt + (l >= 0 && l < n ? l : 0), 1);
    }
}

__global__ void label_scatter(const int32_t *__restrict__ label, int64_t nl, int64_t n,
                              const int64_t *__restrict__ start, int32_t *__restrict__ cursor,
                              int32_t *__restrict__ order) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
        int64_t l = label[i];
        if (l < 0 || l >= n) l = 0;
        order[start[l] + atomicAdd(cursor + l, 1)] = static_cast<int32_t>(i);
    }
}

}  // namespace

// Default visiting order: the heavy rows (degree > kHeavyDeg) spread one per 32 positions at the front —
// one per dynamic claim of the hop kernels (8 groups of 4 rows) — and the light rows in natural order around
// them. A warp that claims a hub gets 31 light rows with it, and no hub is left for the end of a launch
// (the tail a power-law degree sequence otherwise leaves). Pure scheduling: every row's arithmetic and
// output are unchanged (bit-identical for any order).
constexpr int kHeavyDeg = 256;

__global__ void heavy_flags(const int32_t *__restrict__ deg, int64_t nl, int32_t *__restrict__ flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nl) flag[i] = deg[i] > kHeavyDeg ? 1 : 0;
}

// The same spreading for a LIST of rows (the streamed hops, stream.cu): heavy rows every s positions from the front,
// s = min(32, count / H) (>= 1), the light rows in list order around them. H is read on the device (no host sync).
__global__ void heavy_flags_list(const int32_t *__restrict__ rows, int64_t count, const int32_t *__restrict__ deg,
                                 int32_t *__restrict__ flag) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
        flag[t] = deg[rows[t]] > kHeavyDeg ? 1 : 0;
}

__global__ void heavy_place_list(const int32_t *__restrict__ rows, const int32_t *__restrict__ flag,
                                 const int64_t *__restrict__ hrank, int64_t count, int32_t *__restrict__ out) {
    const int64_t H = hrank[count];
    const int64_t sp = H > 0 ? (count / H < 32 ? count / H : 32) : 32;   // >= 1 since H <= count
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = hrank[t];
        int64_t pos;
        if (flag[t]) {
            pos = sp * h;
        } else {
            const int64_t j = t - h;   // light index
            pos = (sp > 1 && j < (sp - 1) * H) ? (j / (sp - 1)) * sp + j % (sp - 1) + 1 : j + H;
        }
        out[pos] = rows ? rows[t] : (int32_t)t;
    }
}

raftgp_status spread_heavy_list(raftgp_ctx ctx, const int32_t *rows, int64_t count, const int32_t *deg, int32_t *out) {
    if (count <= 0) return RAFTGP_OK;
    int32_t *flag = nullptr;
    int64_t *hrank = nullptr;
    RG_TRY(dalloc_t(ctx, &flag, (size_t)count));
    RG_TRY(dalloc_t(ctx, &hrank, (size_t)count + 1));
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(count, 256), (int64_t)ctx->sm_count * 8);
    {
        LaunchScope L(ctx, K_ORDER);
        heavy_flags_list<<<grid, 256, 0, ctx->stream>>>(rows, count, deg, flag);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(scan_i32_to_i64(ctx, flag, hrank, count));
    {
        LaunchScope L(ctx, K_ORDER);
        heavy_place_list<<<grid, 256, 0, ctx->stream>>>(rows, flag, hrank, count, out);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, flag);
    dfree(ctx, hrank);
    return RAFTGP_OK;
}

namespace {
// order validation: cnt[v] += 1 for every listed row (err if out of range), then err if any cnt != 1
__global__ void order_count(const int32_t *__restrict__ order, int64_t nl, int32_t *cnt, int32_t *err) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nl; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = order[t];
        if (v < 0 || (int64_t)v >= nl) atomicOr(err, 1);
        else atomicAdd(cnt + v, 1);
    }
}
__global__ void order_check(const int32_t *__restrict__ cnt, int64_t nl, int32_t *err) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nl; t += (int64_t)gridDim.x * blockDim.x)
        if (cnt[t] != 1) atomicOr(err, 2);
}
}  // namespace

raftgp_status order_is_permutation(raftgp_ctx ctx, const int32_t *order, int64_t nl, bool *ok) {
    *ok = true;
    if (nl == 0) return RAFTGP_OK;
    int32_t *cnt = nullptr;
    RG_TRY(dalloc_t(ctx, &cnt, (size_t)nl + 1));
    RG_TRY(dzero(ctx, cnt, sizeof(int32_t) * ((size_t)nl + 1)));
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nl, 256), (int64_t)ctx->sm_count * 8);
    {
        LaunchScope L(ctx, K_MISC);
        order_count<<<grid, 256, 0, ctx->stream>>>(order, nl, cnt, cnt + nl);
    }
    RG_CHECK_LAUNCH(ctx);
    {
        LaunchScope L(ctx, K_MISC);
        order_check<<<grid, 256, 0, ctx->stream>>>(cnt, nl, cnt + nl);
    }
    RG_CHECK_LAUNCH(ctx);
    int32_t err = 0;
    RG_TRY(dread(ctx, &err, cnt + nl, sizeof(int32_t)));
    dfree(ctx, cnt);
    *ok = err == 0;
    return RAFTGP_OK;
}

raftgp_status compute_order(raftgp_graph g) {
    static const int rounds = [] {
        const char *e = getenv("RAFTGP_ORDER_ROUNDS");
        return e ? atoi(e) : 0;   // off by default: measured gain < cost at C4
    }();
    raftgp_ctx ctx = g->ctx;
    if (g->nl == 0) return RAFTGP_OK;
    if (rounds <= 0) {
        static const bool spread = [] {   // RAFTGP_HEAVY_SPREAD=0: natural order
            const char *e = getenv("RAFTGP_HEAVY_SPREAD");
            return !(e && e[0] == '0');
        }();
        if (!spread) return RAFTGP_OK;
        cudaStream_t st = ctx->stream;
        const int64_t nl = g->nl;
        int32_t *flag = nullptr;
        int64_t *hrank = nullptr;
        RG_TRY(dalloc_t(ctx, &flag, (size_t)nl));
        RG_TRY(dalloc_t(ctx, &hrank, (size_t)nl + 1));
        const unsigned grid = (unsigned)ceil_div(nl, 256);
        {
            LaunchScope L(ctx, K_ORDER);
            heavy_flags<<<grid, 256, 0, st>>>(g->deg_local, nl, flag);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, flag, hrank, nl));
        // the heavy count H stays on the device (no host read-back): the placement reads it and spaces the heavy rows
        // min(32, nl / H) apart (every 32nd position for C4's 1.8 % heavy rows; identity order when H = 0)
        if (g->order == nullptr) RG_TRY(dalloc_t(ctx, &g->order, (size_t)nl));
        {
            LaunchScope L(ctx, K_ORDER);
            const unsigned pg = (unsigned)std::min<int64_t>(grid, (int64_t)ctx->sm_count * 16);
            heavy_place_list<<<pg, 256, 0, st>>>(nullptr, flag, hrank, nl, g->order);
        }
        RG_CHECK_LAUNCH(ctx);
        dfree(ctx, flag);
        dfree(ctx, hrank);
        return RAFTGP_OK;
    }
    cudaStream_t st = ctx->stream;
    const int64_t nl = g->nl, n = g->n;
    int32_t *label = nullptr, *cnt = nullptr;
    int64_t *start = nullptr;
    RG_TRY(dalloc_t(ctx, &label, (size_t)nl));
    RG_TRY(dalloc_t(ctx, &cnt, (size_t)n));
    RG_TRY(dalloc_t(ctx, &start, (size_t)n + 1));
    if (g->order == nullptr) RG_TRY(dalloc_t(ctx, &g->order, (size_t)nl));
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nl, 256), (int64_t)ctx->sm_count * 8));
    const int wgrid = static_cast<int>(std::min<int64_t>(ceil_div(nl, 8), (int64_t)ctx->sm_count * 8));
    {
        LaunchScope L(ctx, K_ORDER);
        init_labels<<<grid, 256, 0, st>>>(label, nl, g->row_begin);
    }
    RG_CHECK_LAUNCH(ctx);
    for (int it = 0; it < rounds; ++it) {
        LaunchScope L(ctx, K_ORDER);
        label_prop<<<wgrid, 256, 0, st>>>(g->row_ptr, g->col, nl, g->row_begin, label);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(dzero(ctx, cnt, sizeof(int32_t) * n, st));
    {
        LaunchScope L(ctx, K_ORDER);
        label_hist<<<grid, 256, 0, st>>>(label, nl, g->row_begin, n, cnt);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(scan_i32_to_i64(ctx, cnt, start, n));
    RG_TRY(dzero(ctx, cnt, sizeof(int32_t) * n, st));
    {
        LaunchScope L(ctx, K_ORDER);
        label_scatter<<<grid, 256, 0, st>>>(label, nl, n, start, cnt, g->order);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, label);
    dfree(ctx, cnt);
    dfree(ctx, start);
    return RAFTGP_OK;
}

}  // namespace raftgp
