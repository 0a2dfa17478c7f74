// relabel.cu — slot layout of the hop operands (a scheduling / layout choice: every row's arithmetic is unchanged).
//
// The hops gather one operand row per CSR entry (Eq. 5-6); on the power-law graphs of the
// workloads a few rows are gathered very often (at C4 the 131 K rows of degree >= 186 — 64 MB of 512-byte rows —
// take 29 % of all gathers). In node order those rows are scattered over the 2.56 GB operand and compete for L2 with
// the one-off rows. The slot layout stores node i's operand row at slot[i]: the hubs (the highest degrees, up to
// kHubBytes of rows) first, in node order, then every other row in node order. The hops then gather
// operand[colx[p]] with colx = slot[col] (built once per graph), and load the non-hub slots evict-first, so the hub
// rows stay in L2 (microbenchmark on C4's degree sequence: 13.8 -> 12.1 ms per gather pass). Outputs that are
// embeddings (Z) stay in node order; the sketch writes Theta' into slots, the epilogues write T into slots.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace raftgp {

namespace {

constexpr int kDegBins = 4096;                       // degree histogram (degrees >= kDegBins - 1 share the last bin)
constexpr int64_t kHubBytes = (int64_t)64 << 20;     // operand bytes of hub rows kept in L2 (of 126 MB); RAFTGP_HUB_MB
constexpr int kRowBytes = 512;                       // the widest gathered operand row (128 fp32)

__global__ void slot_hist(const int32_t *__restrict__ deg, int64_t n, unsigned int *__restrict__ hist) {
    __shared__ unsigned int h[kDegBins];
    for (int b = threadIdx.x; b < kDegBins; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[min(deg[i], kDegBins - 1)], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < kDegBins; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], h[b]);
}

// one block: the smallest degree threshold t >= 1 with #(deg >= t) <= kmax (t = kDegBins: no hubs). Suffix counts
// by a block scan over the histogram (one thread walking 4096 bins from the top took 0.23 ms per build)
__global__ void __launch_bounds__(1024) slot_threshold(const unsigned int *__restrict__ hist, int64_t kmax,
                                                       int32_t *__restrict__ thr) {
    constexpr int PER = kDegBins / 1024;
    __shared__ long long wsum[32];
    __shared__ int best;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // thread t owns bins [kDegBins - PER (t + 1), kDegBins - PER t): thread 0 the highest degrees
    long long v[PER], run = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        v[k] = hist[kDegBins - 1 - (PER * t + k)];
        run += v[k];
    }
    long long x = run;   // inclusive scan over threads (highest bins first)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    if (t == 0) best = kDegBins;
    __syncthreads();
    if (w == 0) {
        long long y = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        wsum[lane] = y;
    }
    __syncthreads();
    long long cum = x - run + (w > 0 ? wsum[w - 1] : 0);   // rows of degree above this thread's bins
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int d = kDegBins - 1 - (PER * t + k);
        cum += v[k];
        if (d >= 1 && cum <= kmax) atomicMin(&best, d);   // #(deg >= d) <= kmax
    }
    __syncthreads();
    if (t == 0) thr[0] = best;
}

__global__ void slot_flags(const int32_t *__restrict__ deg, int64_t n, const int32_t *__restrict__ thr,
                           int32_t *__restrict__ flag) {
    const int32_t t = thr[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (t < kDegBins && deg[i] >= t) ? 1 : 0;
}

// stable partition: hubs first in node order, then the rest in node order
__global__ void slot_place(const int32_t *__restrict__ flag, const int64_t *__restrict__ hrank, int64_t n,
                           const float *__restrict__ s_all, int32_t *__restrict__ slot, float *__restrict__ s_slot,
                           int32_t *__restrict__ hubk) {
    const int64_t K = hrank[n];
    if (blockIdx.x == 0 && threadIdx.x == 0) hubk[0] = (int32_t)K;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = hrank[i];
        const int64_t sl = flag[i] ? h : K + (i - h);
        slot[i] = (int32_t)sl;
        s_slot[sl] = s_all[i];
    }
}

// per 32-node word: the hub bitmap and the hubs before the word. An entry's slot is then one 8-byte load from a table
// of n / 4 bytes (1.25 MB at C4, 12.5 MB at C5: L2-resident) instead of a 4-byte load from the n-entry slot map (200 MB
// at C5, whose random reads went to DRAM: 26 ms for C5's 1.9e9 entries)
__global__ void slot_words(const int32_t *__restrict__ flag, const int64_t *__restrict__ hrank, int64_t n,
                           uint2 *__restrict__ words) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (n + 31) / 32;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = w * 32 + lane;
        const unsigned bits = __ballot_sync(0xffffffffu, i < n && flag[i]);
        if (lane == 0) words[w] = make_uint2(bits, (unsigned)hrank[w * 32]);
    }
}

__device__ __forceinline__ int32_t slot_of(int32_t j, const uint2 *__restrict__ words, int64_t K) {
    const uint2 e = __ldg(words + (j >> 5));
    const unsigned b = j & 31;
    const int64_t h = (int64_t)e.y + __popc(e.x & ((1u << b) - 1u));   // hubs before j
    return (int32_t)(((e.x >> b) & 1u) ? h : K + j - h);
}

// four entries per thread (16-byte loads and stores of col / colx, four independent table lookups in flight)
__global__ void slot_cols(const int32_t *__restrict__ col, int64_t nnz, const uint2 *__restrict__ words,
                          const int32_t *__restrict__ hubk, int32_t *__restrict__ colx, bool vec) {
    const int64_t K = hubk[0];
    const int64_t n4 = vec ? nnz >> 2 : 0;
    const int4 *c4 = reinterpret_cast<const int4 *>(col);
    int4 *x4 = reinterpret_cast<int4 *>(colx);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n4; p += (int64_t)gridDim.x * blockDim.x) {
        const int4 j = __ldcs(c4 + p);
        x4[p] = make_int4(slot_of(j.x, words, K), slot_of(j.y, words, K), slot_of(j.z, words, K), slot_of(j.w, words, K));
    }
    for (int64_t p = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (int64_t)gridDim.x * blockDim.x)   // the tail (< 4 entries), or every entry of unaligned arrays
        colx[p] = slot_of(__ldg(col + p), words, K);
}

}  // namespace

// the smallest degree t with #(deg >= t) <= kmax into thr_dev (device int32[1]; kDegBins = no hubs), on the ctx stream
raftgp_status hub_degree_threshold(raftgp_ctx ctx, const int32_t *deg, int64_t n, int64_t kmax, int32_t *thr_dev) {
    unsigned int *hist = nullptr;
    RG_TRY(dalloc_t(ctx, &hist, kDegBins));
    raftgp_status st = dzero(ctx, hist, sizeof(unsigned int) * kDegBins, ctx->stream);
    if (st == RAFTGP_OK) {
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 2));
        LaunchScope L(ctx, K_ORDER);
        slot_hist<<<grid, 256, 0, ctx->stream>>>(deg, n, hist);
        slot_threshold<<<1, 1024, 0, ctx->stream>>>(hist, kmax, thr_dev);
    }
    if (st == RAFTGP_OK) {
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) st = cuda_fail(e, "kernel launch");
    }
    dfree(ctx, hist);
    return st;
}

int64_t slot_hub_bytes() {
    static const int64_t b = [] {
        const char *e = getenv("RAFTGP_HUB_MB");
        return e ? (int64_t)std::max(0, atoi(e)) << 20 : kHubBytes;
    }();
    return b;
}

bool slots_enabled() {
    static const bool on = [] {
        const char *e = getenv("RAFTGP_RELABEL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void drop_slots(raftgp_graph g) {
    raftgp_ctx ctx = g->ctx;
    dfree(ctx, g->slot);
    dfree(ctx, g->colx);
    dfree(ctx, g->s_slot);
    dfree(ctx, g->hubk);
    g->slot = g->colx = g->hubk = nullptr;
    g->s_slot = nullptr;
}

raftgp_status ensure_slots(raftgp_graph g) {
    if (g->slot) return RAFTGP_OK;
    if (g->row_begin != 0 || g->row_end != g->n || g->n == 0) return fail(RAFTGP_ERR_INTERNAL, "slots: whole graph only");
    raftgp_ctx ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t n = g->n, nnz = g->nnz_local;
    unsigned int *hist = nullptr;
    int32_t *thr = nullptr, *flag = nullptr;
    int64_t *hrank = nullptr;
    RG_TRY(dalloc_t(ctx, &g->slot, (size_t)n));
    RG_TRY(dalloc_t(ctx, &g->s_slot, (size_t)n));
    RG_TRY(dalloc_t(ctx, &g->hubk, 1));
    RG_TRY(dalloc_t(ctx, &g->colx, (size_t)std::max<int64_t>(1, nnz)));
    RG_TRY(dalloc_t(ctx, &hist, kDegBins));
    RG_TRY(dalloc_t(ctx, &thr, 1));
    RG_TRY(dalloc_t(ctx, &flag, (size_t)n));
    RG_TRY(dalloc_t(ctx, &hrank, (size_t)n + 1));
    uint2 *words = nullptr;
    RG_TRY(dalloc_t(ctx, &words, (size_t)ceil_div(n, 32)));
    RG_TRY(dzero(ctx, hist, sizeof(unsigned int) * kDegBins, st));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 8));
    {
        LaunchScope L(ctx, K_ORDER);
        slot_hist<<<std::min<unsigned>(grid, (unsigned)ctx->sm_count * 2), 256, 0, st>>>(g->deg_all, n, hist);
        slot_threshold<<<1, 1024, 0, st>>>(hist, slot_hub_bytes() / kRowBytes, thr);
        slot_flags<<<grid, 256, 0, st>>>(g->deg_all, n, thr, flag);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(scan_i32_to_i64(ctx, flag, hrank, n));
    {
        LaunchScope L(ctx, K_ORDER);
        slot_place<<<grid, 256, 0, st>>>(flag, hrank, n, g->s_all, g->slot, g->s_slot, g->hubk);
        if (nnz > 0) {
            const unsigned wg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ceil_div(n, 32), 8), (int64_t)ctx->sm_count * 8));
            slot_words<<<wg, 256, 0, st>>>(flag, hrank, n, words);
            const unsigned cg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nnz, 1024), (int64_t)ctx->sm_count * 16));
            slot_cols<<<cg, 256, 0, st>>>(g->col, nnz, words, g->hubk, g->colx, aligned16(g->col) && aligned16(g->colx));
        }
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, hist);
    dfree(ctx, thr);
    dfree(ctx, flag);
    dfree(ctx, hrank);
    dfree(ctx, words);
    return RAFTGP_OK;
}

}  // namespace raftgp
