// sketch.cu — a3 of the hot path: the Gaussian sketch Theta of Eq. 5 and the random
// weights W^(k) of Eq. 6 (untrained per PAPER.md:151), generated in-kernel from the
// counter-based Philox4x32-10 + Box-Muller spec (docs/SKETCH_SPEC.md, gauss.cuh).
//
// One thread produces one (row, column-quad): one Philox call -> 4 normals -> one 128-bit store.
// The generator is ALU-bound (Philox ~20 IMAD + polynomial FMAs per quad), the store is coalesced.
//
// For the MOD variant the rank-1 term needs g = d^T Theta = sum_j d_j Theta_j (fp64). It is reduced
// deterministically: fixed chunks of kGChunk global rows, each summed sequentially per column by one
// thread (fp64), then the chunk partials combined in a fixed order (g_final). The result depends only on (graph,
// seed, r) — not on the launch configuration or on the number of ranks.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gauss.cuh"
#include "internal.cuh"

namespace raftgp {

namespace {

#ifndef RG_G_CHUNK
#define RG_G_CHUNK 512
#endif
constexpr int kGChunk = RG_G_CHUNK;   // rows per g partial (512: 4x the blocks of round 2's 2048, same bytes)

__global__ void __launch_bounds__(256) gauss_fill(uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows,
                                                  int32_t cols, float sigma, float *__restrict__ out, bool vec4) {
    const int64_t nq = (cols + 3) / 4;
    const int64_t total = rows * nq;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t i = t / nq;
        const uint32_t q = static_cast<uint32_t>(t - i * nq);
        const float4 v = spec_quad(seed, tag, static_cast<uint64_t>(row_begin + i), q, sigma);
        float *o = out + i * cols + 4 * (int64_t)q;
        if (vec4) {
            *reinterpret_cast<float4 *>(o) = v;
        } else {
            const int c0 = 4 * q;
            if (c0 + 0 < cols) o[0] = v.x;
            if (c0 + 1 < cols) o[1] = v.y;
            if (c0 + 2 < cols) o[2] = v.z;
            if (c0 + 3 < cols) o[3] = v.w;
        }
    }
}

// partial[chunk][c] = sum_{j in chunk, sequential} d_j * theta[j][c]   (fp64); rows loaded 16 ahead so the fp64 add
// chain, not the load latency, sets the pace
__global__ void __launch_bounds__(128) g_partials(const float *__restrict__ theta, const int32_t *__restrict__ deg,
                                                  int64_t n, int32_t r, int64_t chunk0, double *__restrict__ partial,
                                                  const int32_t *__restrict__ slot) {
    const int64_t chunk = chunk0 + blockIdx.x;
    const int64_t j0 = chunk * kGChunk, j1 = min(n, j0 + (int64_t)kGChunk);
    // blockIdx.y picks a 128-column slice (wide operands); each (chunk, column) sum stays sequential in j
    for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < r; c += gridDim.y * blockDim.x) {
        double acc = 0.0;
        int64_t j = j0;
        for (; j + 16 <= j1; j += 16) {
            float t[16];
            int32_t d[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {   // row j of theta is at slot[j] in the slot layout (relabel.cu)
                t[u] = __ldg(theta + (slot ? (int64_t)__ldg(slot + j + u) : (j + u)) * r + c);
                d[u] = __ldg(deg + j + u);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc += static_cast<double>(d[u]) * static_cast<double>(t[u]);
        }
        for (; j < j1; ++j)
            acc += static_cast<double>(deg[j]) * static_cast<double>(theta[(slot ? (int64_t)slot[j] : j) * r + c]);
        partial[chunk * r + c] = acc;
    }
}

// g[c] = the chunk partials of column c combined in a FIXED order: block c, thread t sums the chunks t, t + 256, ...
// in sequence, then a fixed shared-memory tree over the 256 threads (deterministic; every path uses this kernel)
constexpr int kGFinalThreads = 256;
__global__ void __launch_bounds__(kGFinalThreads) g_final(const double *__restrict__ partial, int64_t nchunks, int32_t r,
                                                          double *__restrict__ g) {
    __shared__ double red[kGFinalThreads];
    for (int c = blockIdx.x; c < r; c += gridDim.x) {
        double acc = 0.0;
        for (int64_t k = threadIdx.x; k < nchunks; k += kGFinalThreads) acc += __ldg(partial + k * r + c);
        red[threadIdx.x] = acc;
        __syncthreads();
#pragma unroll
        for (int o = kGFinalThreads / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) g[c] = red[0];
        __syncthreads();
    }
}

// Theta' = Theta W1 for all n rows, with Theta generated in shared memory (never written to HBM).
// Every feature operator is linear in Theta, so (X Theta) W1 = X (Theta W1): gathering Theta' instead of
// Theta lets the feature hop skip its per-row GEMM, and one Theta' serves every variant of a call.
// Tile: TM = 128 rows x L1 columns per CTA; Theta is generated KC = 32 columns at a time into shared
// memory and multiplied into the accumulators (256 threads, each an RPT x 8 block, FFMA, W1 resident in
// shared memory), so two CTAs fit per SM and one generates while the other multiplies.
template <int R, int L1>
__global__ void __launch_bounds__(256, 2) sketch_w_kernel(uint64_t seed, int64_t n, float sigma,
                                                          const float *__restrict__ W1, float *__restrict__ out) {
    constexpr int TM = 128, KC = 32, KP = KC + 4;   // padded row stride of the Theta chunk
    constexpr int CG = L1 / 8, RGN = 256 / CG, RPT = TM / RGN;
    extern __shared__ float4 sw4[];
    float *Wsm = reinterpret_cast<float *>(sw4);  // R x L1
    float *Ts = Wsm + R * L1;                     // TM x KP
    for (int t = threadIdx.x; t < R * L1 / 4; t += blockDim.x)
        reinterpret_cast<float4 *>(Wsm)[t] = reinterpret_cast<const float4 *>(W1)[t];
    const int cg = threadIdx.x % CG, rg = threadIdx.x / CG;
    const int64_t ntiles = (n + TM - 1) / TM;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * TM;
        float acc[RPT][8];
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < R; k0 += KC) {
            __syncthreads();
            for (int t = threadIdx.x; t < TM * (KC / 4); t += blockDim.x) {
                const int rr = t / (KC / 4), q = t % (KC / 4);
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r0 + rr < n)
                    v = spec_quad(seed, 0u, static_cast<uint64_t>(r0 + rr), static_cast<uint32_t>(k0 / 4 + q), sigma);
                *reinterpret_cast<float4 *>(Ts + rr * KP + 4 * q) = v;
            }
            __syncthreads();
#pragma unroll 4
            for (int k = 0; k < KC; ++k) {
                const float4 b0 = *reinterpret_cast<const float4 *>(Wsm + (k0 + k) * L1 + cg * 8);
                const float4 b1 = *reinterpret_cast<const float4 *>(Wsm + (k0 + k) * L1 + cg * 8 + 4);
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const float a = Ts[(rg * RPT + i) * KP + k];
                    acc[i][0] = fmaf(a, b0.x, acc[i][0]);
                    acc[i][1] = fmaf(a, b0.y, acc[i][1]);
                    acc[i][2] = fmaf(a, b0.z, acc[i][2]);
                    acc[i][3] = fmaf(a, b0.w, acc[i][3]);
                    acc[i][4] = fmaf(a, b1.x, acc[i][4]);
                    acc[i][5] = fmaf(a, b1.y, acc[i][5]);
                    acc[i][6] = fmaf(a, b1.z, acc[i][6]);
                    acc[i][7] = fmaf(a, b1.w, acc[i][7]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int64_t row = r0 + rg * RPT + i;
            if (row < n) {
                float4 *o = reinterpret_cast<float4 *>(out + row * L1 + cg * 8);
                o[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                o[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
            }
        }
    }
}

template <int R, int L1>
raftgp_status launch_sketch_w(raftgp_ctx ctx, uint64_t seed, int64_t n, float sigma, const float *W1, float *out) {
    const size_t smem = sizeof(float) * ((size_t)R * L1 + 128 * 36);
    static const char attr_key = 0;   // per-(device, instantiation) key
    RG_TRY(per_device(ctx->device, &attr_key, nullptr, [&](int *) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(sketch_w_kernel<R, L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        return RAFTGP_OK;
    }));
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 128), 2 * ctx->sm_count)));
    {
        LaunchScope L(ctx, K_SKETCH);
        sketch_w_kernel<R, L1><<<grid, 256, smem, ctx->stream>>>(seed, n, sigma, W1, out);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

template <int R>
raftgp_status dispatch_sketch_w(raftgp_ctx ctx, uint64_t seed, int64_t n, float sigma, const float *W1, int l1,
                                float *out) {
    switch (l1) {
        case 32: return launch_sketch_w<R, 32>(ctx, seed, n, sigma, W1, out);
        case 64: return launch_sketch_w<R, 64>(ctx, seed, n, sigma, W1, out);
        default: return launch_sketch_w<R, 128>(ctx, seed, n, sigma, W1, out);
    }
}

}  // namespace

raftgp_status sketch_fill(raftgp_ctx ctx, uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows, int32_t cols,
                          int32_t den, float *out) {
    if (rows == 0) return RAFTGP_OK;
    const float sigma = spec_sigma(den);
    const int64_t work = rows * ((cols + 3) / 4);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), (int64_t)ctx->sm_count * 16)));
    const bool vec4 = (cols % 4 == 0) && aligned16(out);
    {
        LaunchScope L(ctx, K_SKETCH);
        gauss_fill<<<grid, 256, 0, ctx->stream>>>(seed, tag, row_begin, rows, cols, sigma, out, vec4);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

bool sketch_w_supported(int32_t r, int32_t l1) {
    return (r == 32 || r == 64 || r == 128) && (l1 == 32 || l1 == 64 || l1 == 128);
}

// tcgen05 path by default (RAFTGP_TC=0 selects the FFMA kernel)
bool sketch_tc_enabled() {   // RAFTGP_TC=0: the FFMA Theta' kernel
    static const bool use_tc = [] {
        const char *e = getenv("RAFTGP_TC");
        return !(e && e[0] == '0');
    }();
    return use_tc;
}

raftgp_status sketch_w_any(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, const float *W1, int32_t l1, float *out) {
    const bool use_tc = sketch_tc_enabled();
    if (n == 0) return RAFTGP_OK;
    if (use_tc) return sketch_w_tc(ctx, seed, n, r, W1, l1, out);
    const float sigma = spec_sigma(r);
    switch (r) {
        case 32: return dispatch_sketch_w<32>(ctx, seed, n, sigma, W1, l1, out);
        case 64: return dispatch_sketch_w<64>(ctx, seed, n, sigma, W1, l1, out);
        default: return dispatch_sketch_w<128>(ctx, seed, n, sigma, W1, l1, out);
    }
}

raftgp_status sketch_theta_w(raftgp_graph g, uint64_t seed, int32_t r, const float *W1, int32_t l1, float *out,
                             double *g_out) {
    RG_TRY(sketch_w_any(g->ctx, seed, g->n, r, W1, l1, out));
    return g_reduce(g, out, l1, g_out);
}

raftgp_status sketch_theta(raftgp_graph g, uint64_t seed, int32_t r, float *theta, double *g_out) {
    raftgp_ctx ctx = g->ctx;
    RG_TRY(sketch_fill(ctx, seed, 0u, 0, g->n, r, r, theta));
    return g_reduce(g, theta, r, g_out);
}

raftgp_status g_reduce(raftgp_graph g, const float *theta, int32_t r, double *g_out) {
    raftgp_ctx ctx = g->ctx;
    if (g_out == nullptr) return RAFTGP_OK;
    const int64_t nchunks = ceil_div(g->n, kGChunk);
    if (nchunks == 0) {
        RG_TRY(dzero(ctx, g_out, sizeof(double) * r, ctx->stream));
        return RAFTGP_OK;
    }
    double *partial = nullptr;
    RG_TRY(dalloc_t(ctx, &partial, (size_t)nchunks * r));
    RG_TRY(g_partials_range(g, theta, r, 0, nchunks, partial));
    RG_TRY(g_final_chunks(ctx, partial, nchunks, r, g_out));
    dfree(ctx, partial);
    return RAFTGP_OK;
}

int64_t g_chunks(int64_t n) { return ceil_div(n, kGChunk); }
int64_t g_chunk_rows() { return kGChunk; }

raftgp_status g_partials_range(raftgp_graph g, const float *theta, int32_t r, int64_t chunk0, int64_t count,
                               double *partial) {
    raftgp_ctx ctx = g->ctx;
    if (count <= 0) return RAFTGP_OK;
    {
        LaunchScope L(ctx, K_SKETCH_G);
        g_partials<<<dim3((unsigned)count, (unsigned)ceil_div(r, 128)), 128, 0, ctx->stream>>>(
            theta, g->deg_all, g->n, r, chunk0, partial, g->slots_active ? g->slot : nullptr);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

raftgp_status g_final_chunks(raftgp_ctx ctx, const double *partial, int64_t nchunks, int32_t r, double *g_out) {
    if (nchunks == 0) return dzero(ctx, g_out, sizeof(double) * r);
    {
        LaunchScope L(ctx, K_G_FINAL);
        g_final<<<(unsigned)r, kGFinalThreads, 0, ctx->stream>>>(partial, nchunks, r, g_out);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

}  // namespace raftgp
