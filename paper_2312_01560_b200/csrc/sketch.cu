// sketch.cu — a3 of the hot path: the Gaussian sketch Theta of Eq. 5 and the random
// weights W^(k) of Eq. 6 (untrained per PAPER.md:151), generated in-kernel from the
// counter-based Philox4x32-10 + Box-Muller spec (docs/SKETCH_SPEC.md, gauss.cuh).
//
// One thread produces one (row, column-quad): one Philox call -> 4 normals -> one 128-bit store.
// The generator is ALU-bound (Philox ~20 IMAD + polynomial FMAs per quad), the store is coalesced.
//
// For the MOD variant the rank-1 term needs g = d^T Theta = sum_j d_j Theta_j (fp64). It is reduced
// deterministically: fixed chunks of kGChunk global rows, each summed sequentially per column by one
// thread (fp64), then the chunk partials summed in chunk order. The result depends only on (graph,
// seed, r) — not on the launch configuration or on the number of ranks.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "gauss.cuh"
#include "internal.cuh"

namespace raftgp {

namespace {

constexpr int kGChunk = 2048;

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

// partial[chunk][c] = sum_{j in chunk, sequential} d_j * theta[j][c]   (fp64)
__global__ void __launch_bounds__(128) g_partials(const float *__restrict__ theta, const int32_t *__restrict__ deg,
                                                  int64_t n, int32_t r, double *__restrict__ partial) {
    const int64_t chunk = blockIdx.x;
    const int64_t j0 = chunk * kGChunk, j1 = min(n, j0 + (int64_t)kGChunk);
    for (int c = threadIdx.x; c < r; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t j = j0; j < j1; ++j) acc += static_cast<double>(deg[j]) * static_cast<double>(theta[j * r + c]);
        partial[chunk * r + c] = acc;
    }
}

__global__ void g_final(const double *__restrict__ partial, int64_t nchunks, int32_t r, double *__restrict__ g) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < r; c += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t k = 0; k < nchunks; ++k) acc += partial[k * r + c];
        g[c] = acc;
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

raftgp_status sketch_theta(raftgp_graph g, uint64_t seed, int32_t r, float *theta, double *g_out) {
    raftgp_ctx ctx = g->ctx;
    RG_TRY(sketch_fill(ctx, seed, 0u, 0, g->n, r, r, theta));
    if (g_out == nullptr) return RAFTGP_OK;
    const int64_t nchunks = ceil_div(g->n, kGChunk);
    if (nchunks == 0) {
        RG_CUDA(cudaMemsetAsync(g_out, 0, sizeof(double) * r, ctx->stream));
        return RAFTGP_OK;
    }
    double *partial = nullptr;
    RG_TRY(dalloc_t(ctx, &partial, (size_t)nchunks * r));
    {
        LaunchScope L(ctx, K_SKETCH_G);
        g_partials<<<(unsigned)nchunks, 128, 0, ctx->stream>>>(theta, g->deg_all, g->n, r, partial);
    }
    RG_CHECK_LAUNCH(ctx);
    {
        LaunchScope L(ctx, K_G_FINAL);
        g_final<<<(unsigned)ceil_div(r, 128), 128, 0, ctx->stream>>>(partial, nchunks, r, g_out);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, partial);
    return RAFTGP_OK;
}

}  // namespace raftgp
