// tc_sketch.cu — Theta' = Theta W1 on the 5th-generation tensor cores (tcgen05, TMEM), fp32-accurate.
//
// The one real dense contraction of the path (N x r by r x L1, r, L1 <= 128; Eq. 5 followed
// by the first GEMM of Eq. 6, applied before aggregation — DESIGN.md reading #13). Theta is generated in
// shared memory (docs/SKETCH_SPEC.md) and never written to HBM; W1 stays in shared memory for the whole
// kernel. fp32 accuracy from TF32 tensor cores by the 3-product split x = hi + lo (hi = x with the low 13
// mantissa bits cleared, lo = x - hi exactly): A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi, accumulated in fp32
// in TMEM (error ~2^-20 relative, far inside the 1e-4 parity bar).
//
// Per CTA (1024 threads, one per SM): a persistent loop over 128-row tiles. For each tile and each
// K-half of at most 64 columns: all threads generate Theta (one Philox call -> 4 normals -> one 16-byte
// K-chunk) and store hi/lo in the canonical no-swizzle K-major layout (8-row x 16-byte core matrices);
// one thread issues tcgen05.mma (M = 128, N = L1, K = 8) x 3 products per K-step into the TMEM
// accumulator and commits to an mbarrier. After the last half, all warps read the accumulator back
// with tcgen05.ld (warp w: lane quarter w % 4, 32-column chunks) and store the rows of Theta'. Every mbarrier wait is bounded (trap on
// timeout) so a descriptor mistake fails loudly instead of hanging the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gauss.cuh"
#include "internal.cuh"
#include "tc.cuh"

namespace raftgp {

namespace {

using namespace tc;

#ifndef RG_TC_THREADS
#define RG_TC_THREADS 1024
#endif
constexpr int kTM = 128;       // rows per tile (MMA M)
constexpr int kKH = 64;        // K columns per half (A buffer)

template <int R, int L1>
__global__ void __launch_bounds__(RG_TC_THREADS, 1) sketch_w_tc_kernel(uint64_t seed, int64_t n, float sigma,
                                                             const float *__restrict__ W1, float *__restrict__ out) {
    constexpr int KH = R < kKH ? R : kKH;              // K columns per half
    constexpr int NH = R / KH;                          // halves
    constexpr int NCOL = L1 < 32 ? 32 : L1;             // TMEM columns (power of two >= 32)
    constexpr uint32_t A_BYTES = kTM * KH * 4;
    constexpr uint32_t B_BYTES = L1 * R * 4;
    // instruction descriptor: D f32, A/B tf32, both K-major, N = L1, M = 128
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(L1 >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);

    extern __shared__ __align__(1024) unsigned char tsm[];
    unsigned char *b_hi = tsm;
    unsigned char *b_lo = b_hi + B_BYTES;
    unsigned char *a_hi = b_lo + B_BYTES;
    unsigned char *a_lo = a_hi + A_BYTES;
    __shared__ __align__(8) uint64_t mma_bar;
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // W1 (R x L1 row-major) -> B operand (L1 x R, K-major) split into hi / lo
    for (int e = tid; e < R * L1; e += blockDim.x) {
        const int k = e / L1, nn = e % L1;
        const float w = W1[e];
        const float hi = tf32_hi(w);
        const uint32_t o = kmajor_off(nn, k, L1);
        *reinterpret_cast<float *>(b_hi + o) = hi;
        *reinterpret_cast<float *>(b_lo + o) = w - hi;
    }
    if (tid == 0) {
        mbar_init(&mma_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base_sh)), "r"(NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;
    uint32_t phase = 0;

    const int64_t ntiles = (n + kTM - 1) / kTM;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * kTM;
        for (int h = 0; h < NH; ++h) {
            // generate Theta[r0 .. r0+127][h*KH .. h*KH+KH-1] as hi/lo K-chunks; GQ independent Philox
            // calls per thread are in flight together (the generator is latency-bound at 16 warps / SM)
            constexpr int NQ = kTM * (KH / 4);
            constexpr int GQ = (NQ / RG_TC_THREADS) < 4 ? ((NQ / RG_TC_THREADS) > 0 ? NQ / RG_TC_THREADS : 1) : 4;
            for (int t0 = tid; t0 < NQ; t0 += RG_TC_THREADS * GQ) {
                float4 v[GQ];
#pragma unroll
                for (int g = 0; g < GQ; ++g) {
                    const int t = t0 + g * RG_TC_THREADS;
                    const int row = t % kTM, q = t / kTM;      // consecutive threads: consecutive rows
                    v[g] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (t < NQ && r0 + row < n)
                        v[g] = spec_quad(seed, 0u, static_cast<uint64_t>(r0 + row), static_cast<uint32_t>(h * (KH / 4) + q),
                                         sigma);
                }
#pragma unroll
                for (int g = 0; g < GQ; ++g) {
                    const int t = t0 + g * RG_TC_THREADS;
                    if (t < NQ) {
                        const int row = t % kTM, q = t / kTM;
                        const float4 hi = make_float4(tf32_hi(v[g].x), tf32_hi(v[g].y), tf32_hi(v[g].z), tf32_hi(v[g].w));
                        const float4 lo = make_float4(v[g].x - hi.x, v[g].y - hi.y, v[g].z - hi.z, v[g].w - hi.w);
                        const uint32_t o = kmajor_off(row, 4 * q, kTM);
                        *reinterpret_cast<float4 *>(a_hi + o) = hi;
                        *reinterpret_cast<float4 *>(a_lo + o) = lo;
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
                const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
                constexpr uint32_t A_LBO = (kTM / 8) * 128, B_LBO = (L1 / 8) * 128, SBO = 128;
#pragma unroll
                for (int s = 0; s < KH / 8; ++s) {
                    const uint32_t aoff = s * 2 * A_LBO;
                    const uint32_t boff = (h * (KH / 8) + s) * 2 * B_LBO;
                    const uint64_t dah = smem_desc(ah + aoff, A_LBO, SBO), dal = smem_desc(al + aoff, A_LBO, SBO);
                    const uint64_t dbh = smem_desc(bh + boff, B_LBO, SBO), dbl = smem_desc(bl + boff, B_LBO, SBO);
                    const uint32_t acc0 = (h > 0 || s > 0) ? 1u : 0u;
                    mma_tf32(tmem_d, dah, dbh, IDESC, acc0);
                    mma_tf32(tmem_d, dah, dbl, IDESC, 1u);
                    mma_tf32(tmem_d, dal, dbh, IDESC, 1u);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&mma_bar)) : "memory");
            }
            // the A buffer (and, after the last half, the accumulator) is ready once the MMAs retire
            mbar_wait(&mma_bar, phase);
            phase ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (= tile rows; a warp may only touch the lane
        // quarter of its index mod 4) and the column chunks c = w / 4, w / 4 + NW / 4, ...
        {
            constexpr int NW = RG_TC_THREADS / 32;
            const int lq = warp & 3;
            const int64_t row = r0 + lq * 32 + lane;
            for (int c0 = (warp >> 2) * 32; c0 < L1; c0 += (NW / 4) * 32) {
                float v[32];
                tmem_ld32(tmem_d + (static_cast<uint32_t>(lq * 32) << 16) + c0, v);
                if (row < n) {
                    float4 *o = reinterpret_cast<float4 *>(out + row * L1 + c0);
#pragma unroll
                    for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(NCOL));
}

template <int R, int L1>
raftgp_status launch_tc(raftgp_ctx ctx, uint64_t seed, int64_t n, float sigma, const float *W1, float *out) {
    constexpr int KH = R < kKH ? R : kKH;
    const size_t smem = 2 * (size_t)L1 * R * 4 + 2 * (size_t)kTM * KH * 4;
    static bool attr = false;
    if (!attr) {
        RG_CUDA(cudaFuncSetAttribute(sketch_w_tc_kernel<R, L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kTM), ctx->sm_count)));
    {
        LaunchScope L(ctx, K_SKETCH);
        sketch_w_tc_kernel<R, L1><<<grid, RG_TC_THREADS, smem, ctx->stream>>>(seed, n, sigma, W1, out);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

template <int R>
raftgp_status dispatch_tc(raftgp_ctx ctx, uint64_t seed, int64_t n, float sigma, const float *W1, int l1, float *out) {
    switch (l1) {
        case 32: return launch_tc<R, 32>(ctx, seed, n, sigma, W1, out);
        case 64: return launch_tc<R, 64>(ctx, seed, n, sigma, W1, out);
        default: return launch_tc<R, 128>(ctx, seed, n, sigma, W1, out);
    }
}

}  // namespace

raftgp_status sketch_w_tc(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, const float *W1, int32_t l1, float *out) {
    if (n == 0) return RAFTGP_OK;
    const float sigma = spec_sigma(r);
    switch (r) {
        case 32: return dispatch_tc<32>(ctx, seed, n, sigma, W1, l1, out);
        case 64: return dispatch_tc<64>(ctx, seed, n, sigma, W1, l1, out);
        default: return dispatch_tc<128>(ctx, seed, n, sigma, W1, l1, out);
    }
}

}  // namespace raftgp
