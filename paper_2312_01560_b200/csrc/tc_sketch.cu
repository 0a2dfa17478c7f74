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
// K-quarter of at most 32 columns: all threads generate Theta (one Philox call -> 4 normals -> one 16-byte
// K-chunk) and store hi/lo in the canonical no-swizzle K-major layout (8-row x 16-byte core matrices) into
// one of two A buffers; one thread issues tcgen05.mma (M = 128, N = L1, K = 8) x 3 products per K-step into
// one of two TMEM accumulators and commits to that buffer's mbarrier, so generating quarter g overlaps the
// MMAs of quarter g - 1. All warps read the previous tile's accumulator back with tcgen05.ld (warp w: lane
// quarter w % 4, 32-column chunks) and store its rows of Theta' while the next tile's first MMAs run. Every mbarrier wait is bounded (trap on
// timeout) so a descriptor mistake fails loudly instead of hanging the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

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
constexpr int kKQ = 32;        // K columns per quarter (one of two A buffers)

// Global rows row0 .. row0 + n - 1 of Theta' (Theta's generator row = the global row); each finished row is stored at
// its global row into every one of the nout output copies (nout > 1: the row-partitioned path pushes its share of
// Theta' into every rank's copy over NVLink, dist.cu).
struct SketchOut {
    float *out[kMaxPush];
    int nout;
};

template <int R, int L1>
__global__ void __launch_bounds__(RG_TC_THREADS, 1) sketch_w_tc_kernel(uint64_t seed, int64_t row0, int64_t n, float sigma,
                                                             const float *__restrict__ W1, SketchOut outs) {
    constexpr int KQ = R < kKQ ? R : kKQ;              // K columns per quarter (one A buffer)
    constexpr int NQK = R / KQ;                         // quarters per tile
    constexpr int NCOL = L1 < 32 ? 32 : L1;             // TMEM columns of one accumulator (power of two >= 32)
    constexpr uint32_t A_BYTES = kTM * KQ * 4;
    constexpr uint32_t B_BYTES = L1 * R * 4;
    // instruction descriptor: D f32, A/B tf32, both K-major, N = L1, M = 128
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(L1 >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);

    extern __shared__ __align__(1024) unsigned char tsm[];
    unsigned char *b_hi = tsm;
    unsigned char *b_lo = b_hi + B_BYTES;
    unsigned char *a_base = b_lo + B_BYTES;             // two A buffers, each hi | lo
    __shared__ __align__(8) uint64_t mma_bar[2];        // completion of the MMAs reading A buffer 0 / 1
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
        mbar_init(&mma_bar[0], 1);
        mbar_init(&mma_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {   // two accumulators: tile t accumulates into t & 1 while tile t - 1 is read back
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base_sh)), "r"(2 * NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;

    // Pipeline over quarters g = (local tile) * NQK + q, A buffer g & 1: generating quarter g overlaps the
    // MMAs of quarter g - 1, and tile t - 1 is read back from TMEM while the MMAs of tile t's first quarter
    // run. Quarter g's commit is the (g >> 1)-th completion of mma_bar[g & 1] (parity (g >> 1) & 1); every
    // wait happens before that barrier can complete again, so the parity test is unambiguous.
    auto wait_quarter = [&](int64_t g) { mbar_wait(&mma_bar[g & 1], (uint32_t)((g >> 1) & 1)); };
    auto epilogue = [&](int64_t tile_prev, int acc) {
        // warp w reads TMEM lanes 32 (w % 4) .. + 31 (= tile rows; a warp may only touch the lane quarter of
        // its index mod 4) and the column chunks c = w / 4, w / 4 + NW / 4, ...
        constexpr int NW = RG_TC_THREADS / 32;
        const int lq = warp & 3;
        const int64_t row = tile_prev * kTM + lq * 32 + lane;
        for (int c0 = (warp >> 2) * 32; c0 < L1; c0 += (NW / 4) * 32) {
            float v[32];
            tmem_ld32(tmem_d + (static_cast<uint32_t>(lq * 32) << 16) + (uint32_t)(acc * NCOL + c0), v);
            if (row < n) {
                for (int q = 0; q < outs.nout; ++q) {
                    float4 *o = reinterpret_cast<float4 *>(outs.out[q] + (row0 + row) * L1 + c0);
#pragma unroll
                    for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
        }
    };

    const int64_t ntiles = (n + kTM - 1) / kTM;
    int64_t it = 0, prev_tile = -1;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t r0 = tile * kTM;
        const int acc = (int)(it & 1);
        for (int q = 0; q < NQK; ++q) {
            const int64_t g = it * NQK + q;
            unsigned char *a_hi = a_base + (size_t)(g & 1) * 2 * A_BYTES;
            unsigned char *a_lo = a_hi + A_BYTES;
            if (g >= 2) wait_quarter(g - 2);   // the MMAs that read this buffer have retired
            // generate Theta[r0 .. r0+127][q*KQ .. q*KQ+KQ-1] as hi/lo K-chunks (one Philox call per 4 columns)
            constexpr int NQ = kTM * (KQ / 4);
            for (int t = tid; t < NQ; t += RG_TC_THREADS) {
                const int row = t % kTM, qq = t / kTM;      // consecutive threads: consecutive rows
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r0 + row < n)
                    v = spec_quad(seed, 0u, static_cast<uint64_t>(row0 + r0 + row),
                                  static_cast<uint32_t>(q * (KQ / 4) + qq), sigma);
                const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                const float4 lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
                const uint32_t o = kmajor_off(row, 4 * qq, kTM);
                *reinterpret_cast<float4 *>(a_hi + o) = hi;
                *reinterpret_cast<float4 *>(a_lo + o) = lo;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
                const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
                constexpr uint32_t A_LBO = (kTM / 8) * 128, B_LBO = (L1 / 8) * 128, SBO = 128;
                const uint32_t dacc = tmem_d + (uint32_t)(acc * NCOL);
#pragma unroll
                for (int s = 0; s < KQ / 8; ++s) {
                    const uint32_t aoff = s * 2 * A_LBO;
                    const uint32_t boff = (q * (KQ / 8) + s) * 2 * B_LBO;
                    const uint64_t dah = smem_desc(ah + aoff, A_LBO, SBO), dal = smem_desc(al + aoff, A_LBO, SBO);
                    const uint64_t dbh = smem_desc(bh + boff, B_LBO, SBO), dbl = smem_desc(bl + boff, B_LBO, SBO);
                    const uint32_t acc0 = (q > 0 || s > 0) ? 1u : 0u;
                    mma_tf32(dacc, dah, dbh, IDESC, acc0);
                    mma_tf32(dacc, dah, dbl, IDESC, 1u);
                    mma_tf32(dacc, dal, dbh, IDESC, 1u);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&mma_bar[g & 1])) : "memory");
            }
            if (q == 0 && prev_tile >= 0) {
                // the previous tile's accumulator is complete once its last quarter's MMAs retired (they
                // were issued before this tile's first quarter, which now runs on the other accumulator)
                wait_quarter(g - 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                epilogue(prev_tile, acc ^ 1);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            }
        }
        prev_tile = tile;
    }
    if (prev_tile >= 0) {
        wait_quarter(it * NQK - 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        epilogue(prev_tile, (int)((it - 1) & 1));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(2 * NCOL));
    if (outs.nout > 1) __threadfence_system();   // rows stored into the peers' copies are visible to them
}

template <int R, int L1>
raftgp_status launch_tc(raftgp_ctx ctx, uint64_t seed, int64_t row0, int64_t n, float sigma, const float *W1,
                        const SketchOut &outs) {
    constexpr int KQ = R < kKQ ? R : kKQ;
    const size_t smem = 2 * (size_t)L1 * R * 4 + 2 * 2 * (size_t)kTM * KQ * 4;
    static const char attr_key = 0;   // per-(device, instantiation) key
    RG_TRY(per_device(ctx->device, &attr_key, nullptr, [&](int *) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(sketch_w_tc_kernel<R, L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        return RAFTGP_OK;
    }));
    // CTAs (one per SM while resident): ctx->sketch_ctas if set (raftgp_build_embed leaves SMs to the concurrent CSR
    // build), else every SM; RAFTGP_TC_GRID overrides (A/B runs)
    static const int env_grid = [] {
        const char *e = getenv("RAFTGP_TC_GRID");
        return e ? atoi(e) : 0;
    }();
    const int want = env_grid > 0 ? env_grid : (ctx->sketch_ctas > 0 ? ctx->sketch_ctas : ctx->sm_count);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kTM), want)));
    {
        LaunchScope L(ctx, K_SKETCH);
        sketch_w_tc_kernel<R, L1><<<grid, RG_TC_THREADS, smem, ctx->stream>>>(seed, row0, n, sigma, W1, outs);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

template <int R>
raftgp_status dispatch_tc(raftgp_ctx ctx, uint64_t seed, int64_t row0, int64_t n, float sigma, const float *W1, int l1,
                          const SketchOut &outs) {
    switch (l1) {
        case 32: return launch_tc<R, 32>(ctx, seed, row0, n, sigma, W1, outs);
        case 64: return launch_tc<R, 64>(ctx, seed, row0, n, sigma, W1, outs);
        default: return launch_tc<R, 128>(ctx, seed, row0, n, sigma, W1, outs);
    }
}

}  // namespace

raftgp_status sketch_w_tc_rows(raftgp_ctx ctx, uint64_t seed, int64_t row0, int64_t rows, int32_t r, const float *W1,
                               int32_t l1, float *const *outs, int nout) {
    if (rows == 0) return RAFTGP_OK;
    if (nout < 1 || nout > kMaxPush) return fail(RAFTGP_ERR_INTERNAL, "sketch_w_tc_rows: 1..8 outputs");
    SketchOut so{};
    so.nout = nout;
    for (int q = 0; q < nout; ++q) so.out[q] = outs[q];
    const float sigma = spec_sigma(r);
    switch (r) {
        case 32: return dispatch_tc<32>(ctx, seed, row0, rows, sigma, W1, l1, so);
        case 64: return dispatch_tc<64>(ctx, seed, row0, rows, sigma, W1, l1, so);
        default: return dispatch_tc<128>(ctx, seed, row0, rows, sigma, W1, l1, so);
    }
}

raftgp_status sketch_w_tc(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, const float *W1, int32_t l1, float *out) {
    return sketch_w_tc_rows(ctx, seed, 0, n, r, W1, l1, &out, 1);
}

}  // namespace raftgp
