// tc_sketch.cu — Theta' = Theta W1 on the 5th-generation tensor cores (tcgen05, TMEM), fp32-accurate.
//
// The one real dense contraction of the path (N x r by r x L1, r, L1 <= 128; Eq. 5 followed
// by the first GEMM of Eq. 6, applied before aggregation — DESIGN.md reading #13). Theta is generated in
// shared memory (docs/SKETCH_SPEC.md) and never written to HBM; W1 stays in shared memory for the whole
// kernel. fp32 accuracy from TF32 tensor cores by the 3-product split x = hi + lo (hi = x with the low 13
// mantissa bits cleared, lo = x - hi exactly): A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi, accumulated in fp32
// in TMEM (error ~2^-20 relative, far inside the 1e-4 parity bar).
//
// Per CTA (512 threads, one per SM): a persistent loop over 128-row tiles, each split into K-quarters of at most
// 32 columns. Every thread generates two Philox quads (8 normals) per quarter and stores their hi / lo tf32 parts in
// the canonical no-swizzle K-major layout (8-row x 16-byte core matrices) into a ring of NS quarter stages; one
// thread issues tcgen05.mma (M = 128, N = L1, K = 8) x 3 products per K-step into one of two TMEM accumulators as
// soon as a stage is complete; four warps drain the previous tile's accumulator with tcgen05.ld, one 32-column chunk
// per quarter of the next tile, and store its rows of Theta'. The warps meet only at the ring's mbarriers (see the kernel). Every mbarrier wait is bounded (trap on
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
#define RG_TC_THREADS 512   // 16 warps, 2 independent Philox quads per thread per quarter (1024 / 256: 2.37 / 2.33 ms vs 2.21 at C4)
#endif
#ifndef RG_TC_MMA_WARP
#define RG_TC_MMA_WARP 1   // 1: a 17th warp only issues the MMAs (0: warp 0's lane 0 issues them between its own quarters)
#endif
constexpr int kTcBlock = RG_TC_THREADS + (RG_TC_MMA_WARP ? 32 : 0);
constexpr int kTM = 128;       // rows per tile (MMA M)
constexpr int kKQ = 32;        // K columns per quarter (one of two A buffers)
#ifndef RG_TC_DRAIN_SPREAD
#define RG_TC_DRAIN_SPREAD 1
#endif
#ifndef RG_TC_NO_STORE
#define RG_TC_NO_STORE 0   // timing experiments only: the drain skips its stores (Theta' is NOT written)
#endif

// Global rows row0 .. row0 + n - 1 of Theta' (Theta's generator row = the global row); each finished row is stored at
// its global row into every one of the nout output copies (nout > 1: the row-partitioned path pushes its share of
// Theta' into every rank's copy over NVLink, dist.cu).
struct SketchOut {
    float *out[kMaxPush];
    int nout;
    const int32_t *slot;   // slot layout (relabel.cu): row i stored at slot[i]; null = row order
};

template <int R, int L1>
struct TcCfg {
    static constexpr int KQ = R < kKQ ? R : kKQ;                 // K columns per quarter (one A stage)
    static constexpr int NQK = R / KQ;                            // quarters per tile
    static constexpr int NCOL = L1 < 32 ? 32 : L1;                // TMEM columns of one accumulator
    static constexpr uint32_t A_BYTES = kTM * KQ * 4;             // one of hi / lo of one stage
    static constexpr uint32_t B_BYTES = L1 * R * 4;
    // A ring depth: as many stages as fit next to W1 (hi + lo), at most 4
    static constexpr int NS0 = (int)((224u * 1024u - 2u * B_BYTES) / (2u * A_BYTES));
    static constexpr int NS = NS0 > 4 ? 4 : NS0;
    static constexpr size_t SMEM = 2 * (size_t)B_BYTES + (size_t)NS * 2 * A_BYTES;
    static_assert(NS >= 2, "A ring needs two stages");
};

// Warp roles inside one CTA (RG_TC_THREADS = 512, 16 warps; QPT = 2 quads per thread per quarter):
//   every warp generates: QPT Philox calls -> 4 QPT normals per thread per quarter (128 rows x KQ columns = 1024 quads),
//     stored as hi / lo K-chunks into the quarter's ring stage, then the warp arrives on full[stage];
//   warp 0, lane 0 also issues the MMAs of each quarter as soon as full[stage] completes (all NW warps' stores are
//     in), and commits them to empty[stage] (the stage may be rewritten) and, after a tile's last quarter, to
//     accf[acc];
//   the last 4 warps (lane quarters 0..3 of TMEM) also drain the previous tile's accumulator into Theta', one
//     32-column chunk after each quarter they generate (wait accf before the first, tcgen05.ld, store; arrive on
//     acce[acc] after the last).
// No block-wide barrier inside the loop: the warps only meet at the ring's mbarriers, so generation is never held
// up by the MMA issue or the drain (the round-1 version's per-quarter __syncthreads was its largest stall).
template <int R, int L1>
__global__ void __launch_bounds__(kTcBlock, 1) sketch_w_tc_kernel(uint64_t seed, int64_t row0, int64_t n, float sigma,
                                                             const float *__restrict__ W1, SketchOut outs) {
    using C = TcCfg<R, L1>;
    constexpr int KQ = C::KQ, NQK = C::NQK, NCOL = C::NCOL, NS = C::NS;
    constexpr uint32_t A_BYTES = C::A_BYTES, B_BYTES = C::B_BYTES;
    constexpr int NW = RG_TC_THREADS / 32;
    constexpr int EPI0 = NW - 4;                          // first drain warp (its index is 0 mod 4)
    constexpr int QPT = kTM * (KQ / 4) / RG_TC_THREADS;   // Philox quads per thread per quarter (independent chains)
    static_assert(NW % 4 == 0 && QPT >= 1 && QPT * RG_TC_THREADS == kTM * (KQ / 4), "whole quads per thread per quarter");
    // instruction descriptor: D f32, A/B tf32, both K-major, N = L1, M = 128
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(L1 >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);

    extern __shared__ __align__(1024) unsigned char tsm[];
    unsigned char *b_hi = tsm;
    unsigned char *b_lo = b_hi + B_BYTES;
    unsigned char *a_base = b_lo + B_BYTES;             // NS stages, each hi | lo
    __shared__ __align__(8) uint64_t full[NS], empty[NS], accf[2], acce[2];
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
        for (int q = 0; q < NS; ++q) {
            mbar_init(&full[q], NW);
            mbar_init(&empty[q], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&accf[a], 1);
            mbar_init(&acce[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {   // two accumulators: tile t accumulates into t & 1 while tile t - 1 is drained
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base_sh)), "r"(2 * NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;

    // drain the accumulator of local tile `it` (global tile index `tile`) into Theta' (drain warps only)
    // drain of local tile `it` (global tile index `tile`) into Theta', spread over the next tile's quarters: at quarter
    // q the drain warps store the 32-column chunks [q CPQ, (q + 1) CPQ) (RG_TC_DRAIN_SPREAD=0: all chunks at q = 0),
    // so they never fall a whole accumulator behind the generating warps (the ring waits for every warp's arrival)
    constexpr int NCH = L1 / 32 > 0 ? L1 / 32 : 1;                 // 32-column chunks of one accumulator
    constexpr int CPQ = RG_TC_DRAIN_SPREAD ? (NCH + NQK - 1) / NQK : NCH;
    auto drain = [&](int64_t it, int64_t tile, int q) {
        const int acc = (int)(it & 1);
        const int k0 = q * CPQ, k1 = min(NCH, k0 + CPQ);
        if (k0 >= k1) return;
        if (k0 == 0) {
            mbar_wait(&accf[acc], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const int lq = warp & 3;
        const int64_t row = tile * kTM + lq * 32 + lane;
#pragma unroll 1
        for (int kc = k0; kc < k1; ++kc) {
            const int c0 = kc * 32;
            float v[32];
            tmem_ld32(tmem_d + (static_cast<uint32_t>(lq * 32) << 16) + (uint32_t)(acc * NCOL + c0), v);
            if (row < n && c0 < L1 && !RG_TC_NO_STORE) {
                for (int o = 0; o < outs.nout; ++o) {
                    const int64_t orow = outs.slot ? (int64_t)__ldg(outs.slot + row0 + row) : row0 + row;
                    float4 *dst = reinterpret_cast<float4 *>(outs.out[o] + orow * L1 + c0);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (c0 + 4 * i < L1) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
        }
        if (k1 == NCH) {   // the accumulator is free for tile it + 2
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[acc]);
        }
    };

    // the MMAs of quarter q of local tile it (ring stage st, quarter counter g): one thread
    auto issue = [&](int64_t it, int q, int64_t g, int st) {
        const int acc = (int)(it & 1);
        unsigned char *a_hi = a_base + (size_t)st * 2 * A_BYTES;
        unsigned char *a_lo = a_hi + A_BYTES;
        if (q == 0 && it >= 2) mbar_wait(&acce[acc], (uint32_t)(((it - 2) >> 1) & 1));   // drained
        mbar_wait(&full[st], (uint32_t)((g / NS) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
        const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
        constexpr uint32_t A_LBO = (kTM / 8) * 128, B_LBO = (L1 / 8) * 128, SBO = 128;
        const uint32_t dacc = tmem_d + (uint32_t)(acc * NCOL);
#pragma unroll
        for (int s8 = 0; s8 < KQ / 8; ++s8) {
            const uint32_t aoff = s8 * 2 * A_LBO;
            const uint32_t boff = (q * (KQ / 8) + s8) * 2 * B_LBO;
            const uint64_t dah = smem_desc(ah + aoff, A_LBO, SBO), dal = smem_desc(al + aoff, A_LBO, SBO);
            const uint64_t dbh = smem_desc(bh + boff, B_LBO, SBO), dbl = smem_desc(bl + boff, B_LBO, SBO);
            const uint32_t acc0 = (q > 0 || s8 > 0) ? 1u : 0u;
            mma_tf32(dacc, dah, dbh, IDESC, acc0);
            mma_tf32(dacc, dah, dbl, IDESC, 1u);
            mma_tf32(dacc, dal, dbh, IDESC, 1u);
        }
        mma_commit(&empty[st]);
        if (q == NQK - 1) mma_commit(&accf[acc]);
    };

    const int64_t ntiles = (n + kTM - 1) / kTM;
    if (RG_TC_MMA_WARP && warp == NW) {   // the MMA warp: issue every quarter as soon as its stage is complete
        if (lane == 0) {
            int64_t itm = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++itm)
                for (int q = 0; q < NQK; ++q) {
                    const int64_t g = itm * NQK + q;
                    issue(itm, q, g, (int)(g % NS));
                }
        }
        __syncwarp();
    }
    const PhiloxKeys keys = philox_keys(seed);
    int64_t it = 0;
    for (int64_t tile = (RG_TC_MMA_WARP && warp == NW) ? ntiles : blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t r0 = tile * kTM;
        const int acc = (int)(it & 1);
        for (int q = 0; q < NQK; ++q) {
            const int64_t g = it * NQK + q;                    // this CTA's quarter counter
            const int st = (int)(g % NS);
            unsigned char *a_hi = a_base + (size_t)st * 2 * A_BYTES;
            unsigned char *a_lo = a_hi + A_BYTES;
            if (g >= NS) mbar_wait(&empty[st], (uint32_t)(((g / NS) - 1) & 1));   // its previous MMAs retired
#pragma unroll
            for (int j = 0; j < QPT; ++j) {   // Theta[r0 .. r0+127][q*KQ .. q*KQ+KQ-1]: quad t -> row t % 128, column quad t / 128
                const int t = tid + j * RG_TC_THREADS;
                const int row = t % kTM, qq = t / kTM;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r0 + row < n)
                    v = spec_quad(keys, 0u, static_cast<uint64_t>(row0 + r0 + row),
                                  static_cast<uint32_t>(q * (KQ / 4) + qq), sigma);
                const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                const float4 lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
                const uint32_t o = kmajor_off(row, 4 * qq, kTM);
                *reinterpret_cast<float4 *>(a_hi + o) = hi;
                *reinterpret_cast<float4 *>(a_lo + o) = lo;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic stores -> async proxy (MMA)
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[st]);
            if (!RG_TC_MMA_WARP && warp == 0) {
                if (lane == 0) issue(it, q, g, st);
                __syncwarp();
            }
            if (warp >= EPI0 && warp < NW && it >= 1) drain(it - 1, tile - gridDim.x, q);
        }
    }
    if (warp >= EPI0 && warp < NW && it >= 1)
        for (int q = 0; q < NQK; ++q) drain(it - 1, (int64_t)blockIdx.x + (it - 1) * gridDim.x, q);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(2 * NCOL));
    if (outs.nout > 1) __threadfence_system();   // rows stored into the peers' copies are visible to them
}

template <int R, int L1>
raftgp_status launch_tc(raftgp_ctx ctx, uint64_t seed, int64_t row0, int64_t n, float sigma, const float *W1,
                        const SketchOut &outs) {
    const size_t smem = TcCfg<R, L1>::SMEM;
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
        sketch_w_tc_kernel<R, L1><<<grid, kTcBlock, smem, ctx->stream>>>(seed, row0, n, sigma, W1, outs);
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
                               int32_t l1, float *const *outs, int nout, const int32_t *slot) {
    if (rows == 0) return RAFTGP_OK;
    if (nout < 1 || nout > kMaxPush) return fail(RAFTGP_ERR_INTERNAL, "sketch_w_tc_rows: 1..8 outputs");
    SketchOut so{};
    so.nout = nout;
    so.slot = slot;
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
