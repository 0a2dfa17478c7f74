// wide.cu — NEXT-2: the paper's Table I layer widths (L up to 4096, GNN 4096 -> 2048 ->
// 1024 -> 512 -> 256). At these widths the per-layer transforms of Eq. 6 (and Theta W^(1) of the feature
// hop, reading #13) are real GEMMs (N x 4096 x 2048), so they run on the tcgen05 tensor cores, fp32-accurate
// by the 3xTF32 split (x = hi + lo, hi = x with the low 13 mantissa bits cleared; A B ~ Ah Bh + Ah Bl + Al Bh,
// fp32 accumulation in TMEM; error ~2^-20 relative, far inside the 1e-4 bar).
//
// Operands live in HBM pre-split and pre-tiled in the canonical no-swizzle K-major layout (tc.cuh): chunk
// (tile, kb) holds rows [128 tile, +128) (A) or output columns [NT tile, +NT) (B) x K columns [32 kb, +32),
// contiguous, so one 1-D bulk copy (TMA engine) moves a whole operand chunk into shared memory with no
// reformatting. Producers of A (the Theta generator, the wide GCN hop) write this layout directly.
//
// GEMM kernel (one CTA per 128 x NT output tile, n-tiles of one m-tile adjacent in the grid so they share A
// through L2): warp 0 lane 0 streams k-blocks through an NS-stage ring (full/empty mbarriers), warp 1 lane 0
// issues 3 x 4 MMAs (M = 128, N = NT, K = 8) per k-block and releases each stage with tcgen05.commit; the four
// warps then read the accumulator back (warp w owns TMEM lanes 32w..32w+31 = tile rows), apply the optional
// row scale (s^ of Eq. 6) and store C row-major.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "gauss.cuh"
#include "internal.cuh"
#include "tc.cuh"

namespace raftgp {

namespace {

using namespace tc;

constexpr int kGM = 128;   // MMA M (rows per output tile)
#ifndef RG_KB
#define RG_KB 32
#endif
#ifndef RG_GEMM_NS
#define RG_GEMM_NS 4
#endif
constexpr int kKB = RG_KB;    // K columns per k-block (one bulk-copied chunk)
constexpr int kGemmThreads = 128;

__host__ __device__ constexpr uint32_t chunk_bytes(int rows) { return (uint32_t)rows * kKB * 4u; }

// ---------------------------------------------------------------- operand tiling (split into hi / lo)
// A operand from a row-major M x K matrix X (leading dimension ldx): rows padded to a multiple of 128, K to
// a multiple of 32, padding zero. Thread per (row, 4-column group).
__global__ void tile_rows_split(const float *__restrict__ X, int64_t M, int K, int64_t ldx, int64_t Mp, int Kp,
                                float *__restrict__ hi, float *__restrict__ lo) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t groups = (int64_t)Kp / 4;
    if (t >= Mp * groups) return;
    const int64_t row = t / groups;
    const int k = (int)(t % groups) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < M) {
        const float *x = X + row * ldx + k;
        v.x = k < K ? x[0] : 0.f;
        v.y = k + 1 < K ? x[1] : 0.f;
        v.z = k + 2 < K ? x[2] : 0.f;
        v.w = k + 3 < K ? x[3] : 0.f;
    }
    const int64_t KBn = Kp / kKB;
    const int64_t chunk = (row / kGM) * KBn + k / kKB;
    const size_t off = (size_t)chunk * chunk_bytes(kGM) + kmajor_off((int)(row % kGM), k % kKB, kGM);
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(hi) + off) = h;
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(lo) + off) =
        make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// B operand from a row-major K x N matrix W: B row n (= output column) is W's column n. Output columns padded
// to a multiple of NT, K to a multiple of 32. Thread per (column n, 4-k group).
__global__ void tile_cols_split(const float *__restrict__ W, int K, int N, int Np, int Kp, int NT,
                                float *__restrict__ hi, float *__restrict__ lo) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t groups = (int64_t)Kp / 4;
    if (t >= (int64_t)Np * groups) return;
    const int n = (int)(t % Np);   // consecutive threads: consecutive columns (coalesced reads of W rows)
    const int k = (int)(t / Np) * 4;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (n < N && k + j < K) ? W[(int64_t)(k + j) * N + n] : 0.f;
    const int KBn = Kp / kKB;
    const int64_t chunk = (int64_t)(n / NT) * KBn + k / kKB;
    const size_t off = (size_t)chunk * chunk_bytes(NT) + kmajor_off(n % NT, k % kKB, NT);
    const float4 h = make_float4(tf32_hi(v[0]), tf32_hi(v[1]), tf32_hi(v[2]), tf32_hi(v[3]));
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(hi) + off) = h;
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(lo) + off) =
        make_float4(v[0] - h.x, v[1] - h.y, v[2] - h.z, v[3] - h.w);
}

// Theta of Eq. 5 (docs/SKETCH_SPEC.md, tag 0, den r) generated straight into the tiled A layout (hi / lo):
// thread per (row, column quad), one Philox call -> 4 normals. Rows >= n are zero.
__global__ void theta_tiles(uint64_t seed, int64_t n, int r, int64_t Mp, float sigma, float *__restrict__ hi,
                            float *__restrict__ lo) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t quads = r / 4;
    if (t >= Mp * quads) return;
    const int64_t row = t % Mp;    // consecutive threads: consecutive rows (16-B stores within a core matrix)
    const int q = (int)(t / Mp);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < n) v = spec_quad(seed, 0u, (uint64_t)row, (uint32_t)q, sigma);
    const int k = 4 * q;
    const int64_t chunk = (row / kGM) * (r / kKB) + k / kKB;
    const size_t off = (size_t)chunk * chunk_bytes(kGM) + kmajor_off((int)(row % kGM), k % kKB, kGM);
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(hi) + off) = h;
    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(lo) + off) =
        make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// ---------------------------------------------------------------- the 3xTF32 GEMM
template <int NT>
struct GemmCfg {
    static constexpr uint32_t A_CH = chunk_bytes(kGM);
    static constexpr uint32_t B_CH = chunk_bytes(NT);
    static constexpr uint32_t STAGE = 2 * A_CH + 2 * B_CH;
    static constexpr int NS = (int)((220u * 1024u) / STAGE) > RG_GEMM_NS ? RG_GEMM_NS : (int)((220u * 1024u) / STAGE);
    static constexpr size_t SMEM = (size_t)NS * STAGE + 1024;   // + alignment slack
    // NACC accumulators in TMEM (512 columns in all), k-block kb accumulating into kb % NACC: the tensor
    // cores' fp32 accumulation error grows with the number of accumulated terms (measured: relative error
    // ~2^-27 K with one accumulator), so the K terms are spread over NACC partial sums added in fp32 at the end
    static constexpr int NACC = 512 / NT;
    static constexpr int NCOL = 512;
    // D f32, A/B tf32, both K-major, N = NT, M = 128
    static constexpr uint32_t IDESC =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);
};

template <int NT>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_tf32x3(const float *__restrict__ Ahi, const float *__restrict__ Alo,
                                                               const float *__restrict__ Bhi, const float *__restrict__ Blo,
                                                               int64_t M, int Kp, int N, int ntn,
                                                               const float *__restrict__ row_scale, float *__restrict__ C,
                                                               int64_t ldc) {
    using G = GemmCfg<NT>;
    extern __shared__ unsigned char gsm_raw[];
    unsigned char *gsm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[G::NS], empty[G::NS], done;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nt = (int)(blockIdx.x % ntn);
    const int64_t mt = blockIdx.x / ntn;
    const int KBn = Kp / kKB;

    if (tid == 0) {
        for (int s = 0; s < G::NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(G::NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;

    const char *a_hi = reinterpret_cast<const char *>(Ahi) + (size_t)mt * KBn * G::A_CH;
    const char *a_lo = reinterpret_cast<const char *>(Alo) + (size_t)mt * KBn * G::A_CH;
    const char *b_hi = reinterpret_cast<const char *>(Bhi) + (size_t)nt * KBn * G::B_CH;
    const char *b_lo = reinterpret_cast<const char *>(Blo) + (size_t)nt * KBn * G::B_CH;

    if (warp == 0 && lane == 0) {
        // producer: k-block kb -> stage kb % NS
        for (int kb = 0; kb < KBn; ++kb) {
            const int s = kb % G::NS;
            if (kb >= G::NS) mbar_wait(&empty[s], ((kb / G::NS) - 1) & 1);
            unsigned char *st = gsm + (size_t)s * G::STAGE;
            mbar_expect_tx(&full[s], G::STAGE);
            bulk_g2s(st, a_hi + (size_t)kb * G::A_CH, G::A_CH, &full[s]);
            bulk_g2s(st + G::A_CH, a_lo + (size_t)kb * G::A_CH, G::A_CH, &full[s]);
            bulk_g2s(st + 2 * G::A_CH, b_hi + (size_t)kb * G::B_CH, G::B_CH, &full[s]);
            bulk_g2s(st + 2 * G::A_CH + G::B_CH, b_lo + (size_t)kb * G::B_CH, G::B_CH, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        // MMA issuer
        constexpr uint32_t A_LBO = (kGM / 8) * 128, B_LBO = (NT / 8) * 128, SBO = 128;
        for (int kb = 0; kb < KBn; ++kb) {
            const int s = kb % G::NS;
            mbar_wait(&full[s], (kb / G::NS) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t st = smem_u32(gsm + (size_t)s * G::STAGE);
            const uint32_t ah = st, al = st + G::A_CH, bh = st + 2 * G::A_CH, bl = bh + G::B_CH;
#pragma unroll
            for (int k8 = 0; k8 < kKB / 8; ++k8) {
                const uint32_t ao = k8 * 2 * A_LBO, bo = k8 * 2 * B_LBO;
                const uint64_t dah = smem_desc(ah + ao, A_LBO, SBO), dal = smem_desc(al + ao, A_LBO, SBO);
                const uint64_t dbh = smem_desc(bh + bo, B_LBO, SBO), dbl = smem_desc(bl + bo, B_LBO, SBO);
                const uint32_t acc = tmem_d + (uint32_t)((kb % G::NACC) * NT);
                mma_tf32(acc, dah, dbh, G::IDESC, (kb >= G::NACC || k8 > 0) ? 1u : 0u);
                mma_tf32(acc, dah, dbl, G::IDESC, 1u);
                mma_tf32(acc, dal, dbh, G::IDESC, 1u);
            }
            mma_commit(&empty[s]);   // stage s is free once these MMAs have read it
        }
        mma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // epilogue: warp w reads TMEM lanes 32w..32w+31 (tile rows), 32 columns at a time
    const int64_t row = mt * kGM + warp * 32 + lane;
    const float sc = (row_scale && row < M) ? row_scale[row] : 1.0f;
    const int nacc = KBn < G::NACC ? KBn : G::NACC;   // accumulators that received at least one k-block
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 32) {
        float v[32];
        tmem_ld32(tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        for (int a = 1; a < nacc; ++a) {
            float w[32];
            tmem_ld32(tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * NT + c0), w);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += w[i];
        }
        const int col0 = nt * NT + c0;
        if (row < M && col0 < N) {
            float *o = C + row * ldc + col0;
            if (col0 + 32 <= N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    reinterpret_cast<float4 *>(o)[i] =
                        make_float4(v[4 * i] * sc, v[4 * i + 1] * sc, v[4 * i + 2] * sc, v[4 * i + 3] * sc);
            } else {
                for (int i = 0; i < 32 && col0 + i < N; ++i) o[i] = v[i] * sc;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(G::NCOL));
}

// ---------------------------------------------------------------- wide hops (rows of 1-8 KB)
// One warp per (row, column slice of CW = 128 V floats): lane l owns float4 columns l, l + 32, ..., l + 32 (V-1)
// of the slice, so every gathered neighbour slice is V fully coalesced 512-B requests; col_idx is read 32
// entries at a time and broadcast by shuffle; U neighbours are in flight per lane (U x V x 16 B). The NW = W /
// CW slices of one row are the NW warps of one CTA; the GCN kind combines their l2-norm partials in shared
// memory. Per-row sum order is fixed (neighbour order, then the per-lane columns are independent), so results
// are deterministic.
enum WideKind : int { W_NCUT = 0, W_MOD = 1, W_MOD_REDUCED = 2, W_DUAL = 3, W_GCN = 4 };

struct WideArgs {
    int64_t n;
    const int64_t *row_ptr;
    const int32_t *col;
    const float *X;          // gathered operand, n x W row-major
    const float *s_all, *sh_all;
    const int32_t *deg_all;
    const double *gvec;      // MOD: g' = d^T X (W doubles)
    double inv2e;
    int W;
    float *out;              // feature kinds: T = s^ (.) y (n x W); GCN: Z row-major (may be null)
    float *out2;             // W_DUAL: the MOD variant's T
    float *zhi, *zlo;        // GCN: Z split and tiled as the next GEMM's A operand (may be null)
    float *ssq;              // GCN, deferred normalisation: per-row, per-slice sums of squares (n x NW) or null
    unsigned long long *ctr; // zeroed row counter: CTAs claim rows dynamically (degree skew), or null (grid-stride)
    const int32_t *order;    // visiting order of the rows (heavy rows spread, order.cu), or null
    const int32_t *hub_thr;  // device int32[1]: gathered rows of degree >= *hub_thr are loaded L2-evict-last, the
                             // others evict-first (the hub rows then stay in L2), or null: plain loads
};

#ifndef RG_WIDE_STCS
#define RG_WIDE_STCS 1
#endif
__device__ __forceinline__ void wst4(float4 *p, const float4 &v, bool hinted) {
    if (RG_WIDE_STCS && hinted) __stcs(p, v);
    else *p = v;
}
__device__ __forceinline__ float4 ldg4_hint(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}

template <int KIND, int V, int U>
__global__ void __launch_bounds__(512) hop_wide(WideArgs a) {
    constexpr int CW = 128 * V;
    // hub rows (degree >= *hub_thr, a byte budget of the widest rows) are loaded evict-last and the rest evict-first,
    // so the often-gathered rows stay in L2 (Table I leg at 2E5: wide hops 50.4 -> 48.4 ms)
    const bool hinted = a.hub_thr != nullptr;
    const int32_t hthr = hinted ? __ldg(a.hub_thr) : 0x7fffffff;
    uint64_t pol_last = 0, pol_first = 0;
    if (hinted) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int NW = a.W / CW;                 // warps (slices) per row
    const int rpc = (int)(blockDim.x >> 5) / NW;   // rows per CTA iteration
    const int rsub = wib / NW, slice = wib % NW;
    __shared__ float ssq[16];
    const float4 *X4 = reinterpret_cast<const float4 *>(a.X);
    const int64_t W4 = a.W / 4;
    const int64_t cbase = (int64_t)slice * (CW / 4);   // first float4 column of this slice
    __shared__ long long claim;
    for (int64_t r0 = (int64_t)blockIdx.x * rpc;; r0 += (int64_t)gridDim.x * rpc) {
        if (a.ctr) {   // dynamic: the CTA's next rpc rows (a hub row no longer delays a statically assigned range)
            if (threadIdx.x == 0) claim = (long long)atomicAdd(a.ctr, (unsigned long long)rpc);
            __syncthreads();
            r0 = claim;
        }
        if (r0 >= a.n) break;
        const int64_t ii = r0 + rsub;
        const bool valid = ii < a.n;
        const int64_t i = (valid && a.order) ? (int64_t)__ldg(a.order + ii) : ii;
        float4 acc[V], acc2[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = acc2[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            const int64_t beg = a.row_ptr[i], end = a.row_ptr[i + 1];
            for (int64_t base = beg; base < end; base += 32) {
                const int cnt = (int)min((int64_t)32, end - base);
                const int32_t myj = lane < cnt ? __ldg(a.col + base + lane) : 0;
                const int myhub = (hinted && lane < cnt) ? (__ldg(a.deg_all + myj) >= hthr) : 0;
                float myw = 0.f;
                if (KIND == W_NCUT || KIND == W_DUAL) myw = lane < cnt ? __ldg(a.s_all + myj) : 0.f;
                if (KIND == W_MOD_REDUCED) myw = lane < cnt ? (float)__ldg(a.deg_all + myj) : 0.f;
                for (int k0 = 0; k0 < cnt; k0 += U) {
                    float4 x[U][V];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int k = k0 + u;
                        const int32_t j = __shfl_sync(0xffffffffu, myj, k & 31);
                        const int hub = __shfl_sync(0xffffffffu, myhub, k & 31);
                        if (hinted) {
                            const uint64_t pol = hub ? pol_last : pol_first;
#pragma unroll
                            for (int v = 0; v < V; ++v)
                                x[u][v] = k < cnt ? ldg4_hint(X4 + (int64_t)j * W4 + cbase + v * 32 + lane, pol)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                        } else {
#pragma unroll
                            for (int v = 0; v < V; ++v)
                                x[u][v] = k < cnt ? __ldg(X4 + (int64_t)j * W4 + cbase + v * 32 + lane)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const float w = __shfl_sync(0xffffffffu, myw, (k0 + u) & 31);
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            if (KIND == W_NCUT) {
                                acc[v].x = fmaf(w, x[u][v].x, acc[v].x); acc[v].y = fmaf(w, x[u][v].y, acc[v].y);
                                acc[v].z = fmaf(w, x[u][v].z, acc[v].z); acc[v].w = fmaf(w, x[u][v].w, acc[v].w);
                            } else {
                                acc[v].x += x[u][v].x; acc[v].y += x[u][v].y; acc[v].z += x[u][v].z; acc[v].w += x[u][v].w;
                                if (KIND == W_DUAL || KIND == W_MOD_REDUCED) {
                                    acc2[v].x = fmaf(w, x[u][v].x, acc2[v].x); acc2[v].y = fmaf(w, x[u][v].y, acc2[v].y);
                                    acc2[v].z = fmaf(w, x[u][v].z, acc2[v].z); acc2[v].w = fmaf(w, x[u][v].w, acc2[v].w);
                                }
                            }
                        }
                    }
                }
            }
        }
        float4 y[V], y2[V];
        if (KIND == W_GCN) {
            float ss = 0.f;
            const float shi = valid ? __ldg(a.sh_all + i) : 0.f;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                float4 self = valid ? __ldg(X4 + i * W4 + cbase + v * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
                acc[v].x += self.x; acc[v].y += self.y; acc[v].z += self.z; acc[v].w += self.w;
                y[v] = make_float4(tanhf(shi * acc[v].x), tanhf(shi * acc[v].y), tanhf(shi * acc[v].z),
                                   tanhf(shi * acc[v].w));
                ss += y[v].x * y[v].x + y[v].y * y[v].y + y[v].z * y[v].z + y[v].w * y[v].w;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            if (a.ssq) {
                // deferred: the row's 1/||y|| is folded into the next GEMM's row scale (no CTA barrier here)
                if (valid && lane == 0) a.ssq[i * NW + slice] = ss;
            } else {
                if (NW > 1) {
                    if (lane == 0) ssq[wib] = ss;
                    __syncthreads();
                    ss = 0.f;
                    for (int q = 0; q < NW; ++q) ss += ssq[rsub * NW + q];
                    __syncthreads();
                }
                if (ss > 0.f) {
                    const float nrm = sqrtf(ss);
#pragma unroll
                    for (int v = 0; v < V; ++v) y[v] = make_float4(y[v].x / nrm, y[v].y / nrm, y[v].z / nrm, y[v].w / nrm);
                }
            }
        } else if (valid) {
            const float shi = __ldg(a.sh_all + i);
            const float si = __ldg(a.s_all + i);
            const double c = (double)__ldg(a.deg_all + i) * a.inv2e;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                float4 t;
                if (KIND == W_NCUT) {
                    t = make_float4(si * acc[v].x, si * acc[v].y, si * acc[v].z, si * acc[v].w);
                } else if (KIND == W_MOD_REDUCED) {
                    t = make_float4((float)(acc[v].x - c * acc2[v].x), (float)(acc[v].y - c * acc2[v].y),
                                    (float)(acc[v].z - c * acc2[v].z), (float)(acc[v].w - c * acc2[v].w));
                } else {   // MOD (and the MOD half of DUAL): sum_j X_j - d_i g' / 2e
                    const int64_t c4 = cbase + v * 32 + lane;
                    const double2 ga = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * c4);
                    const double2 gb = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * c4 + 1);
                    t = make_float4((float)(acc[v].x - c * ga.x), (float)(acc[v].y - c * ga.y),
                                    (float)(acc[v].z - c * gb.x), (float)(acc[v].w - c * gb.y));
                }
                y[v] = make_float4(shi * t.x, shi * t.y, shi * t.z, shi * t.w);
                if (KIND == W_DUAL) {   // same op order as W_NCUT: s^_i (s_i acc)
                    const float4 t2 = make_float4(si * acc2[v].x, si * acc2[v].y, si * acc2[v].z, si * acc2[v].w);
                    y2[v] = make_float4(shi * t2.x, shi * t2.y, shi * t2.z, shi * t2.w);
                }
            }
        }
        if (valid) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int64_t c4 = cbase + v * 32 + lane;
                // outputs are written once and read by a later launch: streamed (evict-first) when the gathers
                // keep hub rows in L2 (RG_WIDE_STCS)
                if (KIND == W_DUAL) {
                    // DUAL: out = NCut's T (acc2 path), out2 = MOD's T
                    if (a.out) wst4(reinterpret_cast<float4 *>(a.out) + i * W4 + c4, y2[v], hinted);
                    if (a.out2) wst4(reinterpret_cast<float4 *>(a.out2) + i * W4 + c4, y[v], hinted);
                } else if (a.out) {
                    wst4(reinterpret_cast<float4 *>(a.out) + i * W4 + c4, y[v], hinted);
                }
                if (KIND == W_GCN && a.zhi) {
                    const int k = (int)(c4 * 4);
                    const int64_t chunk = (i / kGM) * (a.W / kKB) + k / kKB;
                    const size_t off = (size_t)chunk * chunk_bytes(kGM) + kmajor_off((int)(i % kGM), k % kKB, kGM);
                    const float4 h = make_float4(tf32_hi(y[v].x), tf32_hi(y[v].y), tf32_hi(y[v].z), tf32_hi(y[v].w));
                    wst4(reinterpret_cast<float4 *>(reinterpret_cast<char *>(a.zhi) + off), h, hinted);
                    wst4(reinterpret_cast<float4 *>(reinterpret_cast<char *>(a.zlo) + off),
                         make_float4(y[v].x - h.x, y[v].y - h.y, y[v].z - h.z, y[v].w - h.w), hinted);
                }
            }
        }
        if (a.ctr) __syncthreads();   // every warp has read `claim` before thread 0 overwrites it
    }
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, ceil_div(n, t)); }

// Wide hop with the neighbour rows streamed by the TMA engine (W in {512, 1024, 2048}). CTA = 4 consumer
// warps (warp c owns columns [c W/4, (c+1) W/4): V = W/512 float4 per lane) + 1 producer warp. The producer
// walks the CTA's rows (grid-stride) and their neighbours in CSR order (the GCN self row last), reads col_idx
// 32 at a time (coalesced), and for every item bulk-copies the whole W-float row into the next slot of an
// S-slot shared-memory ring (full/empty mbarriers; the item's weight s_j / d_j travels in a slot array). The
// consumers accumulate straight from shared memory. Memory parallelism is the ring depth (S x 4W bytes per
// CTA), not registers: no per-lane load staging at all. Same per-column summation order as hop_wide.
constexpr int kRingThreads = 160;
#ifndef RG_RING_BYTES
#define RG_RING_BYTES (96 * 1024)
#endif

template <int W>
struct RingCfg {
    static constexpr int S = RG_RING_BYTES / (4 * W);   // ring slots (one W-float row each)
    static constexpr int V = W / 512;
    static constexpr size_t SMEM = (size_t)S * W * 4 + 128;
};

template <int KIND, int W>
__global__ void __launch_bounds__(kRingThreads) hop_wide_ring(WideArgs a) {
    using R = RingCfg<W>;
    constexpr int S = R::S, V = R::V;
    extern __shared__ __align__(128) float ring[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ float item_w[S];
    __shared__ float ssq_sh[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const bool gcn = KIND == W_GCN;
    if (warp == 4) {
        // ---------------- producer
        uint32_t it = 0;
        for (int64_t i = blockIdx.x; i < a.n; i += gridDim.x) {
            const int64_t beg = a.row_ptr[i], end = a.row_ptr[i + 1];
            const int64_t total = (end - beg) + (gcn ? 1 : 0);
            for (int64_t base = 0; base < total; base += 32) {
                const int cnt = (int)min((int64_t)32, total - base);
                int32_t myj = 0;
                float myw = 1.f;
                if (lane < cnt) {
                    const int64_t p = beg + base + lane;
                    myj = p < end ? __ldg(a.col + p) : (int32_t)i;   // the GCN self row comes last
                    if (KIND == W_NCUT || KIND == W_DUAL) myw = __ldg(a.s_all + myj);
                    if (KIND == W_MOD_REDUCED) myw = (float)__ldg(a.deg_all + myj);
                }
                for (int k = 0; k < cnt; ++k, ++it) {
                    const int32_t j = __shfl_sync(0xffffffffu, myj, k);
                    const float w = __shfl_sync(0xffffffffu, myw, k);
                    if (lane == 0) {
                        const int q = (int)(it % S);
                        if (it >= (uint32_t)S) mbar_wait(&empty[q], ((it / S) - 1) & 1);
                        item_w[q] = w;
                        mbar_expect_tx(&full[q], W * 4);
                        bulk_g2s(ring + (size_t)q * W, a.X + (int64_t)j * W, W * 4, &full[q]);
                    }
                }
            }
        }
        return;
    }
    // ---------------- consumers: warp c, columns c * W/4 + (v * 32 + lane) * 4
    uint32_t it = 0;
    const int cbase4 = warp * (W / 16);   // first float4 column of this warp's slice
    for (int64_t i = blockIdx.x; i < a.n; i += gridDim.x) {
        const int64_t total = (a.row_ptr[i + 1] - a.row_ptr[i]) + (gcn ? 1 : 0);
        float4 acc[V], acc2[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = acc2[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t k = 0; k < total; ++k, ++it) {
            const int q = (int)(it % S);
            mbar_wait(&full[q], (it / S) & 1);
            const float w = item_w[q];
            const float4 *row = reinterpret_cast<const float4 *>(ring + (size_t)q * W) + cbase4;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const float4 x = row[v * 32 + lane];
                if (KIND == W_NCUT) {
                    acc[v].x = fmaf(w, x.x, acc[v].x); acc[v].y = fmaf(w, x.y, acc[v].y);
                    acc[v].z = fmaf(w, x.z, acc[v].z); acc[v].w = fmaf(w, x.w, acc[v].w);
                } else {
                    acc[v].x += x.x; acc[v].y += x.y; acc[v].z += x.z; acc[v].w += x.w;
                    if (KIND == W_DUAL || KIND == W_MOD_REDUCED) {
                        acc2[v].x = fmaf(w, x.x, acc2[v].x); acc2[v].y = fmaf(w, x.y, acc2[v].y);
                        acc2[v].z = fmaf(w, x.z, acc2[v].z); acc2[v].w = fmaf(w, x.w, acc2[v].w);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q]);
        }
        // epilogue (same arithmetic as hop_wide)
        float4 y[V], y2[V];
        if (KIND == W_GCN) {
            float ss = 0.f;
            const float shi = __ldg(a.sh_all + i);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                y[v] = make_float4(tanhf(shi * acc[v].x), tanhf(shi * acc[v].y), tanhf(shi * acc[v].z),
                                   tanhf(shi * acc[v].w));
                ss += y[v].x * y[v].x + y[v].y * y[v].y + y[v].z * y[v].z + y[v].w * y[v].w;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            if (a.ssq) {
                if (lane == 0) a.ssq[i * 4 + warp] = ss;
            } else {
                if (lane == 0) ssq_sh[warp] = ss;
                asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 consumer warps only
                ss = ssq_sh[0] + ssq_sh[1] + ssq_sh[2] + ssq_sh[3];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (ss > 0.f) {
                    const float nrm = sqrtf(ss);
#pragma unroll
                    for (int v = 0; v < V; ++v) y[v] = make_float4(y[v].x / nrm, y[v].y / nrm, y[v].z / nrm, y[v].w / nrm);
                }
            }
        } else {
            const float shi = __ldg(a.sh_all + i);
            const float si = __ldg(a.s_all + i);
            const double c = (double)__ldg(a.deg_all + i) * a.inv2e;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                float4 t;
                if (KIND == W_NCUT) {
                    t = make_float4(si * acc[v].x, si * acc[v].y, si * acc[v].z, si * acc[v].w);
                } else if (KIND == W_MOD_REDUCED) {
                    t = make_float4((float)(acc[v].x - c * acc2[v].x), (float)(acc[v].y - c * acc2[v].y),
                                    (float)(acc[v].z - c * acc2[v].z), (float)(acc[v].w - c * acc2[v].w));
                } else {
                    const int64_t c4 = cbase4 + v * 32 + lane;
                    const double2 ga = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * c4);
                    const double2 gb = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * c4 + 1);
                    t = make_float4((float)(acc[v].x - c * ga.x), (float)(acc[v].y - c * ga.y),
                                    (float)(acc[v].z - c * gb.x), (float)(acc[v].w - c * gb.y));
                }
                y[v] = make_float4(shi * t.x, shi * t.y, shi * t.z, shi * t.w);
                if (KIND == W_DUAL) {
                    const float4 t2 = make_float4(si * acc2[v].x, si * acc2[v].y, si * acc2[v].z, si * acc2[v].w);
                    y2[v] = make_float4(shi * t2.x, shi * t2.y, shi * t2.z, shi * t2.w);
                }
            }
        }
        const int64_t W4 = W / 4;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int64_t c4 = cbase4 + v * 32 + lane;
            if (KIND == W_DUAL) {
                if (a.out) reinterpret_cast<float4 *>(a.out)[i * W4 + c4] = y2[v];
                if (a.out2) reinterpret_cast<float4 *>(a.out2)[i * W4 + c4] = y[v];
            } else if (a.out) {
                reinterpret_cast<float4 *>(a.out)[i * W4 + c4] = y[v];
            }
            if (KIND == W_GCN && a.zhi) {
                const int kk = (int)(c4 * 4);
                const int64_t chunk = (i / kGM) * (W / kKB) + kk / kKB;
                const size_t off = (size_t)chunk * chunk_bytes(kGM) + kmajor_off((int)(i % kGM), kk % kKB, kGM);
                const float4 h = make_float4(tf32_hi(y[v].x), tf32_hi(y[v].y), tf32_hi(y[v].z), tf32_hi(y[v].w));
                *reinterpret_cast<float4 *>(reinterpret_cast<char *>(a.zhi) + off) = h;
                *reinterpret_cast<float4 *>(reinterpret_cast<char *>(a.zlo) + off) =
                    make_float4(y[v].x - h.x, y[v].y - h.y, y[v].z - h.z, y[v].w - h.w);
            }
        }
    }
}

// Row scale of the GEMM after a deferred-normalisation hop: s^_i / ||y_i|| (y_i = 0 rows keep s^_i).
__global__ void wide_row_scale(const float *__restrict__ ssq, int nw, int64_t n, const float *__restrict__ sh,
                               float *__restrict__ scale) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float ss = 0.f;
    for (int q = 0; q < nw; ++q) ss += ssq[i * nw + q];
    scale[i] = ss > 0.f ? sh[i] / sqrtf(ss) : sh[i];
}

#ifndef RG_WIDE_U   // neighbours in flight per lane; U = 6 / U_DUAL = 4: Table I wide hops 51.3 vs 54.1 ms with 4 / 2
#define RG_WIDE_U 6
#endif
#ifndef RG_WIDE_U_DUAL
#define RG_WIDE_U_DUAL 4
#endif

int wide_ssq_slices(int32_t w);

bool wide_width(int32_t w) { return w == 256 || w == 512 || w == 1024 || w == 2048; }

// The bulk-copy ring is off by default (RAFTGP_WIDE_RING=1 selects it): measured at 2E5 with Table I widths
// it is slower than the register-staged hop_wide (wide hops 85 ms with a 96-KB ring, 120 ms with 192 KB,
// vs 66-69 ms), see DESIGN.md "tried and rejected".
bool wide_ring_enabled() {
    static const bool on = [] {
        const char *e = getenv("RAFTGP_WIDE_RING");
        return e && e[0] == '1';
    }();
    return on;
}

// slices (partial sums of squares) per row written by a deferred-normalisation GCN hop of width w
int wide_ssq_slices(int32_t w) {
    if (wide_ring_enabled() && w >= 512) return 4;
    const char *e = getenv("RAFTGP_WIDE_V");
    const int v = (e && e[0] == '1') ? 1 : (w == 256 ? 2 : 4);
    return w / (128 * v);
}

template <int KIND>
raftgp_status launch_wide(raftgp_ctx ctx, const WideArgs &a) {
    const bool use_ring = wide_ring_enabled();
    if (use_ring && a.W >= 512) {
        auto go = [&](auto wtag) -> raftgp_status {
            constexpr int W = decltype(wtag)::value;
            using R = RingCfg<W>;
            static const char ring_key = 0;
            int per_sm = 1;
            RG_TRY(per_device(ctx->device, &ring_key, &per_sm, [&](int *v) -> raftgp_status {
                RG_CUDA(cudaFuncSetAttribute(hop_wide_ring<KIND, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)R::SMEM));
                RG_CUDA(cudaFuncSetAttribute(hop_wide_ring<KIND, W>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             100));
                int b = 0;
                RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, hop_wide_ring<KIND, W>, kRingThreads,
                                                                      R::SMEM));
                *v = std::max(1, b);
                return RAFTGP_OK;
            }));
            const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.n, (int64_t)ctx->sm_count * per_sm));
            LaunchScope LS(ctx, K_WIDE_HOP);
            hop_wide_ring<KIND, W><<<grid, kRingThreads, R::SMEM, ctx->stream>>>(a);
            return RAFTGP_OK;
        };
        switch (a.W) {
            case 512: return go(std::integral_constant<int, 512>());
            case 1024: return go(std::integral_constant<int, 1024>());
            default: return go(std::integral_constant<int, 2048>());
        }
    }
    // V float4 per lane per slice: 4 = 512-column slices (default; 256-wide rows use V = 2); RAFTGP_WIDE_V=1 =
    // 128-column slices, W/128 warps per row at 64 registers (measured slower at 2E5: 77 vs 69 ms of wide hops)
    static const int Vsel = [] {
        const char *e = getenv("RAFTGP_WIDE_V");
        return (e && e[0] == '1') ? 1 : 4;
    }();
    const int V = a.W == 256 ? (Vsel == 4 ? 2 : 1) : Vsel;
    const int NW = a.W / (128 * V);
    const int warps = std::max(4, NW);
    const int rpc = warps / NW;
    const int64_t per_sm = 2048 / (32 * warps);   // CTAs per SM in the grid (grid-stride over rows)
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.n, rpc), ctx->sm_count * per_sm));
    WideArgs b = a;
    b.ctr = nullptr;
    // hub threshold for this width: the highest-degree rows up to RAFTGP_WIDE_HUB_MB (default 64) MB of operand rows
    static const int64_t hub_mb = [] {
        const char *e = getenv("RAFTGP_WIDE_HUB_MB");
        return e ? (int64_t)std::max(0, atoi(e)) : (int64_t)64;
    }();
    int32_t *thr = nullptr;
    if (hub_mb > 0 && a.deg_all && a.n > 0) {
        RG_TRY(dalloc_t(ctx, &thr, 1));
        RG_TRY(hub_degree_threshold(ctx, a.deg_all, a.n, (hub_mb << 20) / ((int64_t)a.W * 4), thr));
        b.hub_thr = thr;
    }
    static const bool dyn = [] {   // RAFTGP_WIDE_DYN=0: static grid-stride rows
        const char *e = getenv("RAFTGP_WIDE_DYN");
        return !(e && e[0] == '0');
    }();
    if (dyn) {
        RG_TRY(dalloc_t(ctx, &b.ctr, 1));
        RG_TRY(dzero(ctx, b.ctr, sizeof(unsigned long long), ctx->stream));
    }
    {
        LaunchScope LS(ctx, K_WIDE_HOP);
        // neighbours in flight per lane: U x V float4 (DUAL keeps two accumulator sets, so a smaller U)
        constexpr int U4 = KIND == W_DUAL ? RG_WIDE_U_DUAL : RG_WIDE_U;
        if (V == 1) hop_wide<KIND, 1, 2 * U4><<<grid, 32 * warps, 0, ctx->stream>>>(b);
        else if (V == 2) hop_wide<KIND, 2, 2 * U4><<<grid, 32 * warps, 0, ctx->stream>>>(b);
        else hop_wide<KIND, 4, U4><<<grid, 32 * warps, 0, ctx->stream>>>(b);
    }
    dfree(ctx, b.ctr);
    dfree(ctx, thr);
    return RAFTGP_OK;
}

template <int NT>
raftgp_status launch_gemm(raftgp_ctx ctx, const float *Ahi, const float *Alo, const float *Bhi, const float *Blo,
                          int64_t M, int Kp, int N, const float *row_scale, float *C, int64_t ldc) {
    using G = GemmCfg<NT>;
    static const char attr_key = 0;   // per-(device, instantiation) key
    RG_TRY(per_device(ctx->device, &attr_key, nullptr, [&](int *) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(gemm_tf32x3<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
        return RAFTGP_OK;
    }));
    const int ntn = (int)ceil_div(N, NT);
    const int64_t mtn = ceil_div(M, kGM);
    if (M == 0 || N == 0) return RAFTGP_OK;
    {
        LaunchScope LS(ctx, K_GEMM);
        gemm_tf32x3<NT><<<(unsigned)(mtn * ntn), kGemmThreads, G::SMEM, ctx->stream>>>(Ahi, Alo, Bhi, Blo, M, Kp, N, ntn,
                                                                                     row_scale, C, ldc);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

}  // namespace

// N-tile width used for an output of N columns (a power of two in [32, 128]: at least 4 accumulators)
#ifndef RG_GEMM_NT_MAX   // 256-column output tiles: Table I GEMMs 22.3 vs 25.1 ms with 128 (fewer operand bytes per MAC)
#define RG_GEMM_NT_MAX 256
#endif
int gemm_nt(int N) {
    int nt = 32;
    while (nt < N && nt < RG_GEMM_NT_MAX) nt <<= 1;
    return nt;
}

int64_t gemm_pad_rows(int64_t M) { return ceil_div(M, kGM) * kGM; }
int gemm_pad_k(int K) { return (int)ceil_div(K, kKB) * kKB; }

raftgp_status gemm_tile_a(raftgp_ctx ctx, const float *X, int64_t M, int K, int64_t ldx, float *hi, float *lo) {
    const int64_t Mp = gemm_pad_rows(M);
    const int Kp = gemm_pad_k(K);
    if (Mp == 0) return RAFTGP_OK;
    {
        LaunchScope LS(ctx, K_GEMM_TILE);
        tile_rows_split<<<blocks_for(Mp * (Kp / 4), 256), 256, 0, ctx->stream>>>(X, M, K, ldx, Mp, Kp, hi, lo);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

raftgp_status gemm_tile_b(raftgp_ctx ctx, const float *W, int K, int N, float *hi, float *lo) {
    const int NT = gemm_nt(N);
    const int Np = (int)ceil_div(N, NT) * NT;
    const int Kp = gemm_pad_k(K);
    {
        LaunchScope LS(ctx, K_GEMM_TILE);
        tile_cols_split<<<blocks_for((int64_t)Np * (Kp / 4), 256), 256, 0, ctx->stream>>>(W, K, N, Np, Kp, NT, hi, lo);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

raftgp_status gemm_theta_tiles(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, float *hi, float *lo) {
    const int64_t Mp = gemm_pad_rows(n);
    if (Mp == 0) return RAFTGP_OK;
    {
        LaunchScope LS(ctx, K_GEMM_TILE);
        theta_tiles<<<blocks_for(Mp * (r / 4), 256), 256, 0, ctx->stream>>>(seed, n, r, Mp, spec_sigma(r), hi, lo);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

raftgp_status gemm_tiled(raftgp_ctx ctx, const float *Ahi, const float *Alo, const float *Bhi, const float *Blo,
                         int64_t M, int K, int N, const float *row_scale, float *C, int64_t ldc) {
    const int Kp = gemm_pad_k(K);
    switch (gemm_nt(N)) {
        case 32: return launch_gemm<32>(ctx, Ahi, Alo, Bhi, Blo, M, Kp, N, row_scale, C, ldc);
        case 64: return launch_gemm<64>(ctx, Ahi, Alo, Bhi, Blo, M, Kp, N, row_scale, C, ldc);
#if RG_GEMM_NT_MAX >= 256
        case 256: return launch_gemm<256>(ctx, Ahi, Alo, Bhi, Blo, M, Kp, N, row_scale, C, ldc);
#endif
        default: return launch_gemm<128>(ctx, Ahi, Alo, Bhi, Blo, M, Kp, N, row_scale, C, ldc);
    }
}

// C = diag(row_scale) A B for row-major A (M x K), B (K x N): tiles both operands, then the tensor-core GEMM.
raftgp_status gemm_rowmajor(raftgp_ctx ctx, const float *A, int64_t M, int K, const float *B, int N,
                            const float *row_scale, float *C) {
    if (M == 0 || N == 0) return RAFTGP_OK;
    const int64_t Mp = gemm_pad_rows(M);
    const int Kp = gemm_pad_k(K);
    const int NT = gemm_nt(N);
    const int64_t Np = ceil_div(N, NT) * NT;
    float *ah = nullptr, *al = nullptr, *bh = nullptr, *bl = nullptr;
    raftgp_status st = dalloc_t(ctx, &ah, (size_t)Mp * Kp);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &al, (size_t)Mp * Kp);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &bh, (size_t)Np * Kp);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &bl, (size_t)Np * Kp);
    if (st == RAFTGP_OK) st = gemm_tile_a(ctx, A, M, K, K, ah, al);
    if (st == RAFTGP_OK) st = gemm_tile_b(ctx, B, K, N, bh, bl);
    if (st == RAFTGP_OK) st = gemm_tiled(ctx, ah, al, bh, bl, M, K, N, row_scale, C, N);
    dfree(ctx, ah);
    dfree(ctx, al);
    dfree(ctx, bh);
    dfree(ctx, bl);
    return st;
}

bool wide_supported(int32_t layers, const int32_t *dims) {
    bool any_wide = dims[0] > 128;
    if (dims[0] % 32 != 0) return false;
    for (int k = 1; k <= layers; ++k) {
        const int32_t w = dims[k];
        if (!(w == 32 || w == 64 || w == 128 || wide_width(w))) return false;
        any_wide |= w > 128;
    }
    return any_wide;
}

// The whole embedding (feature hop + GCN) for Table I widths, Y not materialised (Theta W^(1) before the
// aggregation, reading #13). Narrow layers (<= 128) reuse spmm.cu's fused hops; a transform next to a wide
// layer is the tensor-core GEMM on the hop's tiled output.
raftgp_status embed_wide(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                         const int32_t *dims, uint64_t seed, float *const *Z_dev, const int where[3]) {
    raftgp_ctx ctx = g->ctx;
    const int64_t n = g->n, Mp = gemm_pad_rows(n);
    const int32_t r = dims[0], l1 = dims[1];
    std::vector<void *> pool;
    auto take = [&](void **p, size_t bytes) -> raftgp_status {
        raftgp_status st = dalloc(ctx, p, bytes);
        if (st == RAFTGP_OK) pool.push_back(*p);
        return st;
    };
    auto release = [&](void *p) {
        for (auto &q : pool)
            if (q == p) q = nullptr;
        dfree(ctx, p);
    };
    auto weights_tiled = [&](uint32_t tag, int32_t fin, int32_t fout, float **bhi, float **blo) -> raftgp_status {
        const int NT = gemm_nt(fout);
        const size_t bn = (size_t)ceil_div(fout, NT) * NT * gemm_pad_k(fin);
        float *w = nullptr;
        RG_TRY(dalloc_t(ctx, &w, (size_t)fin * fout));
        raftgp_status st = sketch_fill(ctx, seed, tag, 0, fin, fout, fin, w);
        if (st == RAFTGP_OK) st = take(reinterpret_cast<void **>(bhi), bn * 4);
        if (st == RAFTGP_OK) st = take(reinterpret_cast<void **>(blo), bn * 4);
        if (st == RAFTGP_OK) st = gemm_tile_b(ctx, w, fin, fout, *bhi, *blo);
        dfree(ctx, w);
        return st;
    };
    raftgp_status st = RAFTGP_OK;
    auto cleanup = [&]() {
        for (auto q : pool)
            if (q) dfree(ctx, q);
    };
    // ---- Theta' = Theta W1 (n x l1) and g' = d^T Theta' for MOD
    float *thw = nullptr;
    double *gw = nullptr;
    st = take(reinterpret_cast<void **>(&thw), (size_t)n * l1 * 4);
    if (st == RAFTGP_OK && sketch_w_supported(r, l1)) {
        float *w1 = nullptr;
        st = take(reinterpret_cast<void **>(&w1), (size_t)r * l1 * 4);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, r, l1, r, w1);
        if (st == RAFTGP_OK) st = sketch_w_any(ctx, seed, n, r, w1, l1, thw);
        release(w1);
    } else if (st == RAFTGP_OK) {
        float *th_hi = nullptr, *th_lo = nullptr, *b_hi = nullptr, *b_lo = nullptr;
        st = take(reinterpret_cast<void **>(&th_hi), (size_t)Mp * r * 4);
        if (st == RAFTGP_OK) st = take(reinterpret_cast<void **>(&th_lo), (size_t)Mp * r * 4);
        if (st == RAFTGP_OK) st = gemm_theta_tiles(ctx, seed, n, r, th_hi, th_lo);
        if (st == RAFTGP_OK) st = weights_tiled(1u, r, l1, &b_hi, &b_lo);
        if (st == RAFTGP_OK) st = gemm_tiled(ctx, th_hi, th_lo, b_hi, b_lo, n, r, l1, nullptr, thw, l1);
        release(th_hi);
        release(th_lo);
        release(b_hi);
        release(b_lo);
    }
    if (st == RAFTGP_OK && (where[RAFTGP_MOD] >= 0)) {
        st = take(reinterpret_cast<void **>(&gw), (size_t)l1 * sizeof(double));
        if (st == RAFTGP_OK) st = g_reduce(g, thw, l1, gw);
    }
    // ---- feature hop: T1 = s^ (.) (X Theta')
    std::vector<float *> T1(nvariants, nullptr);
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) st = take(reinterpret_cast<void **>(&T1[v]), (size_t)n * l1 * 4);
    const bool dual = where[RAFTGP_NCUT] >= 0 && where[RAFTGP_MOD] >= 0;
    if (st == RAFTGP_OK) {
        if (l1 <= 128) {
            if (dual) st = feature_hop_pre(g, -1, l1, thw, gw, T1[where[RAFTGP_NCUT]], T1[where[RAFTGP_MOD]]);
            for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
                if (dual && (variants[v] == RAFTGP_NCUT || variants[v] == RAFTGP_MOD)) continue;
                st = feature_hop_pre(g, variants[v], l1, thw, gw, T1[v], nullptr);
            }
        } else {
            WideArgs a{};
            a.n = n; a.row_ptr = g->row_ptr; a.col = g->col; a.X = thw; a.s_all = g->s_all; a.sh_all = g->sh_all;
            a.deg_all = g->deg_all; a.gvec = gw; a.inv2e = g->two_e > 0 ? 1.0 / (double)g->two_e : 0.0; a.W = l1;
            a.order = g->order;
            if (dual) {
                a.out = T1[where[RAFTGP_NCUT]];
                a.out2 = T1[where[RAFTGP_MOD]];
                st = launch_wide<W_DUAL>(ctx, a);
                if (st == RAFTGP_OK) { RG_CHECK_LAUNCH(ctx); }
            }
            for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
                if (dual && (variants[v] == RAFTGP_NCUT || variants[v] == RAFTGP_MOD)) continue;
                a.out = T1[v];
                a.out2 = nullptr;
                st = variants[v] == RAFTGP_NCUT ? launch_wide<W_NCUT>(ctx, a)
                     : variants[v] == RAFTGP_MOD ? launch_wide<W_MOD>(ctx, a) : launch_wide<W_MOD_REDUCED>(ctx, a);
                if (st == RAFTGP_OK) { RG_CHECK_LAUNCH(ctx); }
            }
        }
    }
    release(thw);
    if (gw) release(gw);
    // ---- GCN layers (Eq. 6 + l2 normalisation), GEMM-first: T_{k+1} = s^ (.) (Z^(k) W^(k+1))
    std::vector<float *> Bhi(layers + 2, nullptr), Blo(layers + 2, nullptr), Wrm(layers + 2, nullptr);
    for (int k = 1; k < layers && st == RAFTGP_OK; ++k) {
        const int32_t w = dims[k], wn = dims[k + 1];
        if (w <= 128 && wn <= 128) {
            st = take(reinterpret_cast<void **>(&Wrm[k + 1]), (size_t)w * wn * 4);
            if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, (uint32_t)(k + 1), 0, w, wn, w, Wrm[k + 1]);
        } else {
            st = weights_tiled((uint32_t)(k + 1), w, wn, &Bhi[k + 1], &Blo[k + 1]);
        }
    }
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
        float *T = T1[v];
        for (int k = 1; k <= layers && st == RAFTGP_OK; ++k) {
            const int32_t w = dims[k];
            const bool last = k == layers;
            const int32_t wn = last ? 0 : dims[k + 1];
            float *Tn = nullptr;
            if (!last) st = take(reinterpret_cast<void **>(&Tn), (size_t)n * wn * 4);
            if (st != RAFTGP_OK) break;
            if (w <= 128 && (last || wn <= 128)) {
                st = gcn_hop(g, T, w, last ? Z_dev[v] : nullptr, last ? nullptr : Wrm[k + 1], wn, Tn);
            } else {
                float *zhi = nullptr, *zlo = nullptr, *rscale = nullptr;
                if (!last) {
                    st = take(reinterpret_cast<void **>(&zhi), (size_t)Mp * w * 4);
                    if (st == RAFTGP_OK) st = take(reinterpret_cast<void **>(&zlo), (size_t)Mp * w * 4);
                }
                if (st == RAFTGP_OK && w <= 128) {
                    // narrow hop, wide next layer: Z^(k) row-major, then tiled for the GEMM
                    float *zr = nullptr;
                    st = take(reinterpret_cast<void **>(&zr), (size_t)n * w * 4);
                    if (st == RAFTGP_OK) st = gcn_hop(g, T, w, zr, nullptr, 0, nullptr);
                    if (st == RAFTGP_OK) st = gemm_tile_a(ctx, zr, n, w, w, zhi, zlo);
                    release(zr);
                } else if (st == RAFTGP_OK) {
                    if (!last && Mp > n) {   // padding rows of the last row tile are zero
                        const size_t tile = (size_t)(w / kKB) * chunk_bytes(kGM);
                        RG_TRY(dzero(ctx, reinterpret_cast<char *>(zhi) + (size_t)(Mp / kGM - 1) * tile, tile));
                        RG_TRY(dzero(ctx, reinterpret_cast<char *>(zlo) + (size_t)(Mp / kGM - 1) * tile, tile));
                    }
                    WideArgs a{};
                    a.n = n; a.row_ptr = g->row_ptr; a.col = g->col; a.X = T; a.s_all = g->s_all; a.sh_all = g->sh_all;
                    a.deg_all = g->deg_all; a.W = w; a.out = last ? Z_dev[v] : nullptr; a.zhi = zhi; a.zlo = zlo;
                    a.order = g->order;
                    const int nw = wide_ssq_slices(w);
                    if (!last) {   // deferred row normalisation: y = tanh(.) tiled, 1/||y|| goes to the GEMM row scale
                        st = take(reinterpret_cast<void **>(&a.ssq), (size_t)n * nw * 4);
                        if (st == RAFTGP_OK) st = take(reinterpret_cast<void **>(&rscale), (size_t)n * 4);
                    }
                    if (st == RAFTGP_OK) st = launch_wide<W_GCN>(ctx, a);
                    if (st == RAFTGP_OK) { RG_CHECK_LAUNCH(ctx); }
                    if (st == RAFTGP_OK && !last) {
                        {
                            LaunchScope LS(ctx, K_WIDE_HOP);
                            wide_row_scale<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a.ssq, nw, n, g->sh_all, rscale);
                        }
                        RG_CHECK_LAUNCH(ctx);
                    }
                    if (a.ssq) release(a.ssq);
                }
                if (st == RAFTGP_OK && !last)
                    st = gemm_tiled(ctx, zhi, zlo, Bhi[k + 1], Blo[k + 1], n, w, wn, rscale ? rscale : g->sh_all, Tn, wn);
                if (rscale) release(rscale);
                if (zhi) release(zhi);
                if (zlo) release(zlo);
            }
            if (T != T1[v]) release(T);
            T = Tn;
        }
        if (T && T != T1[v]) release(T);
    }
    cleanup();
    return st;
}

}  // namespace raftgp
