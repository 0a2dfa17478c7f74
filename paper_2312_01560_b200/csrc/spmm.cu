// spmm.cu — a4/a5 of the hot path: the sparse-times-dense hops with fused epilogues.
//
//   feature hop (Eq. 5):  Y = X Theta, X in {M, Q, Q~}
//   GCN hop     (Eq. 6):  Z'_i = rownorm(tanh(s^_i (T_i + sum_{j in N(i)} T_j))),
//                                           T = s^ (.) (Z W) produced by the previous hop's epilogue
//   transform:                              T = s^ (.) (Z W)   (row GEMM, W in shared memory)
//
// Fast kernel ("hop_kernel"): one warp per row, operand rows gathered with 128-bit loads. A gathered
// row of width W is W/4 lanes wide, so a warp gathers 32/(W/4) neighbours at once and unrolls U such
// steps (U x 16 B in flight per lane); col_idx is read 32 entries at a time, coalesced, and broadcast
// with shuffles. The per-row sum order is fixed (lane sub-slot order, then a fixed xor butterfly), so
// results are deterministic and independent of the grid. After a group of RB rows the warp runs the
// fused epilogue GEMM against W_next held in shared memory (FFMA; Z rows staged per warp in shared
// memory and read as broadcasts). HBM-bound: bytes per edge = 4 (col) + 4W (row), see DESIGN.md.
//
// Generic kernel ("hop_generic"): one block per row, one thread per column, any width / alignment.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "internal.cuh"

namespace raftgp {

namespace {

constexpr unsigned FULL = 0xffffffffu;

#ifndef RG_PREFETCH
#define RG_PREFETCH 0   // 1: load the next row's first col chunk while gathering the current row
#endif

// GCN2: the last GCN hop of two variants at once over an interleaved operand [T_a | T_b] (one 2d-wide
// gather per neighbour instead of two d-wide ones); each half is tanh'd and l2-normalised on its own.
enum Kind : int { KIND_NCUT = 0, KIND_MOD = 1, KIND_MOD_REDUCED = 2, KIND_GCN = 3, KIND_LOAD = 4, KIND_DUAL = 5,
                  KIND_GCN2 = 6, KIND_GCN2H = 7 };
// KIND_GCN2H: KIND_GCN2 restricted to one half of the interleaved operand (HopArgs::half = 1 or 2), a separate
// instantiation so the paired kernel of the one-GPU step carries no half predicate
__host__ __device__ constexpr bool is_pair_kind(int k) { return k == KIND_GCN2 || k == KIND_GCN2H; }

struct HopArgs {
    int64_t nl, rb, n;
    const int64_t *row_ptr;    // local CSR
    const int32_t *order;      // visiting order of the local rows (may be null = natural order)
    const int32_t *col;        // global neighbour ids
    const float *X;            // operand, n x W (global rows); for KIND_LOAD: local rows x W
    const float *s_all;        // deg^-1/2
    const float *sh_all;       // (deg+1)^-1/2
    const int32_t *deg_all;
    const double *gvec;        // MOD: g = d^T Theta (W doubles)
    double inv2e;              // 1 / 2e
    float *out;                // local rows x W (Y or Z'), may be null
    const float *Wn;           // W x WN, may be null
    float *Tn;                 // local rows x WN, may be null
    float *out2;               // KIND_DUAL: second variant's Y (MOD), may be null
    float *Tn2;                // KIND_DUAL: second variant's T
    bool scale_sh;             // multiply the stored rows by s^_i (feature hop on Theta' = Theta W1)
    int32_t tn_ld;             // row stride of Tn in floats (0 = WN)
    unsigned long long *ctr;   // zeroed group counter: warps claim kClaim row groups at a time (degree skew), or
                               // null: static grid-stride
    PushSpec push;             // push.nrep > 0: the T output (out/out2 when WN == 0, Tn/Tn2 when WN > 0) goes to
                               // the replicas at global rows instead of the local buffers
    int claim = 8;             // row groups per dynamic claim (kClaim; 1 for short row lists: every warp gets work)
    const int32_t *colx = nullptr;   // slot layout (relabel.cu): gathered operand rows by slot (colx = slot[col]) ...
    const int32_t *slot = nullptr;   // ... node -> slot (the self term's row; T outputs are written at slots)
    const float *s_slot = nullptr;   // ... s by slot (NCut weights of the gathered rows)
    const int32_t *hubk = nullptr;   // ... number of hub slots: gathers of slots >= *hubk load evict-first
    int half = 0;              // KIND_GCN2H: 1 / 2 only the first / second half of [T_a | T_b] (the other
                               // half's lanes load nothing; each half's arithmetic is unchanged)
};

constexpr int kClaim = 8;      // row groups per dynamic claim

__device__ __forceinline__ float4 ldg4(const float4 *p) { return __ldg(p); }
// read-only load with an L2 eviction-priority policy (createpolicy), for the one-off rows of the slot layout
__device__ __forceinline__ float4 ldg4_pol(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void fma4(float4 &a, float w, const float4 &v) {
    a.x = fmaf(w, v.x, a.x);
    a.y = fmaf(w, v.y, a.y);
    a.z = fmaf(w, v.z, a.z);
    a.w = fmaf(w, v.w, a.w);
}
__device__ __forceinline__ void add4(float4 &a, const float4 &v) {
    a.x += v.x;
    a.y += v.y;
    a.z += v.z;
    a.w += v.w;
}
__device__ __forceinline__ float4 shfl_xor4(const float4 &v, int o) {
    return make_float4(__shfl_xor_sync(FULL, v.x, o), __shfl_xor_sync(FULL, v.y, o), __shfl_xor_sync(FULL, v.z, o),
                       __shfl_xor_sync(FULL, v.w, o));
}

// Gather modes. SUM: acc += X_j. S: acc += s_j X_j. SUM_D: acc += X_j, acc2 += d_j X_j.
// SUM_S: acc += X_j, acc2 += s_j X_j (NCut and full modularity from ONE gather of Theta).
enum Mode : int { M_SUM = 0, M_S = 1, M_SUM_D = 2, M_SUM_S = 3 };

// Gather-sum over the neighbours of one row. Lane layout: sub = lane / LPN picks the neighbour slot,
// cl = lane % LPN the float4 column slice. Returns the full row sums in every sub-slot (xor butterfly).
// `c0` is this row's first 32-entry col chunk, loaded by the caller one row ahead; later chunks are
// prefetched one chunk ahead, so col latency overlaps the row gathers. (L2 eviction-priority hints for
// high-degree rows were measured and made every hop slower; plain read-only loads are used.)
template <int W, int U_REQ, int MODE, bool HALF = false, bool SL = false>
__device__ __forceinline__ void gather_row(const HopArgs &a, int64_t beg, int64_t end, int32_t c0, int lane,
                                           float4 &acc, float4 &acc2, int32_t hk = 0, uint64_t pol = 0) {
    static_assert(!SL || MODE != M_SUM_D, "the slot layout has no by-slot degree vector");
    const int32_t *cg = SL ? a.colx : a.col;   // gathered operand rows: slots or node ids
    const float *sw = SL ? a.s_slot : a.s_all;
    constexpr int LPN = W / 4, NPW = 32 / LPN;
    constexpr int U = (NPW * U_REQ <= 32) ? U_REQ : 32 / NPW;
    static_assert(NPW * U <= 32 && 32 % (NPW * U) == 0, "unroll must tile a 32-entry col chunk");
    const int sub = lane / LPN, cl = lane % LPN;
    const float4 *X4 = reinterpret_cast<const float4 *>(a.X);
    // HALF (KIND_GCN2H): only the lanes of the selected half of the interleaved row load
    const bool act = !HALF || ((cl < LPN / 2) == (a.half == 1));
    acc = make_float4(0.f, 0.f, 0.f, 0.f);
    acc2 = make_float4(0.f, 0.f, 0.f, 0.f);
#if RG_PREFETCH
    int32_t mycur = c0;
#else
    int32_t mycur = (beg + lane < end) ? __ldg(cg + beg + lane) : 0;
    (void)c0;
#endif
    for (int64_t base = beg; base < end; base += 32) {
        const int cnt = (end - base < 32) ? static_cast<int>(end - base) : 32;
        const int64_t nb = base + 32;
        const int32_t mynext = (nb < end && nb + lane < end) ? __ldg(cg + nb + lane) : 0;
        const int32_t myj = mycur;
        float myw = 0.f;
        if (MODE == M_S || MODE == M_SUM_S) myw = lane < cnt ? __ldg(sw + myj) : 0.f;
        if (MODE == M_SUM_D) myw = lane < cnt ? static_cast<float>(__ldg(a.deg_all + myj)) : 0.f;
        for (int k0 = 0; k0 < cnt; k0 += NPW * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + u * NPW + sub;
                const int32_t j = __shfl_sync(FULL, myj, k);
                if constexpr (SL)
                    v[u] = (k < cnt && act) ? (j >= hk ? ldg4_pol(X4 + (int64_t)j * LPN + cl, pol)
                                                       : ldg4(X4 + (int64_t)j * LPN + cl))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                else
                    v[u] = (k < cnt && act) ? ldg4(X4 + (int64_t)j * LPN + cl) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + u * NPW + sub;
                if (MODE == M_S) {
                    fma4(acc, __shfl_sync(FULL, myw, k), v[u]);
                } else {
                    add4(acc, v[u]);
                    if (MODE == M_SUM_D || MODE == M_SUM_S) fma4(acc2, __shfl_sync(FULL, myw, k), v[u]);
                }
            }
        }
        mycur = mynext;
    }
#pragma unroll
    for (int o = LPN; o < 32; o <<= 1) {
        add4(acc, shfl_xor4(acc, o));
        if (MODE == M_SUM_D || MODE == M_SUM_S) add4(acc2, shfl_xor4(acc2, o));
    }
}

#ifndef RG_U_SUM
#define RG_U_SUM 4
#endif
#ifndef RG_U_S
#define RG_U_S 8
#endif
#ifndef RG_U_DUAL
#define RG_U_DUAL 4
#endif
#ifndef RG_U_SUMD
#define RG_U_SUMD 4
#endif
#ifndef RG_WARPS_PER_SM
#define RG_WARPS_PER_SM 32
#endif
#ifndef RG_DUAL_WARPS_PER_SM
#define RG_DUAL_WARPS_PER_SM 32
#endif

template <int KIND>
struct KindTraits {
    static constexpr int NV = KIND == KIND_DUAL ? 2 : 1;   // output rows per input row
    // gather steps in flight per lane (register budget: 64 regs at 32 resident warps per SM)
    static constexpr int U = KIND == KIND_NCUT ? RG_U_S
                             : KIND == KIND_DUAL ? RG_U_DUAL
                             : KIND == KIND_MOD_REDUCED ? RG_U_SUMD : RG_U_SUM;
    // resident warps per SM the kernel is compiled for (sets the register cap)
    static constexpr int WARPS = KIND == KIND_DUAL ? RG_DUAL_WARPS_PER_SM : RG_WARPS_PER_SM;
    [[maybe_unused]] static constexpr int MODE = KIND == KIND_NCUT ? M_S
                                : KIND == KIND_MOD_REDUCED ? M_SUM_D
                                : KIND == KIND_DUAL ? M_SUM_S : M_SUM;
};

// One hop for groups of RB consecutive visiting positions per warp; warps claim kClaim groups at a time from a
// per-launch counter (dynamic, a.ctr) or walk them grid-stride (a.ctr == null).
#ifndef RG_WARPS_SL
#define RG_WARPS_SL 32
#endif
// resident warps per SM a hop kernel is compiled for (the register cap): the slot-layout GCN hops may differ
template <int KIND, bool SL>
__host__ __device__ constexpr int hop_warps() {
    return (SL && (KIND == KIND_GCN || KIND == KIND_GCN2 || KIND == KIND_GCN2H)) ? RG_WARPS_SL : KindTraits<KIND>::WARPS;
}

template <int KIND, int W, int WN, int RB, int U, int THREADS, bool SL = false>
__global__ void __launch_bounds__(THREADS, (hop_warps<KIND, SL>() * 32 / THREADS) > 0 ? hop_warps<KIND, SL>() * 32 / THREADS : 1)
    hop_kernel(HopArgs a) {
    // slot layout: the hub-slot count and the evict-first policy, once per thread
    int32_t hk = 0;
    uint64_t pol = 0;
    if constexpr (SL) {
        hk = __ldg(a.hubk);
        pol = policy_evict_first();
    }
    // operand outputs (the feature hop's T_1, the epilogue's T_next) go to the row's slot; embeddings (Z) keep node
    // order. Each row's slot is loaded one row ahead (with the next row's CSR offsets), so no load waits on it
    constexpr bool FEAT = KIND == KIND_NCUT || KIND == KIND_MOD || KIND == KIND_MOD_REDUCED || KIND == KIND_DUAL;
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    constexpr int LPN = W / 4;
    constexpr int NV = KindTraits<KIND>::NV;
    constexpr int NR = NV * RB;                                     // staged rows per warp
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    float *Wsm = smem;                                              // W x WN
    float *stage = smem + W * WN + wib * NR * W;                    // NR x W
    if constexpr (WN > 0) {
        const float4 *src = reinterpret_cast<const float4 *>(a.Wn);
        float4 *dst = reinterpret_cast<float4 *>(Wsm);
        for (int t = threadIdx.x; t < W * WN / 4; t += blockDim.x) dst[t] = src[t];
        __syncthreads();
    }
    const int sub = lane / LPN, cl = lane % LPN;
    const int64_t ngroups = (a.nl + RB - 1) / RB;
    const int64_t gw = (int64_t)gridDim.x * wpb;
    int64_t grp = (int64_t)blockIdx.x * wpb + wib, glim = 0;
    for (;; grp += a.ctr ? 1 : gw) {
        if (a.ctr && grp >= glim) {   // dynamic: the warp's next kClaim groups
            unsigned long long g0 = 0;
            if (lane == 0) g0 = atomicAdd(a.ctr, (unsigned long long)a.claim);
            grp = (int64_t)__shfl_sync(FULL, g0, 0);
            glim = grp + a.claim;
        }
        if (grp >= ngroups) break;
        const int64_t row0 = grp * RB;
        const int rows_here = (a.nl - row0 < RB) ? static_cast<int>(a.nl - row0) : RB;
        // first col chunk of the group's first row; each row prefetches the next row's first chunk
        int64_t beg = 0, end = 0;
        int32_t c0 = 0, sl_cur = 0, my_sl = 0;
        if constexpr (KIND != KIND_LOAD) {
            const int64_t r = a.order ? static_cast<int64_t>(__ldg(a.order + row0)) : row0;
            beg = a.row_ptr[r];
            end = a.row_ptr[r + 1];
            c0 = (RG_PREFETCH && beg + lane < end) ? __ldg(a.col + beg + lane) : 0;
            if constexpr (SL) sl_cur = __ldg(a.slot + a.rb + r);
        }
        for (int rr = 0; rr < rows_here; ++rr) {
            const int64_t row = a.order ? static_cast<int64_t>(__ldg(a.order + row0 + rr)) : row0 + rr;   // local row
            const int64_t gi = a.rb + row;          // global row id
            const int64_t srow = SL ? (int64_t)sl_cur : gi;   // this row's operand row (self term, T outputs)
            if constexpr (SL) {
                if (lane == rr) my_sl = sl_cur;     // lane rr keeps row rr's slot for the epilogue
            }
            float4 acc, acc2;
            float4 y, y2 = make_float4(0.f, 0.f, 0.f, 0.f);
            if constexpr (KIND == KIND_LOAD) {
                y = ldg4(reinterpret_cast<const float4 *>(a.X) + row * LPN + cl);
            } else {
                int64_t nbeg = end, nend = end;
                int32_t nc0 = 0;
                if (rr + 1 < rows_here) {
                    const int64_t r = a.order ? static_cast<int64_t>(__ldg(a.order + row0 + rr + 1)) : row0 + rr + 1;
                    nbeg = a.row_ptr[r];
                    nend = a.row_ptr[r + 1];
                    if (RG_PREFETCH) nc0 = (nbeg + lane < nend) ? __ldg(a.col + nbeg + lane) : 0;
                    if constexpr (SL) sl_cur = __ldg(a.slot + a.rb + r);
                }
                float4 self = make_float4(0.f, 0.f, 0.f, 0.f);
                if constexpr (KIND == KIND_GCN)
                    self = ldg4(reinterpret_cast<const float4 *>(a.X) + srow * LPN + cl);
                if constexpr (KIND == KIND_GCN2) self = ldg4(reinterpret_cast<const float4 *>(a.X) + srow * LPN + cl);
                if constexpr (KIND == KIND_GCN2H)
                    if ((cl < LPN / 2) == (a.half == 1)) self = ldg4(reinterpret_cast<const float4 *>(a.X) + srow * LPN + cl);
                gather_row<W, U, KindTraits<KIND>::MODE, KIND == KIND_GCN2H, SL>(a, beg, end, c0, lane, acc, acc2, hk, pol);
                beg = nbeg;
                end = nend;
                c0 = nc0;
                if constexpr (KIND == KIND_NCUT) {
                    const float si = __ldg(a.s_all + gi);
                    y = make_float4(si * acc.x, si * acc.y, si * acc.z, si * acc.w);
                } else if constexpr (KIND == KIND_MOD || KIND == KIND_DUAL) {
                    const double c = static_cast<double>(__ldg(a.deg_all + gi)) * a.inv2e;
                    const double2 ga = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * cl);
                    const double2 gb = __ldg(reinterpret_cast<const double2 *>(a.gvec) + 2 * cl + 1);
                    const double g0 = ga.x, g1 = ga.y, g2 = gb.x, g3 = gb.y;
                    const float4 ym = make_float4(static_cast<float>(acc.x - c * g0), static_cast<float>(acc.y - c * g1),
                                                  static_cast<float>(acc.z - c * g2), static_cast<float>(acc.w - c * g3));
                    if constexpr (KIND == KIND_DUAL) {
                        const float si = __ldg(a.s_all + gi);
                        y = make_float4(si * acc2.x, si * acc2.y, si * acc2.z, si * acc2.w);   // NCut
                        y2 = ym;                                                                // modularity
                    } else {
                        y = ym;
                    }
                } else if constexpr (KIND == KIND_MOD_REDUCED) {
                    const double c = static_cast<double>(__ldg(a.deg_all + gi)) * a.inv2e;
                    y = make_float4(static_cast<float>(acc.x - c * acc2.x), static_cast<float>(acc.y - c * acc2.y),
                                    static_cast<float>(acc.z - c * acc2.z), static_cast<float>(acc.w - c * acc2.w));
                } else {   // KIND_GCN(2): H_i = s^_i (T_i + sum_j T_j); tanh; row l2 normalisation
                    add4(acc, self);
                    const float shi = __ldg(a.sh_all + gi);
                    y = make_float4(tanhf(shi * acc.x), tanhf(shi * acc.y), tanhf(shi * acc.z), tanhf(shi * acc.w));
                    float ss = y.x * y.x + y.y * y.y + y.z * y.z + y.w * y.w;
                    constexpr int RL = is_pair_kind(KIND) ? LPN / 2 : LPN;   // lanes of one normalised row
#pragma unroll
                    for (int o = 1; o < RL; o <<= 1) ss += __shfl_xor_sync(FULL, ss, o);
                    if (ss > 0.f) {
                        const float nrm = sqrtf(ss);
                        y = make_float4(y.x / nrm, y.y / nrm, y.z / nrm, y.w / nrm);
                    }
                }
            }
            if constexpr (WN == 0 && KIND != KIND_GCN && !is_pair_kind(KIND) && KIND != KIND_LOAD) {
                if (a.scale_sh) {
                    const float shi = __ldg(a.sh_all + gi);
                    y = make_float4(shi * y.x, shi * y.y, shi * y.z, shi * y.w);
                    y2 = make_float4(shi * y2.x, shi * y2.y, shi * y2.z, shi * y2.w);
                }
            }
            if constexpr (is_pair_kind(KIND)) {
                constexpr int HL = LPN / 2;
                float *o = cl < HL ? a.out : a.out2;
                if (sub == 0 && o != nullptr) reinterpret_cast<float4 *>(o)[row * HL + (cl % HL)] = y;
            } else if (sub == 0) {
                if (WN == 0 && a.push.nrep > 0) {   // fused exchange: this row into every rank's copy of T
                    const int64_t grow = a.push.row0 + row;
                    const int64_t ld4 = a.push.ld > 0 ? a.push.ld / 4 : LPN;
                    // replica loops unrolled over kMaxPush with constant indices: the pointer arrays stay in the
                    // parameter bank (a runtime index made the compiler copy them to local memory and spill)
#pragma unroll
                    for (int r = 0; r < kMaxPush; ++r)
                        if (r < a.push.nrep) reinterpret_cast<float4 *>(a.push.rep[r])[grow * ld4 + cl] = y;
                    if constexpr (NV == 2) {
                        const int n2 = a.push.nrep2 > 0 ? a.push.nrep2 : a.push.nrep;
#pragma unroll
                        for (int r = 0; r < kMaxPush; ++r)
                            if (r < n2) reinterpret_cast<float4 *>(a.push.rep2[r])[grow * ld4 + cl] = y2;
                    }
                } else {
                    const int64_t orow = (SL && FEAT) ? srow : row;   // slot (whole graph) or local row
                    if (a.out != nullptr) reinterpret_cast<float4 *>(a.out)[orow * LPN + cl] = y;
                    if constexpr (NV == 2) {
                        if (a.out2 != nullptr) reinterpret_cast<float4 *>(a.out2)[orow * LPN + cl] = y2;
                    }
                }
                if constexpr (WN > 0) {
                    reinterpret_cast<float4 *>(stage)[rr * LPN + cl] = y;
                    if constexpr (NV == 2) reinterpret_cast<float4 *>(stage)[(RB + rr) * LPN + cl] = y2;
                }
            }
        }
        if constexpr (WN > 0) {
            // fused transform: T_i = s^_i (y_i W_next) for the NR staged rows of this group
            constexpr int OL = WN / 4;        // lanes per output row
            constexpr int RS = 32 / OL;       // rows in parallel
            constexpr int RR = NR / RS;       // rows per lane
            static_assert(RR >= 1 && NR % RS == 0, "staged rows must be a multiple of the parallel row count");
            __syncwarp();
            const int rs = lane / OL, oc = lane % OL;
            const float4 *W4 = reinterpret_cast<const float4 *>(Wsm);
            const float4 *S4 = reinterpret_cast<const float4 *>(stage);
            // rows per lane are processed RC at a time (caps the accumulator registers at 4 x float4)
            constexpr int RC = RR < 4 ? RR : 4;
#pragma unroll 1
            for (int q0 = 0; q0 < RR; q0 += RC) {
                float4 o[RC];
#pragma unroll
                for (int q = 0; q < RC; ++q) o[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
                for (int k = 0; k < W; k += 4) {
                    const float4 w0 = W4[(k + 0) * OL + oc];
                    const float4 w1 = W4[(k + 1) * OL + oc];
                    const float4 w2 = W4[(k + 2) * OL + oc];
                    const float4 w3 = W4[(k + 3) * OL + oc];
#pragma unroll
                    for (int q = 0; q < RC; ++q) {
                        const int rr = rs + (q0 + q) * RS;
                        const float4 z = S4[rr * (W / 4) + k / 4];
                        fma4(o[q], z.x, w0);
                        fma4(o[q], z.y, w1);
                        fma4(o[q], z.z, w2);
                        fma4(o[q], z.w, w3);
                    }
                }
#pragma unroll
                for (int q = 0; q < RC; ++q) {
                    const int rr = rs + (q0 + q) * RS;
                    const int v = rr / RB, r_in = rr % RB;
                    const int32_t tslot = SL ? __shfl_sync(FULL, my_sl, r_in) : 0;   // slot of row r_in
                    if (r_in < rows_here) {
                        const int64_t row = a.order ? static_cast<int64_t>(__ldg(a.order + row0 + r_in)) : row0 + r_in;
                        const float shi = __ldg(a.sh_all + a.rb + row);
                        const float4 t4 = make_float4(shi * o[q].x, shi * o[q].y, shi * o[q].z, shi * o[q].w);
                        if (a.push.nrep > 0) {   // fused exchange (see PushSpec)
                            const int64_t grow = a.push.row0 + row;
                            const int64_t pl4 = a.push.ld > 0 ? a.push.ld / 4 : OL;
                            const int nr = (v == 0 || a.push.nrep2 == 0) ? a.push.nrep : a.push.nrep2;
#pragma unroll
                            for (int r = 0; r < kMaxPush; ++r)
                                if (r < nr)
                                    reinterpret_cast<float4 *>(v == 0 ? a.push.rep[r] : a.push.rep2[r])[grow * pl4 + oc] = t4;
                        } else {
                            float4 *T4 = reinterpret_cast<float4 *>(v == 0 ? a.Tn : a.Tn2);
                            const int64_t ld4 = a.tn_ld > 0 ? a.tn_ld / 4 : OL;
                            T4[(SL ? (int64_t)tslot : row) * ld4 + oc] = t4;
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
    if (a.push.nrep > 1) __threadfence_system();   // the pushed rows are visible to the peers
}

// ---------------------------------------------------------------- generic (any width / alignment)
template <int KIND>
__global__ void __launch_bounds__(128) hop_generic(HopArgs a, int W, int WN) {
    extern __shared__ float gsm[];   // W floats (the finished row) + 32 scratch
    float *rowbuf = gsm;
    float *red = gsm + W;
    for (int64_t t = blockIdx.x; t < a.nl; t += gridDim.x) {
        const int64_t row = a.order ? a.order[t] : t;   // visiting order / row list (streaming), like the fast kernels
        const int64_t gi = a.rb + row;
        float part = 0.f;
        for (int c = threadIdx.x; c < W; c += blockDim.x) {
            float y;
            if (KIND == KIND_LOAD) {
                y = a.X[row * W + c];
            } else {
                const int64_t beg = a.row_ptr[row], end = a.row_ptr[row + 1];
                float acc = 0.f, acc2 = 0.f;
                for (int64_t p = beg; p < end; ++p) {
                    const int32_t j = __ldg(a.col + p);
                    const float v = __ldg(a.X + (int64_t)j * W + c);
                    if (KIND == KIND_NCUT) acc = fmaf(__ldg(a.s_all + j), v, acc);
                    else acc += v;
                    if (KIND == KIND_MOD_REDUCED) acc2 = fmaf(static_cast<float>(__ldg(a.deg_all + j)), v, acc2);
                }
                if (KIND == KIND_NCUT) {
                    y = __ldg(a.s_all + gi) * acc;
                } else if (KIND == KIND_MOD) {
                    const double cc = static_cast<double>(__ldg(a.deg_all + gi)) * a.inv2e;
                    y = static_cast<float>(acc - cc * a.gvec[c]);
                } else if (KIND == KIND_MOD_REDUCED) {
                    const double cc = static_cast<double>(__ldg(a.deg_all + gi)) * a.inv2e;
                    y = static_cast<float>(acc - cc * acc2);
                } else {
                    acc += __ldg(a.X + gi * W + c);
                    y = tanhf(__ldg(a.sh_all + gi) * acc);
                    part += y * y;
                }
            }
            rowbuf[c] = y;
        }
        if (KIND == KIND_GCN) {
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
            __syncthreads();
            float ss = 0.f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ss += red[w];
            __syncthreads();
            if (ss > 0.f) {
                const float nrm = sqrtf(ss);
                for (int c = threadIdx.x; c < W; c += blockDim.x) rowbuf[c] = rowbuf[c] / nrm;
            }
        }
        __syncthreads();
        if (a.out != nullptr)
            for (int c = threadIdx.x; c < W; c += blockDim.x) a.out[row * W + c] = rowbuf[c];
        if (WN > 0) {
            const float shi = __ldg(a.sh_all + gi);
            for (int c = threadIdx.x; c < WN; c += blockDim.x) {
                float acc = 0.f;
                for (int k = 0; k < W; ++k) acc = fmaf(rowbuf[k], __ldg(a.Wn + (int64_t)k * WN + c), acc);
                a.Tn[row * WN + c] = shi * acc;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launch helpers
#ifndef RG_U_SUM_SL
#define RG_U_SUM_SL 8
#endif
template <int KIND, int W, int WN, bool SL>
raftgp_status launch_fast_sl(raftgp_ctx ctx, const HopArgs &a) {
    constexpr int RB = 4;
    // GCN hops on the slot layout: 8 gathers in flight per lane (the L2-resident hub rows leave DRAM latency, not its
    // bandwidth, as the bound: C4 GCN hops 42.4 -> 38.8 ms; in node order U = 8 was slower)
    constexpr bool GCNK = KIND == KIND_GCN || KIND == KIND_GCN2 || KIND == KIND_GCN2H;
    constexpr int U = (SL && GCNK) ? RG_U_SUM_SL : KindTraits<KIND>::U;
    constexpr int THREADS = WN > 0 ? 512 : 256;
    constexpr int WPB = THREADS / 32;
    constexpr int NV = KindTraits<KIND>::NV;
    const size_t smem = sizeof(float) * ((size_t)W * WN + (WN > 0 ? (size_t)WPB * NV * RB * W : 0));
    static const char occ_key = 0;   // per-(device, instantiation) key
    int blocks_per_sm = 1;
    auto kern = hop_kernel<KIND, W, WN, RB, U, THREADS, SL>;
    RG_TRY(per_device(ctx->device, &occ_key, &blocks_per_sm, [&](int *v) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int b = 0;
        RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, THREADS, smem));
        *v = b < 1 ? 1 : b;
        return RAFTGP_OK;
    }));
    const int64_t groups = ceil_div(a.nl, RB);
    const int64_t want = ceil_div(groups, WPB);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count * blocks_per_sm)));
    const int kid = (KIND == KIND_GCN || is_pair_kind(KIND)) ? K_GCN_HOP : (KIND == KIND_LOAD ? K_TRANSFORM : K_FEATURE_HOP);
    HopArgs b = a;
    b.ctr = nullptr;
    static const bool dyn = [] {   // RAFTGP_HOP_DYN=0: static grid-stride groups
        const char *e = getenv("RAFTGP_HOP_DYN");
        return !(e && e[0] == '0');
    }();
    if (dyn && KIND != KIND_LOAD) {
        RG_TRY(dalloc_t(ctx, &b.ctr, 1));
        RG_TRY(dzero(ctx, b.ctr, sizeof(unsigned long long), ctx->stream));
    }
    {
        LaunchScope L(ctx, kid);
        kern<<<grid, THREADS, smem, ctx->stream>>>(b);
    }
    dfree(ctx, b.ctr);
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

// the slot-layout instantiation exists for the kinds of the whole-graph embedding path only
template <int KIND, int W, int WN>
raftgp_status launch_fast(raftgp_ctx ctx, const HopArgs &a) {
    constexpr bool SLOTTABLE = (KIND == KIND_DUAL || KIND == KIND_NCUT || KIND == KIND_MOD || KIND == KIND_GCN ||
                                KIND == KIND_GCN2 || KIND == KIND_GCN2H);
    if constexpr (SLOTTABLE) {
        if (a.colx) {
            if (a.push.nrep > 0) return fail(RAFTGP_ERR_INTERNAL, "hop: slot layout with pushed replicas");
            return launch_fast_sl<KIND, W, WN, true>(ctx, a);
        }
    } else {
        if (a.colx) return fail(RAFTGP_ERR_INTERNAL, "hop: this kind has no slot-layout kernel");
    }
    return launch_fast_sl<KIND, W, WN, false>(ctx, a);
}

template <int KIND, int W>
raftgp_status dispatch_wn(raftgp_ctx ctx, const HopArgs &a, int wn) {
    switch (wn) {
        case 0: return launch_fast<KIND, W, 0>(ctx, a);
        case 32: return launch_fast<KIND, W, 32>(ctx, a);
        case 64: return launch_fast<KIND, W, 64>(ctx, a);
        case 128: return launch_fast<KIND, W, 128>(ctx, a);
        default: return fail(RAFTGP_ERR_INTERNAL, "dispatch_wn: unsupported width");
    }
}

template <int KIND>
raftgp_status dispatch(raftgp_ctx ctx, const HopArgs &a, int w, int wn) {
    const bool fast_w = (w == 32 || w == 64 || w == 128) && (wn == 0 || wn == 32 || wn == 64 || wn == 128);
    const bool al = aligned16(a.X) && (a.out == nullptr || aligned16(a.out)) && (a.Wn == nullptr || aligned16(a.Wn)) &&
                    (a.Tn == nullptr || aligned16(a.Tn));
    if (a.nl == 0) return RAFTGP_OK;
    if (fast_w && al) {
        switch (w) {
            case 32: return dispatch_wn<KIND, 32>(ctx, a, wn);
            case 64: return dispatch_wn<KIND, 64>(ctx, a, wn);
            default: return dispatch_wn<KIND, 128>(ctx, a, wn);
        }
    }
    // the generic kernel implements the plain hop only: the fused exchange, strided T_next and the s^ row scale
    // of the pre-transformed feature hop exist only in the fast kernels (their callers check the fast path first)
    if (a.push.nrep > 0 || a.scale_sh || (a.tn_ld > 0 && a.tn_ld != wn) || a.colx)
        return fail(RAFTGP_ERR_INTERNAL, "hop: push / strided output / s^ scale need the fast kernel");
    const size_t smem = sizeof(float) * ((size_t)w + 32);
    if (smem > 48 * 1024) {
        static const char set_key = 0;   // per-(device, instantiation) key
        RG_TRY(per_device(ctx->device, &set_key, nullptr, [&](int *) -> raftgp_status {
            RG_CUDA(cudaFuncSetAttribute(hop_generic<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            return RAFTGP_OK;
        }));
    }
    const int grid = static_cast<int>(std::min<int64_t>(a.nl, (int64_t)ctx->sm_count * 16));
    {
        LaunchScope L(ctx, K_GENERIC);
        hop_generic<KIND><<<grid, 128, smem, ctx->stream>>>(a, w, wn);
    }
    RG_CHECK_LAUNCH(ctx);
    return RAFTGP_OK;
}

HopArgs base_args(raftgp_graph g, int32_t /*w*/) {
    HopArgs a{};
    a.nl = g->nl;
    a.rb = g->row_begin;
    a.n = g->n;
    a.row_ptr = g->row_ptr;
    a.order = g->order;
    a.col = g->col;
    a.s_all = g->s_all;
    a.sh_all = g->sh_all;
    if (g->slots_active) {   // slot layout of the operands (embed_pre with RAFTGP_RELABEL)
        a.colx = g->colx;
        a.slot = g->slot;
        a.s_slot = g->s_slot;
        a.hubk = g->hubk;
    }
    a.deg_all = g->deg_all;
    a.inv2e = g->two_e > 0 ? 1.0 / static_cast<double>(g->two_e) : 0.0;
    return a;
}

}  // namespace

raftgp_status feature_hop(raftgp_graph g, int variant, int32_t r, const float *theta, const double *gvec, float *Y,
                          const float *W1, int32_t l1, float *T1) {
    HopArgs a = base_args(g, r);
    a.X = theta;
    a.gvec = gvec;
    a.out = Y;
    a.Wn = W1;
    a.Tn = T1;
    const int wn = W1 ? l1 : 0;
    switch (variant) {
        case RAFTGP_NCUT: return dispatch<KIND_NCUT>(g->ctx, a, r, wn);
        case RAFTGP_MOD: return dispatch<KIND_MOD>(g->ctx, a, r, wn);
        default: return dispatch<KIND_MOD_REDUCED>(g->ctx, a, r, wn);
    }
}

raftgp_status feature_hop_dual(raftgp_graph g, int32_t r, const float *theta, const double *gvec, float *Y_ncut,
                               float *Y_mod, const float *W1, int32_t l1, float *T_ncut, float *T_mod) {
    const bool fast = (r == 32 || r == 64 || r == 128) && W1 && (l1 == 32 || l1 == 64 || l1 == 128) &&
                      aligned16(theta) && aligned16(W1) && aligned16(T_ncut) && aligned16(T_mod) &&
                      (!Y_ncut || aligned16(Y_ncut)) && (!Y_mod || aligned16(Y_mod));
    if (!fast) {   // two single-variant hops (same results: per-row arithmetic is identical)
        RG_TRY(feature_hop(g, RAFTGP_NCUT, r, theta, nullptr, Y_ncut, W1, l1, T_ncut));
        return feature_hop(g, RAFTGP_MOD, r, theta, gvec, Y_mod, W1, l1, T_mod);
    }
    if (g->nl == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, r);
    a.X = theta;
    a.gvec = gvec;
    a.out = Y_ncut;
    a.out2 = Y_mod;
    a.Wn = W1;
    a.Tn = T_ncut;
    a.Tn2 = T_mod;
    switch (r) {
        case 32: return dispatch_wn<KIND_DUAL, 32>(g->ctx, a, l1);
        case 64: return dispatch_wn<KIND_DUAL, 64>(g->ctx, a, l1);
        default: return dispatch_wn<KIND_DUAL, 128>(g->ctx, a, l1);
    }
}

raftgp_status feature_hop_pre(raftgp_graph g, int variant_or_dual, int32_t l1, const float *theta_w,
                              const double *gvec_w, float *T_a, float *T_b, const PushSpec *push) {
    if (g->nl == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, l1);
    a.X = theta_w;
    a.gvec = gvec_w;
    a.out = T_a;
    a.out2 = T_b;
    a.scale_sh = true;
    if (push) a.push = *push;
    bool al = aligned16(theta_w) && (push || aligned16(T_a)) && (push || !T_b || aligned16(T_b));
    for (int r = 0; push && r < push->nrep; ++r) al = al && aligned16(push->rep[r]) && (!T_b || aligned16(push->rep2[r]));
    if (!((l1 == 32 || l1 == 64 || l1 == 128) && al))
        return fail(RAFTGP_ERR_INTERNAL, "feature_hop_pre: unsupported width/alignment");
    auto go = [&](auto kind_tag) -> raftgp_status {
        constexpr int K = decltype(kind_tag)::value;
        switch (l1) {
            case 32: return launch_fast<K, 32, 0>(g->ctx, a);
            case 64: return launch_fast<K, 64, 0>(g->ctx, a);
            default: return launch_fast<K, 128, 0>(g->ctx, a);
        }
    };
    switch (variant_or_dual) {
        case RAFTGP_NCUT: return go(std::integral_constant<int, KIND_NCUT>());
        case RAFTGP_MOD: return go(std::integral_constant<int, KIND_MOD>());
        case RAFTGP_MOD_REDUCED: return go(std::integral_constant<int, KIND_MOD_REDUCED>());
        default: return go(std::integral_constant<int, KIND_DUAL>());
    }
}

// Row-list variants (NEXT-4 streaming): the same kernels over `count` local rows listed in `rows` (the
// kernels' visiting-order hook; every row's arithmetic is unchanged, so the rows come out bit-identical).
// Short lists (the changed rows' 1- and 2-hop closures, biased to hubs) are claimed one group at a time so every
// warp gets rows: with 8-group claims a 1,000-row list kept ~34 warps busy, each summing ~32 long rows in turn.
static int row_list_claim(raftgp_ctx ctx, int64_t count) {
    return count < (int64_t)ctx->sm_count * 64 * 4 * 8 ? 1 : kClaim;
}

raftgp_status feature_hop_pre_rows(raftgp_graph g, int variant, int32_t l1, const float *theta_w, const double *gvec_w,
                                   float *T, const int32_t *rows, int64_t count) {
    if (count == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, l1);
    a.nl = count;
    a.order = rows;
    a.claim = row_list_claim(g->ctx, count);
    a.X = theta_w;
    a.gvec = gvec_w;
    a.out = T;
    a.scale_sh = true;
    if (!((l1 == 32 || l1 == 64 || l1 == 128) && aligned16(theta_w) && aligned16(T)))
        return fail(RAFTGP_ERR_INTERNAL, "feature_hop_pre_rows: unsupported width/alignment");
    auto go = [&](auto kind_tag) -> raftgp_status {
        constexpr int K = decltype(kind_tag)::value;
        switch (l1) {
            case 32: return launch_fast<K, 32, 0>(g->ctx, a);
            case 64: return launch_fast<K, 64, 0>(g->ctx, a);
            default: return launch_fast<K, 128, 0>(g->ctx, a);
        }
    };
    switch (variant) {
        case RAFTGP_NCUT: return go(std::integral_constant<int, KIND_NCUT>());
        case RAFTGP_MOD: return go(std::integral_constant<int, KIND_MOD>());
        default: return go(std::integral_constant<int, KIND_MOD_REDUCED>());
    }
}

raftgp_status gcn_hop_rows(raftgp_graph g, const float *Tfull, int32_t w, float *Zout, const float *Wn, int32_t wn,
                           float *Tnext, const int32_t *rows, int64_t count) {
    if (count == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, w);
    a.nl = count;
    a.order = rows;
    a.claim = row_list_claim(g->ctx, count);
    a.X = Tfull;
    a.out = Zout;
    a.Wn = Wn;
    a.Tn = Tnext;
    if (!((w == 32 || w == 64 || w == 128) && (wn == 0 || wn == 32 || wn == 64 || wn == 128) && aligned16(Tfull) &&
          (!Zout || aligned16(Zout)) && (!Wn || aligned16(Wn)) && (!Tnext || aligned16(Tnext))))
        return fail(RAFTGP_ERR_INTERNAL, "gcn_hop_rows: unsupported width/alignment");
    return dispatch<KIND_GCN>(g->ctx, a, w, Wn ? wn : 0);
}

raftgp_status gcn_transform_rows(raftgp_graph g, const float *Z, int32_t lin, const float *W, int32_t lout, float *T,
                                 const int32_t *rows, int64_t count) {
    if (count == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, lin);
    a.nl = count;
    a.order = rows;
    a.X = Z;
    a.out = nullptr;
    a.Wn = W;
    a.Tn = T;
    if (!((lin == 32 || lin == 64 || lin == 128) && (lout == 32 || lout == 64 || lout == 128) && aligned16(Z) &&
          aligned16(W) && aligned16(T)))
        return fail(RAFTGP_ERR_INTERNAL, "gcn_transform_rows: unsupported width/alignment");
    return dispatch<KIND_LOAD>(g->ctx, a, lin, lout);
}

raftgp_status gcn_transform(raftgp_graph g, const float *Z, int32_t lin, const float *W, int32_t lout, float *T) {
    HopArgs a = base_args(g, lin);
    a.X = Z;
    a.out = nullptr;
    a.Wn = W;
    a.Tn = T;
    return dispatch<KIND_LOAD>(g->ctx, a, lin, lout);
}

bool push_fusable(int32_t w, int32_t wn) {
    return (w == 32 || w == 64 || w == 128) && (wn == 0 || wn == 32 || wn == 64 || wn == 128);
}

raftgp_status gcn_hop(raftgp_graph g, const float *Tfull, int32_t w, float *Zout, const float *Wn, int32_t wn,
                      float *Tnext, int32_t tn_ld, const PushSpec *push) {
    HopArgs a = base_args(g, w);
    a.X = Tfull;
    a.out = Zout;
    a.Wn = Wn;
    a.Tn = Tnext;
    a.tn_ld = tn_ld;
    if (push) {
        bool al = aligned16(Tfull) && aligned16(Wn) && (!Zout || aligned16(Zout));
        for (int r = 0; r < push->nrep; ++r) al = al && aligned16(push->rep[r]);
        if (!(Wn && push_fusable(w, wn) && al)) return fail(RAFTGP_ERR_INTERNAL, "gcn_hop: push needs the fast kernel");
        a.push = *push;
        a.Tn = push->rep[0];   // non-null for the dispatcher's alignment checks; the kernel writes the replicas
    }
    if (tn_ld > 0 && tn_ld != wn && !((w == 32 || w == 64 || w == 128) && (wn == 32 || wn == 64 || wn == 128) &&
                                      aligned16(Tfull) && aligned16(Tnext) && aligned16(Wn) && tn_ld % 4 == 0))
        return fail(RAFTGP_ERR_INTERNAL, "gcn_hop: strided T_next needs the fast kernel");
    return dispatch<KIND_GCN>(g->ctx, a, w, Wn ? wn : 0);
}

bool gcn_pair_supported(int32_t d) { return d == 32 || d == 64; }

raftgp_status gcn_final_pair(raftgp_graph g, const float *Tboth, int32_t d, float *Za, float *Zb, int half) {
    if (g->nl == 0) return RAFTGP_OK;
    HopArgs a = base_args(g, 2 * d);
    a.X = Tboth;
    a.out = half == 2 ? nullptr : Za;
    a.out2 = half == 1 ? nullptr : Zb;
    a.half = half;
    if (!(gcn_pair_supported(d) && aligned16(Tboth) && aligned16(Za) && aligned16(Zb)))
        return fail(RAFTGP_ERR_INTERNAL, "gcn_final_pair: unsupported width/alignment");
    if (half != 0)
        return d == 32 ? launch_fast<KIND_GCN2H, 64, 0>(g->ctx, a) : launch_fast<KIND_GCN2H, 128, 0>(g->ctx, a);
    return d == 32 ? launch_fast<KIND_GCN2, 64, 0>(g->ctx, a) : launch_fast<KIND_GCN2, 128, 0>(g->ctx, a);
}

}  // namespace raftgp
