// select.cu — NEXT-1: Alg. 1 hierarchical model selection (§III-C) on the GPU.
//
// The recursion of Alg. 1 is run level by level: every set U of one tree level ("segment") is processed
// by the same launches, so one pass over Z serves all of them. Per level:
//   seeding   (SELECT_SPEC §3.1)  mean pass -> farthest from the mean -> farthest from that point
//   Lloyd     (SELECT_SPEC §3.2)  one fused assign + fixed-point centroid-sum pass per iteration, then a
//                                 per-segment update (segments converge independently)
//   split test (SELECT_SPEC §4)   one pass over the CSR rows of the level: |U_r|, mbar_r, cut; exact
//                                 128-bit integer test  2e * cut > mbar_1 * mbar_2
//   split     stopped segments become blocks; kept ones are stably partitioned into their two children
// Labels are finally made canonical (blocks numbered by their smallest member, SELECT_SPEC §5).
//
// Determinism: every quantity that decides an integer is bit-identical to the oracle's:
//   - centroid sums are exact int64 sums of q(z) = rn(z * 2^32) (order-independent), the centre is
//     (double(S) * 2^-32) / double(count) with explicit round-to-nearest intrinsics;
//   - squared distances are summed sequentially over l with __dsub_rn/__dmul_rn/__dadd_rn (no FMA);
//   - argmax ties go to the smallest node id (max of the distance bits, then min id);
//   - the split test is exact integer arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "internal.cuh"

namespace raftgp {
namespace {

constexpr int kIterChunk = 12;   // Lloyd iterations enqueued per host check

__device__ __forceinline__ long long fixq(float z) { return __double2ll_rn(__dmul_rn((double)z, 4294967296.0)); }

__device__ __forceinline__ double centre(long long S, unsigned long long cnt) {
    return __ddiv_rn(__dmul_rn(__ll2double_rn(S), 0x1p-32), __ull2double_rn(cnt));
}

// SELECT_SPEC §2 squared distance of a row (global memory, float4-aligned) to mu (fp64)
template <int L>
__device__ __forceinline__ double sqdist_smem(const float *row, const double *mu) {
    double d = 0.0;
#pragma unroll 4
    for (int k = 0; k < L / 4; ++k) {
        const float4 v = reinterpret_cast<const float4 *>(row)[k];
        const double2 m01 = __ldg(reinterpret_cast<const double2 *>(mu + 4 * k));
        const double2 m23 = __ldg(reinterpret_cast<const double2 *>(mu + 4 * k + 2));
        double t;
        t = __dsub_rn((double)v.x, m01.x); d = __dadd_rn(d, __dmul_rn(t, t));
        t = __dsub_rn((double)v.y, m01.y); d = __dadd_rn(d, __dmul_rn(t, t));
        t = __dsub_rn((double)v.z, m23.x); d = __dadd_rn(d, __dmul_rn(t, t));
        t = __dsub_rn((double)v.w, m23.y); d = __dadd_rn(d, __dmul_rn(t, t));
    }
    return d;
}

// Both squared distances of one row to the two centres mu[0..L), mu[L..2L): each element is converted once
// and feeds the two sequential sums (the op sequence of each sum is exactly SELECT_SPEC §2's). Global rows
// are loaded in chunks of up to 64 floats with every load issued before the arithmetic (one memory latency
// per chunk instead of one per float4).
template <int L, bool GLOBAL>
__device__ __forceinline__ void sqdist2(const float *row, const double *mu, double &d0, double &d1) {
    d0 = 0.0;
    d1 = 0.0;
    constexpr int CH = L / 4 < 16 ? L / 4 : 16;   // float4 per chunk
#pragma unroll
    for (int c = 0; c < L / 4; c += CH) {
        float4 v[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k)
            v[k] = GLOBAL ? __ldg(reinterpret_cast<const float4 *>(row) + c + k)
                          : reinterpret_cast<const float4 *>(row)[c + k];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const double *m = mu + 4 * (c + k);
            const double2 a01 = __ldg(reinterpret_cast<const double2 *>(m));
            const double2 a23 = __ldg(reinterpret_cast<const double2 *>(m + 2));
            const double2 b01 = __ldg(reinterpret_cast<const double2 *>(m + L));
            const double2 b23 = __ldg(reinterpret_cast<const double2 *>(m + L + 2));
            const double x0 = (double)v[k].x, x1 = (double)v[k].y, x2 = (double)v[k].z, x3 = (double)v[k].w;
            double t;
            t = __dsub_rn(x0, a01.x); d0 = __dadd_rn(d0, __dmul_rn(t, t));
            t = __dsub_rn(x0, b01.x); d1 = __dadd_rn(d1, __dmul_rn(t, t));
            t = __dsub_rn(x1, a01.y); d0 = __dadd_rn(d0, __dmul_rn(t, t));
            t = __dsub_rn(x1, b01.y); d1 = __dadd_rn(d1, __dmul_rn(t, t));
            t = __dsub_rn(x2, a23.x); d0 = __dadd_rn(d0, __dmul_rn(t, t));
            t = __dsub_rn(x2, b23.x); d1 = __dadd_rn(d1, __dmul_rn(t, t));
            t = __dsub_rn(x3, a23.y); d0 = __dadd_rn(d0, __dmul_rn(t, t));
            t = __dsub_rn(x3, b23.y); d1 = __dadd_rn(d1, __dmul_rn(t, t));
        }
    }
}

// Per-segment state of one level (S segments; all device arrays).
struct SegState {
    unsigned long long *acc;   // [S][2][L] fixed-point sums (two's complement int64)
    unsigned long long *cnt;   // [S][2]
    double *mu;                // [S][2][L] centres (slot 0 also holds the mean / first seed)
    unsigned long long *dmax;  // [S] bits of the max distance (d >= 0, so the bit order is the value order)
    int32_t *amin;             // [S] smallest node id attaining dmax
    int32_t *changed;          // [S]
    int32_t *done;             // [S]
    float *delta;              // [S][2] upper bounds of the last centre moves (pruning, see bound_up)
};

// Exact-pruning bounds (Hamerly's algorithm for K = 2, made exact): per row an upper bound u on the TRUE
// Euclidean distance to its own centre and a lower bound l on the distance to the other centre, kept as
// floats with directed rounding and a 2^-40 relative slack over the fp64 distances (whose rounding error is
// < L * 2^-53). After the centres move by at most delta (rounded up), u += delta_own and l -= delta_other.
// A row with u (1 + 2^-20) < l provably keeps its side: the true distances are ordered with a gap of at
// least 2^-20 relative, far above the fp64 error of the spec's sequential squared distances, so the plain
// recomputation (and the oracle) would take the same decision. Only rows that fail the test are read and
// recomputed, and the centroid sums are updated incrementally (exact integers) for the rows that switched.
__device__ __forceinline__ float bound_up(double d2) {
    return __double2float_ru(__dmul_ru(__dsqrt_ru(d2), 1.0 + 0x1p-40));
}
__device__ __forceinline__ float bound_dn(double d2) {
    return __double2float_rd(__dmul_rd(__dsqrt_rd(d2), 1.0 - 0x1p-40));
}

// ---------------------------------------------------------------- row staging by bulk copy (TMA engine)
// Every row a pass needs is brought into shared memory by cp.async.bulk (one 4L-byte copy per row, issued by
// the lane that owns the row, completion counted on a per-warp mbarrier). The rows never pass through
// registers or the L1 data pipe on their way in; lanes then read their own row (distances, a lane per row,
// conflict-free float4 loads thanks to the 16-byte row padding) or one row across the warp (column sums).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init1(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_row(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    for (uint32_t it = 0; it < (1u << 28); ++it) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
        if (done) return;
    }
    __trap();   // a copy never landed: fail loudly instead of hanging
}

// generic-proxy reads of a stage buffer are ordered before the next bulk copy into it
__device__ __forceinline__ void stage_release() {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

constexpr int kRowWarps = 4;    // warps per CTA of sel_rows (two 32-row stages each)
constexpr int kRowRange = 256;  // positions per warp of sel_rows

template <int L>
struct RowAcc {   // per-lane column sums (lane owns columns lane + 32 k) for two sides, run-aggregated
    static constexpr int CPL = (L + 31) / 32;
    long long a0[CPL], a1[CPL];
    long long c0 = 0, c1 = 0;
    int cur = -1;
    __device__ RowAcc() {
#pragma unroll
        for (int k = 0; k < CPL; ++k) a0[k] = a1[k] = 0;
    }
    __device__ __forceinline__ void flush(const SegState &st, int lane) {
        if (cur >= 0) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int col = lane + 32 * k;
                if (col < L) {
                    if (a0[k]) atomicAdd(&st.acc[((size_t)cur * 2 + 0) * L + col], (unsigned long long)a0[k]);
                    if (a1[k]) atomicAdd(&st.acc[((size_t)cur * 2 + 1) * L + col], (unsigned long long)a1[k]);
                }
                a0[k] = a1[k] = 0;
            }
            if (lane == 0) {
                if (c0) atomicAdd(&st.cnt[cur * 2 + 0], (unsigned long long)c0);
                if (c1) atomicAdd(&st.cnt[cur * 2 + 1], (unsigned long long)c1);
            }
        }
        c0 = c1 = 0;
    }
    // add (w = +1) or move (w = 0: side 0 -> 1 when dir > 0, side 1 -> 0 when dir < 0) one row's fixed-point
    // values; s, dir are warp-uniform, the row is in shared memory
    __device__ __forceinline__ void add(const SegState &st, int lane, int s, const float *row, int side, int dir) {
        if (s != cur) {
            flush(st, lane);
            cur = s;
        }
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int col = lane + 32 * k;
            if (col < L) {
                const long long q = fixq(row[col]);
                if (dir == 0) {
                    if (side) a1[k] += q;
                    else a0[k] += q;
                } else if (dir > 0) {
                    a0[k] -= q;
                    a1[k] += q;
                } else {
                    a0[k] += q;
                    a1[k] -= q;
                }
            }
        }
        if (dir == 0) {
            if (side) ++c1;
            else ++c0;
        } else {
            c0 -= dir;
            c1 += dir;
        }
    }
};

// A pass over every row of the level (the positions are contiguous per segment). Each warp streams
// kRowRange positions through two 32-row shared-memory stages (bulk copies of batch k+1 in flight while
// batch k is processed).
//   MODE 0: mean pass (level 1 only; deeper levels inherit their totals from the parent's final sums):
//           every row added to slot 0 (|z| <= 1 checked).
//   MODE 1: Lloyd iteration t = 1: d(z, mu_0) is the one the second seeding pass stored (mu_0 = z_a, same
//           op sequence), so only d(z, mu_1) is computed; bounds initialised; only side-1 rows are summed
//           (slot 1) and sel_update turns the slot-0 total into the side-0 sum (exact integers).
//   MODE 2: seeding: distance to mu[s][0] per row (dpos) and the per-segment maximum (SELECT_SPEC §3.1).
template <int L, int MODE>
__global__ void __launch_bounds__(kRowWarps * 32) sel_rows(const float *__restrict__ Z, const int32_t *__restrict__ perm,
                                                           const int32_t *__restrict__ pseg, int32_t *__restrict__ side,
                                                           float2 *bnd, double *dpos,   // the same buffer (aliased)
                                                           int64_t n_act, SegState st, int32_t *err,
                                                           unsigned long long *rows_read) {
    constexpr int LD = L + 4;
    constexpr uint32_t RB = 4u * L;
    extern __shared__ __align__(16) float sel_smem[];
    __shared__ uint64_t bars[kRowWarps][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *stage = sel_smem + (size_t)warp * 2 * 32 * LD;
    uint64_t *bar = bars[warp];
    const int64_t beg = ((int64_t)blockIdx.x * kRowWarps + warp) * kRowRange;
    if (beg >= n_act) return;
    const int64_t end = min(beg + (int64_t)kRowRange, n_act);
    if (lane == 0) {
        mbar_init1(&bar[0]);
        mbar_init1(&bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    RowAcc<L> acc;
    bool bad = false;
    int sb[2] = {-1, -1};
    uint32_t ph = 0;   // bit k: phase of bar[k]

    auto issue = [&](int64_t b, int buf) {
        const int rows = (int)min((int64_t)32, end - b);
        int s = -1;
        if (lane == 0) mbar_expect(&bar[buf], (uint32_t)rows * RB);
        __syncwarp();
        if (lane < rows) {
            s = pseg[b + lane];
            bulk_row(stage + ((size_t)buf * 32 + lane) * LD, Z + (size_t)(b + lane) * L, RB, &bar[buf]);   // Z in position order
        }
        sb[buf] = s;
    };

    issue(beg, 0);
    int buf = 0;
    for (int64_t b = beg; b < end; b += 32, buf ^= 1) {
        if (b + 32 < end) issue(b + 32, buf ^ 1);
        mbar_wait(&bar[buf], (ph >> buf) & 1u);
        ph ^= 1u << buf;
        const int64_t pos = b + lane;
        const int s = sb[buf];
        const float *srow = stage + (size_t)buf * 32 * LD;
        const float *row = srow + lane * LD;
        int add = 0;
        constexpr int sd = MODE == 1 ? 1 : 0;   // slot the pass sums into (warp-uniform)
        if (s >= 0) {
            if (MODE == 0) {
#pragma unroll 4
                for (int k = 0; k < L / 4; ++k) {
                    const float4 v = reinterpret_cast<const float4 *>(row)[k];
                    bad |= !(fabsf(v.x) <= 1.f && fabsf(v.y) <= 1.f && fabsf(v.z) <= 1.f && fabsf(v.w) <= 1.f);
                }
                add = 1;
            } else if (MODE == 1) {
                const double d0 = dpos[pos];
                const double d1 = sqdist_smem<L>(row, st.mu + ((size_t)s * 2 + 1) * L);
                const int c = d1 < d0 ? 1 : 0;
                bnd[pos] = c ? make_float2(bound_up(d1), bound_dn(d0)) : make_float2(bound_up(d0), bound_dn(d1));
                side[pos] = c;
                add = c;
            }
        }
        if (MODE == 2) {
            double d = 0.0;
            if (s >= 0) {
                d = sqdist_smem<L>(row, st.mu + (size_t)s * 2 * L);
                dpos[pos] = d;
            }
            const int s0 = __shfl_sync(0xffffffffu, s, 0);
            if (__all_sync(0xffffffffu, s == s0) && s0 >= 0) {
                double m = d;
#pragma unroll
                for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                if (lane == 0) atomicMax(&st.dmax[s0], (unsigned long long)__double_as_longlong(m));
            } else if (s >= 0) {
                atomicMax(&st.dmax[s], (unsigned long long)__double_as_longlong(d));
            }
        } else {
            // column sums over the staged rows, in position order (segments are contiguous runs)
            for (unsigned m = __ballot_sync(0xffffffffu, add != 0); m; m &= m - 1) {
                const int r = __ffs(m) - 1;
                acc.add(st, lane, __shfl_sync(0xffffffffu, s, r), srow + r * LD, sd, 0);
            }
        }
        stage_release();
    }
    if (MODE != 2) acc.flush(st, lane);
    if (MODE == 0 && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(err, 1);
    if (MODE == 1 && lane == 0) atomicAdd(&rows_read[blockIdx.x & 63], (unsigned long long)(end - beg));
}

// Lloyd iteration t > 1 with exact pruning. Warps claim kLloydChunk consecutive positions at a time from a
// per-iteration counter (one resident wave of CTAs; the rows failing the bound test cluster, so a static split
// left warps idle behind the busiest range): the bound test
// runs on every position (segment, side and bounds only: 24 B per row); positions that fail it are queued in
// shared memory and recomputed 32 at a time with all lanes busy (a lane per row, rows bulk-copied into a
// shared-memory stage). Rows that switch side then move their fixed-point values between the two sums
// (exact integers), run-aggregated per segment.
constexpr int kPruneWarps = 8;
constexpr int kLloydChunk = 1024;   // positions per dynamic claim (a multiple of 128)

template <int L>
__global__ void __launch_bounds__(kPruneWarps * 32, 3) sel_lloyd_pruned(const float *__restrict__ Z,
                                                                      const int32_t *__restrict__ perm,
                                                                      const int32_t *__restrict__ pseg,
                                                                      int32_t *__restrict__ side,
                                                                      float2 *__restrict__ bnd, int64_t n_act,
                                                                      SegState st, unsigned long long *rows_read,
                                                                      const unsigned long long *__restrict__ prev_active,
                                                                      unsigned long long *__restrict__ claim) {
    constexpr int LD = L + 4;
    constexpr uint32_t RB = 4u * L;
    extern __shared__ __align__(16) float sel_smem[];
    __shared__ int qbuf[kPruneWarps][160];
    __shared__ uint64_t bars[kPruneWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *stage = sel_smem + (size_t)warp * 32 * LD;
    uint64_t *bar = &bars[warp];
    int *q = qbuf[warp];
    if (prev_active[0] == 0) return;   // every segment already converged
    const unsigned lt = (1u << lane) - 1u;
    if (lane == 0) {
        mbar_init1(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    RowAcc<L> acc;
    int qn = 0;
    uint32_t ph = 0;
    unsigned nread = 0;

    // recompute the first k queued positions (k <= 32), lane j takes q[j]
    auto round = [&](int k) {
        nread += k;
        int s = -1;
        int64_t pos = 0;
        if (lane == 0) mbar_expect(bar, (uint32_t)k * RB);
        __syncwarp();
        if (lane < k) {
            pos = q[lane];
            s = pseg[pos];
            bulk_row(stage + lane * LD, Z + (size_t)pos * L, RB, bar);   // Z in position order
        }
        mbar_wait(bar, ph);
        ph ^= 1u;
        int w0 = 0;
        if (lane < k) {
            double d0, d1;
            sqdist2<L, false>(stage + lane * LD, st.mu + (size_t)s * 2 * L, d0, d1);
            const int c = d1 < d0 ? 1 : 0;
            bnd[pos] = c ? make_float2(bound_up(d1), bound_dn(d0)) : make_float2(bound_up(d0), bound_dn(d1));
            if (side[pos] != c) {
                side[pos] = c;
                st.changed[s] = 1;
                w0 = c ? -1 : 1;   // moved 0 -> 1: (-1, +1); moved 1 -> 0: (+1, -1)
            }
        }
        for (unsigned m = __ballot_sync(0xffffffffu, w0 != 0); m; m &= m - 1) {
            const int r = __ffs(m) - 1;
            acc.add(st, lane, __shfl_sync(0xffffffffu, s, r), stage + r * LD, 0, -__shfl_sync(0xffffffffu, w0, r));
        }
        stage_release();
    };

    for (;;) {
        // the warp's next kLloydChunk positions (dynamic: the rows that fail the bound test are not uniform)
        unsigned long long c0 = 0;
        if (lane == 0) c0 = atomicAdd(claim, (unsigned long long)kLloydChunk);
        const int64_t beg = (int64_t)__shfl_sync(0xffffffffu, c0, 0);
        if (beg >= n_act) break;
        const int64_t end = min(beg + (int64_t)kLloydChunk, n_act);
    for (int64_t b = beg; b < end; b += 128) {
        // bound test of 128 positions: lane owns b + 32 j + lane, all loads issued up front
        int sj[4], cj[4];
        float2 ulj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t pos = b + 32 * j + lane;
            sj[j] = pos < end ? pseg[pos] : -1;
            cj[j] = pos < end ? side[pos] : 0;
            ulj[j] = pos < end ? bnd[pos] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t pos = b + 32 * j + lane;
            bool need = false;
            const int s = sj[j];
            if (s >= 0 && !st.done[s]) {
                const int c = cj[j];
                const float2 dl = reinterpret_cast<const float2 *>(st.delta)[s];
                const float u = __fadd_ru(ulj[j].x, c ? dl.y : dl.x);
                const float l = fmaxf(0.f, __fsub_rd(ulj[j].y, c ? dl.x : dl.y));
                if (__fmul_ru(u, 1.0f + 0x1p-20f) < l) bnd[pos] = make_float2(u, l);
                else need = true;
            }
            const unsigned m = __ballot_sync(0xffffffffu, need);
            if (need) q[qn + __popc(m & lt)] = (int)pos;
            qn += __popc(m);
        }
        __syncwarp();
        while (qn >= 32) {
            round(32);
            const int rest = qn - 32;
            int v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = lane + 32 * i < rest ? q[32 + lane + 32 * i] : 0;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < rest) q[lane + 32 * i] = v[i];
            qn = rest;
            __syncwarp();
        }
    }
    }
    if (qn > 0) round(qn);
    acc.flush(st, lane);
    if (lane == 0 && nread) atomicAdd(&rows_read[blockIdx.x & 63], (unsigned long long)nread);
}

// Warp per segment: the mean of U from the slot-0 totals (mean pass at level 1, inherited from the parent's
// final side sums below it); slot 0 keeps the totals, slot 1 and the argmax / Lloyd state are reset.
template <int L>
__global__ void sel_mean(SegState st, int S) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (s >= S) return;
    const unsigned long long n = st.cnt[s * 2];
    for (int l = lane; l < L; l += 32) {
        const size_t i = (size_t)s * 2 * L + l;
        st.mu[i] = n ? centre((long long)st.acc[i], n) : 0.0;
        st.acc[i + L] = 0;
    }
    if (lane == 0) {
        st.cnt[s * 2 + 1] = 0;
        st.dmax[s] = 0;
        st.amin[s] = INT_MAX;
        st.changed[s] = 0;
        st.done[s] = 0;
    }
}

__global__ void sel_argmin(const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg, int64_t n_act,
                           const double *__restrict__ dpos, SegState st) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n_act) return;
    const int s = pseg[pos];
    if ((unsigned long long)__double_as_longlong(dpos[pos]) == st.dmax[s]) atomicMin(&st.amin[s], perm[pos]);
}

// Warp per segment: mu[s][slot] = double(z_amin); reset the argmax state.
template <int L>
__global__ void sel_seed(const float *__restrict__ Z, SegState st, int S, int slot) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (s >= S) return;
    const int a = st.amin[s];
    for (int l = lane; l < L; l += 32) st.mu[((size_t)s * 2 + slot) * L + l] = (double)Z[(size_t)a * L + l];
    __syncwarp();
    if (lane == 0) {
        st.dmax[s] = 0;
        st.amin[s] = INT_MAX;
    }
}

// Warp per segment after Lloyd iteration t (SELECT_SPEC §3.2): converged segments are frozen; the others
// get their new centres (an empty side keeps its centre), an upper bound on how far each centre moved
// (for the pruning bounds), and count as active. The sums and counts are absolute (never reset): MODE 2
// passes update them incrementally.
template <int L>
__global__ void sel_update(SegState st, int S, int t, int max_iter, const int32_t *__restrict__ seg_off,
                           const unsigned long long *__restrict__ prev_active, unsigned long long *active) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (prev_active && prev_active[0] == 0) return;   // every segment converged at an earlier iteration
    if (s >= S || st.done[s]) return;
    if (t == 1) {   // slot 0 held the total over U; the t = 1 pass summed side 1 only
        for (int l = lane; l < L; l += 32) {
            const size_t i0 = (size_t)s * 2 * L + l;
            st.acc[i0] -= st.acc[i0 + L];
        }
        if (lane == 0) st.cnt[s * 2] -= st.cnt[s * 2 + 1];
        __syncwarp();
    }
    if ((t > 1 && st.changed[s] == 0) || t >= max_iter) {
        if (lane == 0) {
            st.done[s] = 1;
            if (t >= max_iter && (t == 1 || st.changed[s] != 0)) {   // stopped by the cap, not converged: counted
                atomicAdd(active, 1ull);                                 // into iteration max_iter's counters
                atomicAdd(active + 1, (unsigned long long)(seg_off[s + 1] - seg_off[s]));
            }
        }
        return;
    }
    const unsigned long long n0 = st.cnt[s * 2], n1 = st.cnt[s * 2 + 1];
    double m0 = 0.0, m1 = 0.0;
    for (int l = lane; l < L; l += 32) {
        const size_t i0 = (size_t)s * 2 * L + l, i1 = i0 + L;
        if (n0) {
            const double v = centre((long long)st.acc[i0], n0), dv = v - st.mu[i0];
            m0 += dv * dv;
            st.mu[i0] = v;
        }
        if (n1) {
            const double v = centre((long long)st.acc[i1], n1), dv = v - st.mu[i1];
            m1 += dv * dv;
            st.mu[i1] = v;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        m0 += __shfl_xor_sync(0xffffffffu, m0, o);
        m1 += __shfl_xor_sync(0xffffffffu, m1, o);
    }
    if (lane == 0) {
        // generous slack (2^-30 relative + an absolute floor) over the rounding of this fp64 sum
        st.delta[2 * s] = __double2float_ru(__dmul_ru(__dsqrt_ru(m0), 1.0 + 0x1p-30) + 0x1p-60);
        st.delta[2 * s + 1] = __double2float_ru(__dmul_ru(__dsqrt_ru(m1), 1.0 + 0x1p-30) + 0x1p-60);
        st.changed[s] = 0;
        atomicAdd(active, 1ull);                                                     // active segments
        atomicAdd(active + 1, (unsigned long long)(seg_off[s + 1] - seg_off[s]));   // and their rows
    }
}

// node_key[node] = 2 * segment + side for every position of the level.
__global__ void sel_mark(const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                         const int32_t *__restrict__ side, int64_t n_act, int32_t *__restrict__ node_key) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < n_act) node_key[perm[pos]] = 2 * pseg[pos] + side[pos];
}

// Split-test statistics (SELECT_SPEC §4): per segment and side |U_r| and mbar_r; cut = edges from U_1
// (side 0) rows into U_2 (side 1), counted once from the U_1 end. A warp takes 32 consecutive positions, a
// lane per row: rows of degree <= kLaneDeg are scanned by their own lane (32 rows' neighbour loads in flight
// at once), longer rows by the whole warp (coalesced). Per-warp sums are reduced in registers and flushed
// with one atomic per (segment, quantity) when the 32 rows share a segment, per lane otherwise.
constexpr int kLaneDeg = 96;

__global__ void __launch_bounds__(256) sel_edges(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                                 const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                                                 const int32_t *__restrict__ side, int64_t n_act,
                                                 const int32_t *__restrict__ node_key,
                                                 unsigned long long *__restrict__ nsz,
                                                 unsigned long long *__restrict__ mbar,
                                                 unsigned long long *__restrict__ cut) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = pos < n_act;
    int s = -1, c = 0;
    int64_t rb = 0, re = 0;
    if (valid) {
        s = pseg[pos];
        c = side[pos];
        const int i = perm[pos];
        rb = row_ptr[i];
        re = row_ptr[i + 1];
    }
    const int64_t deg = re - rb;
    const int want = 2 * s + 1;
    unsigned cnt = 0;
    const bool scan = valid && c == 0;
    if (scan && deg <= kLaneDeg) {
        int64_t p = rb;
        for (; p + 4 <= re; p += 4) {
            const int j0 = __ldg(col + p), j1 = __ldg(col + p + 1), j2 = __ldg(col + p + 2), j3 = __ldg(col + p + 3);
            cnt += (__ldg(node_key + j0) == want) + (__ldg(node_key + j1) == want) + (__ldg(node_key + j2) == want) +
                   (__ldg(node_key + j3) == want);
        }
        for (; p < re; ++p) cnt += (__ldg(node_key + __ldg(col + p)) == want);
    }
    for (unsigned m = __ballot_sync(0xffffffffu, scan && deg > kLaneDeg); m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        const int64_t b0 = __shfl_sync(0xffffffffu, rb, r), e0 = __shfl_sync(0xffffffffu, re, r);
        const int wr = __shfl_sync(0xffffffffu, want, r);
        unsigned k = 0;
        for (int64_t p = b0 + lane; p < e0; p += 32) k += (__ldg(node_key + __ldg(col + p)) == wr);
        k = __reduce_add_sync(0xffffffffu, k);
        if (lane == r) cnt += k;
    }
    const unsigned long long n0 = valid && c == 0, n1 = valid && c == 1;
    const unsigned long long m0 = n0 ? (unsigned long long)deg : 0, m1 = n1 ? (unsigned long long)deg : 0;
    const int s0 = __shfl_sync(0xffffffffu, s, 0);
    if (__all_sync(0xffffffffu, s == s0) && s0 >= 0) {
        const unsigned tn0 = __reduce_add_sync(0xffffffffu, (unsigned)n0);
        const unsigned tn1 = __reduce_add_sync(0xffffffffu, (unsigned)n1);
        unsigned long long tm0 = m0, tm1 = m1, tc = cnt;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            tm0 += __shfl_xor_sync(0xffffffffu, tm0, o);
            tm1 += __shfl_xor_sync(0xffffffffu, tm1, o);
            tc += __shfl_xor_sync(0xffffffffu, tc, o);
        }
        if (lane == 0) {
            if (tn0) atomicAdd(&nsz[2 * s0], (unsigned long long)tn0);
            if (tn1) atomicAdd(&nsz[2 * s0 + 1], (unsigned long long)tn1);
            if (tm0) atomicAdd(&mbar[2 * s0], tm0);
            if (tm1) atomicAdd(&mbar[2 * s0 + 1], tm1);
            if (tc) atomicAdd(&cut[s0], tc);
        }
    } else if (valid) {
        atomicAdd(&nsz[2 * s + c], 1ull);
        if (deg) atomicAdd(&mbar[2 * s + c], (unsigned long long)deg);
        if (cnt) atomicAdd(&cut[s], (unsigned long long)cnt);
    }
}

// Thread per segment: exact split test, keep flag and kept size.
__global__ void sel_decide(const unsigned long long *__restrict__ nsz, const unsigned long long *__restrict__ mbar,
                           const unsigned long long *__restrict__ cut, int S, int32_t eps, int rule,
                           unsigned long long two_E, int32_t *__restrict__ keep, int32_t *__restrict__ ksize) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const unsigned long long n0 = nsz[2 * s], n1 = nsz[2 * s + 1], b0 = mbar[2 * s], b1 = mbar[2 * s + 1];
    const unsigned long long T = b0 + b1;
    const unsigned __int128 two_e = rule == 1 ? (unsigned __int128)T : (unsigned __int128)two_E;
    const bool stop = n0 <= (unsigned long long)eps || n1 <= (unsigned long long)eps || T == 0 ||
                      two_e * (unsigned __int128)cut[s] > (unsigned __int128)b0 * (unsigned __int128)b1;
    keep[s] = stop ? 0 : 1;
    ksize[s] = stop ? 0 : (int32_t)(n0 + n1);
}

// Thread per segment: offsets of the two children of every kept segment.
__global__ void sel_children(const int32_t *__restrict__ keep, const int64_t *__restrict__ krank,
                             const int64_t *__restrict__ base, const unsigned long long *__restrict__ nsz, int S,
                             int32_t *__restrict__ new_off) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s > S) return;
    if (s == S) {
        new_off[2 * krank[S]] = (int32_t)base[S];
        return;
    }
    if (!keep[s]) return;
    const int64_t k = krank[s];
    new_off[2 * k] = (int32_t)base[s];
    new_off[2 * k + 1] = (int32_t)(base[s] + (int64_t)nsz[2 * s]);
}

// Warp per parent segment: the two children of a kept segment inherit its final side sums and counts as their
// slot-0 totals (so no mean pass is needed below level 1).
template <int L>
__global__ void sel_inherit(const int32_t *__restrict__ keep, const int64_t *__restrict__ krank, SegState st, int S,
                            unsigned long long *__restrict__ nacc, unsigned long long *__restrict__ ncnt) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (s >= S || !keep[s]) return;
    const int64_t k = krank[s];
    for (int c = 0; c < 2; ++c) {
        for (int l = lane; l < L; l += 32) nacc[((size_t)(2 * k + c) * 2) * L + l] = st.acc[((size_t)s * 2 + c) * L + l];
        if (lane == 0) ncnt[(2 * k + c) * 2] = st.cnt[s * 2 + c];
    }
}

// Thread per position: stable partition of kept segments into their children; members of stopped
// segments get their (discovery-order) block id and leave the active set.
__global__ void sel_scatter(const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                            const int32_t *__restrict__ side, int64_t n_act, const int32_t *__restrict__ seg_off,
                            const int64_t *__restrict__ ones, const int32_t *__restrict__ keep,
                            const int64_t *__restrict__ krank, const int32_t *__restrict__ new_off, int32_t block_base,
                            int32_t *__restrict__ new_perm, int32_t *__restrict__ new_pseg,
                            int32_t *__restrict__ label_tmp, int32_t *__restrict__ node_key, int32_t *__restrict__ bmin) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int blk = -1, i = INT_MAX;
    if (pos < n_act) {
        const int s = pseg[pos];
        i = perm[pos];
        if (!keep[s]) {
            blk = block_base + (int32_t)(s - krank[s]);
            label_tmp[i] = blk;
            node_key[i] = -1;
        } else {
            const int64_t k = krank[s];
            const int64_t o = ones[pos] - ones[seg_off[s]];
            int64_t np;
            if (side[pos]) np = new_off[2 * k + 1] + o;
            else np = new_off[2 * k] + (pos - seg_off[s]) - o;
            new_perm[np] = i;
            new_pseg[np] = (int32_t)(2 * k + side[pos]);
        }
    }
    // smallest member of every finished block (canonical labels): one atomic per block run of the warp
    const int b0 = __shfl_sync(0xffffffffu, blk, 0);
    if (__all_sync(0xffffffffu, blk == b0)) {
        if (b0 >= 0) {
            const int mn = __reduce_min_sync(0xffffffffu, i);
            if (lane == 0) atomicMin(&bmin[b0], mn);
        }
    } else if (blk >= 0) {
        atomicMin(&bmin[blk], i);
    }
}

__global__ void sel_init(int32_t *__restrict__ perm, int32_t *__restrict__ pseg, int32_t *__restrict__ node_key,
                         int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        perm[i] = (int32_t)i;
        pseg[i] = 0;
        node_key[i] = 0;
    }
}

__global__ void sel_first_flags(const int32_t *__restrict__ label_tmp, const int32_t *__restrict__ bmin, int64_t n,
                                int32_t *__restrict__ first) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) first[i] = bmin[label_tmp[i]] == (int32_t)i;
}

__global__ void sel_canon(const int32_t *__restrict__ label_tmp, const int32_t *__restrict__ bmin,
                          const int64_t *__restrict__ frank, int64_t n, int32_t *__restrict__ labels) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) labels[i] = (int32_t)frank[bmin[label_tmp[i]]];
}

// Z in the level's position order (Zp[pos] = Z[perm[pos]]), so the row passes read rows by position: no
// perm indirection in their dependent load chains, and the rows a pruned pass recomputes (clustered near the
// split) are close together. One coalesced copy per level.
template <int L>
__global__ void sel_gather_rows(const float *__restrict__ Z, const int32_t *__restrict__ perm, int64_t n_act,
                                float *__restrict__ Zp) {
    constexpr int Q = L / 4;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_act * Q) return;
    const int64_t pos = t / Q;
    const int c = (int)(t % Q);
    reinterpret_cast<float4 *>(Zp)[t] = __ldg(reinterpret_cast<const float4 *>(Z + (size_t)perm[pos] * L) + c);
}

__global__ void fill_i32(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)std::max<int64_t>(1, ceil_div(n, threads)); }

// One model selection at compile-time width L.
template <int L>
raftgp_status model_select_L(raftgp_graph g, const float *Z, int32_t eps, int32_t max_iter, int32_t rule,
                             int32_t *labels, int32_t *num_blocks, int64_t *stats) {
    raftgp_ctx ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t n = g->n;
    constexpr size_t kRowSmem = (size_t)kRowWarps * 2 * 32 * (L + 4) * sizeof(float);
    constexpr size_t kPruneSmem = (size_t)kPruneWarps * 32 * (L + 4) * sizeof(float);
    static const char attrs_key = 0;   // per-(device, L) key
    int prune_ctas = 1;
    RG_TRY(per_device(ctx->device, &attrs_key, &prune_ctas, [&](int *v) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(sel_rows<L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem));
        RG_CUDA(cudaFuncSetAttribute(sel_rows<L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem));
        RG_CUDA(cudaFuncSetAttribute(sel_rows<L, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem));
        RG_CUDA(cudaFuncSetAttribute(sel_lloyd_pruned<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kPruneSmem));
        int b = 0;
        RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sel_lloyd_pruned<L>, kPruneWarps * 32, kPruneSmem));
        *v = std::max(1, b);
        return RAFTGP_OK;
    }));

    int32_t *perm = nullptr, *pseg = nullptr, *side = nullptr, *nperm = nullptr, *npseg = nullptr;
    int32_t *node_key = nullptr, *label_tmp = nullptr, *err = nullptr;
    unsigned long long *active = nullptr;
    int64_t *ones = nullptr;
    double *dpos = nullptr;
    RG_TRY(dalloc_t(ctx, &perm, n));
    RG_TRY(dalloc_t(ctx, &pseg, n));
    RG_TRY(dalloc_t(ctx, &side, n));
    RG_TRY(dalloc_t(ctx, &nperm, n));
    RG_TRY(dalloc_t(ctx, &npseg, n));
    RG_TRY(dalloc_t(ctx, &node_key, n));
    RG_TRY(dalloc_t(ctx, &label_tmp, n));
    int32_t *bmin = nullptr;   // smallest member of each finished block (at most n blocks)
    RG_TRY(dalloc_t(ctx, &bmin, n));
    RG_TRY(dalloc_t(ctx, &ones, n + 1));
    RG_TRY(dalloc_t(ctx, &dpos, n));
    float *Zp = nullptr;   // Z in position order (rebuilt per level)
    RG_TRY(dalloc_t(ctx, &Zp, (size_t)std::max<int64_t>(n, 1) * L));
    float2 *bnd = reinterpret_cast<float2 *>(dpos);   // seeding distances, then the Lloyd pruning bounds
    RG_TRY(dalloc_t(ctx, &err, 1));
    RG_TRY(dalloc_t(ctx, &active, 2 + 64));   // [0] active segments, [1] their rows, [2..65] rows read
    RG_TRY(dzero(ctx, active, sizeof(unsigned long long) * 66, st));
    RG_TRY(dzero(ctx, err, sizeof(int32_t), st));
    {
        LaunchScope LS(ctx, K_SELECT);
        sel_init<<<grid_for(n, 256), 256, 0, st>>>(perm, pseg, node_key, n);
    }
    {
        LaunchScope LS(ctx, K_SELECT);
        fill_i32<<<grid_for(n, 256), 256, 0, st>>>(bmin, n, INT_MAX);
    }
    RG_CHECK_LAUNCH(ctx);

    int64_t n_act = n;
    int S = 1;
    std::vector<int32_t> off0 = {0, (int32_t)n};
    int32_t *seg_off = nullptr;
    RG_TRY(dalloc_t(ctx, &seg_off, 2));
    {
        LaunchScope LS(ctx, K_SELECT);
        fill_i32<<<1, 32, 0, st>>>(seg_off, 1, 0);
        fill_i32<<<1, 32, 0, st>>>(seg_off + 1, 1, (int32_t)n);
    }

    int32_t blocks = 0;
    int64_t splits = 0, lloyd_iters = 0, levels = 0, lloyd_rows = 0, seed_rows = 0, act_rows = 0;
    int64_t capped_segs = 0, capped_rows = 0;
    int32_t h_small[2] = {0, 0};
    std::vector<unsigned long long> h_iter(2 * ((size_t)max_iter + 1), 0);
    unsigned long long *iter_act = nullptr;   // [t][2]: active segments / rows after update t
    RG_TRY(dalloc_t(ctx, &iter_act, 2 * ((size_t)max_iter + 1)));
    unsigned long long *claims = nullptr;     // [t]: position counter of Lloyd iteration t (zeroed per level)
    RG_TRY(dalloc_t(ctx, &claims, (size_t)max_iter + 1));
    int64_t h_two[2] = {0, 0};
    raftgp_status rc = RAFTGP_OK;
    // per-level [S][2][L] side sums and [S][2] counts; level 1 fills slot 0 with a mean pass, deeper levels
    // inherit the parent's final side sums (sel_inherit)
    unsigned long long *lvl_acc = nullptr, *lvl_cnt = nullptr;
    RG_TRY(dalloc_t(ctx, &lvl_acc, (size_t)2 * L));
    RG_TRY(dalloc_t(ctx, &lvl_cnt, (size_t)2));
    RG_TRY(dzero(ctx, lvl_acc, sizeof(unsigned long long) * 2 * L, st));
    RG_TRY(dzero(ctx, lvl_cnt, sizeof(unsigned long long) * 2, st));

    while (S > 0 && rc == RAFTGP_OK) {
        ++levels;
        if (n_act > 0) {
            LaunchScope LS(ctx, K_SEL_SEED);
            sel_gather_rows<L><<<grid_for(n_act * (L / 4), 256), 256, 0, st>>>(Z, perm, n_act, Zp);
        }
        // per-segment state of this level
        SegState ss{};
        unsigned long long *nsz = nullptr, *mbar = nullptr, *cut = nullptr;
        int32_t *keep = nullptr, *ksize = nullptr, *new_off = nullptr;
        int64_t *krank = nullptr, *base = nullptr;
        ss.acc = lvl_acc;
        ss.cnt = lvl_cnt;
        RG_TRY(dalloc_t(ctx, &ss.mu, (size_t)S * 2 * L));
        RG_TRY(dalloc_t(ctx, &ss.dmax, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.amin, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.changed, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.done, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.delta, (size_t)S * 2));
        RG_TRY(dalloc_t(ctx, &nsz, (size_t)S * 5));
        mbar = nsz + 2 * (size_t)S;
        cut = nsz + 4 * (size_t)S;
        RG_TRY(dalloc_t(ctx, &keep, (size_t)S * 2));
        ksize = keep + S;
        RG_TRY(dalloc_t(ctx, &krank, (size_t)S + 1));
        RG_TRY(dalloc_t(ctx, &base, (size_t)S + 1));
        RG_TRY(dalloc_t(ctx, &new_off, (size_t)2 * S + 1));
        RG_TRY(dzero(ctx, nsz, sizeof(unsigned long long) * (size_t)S * 5, st));

        const unsigned rgrid = grid_for(ceil_div(n_act, kRowRange), kRowWarps);
        // pruned passes: one wave of resident CTAs claiming kLloydChunk positions per warp at a time
        const unsigned qgrid = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)ctx->sm_count * prune_ctas, ceil_div(ceil_div(n_act, kLloydChunk), kPruneWarps)));
        act_rows = n_act;
        seed_rows += n_act;
        const unsigned sgrid = grid_for((int64_t)S * 32, 256);
        // seeding: mean, farthest from the mean, farthest from that
        if (levels == 1) {
            LaunchScope LS(ctx, K_SEL_SEED);
            sel_rows<L, 0><<<rgrid, kRowWarps * 32, kRowSmem, st>>>(Zp, perm, pseg, side, bnd, dpos, n_act, ss, err,
                                                                    active + 2);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SEL_SEED);
            sel_mean<L><<<sgrid, 256, 0, st>>>(ss, S);
        }
        RG_CHECK_LAUNCH(ctx);
        if (levels == 1) {
            RG_TRY(dread(ctx, h_small, err, sizeof(int32_t), st));
            if (h_small[0]) {
                rc = fail(RAFTGP_ERR_DATA, "raftgp_model_select: Z has an entry with |z| > 1 or NaN (SELECT_SPEC §1)");
            }
        }
        for (int slot = 0; slot < 2 && rc == RAFTGP_OK; ++slot) {
            {
                LaunchScope LS(ctx, K_SEL_SEED);
                sel_rows<L, 2><<<rgrid, kRowWarps * 32, kRowSmem, st>>>(Zp, perm, pseg, side, bnd, dpos, n_act, ss,
                                                                        err, active + 2);
            }
            RG_CHECK_LAUNCH(ctx);
            {
                LaunchScope LS(ctx, K_SEL_SEED);
                sel_argmin<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, n_act, dpos, ss);
            }
            RG_CHECK_LAUNCH(ctx);
            {
                LaunchScope LS(ctx, K_SEL_SEED);
                // first seed a overwrites the mean in slot 0; the second seed b goes to slot 1
                sel_seed<L><<<sgrid, 256, 0, st>>>(Z, ss, S, slot);
            }
            RG_CHECK_LAUNCH(ctx);
        }
        // Lloyd iterations, all segments in lock step (converged ones frozen). Iterations are enqueued in chunks
        // of kIterChunk without host round trips: update t counts the still-active segments (and their rows)
        // into iter_act[t], and the kernels of iteration t + 1 exit at once when that count is 0. The host
        // reads the counters once per chunk.
        RG_TRY(dzero(ctx, iter_act, sizeof(unsigned long long) * 2 * ((size_t)max_iter + 1), st));
        RG_TRY(dzero(ctx, claims, sizeof(unsigned long long) * ((size_t)max_iter + 1), st));
        for (int t0 = 1; t0 <= max_iter && rc == RAFTGP_OK; t0 += kIterChunk) {
            const int t1 = std::min(max_iter, t0 + kIterChunk - 1);
            for (int t = t0; t <= t1; ++t) {
                const unsigned long long *prev = t > 1 ? iter_act + 2 * (t - 1) : nullptr;
                {
                    LaunchScope LS(ctx, K_SEL_LLOYD);
                    if (t == 1)
                        sel_rows<L, 1><<<rgrid, kRowWarps * 32, kRowSmem, st>>>(Zp, perm, pseg, side, bnd, dpos, n_act,
                                                                                ss, err, active + 2);
                    else
                        sel_lloyd_pruned<L><<<qgrid, kPruneWarps * 32, kPruneSmem, st>>>(Zp, perm, pseg, side, bnd,
                                                                                       n_act, ss, active + 2, prev,
                                                                                       claims + t);
                }
                RG_CHECK_LAUNCH(ctx);
                {
                    LaunchScope LS(ctx, K_SEL_LLOYD);
                    sel_update<L><<<sgrid, 256, 0, st>>>(ss, S, t, max_iter, seg_off, prev, iter_act + 2 * t);
                }
                RG_CHECK_LAUNCH(ctx);
            }
            RG_TRY(dread(ctx, h_iter.data() + 2 * t0, iter_act + 2 * t0,
                         sizeof(unsigned long long) * 2 * (size_t)(t1 - t0 + 1), st));
            bool stop = false;
            for (int t = t0; t <= t1 && !stop; ++t) {
                ++lloyd_iters;
                lloyd_rows += act_rows;
                act_rows = (int64_t)h_iter[2 * t + 1];
                stop = h_iter[2 * t] == 0;
                if (t == max_iter) {   // the segments the cap stopped before convergence, and their rows
                    capped_segs += (int64_t)h_iter[2 * t];
                    capped_rows += (int64_t)h_iter[2 * t + 1];
                }
            }
            if (stop) break;
        }
        if (rc != RAFTGP_OK) {
            dfree(ctx, ss.mu); dfree(ctx, ss.dmax); dfree(ctx, ss.amin); dfree(ctx, ss.changed); dfree(ctx, ss.done);
            dfree(ctx, ss.delta); dfree(ctx, nsz); dfree(ctx, keep); dfree(ctx, krank); dfree(ctx, base);
            dfree(ctx, new_off);
            break;
        }
        // split test
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_mark<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, side, n_act, node_key);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_edges<<<grid_for(n_act, 256), 256, 0, st>>>(
                g->row_ptr, g->col, perm, pseg, side, n_act, node_key, nsz, mbar, cut);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_decide<<<grid_for(S, 256), 256, 0, st>>>(nsz, mbar, cut, S, eps, rule,
                                                         (unsigned long long)g->two_e, keep, ksize);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, keep, krank, S));
        RG_TRY(scan_i32_to_i64(ctx, ksize, base, S));
        RG_TRY(scan_i32_to_i64(ctx, side, ones, n_act));
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_children<<<grid_for((int64_t)S + 1, 256), 256, 0, st>>>(keep, krank, base, nsz, S, new_off);
        }
        RG_CHECK_LAUNCH(ctx);
        unsigned long long *nacc = nullptr, *ncnt = nullptr;
        RG_TRY(dalloc_t(ctx, &nacc, (size_t)S * 4 * L));
        RG_TRY(dalloc_t(ctx, &ncnt, (size_t)S * 4));
        RG_TRY(dzero(ctx, nacc, sizeof(unsigned long long) * (size_t)S * 4 * L, st));
        RG_TRY(dzero(ctx, ncnt, sizeof(unsigned long long) * (size_t)S * 4, st));
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_inherit<L><<<sgrid, 256, 0, st>>>(keep, krank, ss, S, nacc, ncnt);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SEL_SPLIT);
            sel_scatter<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, side, n_act, seg_off, ones, keep, krank,
                                                              new_off, blocks, nperm, npseg, label_tmp, node_key,
                                                              bmin);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(dread(ctx, &h_two[0], krank + S, sizeof(int64_t), st));
        RG_TRY(dread(ctx, &h_two[1], base + S, sizeof(int64_t), st));
        const int64_t kept = h_two[0];
        blocks += (int32_t)(S - kept);
        splits += kept;
        dfree(ctx, ss.acc); dfree(ctx, ss.cnt);
        lvl_acc = nacc;
        lvl_cnt = ncnt;
        dfree(ctx, ss.mu); dfree(ctx, ss.dmax); dfree(ctx, ss.amin);
        dfree(ctx, ss.changed); dfree(ctx, ss.done); dfree(ctx, ss.delta); dfree(ctx, nsz); dfree(ctx, keep); dfree(ctx, krank);
        dfree(ctx, base);
        dfree(ctx, seg_off);
        seg_off = new_off;
        std::swap(perm, nperm);
        std::swap(pseg, npseg);
        n_act = h_two[1];
        S = (int)(2 * kept);
    }
    if (rc == RAFTGP_OK && n > 0) {
        // canonical labels: blocks ordered by their smallest member (SELECT_SPEC §5)
        int32_t *first = nullptr;
        RG_TRY(dalloc_t(ctx, &first, n));
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_first_flags<<<grid_for(n, 256), 256, 0, st>>>(label_tmp, bmin, n, first);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, first, ones, n));
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_canon<<<grid_for(n, 256), 256, 0, st>>>(label_tmp, bmin, ones, n, labels);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_CUDA(cudaStreamSynchronize(st));
        dfree(ctx, first);
    }
    dfree(ctx, seg_off);
    dfree(ctx, lvl_acc);
    dfree(ctx, lvl_cnt);
    dfree(ctx, iter_act);
    dfree(ctx, claims);
    dfree(ctx, Zp);
    dfree(ctx, perm); dfree(ctx, pseg); dfree(ctx, side); dfree(ctx, nperm); dfree(ctx, npseg);
    dfree(ctx, node_key); dfree(ctx, label_tmp); dfree(ctx, bmin); dfree(ctx, ones); dfree(ctx, dpos); dfree(ctx, err);
    unsigned long long h_read[64] = {0};
    if (rc == RAFTGP_OK) {
        RG_TRY(dread(ctx, h_read, active + 2, sizeof(h_read), st));
    }
    dfree(ctx, active);
    if (rc != RAFTGP_OK) return rc;
    int64_t rows_read = 0;
    for (int i = 0; i < 64; ++i) rows_read += (int64_t)h_read[i];
    *num_blocks = blocks;
    if (stats) {
        stats[0] = blocks;
        stats[1] = splits;
        stats[2] = lloyd_iters;
        stats[3] = levels;
        stats[4] = lloyd_rows;   // rows of not-yet-converged segments visited by the Lloyd passes
        stats[5] = seed_rows;    // rows visited per seeding pass (3 passes: mean, 2 x farthest)
        stats[6] = rows_read;    // Z rows actually read by the Lloyd passes (the rest were pruned by bounds)
        stats[7] = capped_segs;  // segments whose Lloyd iteration stopped at max_iter without converging (all levels)
        stats[8] = capped_rows;  // their rows
    }
    return RAFTGP_OK;
}

}  // namespace

raftgp_status model_select(raftgp_graph g, const float *Z, int32_t L, int32_t eps, int32_t max_iter, int32_t rule,
                           int32_t *labels, int32_t *num_blocks, int64_t *stats) {
    switch (L) {
        case 8: return model_select_L<8>(g, Z, eps, max_iter, rule, labels, num_blocks, stats);
        case 16: return model_select_L<16>(g, Z, eps, max_iter, rule, labels, num_blocks, stats);
        case 32: return model_select_L<32>(g, Z, eps, max_iter, rule, labels, num_blocks, stats);
        case 64: return model_select_L<64>(g, Z, eps, max_iter, rule, labels, num_blocks, stats);
        case 128: return model_select_L<128>(g, Z, eps, max_iter, rule, labels, num_blocks, stats);
        default: return fail(RAFTGP_ERR_PARAM, "raftgp_model_select: L must be 8, 16, 32, 64 or 128");
    }
}

}  // namespace raftgp
