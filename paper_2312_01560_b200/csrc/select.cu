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

constexpr int kSelRange = 128;   // positions per warp in the fused Lloyd / mean passes
constexpr int kEdgeRange = 16;   // rows per warp in the split-test pass

__device__ __forceinline__ long long fixq(float z) { return __double2ll_rn(__dmul_rn((double)z, 4294967296.0)); }

__device__ __forceinline__ double centre(long long S, unsigned long long cnt) {
    return __ddiv_rn(__dmul_rn(__ll2double_rn(S), 0x1p-32), __ull2double_rn(cnt));
}

// SELECT_SPEC §2 squared distance of a row held in shared memory (float4-aligned) to mu (global, fp64)
template <int L>
__device__ __forceinline__ double sqdist_smem(const float *row, const double *mu) {
    double d = 0.0;
#pragma unroll 4
    for (int k = 0; k < L / 4; ++k) {
        const float4 v = *reinterpret_cast<const float4 *>(row + 4 * k);
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

template <int L>
__device__ __forceinline__ double sqdist_global(const float *row, const double *mu) {
    double d = 0.0;
#pragma unroll 4
    for (int k = 0; k < L / 4; ++k) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(row + 4 * k));
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

// Per-segment state of one level (S segments; all device arrays).
struct SegState {
    unsigned long long *acc;   // [S][2][L] fixed-point sums (two's complement int64)
    unsigned long long *cnt;   // [S][2]
    double *mu;                // [S][2][L] centres (slot 0 also holds the mean / first seed)
    unsigned long long *dmax;  // [S] bits of the max distance (d >= 0, so the bit order is the value order)
    int32_t *amin;             // [S] smallest node id attaining dmax
    int32_t *changed;          // [S]
    int32_t *done;             // [S]
};

// Fused pass over the positions of a level. MODE 0: mean pass (every member into slot 0, |z| <= 1 check).
// MODE 1: Lloyd iteration t: assign side by distance to mu[s][0], mu[s][1], then accumulate q(z) per side.
// Each warp handles kSelRange consecutive positions; rows are staged 32 at a time in shared memory, then
// lane-per-column integer sums run along the staged rows and are flushed with one atomic per (segment,
// side, column) whenever the segment changes.
template <int L, int MODE>
__global__ void __launch_bounds__(L >= 128 ? 128 : 256) sel_pass(const float *__restrict__ Z, const int32_t *__restrict__ perm,
                                                          const int32_t *__restrict__ pseg, int32_t *__restrict__ side,
                                                          int64_t n_act, int t, SegState st, int32_t *err) {
    constexpr int LD = L + 4;
    constexpr int CPL = (L + 31) / 32;   // columns per lane
    extern __shared__ __align__(16) float sel_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *stage = sel_smem + (size_t)warp * 32 * LD;
    __shared__ int2 meta_all[8][32];
    int2 *meta = meta_all[warp];
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const int64_t beg = w * kSelRange;
    if (beg >= n_act) return;
    const int64_t end = min(beg + (int64_t)kSelRange, n_act);

    long long a0[CPL], a1[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) a0[k] = a1[k] = 0;
    unsigned long long c0 = 0, c1 = 0;
    int cur = -1;
    bool bad = false;

    auto flush = [&]() {
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
                if (c0) atomicAdd(&st.cnt[cur * 2 + 0], c0);
                if (c1) atomicAdd(&st.cnt[cur * 2 + 1], c1);
            }
        }
        c0 = c1 = 0;
    };

    for (int64_t b = beg; b < end; b += 32) {
        const int64_t pos = b + lane;
        int s = -1, c = 0;
        if (pos < end) {
            s = pseg[pos];
            if (MODE == 1 && st.done[s]) s = -1;
        }
        if (s >= 0) {
            const float4 *src = reinterpret_cast<const float4 *>(Z + (size_t)perm[pos] * L);
            float4 *dst = reinterpret_cast<float4 *>(stage + lane * LD);
#pragma unroll 4
            for (int k = 0; k < L / 4; ++k) {
                const float4 v = __ldg(src + k);
                if (MODE == 0)
                    bad |= !(fabsf(v.x) <= 1.f && fabsf(v.y) <= 1.f && fabsf(v.z) <= 1.f && fabsf(v.w) <= 1.f);
                dst[k] = v;
            }
            if (MODE == 1) {
                const double *m0 = st.mu + (size_t)s * 2 * L;
                const double d0 = sqdist_smem<L>(stage + lane * LD, m0);
                const double d1 = sqdist_smem<L>(stage + lane * LD, m0 + L);
                c = d1 < d0 ? 1 : 0;
                if (t > 1 && side[pos] != c) st.changed[s] = 1;
                side[pos] = c;
            }
        }
        meta[lane] = make_int2(s, c);
        __syncwarp();
        const int rows = (int)min((int64_t)32, end - b);
        for (int r = 0; r < rows; ++r) {
            const int2 mr = meta[r];
            if (mr.x != cur) {
                flush();
                cur = mr.x;
            }
            if (mr.x < 0) continue;
            const float *row = stage + r * LD;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int col = lane + 32 * k;
                if (col < L) {
                    const long long q = fixq(row[col]);
                    if (mr.y) a1[k] += q;
                    else a0[k] += q;
                }
            }
            if (mr.y) ++c1;
            else ++c0;
        }
        __syncwarp();
    }
    flush();
    if (MODE == 0 && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(err, 1);
}

// Warp per segment: slot-0 mean from the mean pass, reset the accumulators and the argmax state.
template <int L>
__global__ void sel_mean(SegState st, int S) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (s >= S) return;
    const unsigned long long n = st.cnt[s * 2];
    for (int l = lane; l < L; l += 32) {
        const size_t i = (size_t)s * 2 * L + l;
        st.mu[i] = n ? centre((long long)st.acc[i], n) : 0.0;
        st.acc[i] = 0;
        st.acc[i + L] = 0;
    }
    if (lane == 0) {
        st.cnt[s * 2] = st.cnt[s * 2 + 1] = 0;
        st.dmax[s] = 0;
        st.amin[s] = INT_MAX;
        st.changed[s] = 0;
        st.done[s] = 0;
    }
}

// Farthest member from the reference point mu[s][slot] (SELECT_SPEC §3.1): distances kept per position,
// maximum bits per segment.
template <int L>
__global__ void sel_far(const float *__restrict__ Z, const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                        int64_t n_act, int slot, SegState st, double *__restrict__ dpos) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int s = -1;
    double d = 0.0;
    if (pos < n_act) {
        s = pseg[pos];
        d = sqdist_global<L>(Z + (size_t)perm[pos] * L, st.mu + ((size_t)s * 2 + slot) * L);
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
// get their new centres (an empty side keeps its centre) and count as active.
template <int L>
__global__ void sel_update(SegState st, int S, int t, int max_iter, int32_t *active) {
    const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (s >= S || st.done[s]) return;
    if ((t > 1 && st.changed[s] == 0) || t >= max_iter) {
        if (lane == 0) st.done[s] = 1;
        return;
    }
    const unsigned long long n0 = st.cnt[s * 2], n1 = st.cnt[s * 2 + 1];
    for (int l = lane; l < L; l += 32) {
        const size_t i0 = (size_t)s * 2 * L + l, i1 = i0 + L;
        if (n0) st.mu[i0] = centre((long long)st.acc[i0], n0);
        if (n1) st.mu[i1] = centre((long long)st.acc[i1], n1);
        st.acc[i0] = 0;
        st.acc[i1] = 0;
    }
    __syncwarp();
    if (lane == 0) {
        st.cnt[s * 2] = st.cnt[s * 2 + 1] = 0;
        st.changed[s] = 0;
        atomicAdd(active, 1);
    }
}

// node_key[node] = 2 * segment + side for every position of the level.
__global__ void sel_mark(const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                         const int32_t *__restrict__ side, int64_t n_act, int32_t *__restrict__ node_key) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < n_act) node_key[perm[pos]] = 2 * pseg[pos] + side[pos];
}

// Split-test statistics (SELECT_SPEC §4): per segment and side |U_r| and mbar_r; cut = edges from U_1
// (side 0) rows into U_2 (side 1), counted once from the U_1 end. Warp per row, kEdgeRange rows per warp,
// run-aggregated atomics.
__global__ void sel_edges(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                          const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                          const int32_t *__restrict__ side, int64_t n_act, const int32_t *__restrict__ node_key,
                          unsigned long long *__restrict__ nsz, unsigned long long *__restrict__ mbar,
                          unsigned long long *__restrict__ cut) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t beg = w * kEdgeRange;
    if (beg >= n_act) return;
    const int64_t end = min(beg + (int64_t)kEdgeRange, n_act);
    int cur = -1;
    unsigned long long n0 = 0, n1 = 0, m0 = 0, m1 = 0, cu = 0;
    auto flush = [&]() {
        if (cur >= 0 && lane == 0) {
            if (n0) atomicAdd(&nsz[cur * 2], n0);
            if (n1) atomicAdd(&nsz[cur * 2 + 1], n1);
            if (m0) atomicAdd(&mbar[cur * 2], m0);
            if (m1) atomicAdd(&mbar[cur * 2 + 1], m1);
            if (cu) atomicAdd(&cut[cur], cu);
        }
        n0 = n1 = m0 = m1 = cu = 0;
    };
    for (int64_t pos = beg; pos < end; ++pos) {
        const int s = pseg[pos], c = side[pos], i = perm[pos];
        if (s != cur) {
            flush();
            cur = s;
        }
        const int64_t rb = row_ptr[i], re = row_ptr[i + 1];
        if (c) {
            ++n1;
            m1 += (unsigned long long)(re - rb);
            continue;
        }
        ++n0;
        m0 += (unsigned long long)(re - rb);
        const int want = 2 * s + 1;
        unsigned cnt = 0;
        for (int64_t p = rb + lane; p < re; p += 32) cnt += (__ldg(node_key + __ldg(col + p)) == want);
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        cu += cnt;
    }
    flush();
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

// Thread per position: stable partition of kept segments into their children; members of stopped
// segments get their (discovery-order) block id and leave the active set.
__global__ void sel_scatter(const int32_t *__restrict__ perm, const int32_t *__restrict__ pseg,
                            const int32_t *__restrict__ side, int64_t n_act, const int32_t *__restrict__ seg_off,
                            const int64_t *__restrict__ ones, const int32_t *__restrict__ keep,
                            const int64_t *__restrict__ krank, const int32_t *__restrict__ new_off, int32_t block_base,
                            int32_t *__restrict__ new_perm, int32_t *__restrict__ new_pseg,
                            int32_t *__restrict__ label_tmp, int32_t *__restrict__ node_key) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n_act) return;
    const int s = pseg[pos], i = perm[pos];
    if (!keep[s]) {
        label_tmp[i] = block_base + (int32_t)(s - krank[s]);
        node_key[i] = -1;
        return;
    }
    const int64_t k = krank[s];
    const int64_t o = ones[pos] - ones[seg_off[s]];
    int64_t np;
    if (side[pos]) np = new_off[2 * k + 1] + o;
    else np = new_off[2 * k] + (pos - seg_off[s]) - o;
    new_perm[np] = i;
    new_pseg[np] = (int32_t)(2 * k + side[pos]);
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

__global__ void sel_block_min(const int32_t *__restrict__ label_tmp, int64_t n, int32_t *__restrict__ bmin) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMin(&bmin[label_tmp[i]], (int32_t)i);
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
    constexpr int kWarps = L >= 128 ? 4 : 8;
    constexpr size_t kSmem = (size_t)kWarps * 32 * (L + 4) * sizeof(float);
    static bool attrs = false;
    if (!attrs) {
        RG_CUDA(cudaFuncSetAttribute(sel_pass<L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
        RG_CUDA(cudaFuncSetAttribute(sel_pass<L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
        attrs = true;
    }

    int32_t *perm = nullptr, *pseg = nullptr, *side = nullptr, *nperm = nullptr, *npseg = nullptr;
    int32_t *node_key = nullptr, *label_tmp = nullptr, *err = nullptr, *active = nullptr;
    int64_t *ones = nullptr;
    double *dpos = nullptr;
    RG_TRY(dalloc_t(ctx, &perm, n));
    RG_TRY(dalloc_t(ctx, &pseg, n));
    RG_TRY(dalloc_t(ctx, &side, n));
    RG_TRY(dalloc_t(ctx, &nperm, n));
    RG_TRY(dalloc_t(ctx, &npseg, n));
    RG_TRY(dalloc_t(ctx, &node_key, n));
    RG_TRY(dalloc_t(ctx, &label_tmp, n));
    RG_TRY(dalloc_t(ctx, &ones, n + 1));
    RG_TRY(dalloc_t(ctx, &dpos, n));
    RG_TRY(dalloc_t(ctx, &err, 2));
    active = err + 1;
    RG_CUDA(cudaMemsetAsync(err, 0, 2 * sizeof(int32_t), st));
    {
        LaunchScope LS(ctx, K_SELECT);
        sel_init<<<grid_for(n, 256), 256, 0, st>>>(perm, pseg, node_key, n);
    }
    RG_CHECK_LAUNCH(ctx);

    int64_t n_act = n;
    int S = 1;
    std::vector<int32_t> off0 = {0, (int32_t)n};
    int32_t *seg_off = nullptr;
    RG_TRY(dalloc_t(ctx, &seg_off, 2));
    RG_CUDA(cudaMemcpyAsync(seg_off, off0.data(), 2 * sizeof(int32_t), cudaMemcpyHostToDevice, st));

    int32_t blocks = 0;
    int64_t splits = 0, lloyd_iters = 0, levels = 0;
    int32_t h_small[2] = {0, 0};
    int64_t h_two[2] = {0, 0};
    raftgp_status rc = RAFTGP_OK;

    while (S > 0 && rc == RAFTGP_OK) {
        ++levels;
        // per-segment state of this level
        SegState ss{};
        unsigned long long *nsz = nullptr, *mbar = nullptr, *cut = nullptr;
        int32_t *keep = nullptr, *ksize = nullptr, *new_off = nullptr;
        int64_t *krank = nullptr, *base = nullptr;
        RG_TRY(dalloc_t(ctx, &ss.acc, (size_t)S * 2 * L));
        RG_TRY(dalloc_t(ctx, &ss.cnt, (size_t)S * 2));
        RG_TRY(dalloc_t(ctx, &ss.mu, (size_t)S * 2 * L));
        RG_TRY(dalloc_t(ctx, &ss.dmax, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.amin, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.changed, (size_t)S));
        RG_TRY(dalloc_t(ctx, &ss.done, (size_t)S));
        RG_TRY(dalloc_t(ctx, &nsz, (size_t)S * 5));
        mbar = nsz + 2 * (size_t)S;
        cut = nsz + 4 * (size_t)S;
        RG_TRY(dalloc_t(ctx, &keep, (size_t)S * 2));
        ksize = keep + S;
        RG_TRY(dalloc_t(ctx, &krank, (size_t)S + 1));
        RG_TRY(dalloc_t(ctx, &base, (size_t)S + 1));
        RG_TRY(dalloc_t(ctx, &new_off, (size_t)2 * S + 1));
        RG_CUDA(cudaMemsetAsync(ss.acc, 0, sizeof(unsigned long long) * (size_t)S * 2 * L, st));
        RG_CUDA(cudaMemsetAsync(ss.cnt, 0, sizeof(unsigned long long) * (size_t)S * 2, st));
        RG_CUDA(cudaMemsetAsync(nsz, 0, sizeof(unsigned long long) * (size_t)S * 5, st));

        const int64_t nwarps = ceil_div(n_act, kSelRange);
        const unsigned pgrid = grid_for(nwarps, kWarps);
        const unsigned sgrid = grid_for((int64_t)S * 32, 256);
        // seeding: mean, farthest from the mean, farthest from that
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_pass<L, 0><<<pgrid, kWarps * 32, kSmem, st>>>(Z, perm, pseg, side, n_act, 0, ss, err);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_mean<L><<<sgrid, 256, 0, st>>>(ss, S);
        }
        RG_CHECK_LAUNCH(ctx);
        if (levels == 1) {
            RG_CUDA(cudaMemcpyAsync(h_small, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            RG_CUDA(cudaStreamSynchronize(st));
            if (h_small[0]) {
                rc = fail(RAFTGP_ERR_DATA, "raftgp_model_select: Z has an entry with |z| > 1 or NaN (SELECT_SPEC §1)");
            }
        }
        for (int slot = 0; slot < 2 && rc == RAFTGP_OK; ++slot) {
            {
                LaunchScope LS(ctx, K_SELECT);
                sel_far<L><<<grid_for(n_act, 256), 256, 0, st>>>(Z, perm, pseg, n_act, 0, ss, dpos);
            }
            RG_CHECK_LAUNCH(ctx);
            {
                LaunchScope LS(ctx, K_SELECT);
                sel_argmin<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, n_act, dpos, ss);
            }
            RG_CHECK_LAUNCH(ctx);
            {
                LaunchScope LS(ctx, K_SELECT);
                // first seed a overwrites the mean in slot 0; the second seed b goes to slot 1
                sel_seed<L><<<sgrid, 256, 0, st>>>(Z, ss, S, slot);
            }
            RG_CHECK_LAUNCH(ctx);
        }
        // Lloyd iterations, all segments in lock step (converged ones frozen)
        for (int t = 1; t <= max_iter && rc == RAFTGP_OK; ++t) {
            ++lloyd_iters;
            {
                LaunchScope LS(ctx, K_SELECT);
                sel_pass<L, 1><<<pgrid, kWarps * 32, kSmem, st>>>(Z, perm, pseg, side, n_act, t, ss, err);
            }
            RG_CHECK_LAUNCH(ctx);
            RG_CUDA(cudaMemsetAsync(active, 0, sizeof(int32_t), st));
            {
                LaunchScope LS(ctx, K_SELECT);
                sel_update<L><<<sgrid, 256, 0, st>>>(ss, S, t, max_iter, active);
            }
            RG_CHECK_LAUNCH(ctx);
            RG_CUDA(cudaMemcpyAsync(h_small + 1, active, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            RG_CUDA(cudaStreamSynchronize(st));
            if (h_small[1] == 0) break;
        }
        if (rc != RAFTGP_OK) break;
        // split test
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_mark<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, side, n_act, node_key);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_edges<<<grid_for(ceil_div(n_act, kEdgeRange) * 32, 256), 256, 0, st>>>(
                g->row_ptr, g->col, perm, pseg, side, n_act, node_key, nsz, mbar, cut);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_decide<<<grid_for(S, 256), 256, 0, st>>>(nsz, mbar, cut, S, eps, rule,
                                                         (unsigned long long)g->two_e, keep, ksize);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, keep, krank, S));
        RG_TRY(scan_i32_to_i64(ctx, ksize, base, S));
        RG_TRY(scan_i32_to_i64(ctx, side, ones, n_act));
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_children<<<grid_for((int64_t)S + 1, 256), 256, 0, st>>>(keep, krank, base, nsz, S, new_off);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_scatter<<<grid_for(n_act, 256), 256, 0, st>>>(perm, pseg, side, n_act, seg_off, ones, keep, krank,
                                                              new_off, blocks, nperm, npseg, label_tmp, node_key);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_CUDA(cudaMemcpyAsync(&h_two[0], krank + S, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaMemcpyAsync(&h_two[1], base + S, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
        const int64_t kept = h_two[0];
        blocks += (int32_t)(S - kept);
        splits += kept;
        dfree(ctx, ss.acc); dfree(ctx, ss.cnt); dfree(ctx, ss.mu); dfree(ctx, ss.dmax); dfree(ctx, ss.amin);
        dfree(ctx, ss.changed); dfree(ctx, ss.done); dfree(ctx, nsz); dfree(ctx, keep); dfree(ctx, krank);
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
        int32_t *bmin = nullptr, *first = nullptr;
        RG_TRY(dalloc_t(ctx, &bmin, std::max<int32_t>(1, blocks)));
        RG_TRY(dalloc_t(ctx, &first, n));
        {
            LaunchScope LS(ctx, K_SELECT);
            fill_i32<<<grid_for(blocks, 256), 256, 0, st>>>(bmin, blocks, INT_MAX);
        }
        {
            LaunchScope LS(ctx, K_SELECT);
            sel_block_min<<<grid_for(n, 256), 256, 0, st>>>(label_tmp, n, bmin);
        }
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
        dfree(ctx, bmin);
        dfree(ctx, first);
    }
    dfree(ctx, seg_off);
    dfree(ctx, perm); dfree(ctx, pseg); dfree(ctx, side); dfree(ctx, nperm); dfree(ctx, npseg);
    dfree(ctx, node_key); dfree(ctx, label_tmp); dfree(ctx, ones); dfree(ctx, dpos); dfree(ctx, err);
    if (rc != RAFTGP_OK) return rc;
    *num_blocks = blocks;
    if (stats) {
        stats[0] = blocks;
        stats[1] = splits;
        stats[2] = lloyd_iters;
        stats[3] = levels;
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
