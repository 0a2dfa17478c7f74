// sbm.cu — NEXT-3: Alg. 2 (§IV), the exact degree-corrected SBM sampler, per
// docs/SBM_SPEC.md. The walk of every block pair is cut into fixed chunks of 2^q cells (independent Poisson
// events, so the distribution is the exact SBM one), and every chunk is one GPU thread:
//   members   block member lists in ascending id: a stable counting sort by block (K <= 4096), else the CSR
//             build (csr.cu) of the bipartite edge list (i, N + c_i), keeping only the block rows N..N+K-1
//   tables    P_r (theta prefix sums) and Q_r (upper-triangle row-sum prefixes), one thread per block,
//             sequential fp64 in the spec's order
//   chunks    per pair (r <= s): T_rs cells -> ceil(T / 2^q) chunks; exclusive scan -> chunk ids
//   count     persistent walk, one chunk per lane at a time (draw u, E = -ln_spec64(u), binary search of the
//             first cell whose RangeSum exceeds E), counting edges and recording the first kSlots event
//             cells of every chunk
//   write     scan of the counts, then the recorded cells (and the logged events past them) are emitted as
//             (src, dst) at the chunk's offset; without room for the log, the chunks with more than nslot
//             events are walked again
// Every floating-point value that decides an integer (RangeSum bits, E) is computed with the spec's operation
// sequence (explicit round-to-nearest intrinsics, no contraction), so the edge list is bit-identical to the
// oracle's, in (pair, chunk, cell) order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gauss.cuh"
#include "internal.cuh"

namespace raftgp {

namespace {

// ---------------------------------------------------------------- SBM_SPEC §5, §6
__device__ __forceinline__ double sbm_uniform(uint64_t seed, uint32_t p, uint32_t k, uint32_t d) {
    const Words4 x = philox10(p, k, d, 0x53424D31u, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t v = ((uint64_t)(x.x0 >> 5) << 26) + (uint64_t)(x.x1 >> 6) + 1ull;
    return __dmul_rn(__ull2double_rn(v), 0x1p-53);
}

__device__ __forceinline__ double ln_spec64(double u) {
    const uint64_t bits = (uint64_t)__double_as_longlong(u);
    int e = (int)((bits >> 52) & 0x7FF) - 1023;
    double m = __longlong_as_double((long long)((bits & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = __dmul_rn(m, 0.5);
        e = e + 1;
    }
    const double t = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
    const double t2 = __dmul_rn(t, t);
    double s = 2.0 / 25.0;
#pragma unroll
    for (int k = 11; k >= 0; --k) s = __fma_rn(t2, s, 2.0 / (double)(2 * k + 1));
    const double lnm = __dmul_rn(t, s);
    return __fma_rn((double)e, 0x1.62e42fefa39efp-1, __fma_rn((double)e, 0x1.abc9e3b39803fp-56, lnm));
}

struct SbmArgs {
    int32_t K;
    const int64_t *boff;     // [K+1] member offsets
    const int32_t *mem;      // members, ascending id per block
    const double *thm;       // theta of the members, in member order (thm[boff[r] + a] = theta[C_r[a]])
    const double *omega;     // [K*K]
    const double *P, *Q;     // tables: block r at boff[r] + r, length n_r + 1
    const int64_t *choff;    // [npairs+1] chunk offsets per pair
    const int8_t *qp;        // [npairs] log2 chunk size of each pair (SBM_SPEC §4)
    int64_t npairs, nchunks;
    uint64_t seed;
    int q;
    int nslot;               // event cells recorded per chunk by the count walk (0: the write pass walks again)
};

struct PairView {
    bool diag;
    int64_t nr, ns;
    const int32_t *Cr, *Cs;
    const double *Tr;        // theta of the row block's members
    const double *Pr, *Ps, *Qr;
    double omega;
};

__device__ __forceinline__ void pair_of(int64_t p, int32_t K, int32_t &r, int32_t &s) {
    // pairs r-major: pair index of (r, r) is r K - r (r - 1) / 2
    int32_t lo = 0, hi = K - 1;
    while (lo < hi) {
        const int32_t mid = (lo + hi + 1) / 2;
        const int64_t start = (int64_t)mid * K - (int64_t)mid * (mid - 1) / 2;
        if (start <= p) lo = mid;
        else hi = mid - 1;
    }
    r = lo;
    s = (int32_t)(r + (p - ((int64_t)r * K - (int64_t)r * (r - 1) / 2)));
}

__device__ __forceinline__ int64_t tri_start(int64_t n, int64_t a) { return a * n - a * (a + 1) / 2; }

// SBM_SPEC §3: cell -> (a, b). The diagonal row is the unique largest a with O(a) <= x (found from a fp64
// estimate, then fixed up in exact integers: any method yields the same row).
__device__ __forceinline__ void cell_ab(const PairView &v, int64_t x, int64_t &a, int64_t &b) {
    if (!v.diag) {
        a = x / v.ns;
        b = x - a * v.ns;
        return;
    }
    const int64_t n = v.nr;
    const double nn = (double)n - 0.5;
    int64_t g = (int64_t)(nn - sqrt(fmax(0.0, nn * nn - 2.0 * (double)x)));
    g = max((int64_t)0, min(g, n - 2));
    while (g > 0 && tri_start(n, g) > x) --g;
    while (g < n - 2 && tri_start(n, g + 1) <= x) ++g;
    a = g;
    b = g + 1 + (x - tri_start(n, g));
}

// SBM_SPEC §3 RangeSum(x, y) with x's row/column precomputed
__device__ __forceinline__ double range_sum(const SbmArgs &A, const PairView &v, int64_t a1, int64_t b1, int64_t y) {
    int64_t a2, b2;
    cell_ab(v, y, a2, b2);
    const double t1 = v.Tr[a1];
    if (!v.diag) {
        if (a1 == a2) return __dmul_rn(v.omega, __dmul_rn(t1, __dsub_rn(v.Ps[b2 + 1], v.Ps[b1])));
        const double t2 = v.Tr[a2];
        const double u1 = __dmul_rn(t1, __dsub_rn(v.Ps[v.ns], v.Ps[b1]));
        const double u2 = __dmul_rn(__dsub_rn(v.Pr[a2], v.Pr[a1 + 1]), v.Ps[v.ns]);
        const double u3 = __dmul_rn(t2, v.Ps[b2 + 1]);
        return __dmul_rn(v.omega, __dadd_rn(__dadd_rn(u1, u2), u3));
    }
    const int64_t n = v.nr;
    if (a1 == a2) return __dmul_rn(v.omega, __dmul_rn(t1, __dsub_rn(v.Pr[b2 + 1], v.Pr[b1])));
    const double t2 = v.Tr[a2];
    const double u1 = __dmul_rn(t1, __dsub_rn(v.Pr[n], v.Pr[b1]));
    const double u2 = __dsub_rn(v.Qr[a2], v.Qr[a1 + 1]);
    const double u3 = __dmul_rn(t2, __dsub_rn(v.Pr[b2 + 1], v.Pr[a2 + 1]));
    return __dmul_rn(v.omega, __dadd_rn(__dadd_rn(u1, u2), u3));
}

// Chunk set-up: pair of the chunk, its cell range [x0, x1) and the row/column of x0 (SBM_SPEC §3, §4)
__device__ __forceinline__ void chunk_setup(const SbmArgs &A, int64_t chunk, int64_t &p, int64_t &k, PairView &v,
                                            int64_t &x1, int64_t &mm) {
    // pair of this chunk: largest p with choff[p] <= chunk
    int64_t lo = 0, hi = A.npairs - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (A.choff[mid] <= chunk) lo = mid;
        else hi = mid - 1;
    }
    p = lo;
    k = chunk - A.choff[p];
    int32_t r, s;
    pair_of(p, A.K, r, s);
    v.diag = r == s;
    v.nr = A.boff[r + 1] - A.boff[r];
    v.ns = A.boff[s + 1] - A.boff[s];
    v.Cr = A.mem + A.boff[r];
    v.Cs = A.mem + A.boff[s];
    v.Tr = A.thm + A.boff[r];
    v.Pr = A.P + A.boff[r] + r;
    v.Ps = A.P + A.boff[s] + s;
    v.Qr = A.Q + A.boff[r] + r;
    v.omega = A.omega[(int64_t)r * A.K + s];
    const int64_t T = v.diag ? v.nr * (v.nr - 1) / 2 : v.nr * v.ns;
    const int q = A.qp[p];
    mm = k << q;
    x1 = min(T, (k + 1) << q);
}

// The walks (SBM_SPEC §4) as a persistent kernel: every lane owns one chunk at a time and performs ONE event
// attempt per loop iteration (draw, test, binary search, emit); a lane whose chunk ends takes the next
// unclaimed chunk (warp-aggregated claim on a global counter). The per-chunk event counts are Poisson, so a
// thread-per-chunk walk leaves most lanes of a warp idle behind the longest chunk; here they stay busy. A
// chunk's events depend only on the chunk, so the output (in (pair, chunk, cell) order via the count scan) is
// the same for any assignment of chunks to lanes. WRITE = false counts (cnt[chunk]), true writes at off[chunk].
constexpr int kSlots = 16;   // default event cells recorded per chunk by the count walk (expected <= 8 per chunk)

// Events past a chunk's nslot recorded cells (the hub rows of dense diagonal pairs hold hundreds per chunk)
// go to an append-only log, staged per warp in shared memory and flushed with one atomic per kWarpLog entries.
struct LogEnt {
    int64_t chunk;
    uint32_t c;      // event index within the chunk
    uint32_t cell;   // cell offset from the chunk start
};
constexpr int kWarpLog = 64;

template <bool WRITE>
__global__ void __launch_bounds__(128) sbm_walk(SbmArgs A, unsigned long long *next, int32_t *cnt,
                                                const int64_t *off, int32_t *src, int32_t *dst,
                                                uint32_t *slots, int64_t *ovf, unsigned long long *novf,
                                                LogEnt *log, unsigned long long *nlog, int64_t log_cap,
                                                const int64_t *list, int64_t nlist) {
    __shared__ LogEnt wbuf[WRITE ? 1 : 4][WRITE ? 1 : kWarpLog];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t chunk = -1, p = 0, k = 0, x0 = 0, x1 = 0, mm = 0, a1 = 0, b1 = 0, c = 0, o = 0;
    uint32_t d = 0;
    PairView v{};
    bool exhausted = false;
    int wc = 0;   // staged log entries of this warp (warp-uniform)
    auto flush = [&]() {
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(nlog, (unsigned long long)wc);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < wc; i += 32)
            if ((int64_t)(base + i) < log_cap) log[base + i] = wbuf[w][i];
        __syncwarp();
        wc = 0;
    };
    for (;;) {
        const bool need = chunk < 0 && !exhausted;
        const unsigned nm = __ballot_sync(0xffffffffu, need);
        if (nm) {
            const int leader = __ffs(nm) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(next, (unsigned long long)__popc(nm));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (need) {
                const int64_t cid = (int64_t)base + __popc(nm & ((1u << lane) - 1u));
                if (cid >= nlist) {
                    exhausted = true;
                } else {
                    chunk = list ? list[cid] : cid;
                    chunk_setup(A, chunk, p, k, v, x1, mm);
                    cell_ab(v, mm, a1, b1);
                    d = 0;
                    c = 0;
                    x0 = mm;
                    if (WRITE) o = off[chunk];
                }
            }
        }
        if (__all_sync(0xffffffffu, exhausted)) break;
        bool lg = false;
        LogEnt ent;
        if (chunk >= 0) {
            const double u = sbm_uniform(A.seed, (uint32_t)p, (uint32_t)k, d++);
            const double E = -ln_spec64(u);
            bool end = !(range_sum(A, v, a1, b1, x1 - 1) > E);
            if (!end) {
                int64_t l = mm, h = x1 - 1;
                while (l < h) {
                    const int64_t mid = l + (h - l) / 2;
                    if (range_sum(A, v, a1, b1, mid) > E) h = mid;
                    else l = mid + 1;
                }
                if (WRITE) {
                    int64_t a, b;
                    cell_ab(v, l, a, b);
                    src[o + c] = v.Cr[a];
                    dst[o + c] = v.diag ? v.Cr[b] : v.Cs[b];
                } else if (slots) {
                    if (c < A.nslot) {
                        slots[chunk * A.nslot + c] = (uint32_t)(l - x0);   // < 2^q <= 2^30
                    } else if (log) {
                        lg = true;
                        ent.chunk = chunk;
                        ent.c = (uint32_t)c;
                        ent.cell = (uint32_t)(l - x0);
                    }
                }
                ++c;
                mm = l + 1;
                end = mm >= x1;
                if (!end) cell_ab(v, mm, a1, b1);
            }
            if (end) {
                if (!WRITE) {
                    cnt[chunk] = (int32_t)c;
                    if (slots && c > A.nslot) ovf[atomicAdd(novf, 1ull)] = chunk;
                }
                chunk = -1;
            }
        }
        if (!WRITE && log) {   // converged: stage this iteration's log entries
            const unsigned lm = __ballot_sync(0xffffffffu, lg);
            if (lm) {
                const int nn = __popc(lm);
                if (wc + nn > kWarpLog) flush();
                if (lg) wbuf[w][wc + __popc(lm & ((1u << lane) - 1u))] = ent;
                wc += nn;
            }
        }
    }
    if (!WRITE && log && wc > 0) flush();
}

// Emit the recorded cells of every chunk as (src, dst) at the chunk's offset (thread per chunk; a chunk's
// cells are in increasing order, as the walk found them): all of them for chunks with at most nslot events,
// the first nslot of the others when the log holds the rest (with_log), none of those otherwise.
__global__ void __launch_bounds__(128) sbm_emit(SbmArgs A, const int32_t *cnt, const int64_t *off,
                                                const uint32_t *slots, bool with_log, int32_t *src, int32_t *dst) {
    for (int64_t chunk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; chunk < A.nchunks;
         chunk += (int64_t)gridDim.x * blockDim.x) {
        const int call = cnt[chunk];
        if (call == 0 || (call > A.nslot && !with_log)) continue;
        const int c = min(call, A.nslot);
        int64_t p, k, x1, x0;
        PairView v;
        chunk_setup(A, chunk, p, k, v, x1, x0);
        const int64_t o = off[chunk];
        for (int i = 0; i < c; ++i) {
            int64_t a, b;
            cell_ab(v, x0 + slots[chunk * A.nslot + i], a, b);
            src[o + i] = v.Cr[a];
            dst[o + i] = v.diag ? v.Cr[b] : v.Cs[b];
        }
    }
}

// Emit the logged events (thread per entry) at off[chunk] + c.
__global__ void __launch_bounds__(128) sbm_emit_log(SbmArgs A, const LogEnt *log, int64_t nlog, const int64_t *off,
                                                    int32_t *src, int32_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlog; i += (int64_t)gridDim.x * blockDim.x) {
        const LogEnt e = log[i];
        int64_t p, k, x1, x0;
        PairView v;
        chunk_setup(A, e.chunk, p, k, v, x1, x0);
        int64_t a, b;
        cell_ab(v, x0 + e.cell, a, b);
        const int64_t o = off[e.chunk] + e.c;
        src[o] = v.Cr[a];
        dst[o] = v.diag ? v.Cr[b] : v.Cs[b];
    }
}

__global__ void sbm_gather_theta(const int32_t *mem, const double *theta, int64_t n, double *thm) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) thm[t] = theta[mem[t]];
}

// SBM_SPEC §2: one thread per block, sequential fp64 sums in member order (over the contiguous member thetas)
// P_r and Q_r (SBM_SPEC §2): one warp per block. The sums are sequential in a (the spec's order), so one lane
// runs the add chain; the warp streams the operands through shared memory 256 at a time, loading the next
// tile into registers while the chain consumes the current one, and writes the results back coalesced.
constexpr int kTabTile = 256;

template <bool QPASS>
__device__ __forceinline__ void tables_pass(const double *__restrict__ thm, const double *__restrict__ Pin,
                                            int64_t b0, int64_t nr, int64_t o, double tot, double *__restrict__ out,
                                            double *sth, double *spp, double *sout, double &acc) {
    const int lane = threadIdx.x;
    double rt[kTabTile / 32], rp[kTabTile / 32];
    auto load = [&](int64_t a0) {
#pragma unroll
        for (int j = 0; j < kTabTile / 32; ++j) {
            const int64_t a = a0 + j * 32 + lane;
            rt[j] = a < nr ? thm[b0 + a] : 0.0;
            if (QPASS) rp[j] = a < nr ? Pin[o + a + 1] : 0.0;
        }
    };
    load(0);
    for (int64_t a0 = 0; a0 < nr; a0 += kTabTile) {
#pragma unroll
        for (int j = 0; j < kTabTile / 32; ++j) {
            sth[j * 32 + lane] = rt[j];
            if (QPASS) spp[j * 32 + lane] = rp[j];
        }
        __syncwarp();
        if (a0 + kTabTile < nr) load(a0 + kTabTile);   // in flight while the chain runs
        if (lane == 0) {
            const int cnt = (int)min((int64_t)kTabTile, nr - a0);
            for (int i0 = 0; i0 < cnt; i0 += 8) {
                double t[8], pp[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    t[j] = sth[i0 + j];
                    if (QPASS) pp[j] = spp[i0 + j];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (i0 + j < cnt) {
                        if (QPASS) acc = __dadd_rn(acc, __dmul_rn(t[j], __dsub_rn(tot, pp[j])));
                        else acc = __dadd_rn(acc, t[j]);
                        sout[i0 + j] = acc;
                    }
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kTabTile / 32; ++j) {
            const int64_t a = a0 + j * 32 + lane;
            if (a < nr) out[o + a + 1] = sout[j * 32 + lane];
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(32) sbm_tables(int32_t K, const int64_t *boff, const double *thm, double *P,
                                                 double *Q) {
    __shared__ double sth[kTabTile], spp[kTabTile], sout[kTabTile];
    const int32_t r = blockIdx.x;
    if (r >= K) return;
    const int64_t b0 = boff[r], nr = boff[r + 1] - b0, o = b0 + r;
    if (threadIdx.x == 0) {
        P[o] = 0.0;
        Q[o] = 0.0;
    }
    double acc = 0.0;
    tables_pass<false>(thm, nullptr, b0, nr, o, 0.0, P, sth, spp, sout, acc);
    __syncwarp();
    const double tot = __shfl_sync(0xffffffffu, acc, 0);
    __threadfence_block();
    double q = 0.0;
    tables_pass<true>(thm, P, b0, nr, o, tot, Q, sth, spp, sout, q);
}

// chunks per pair (0 when omega_rs = 0 or the pair has no cells) and the pair's chunk size 2^q_p:
// the largest q_p in [4, q] with R_p 2^q_p <= 8 T, R_p = RangeSum(0, T - 1) (SBM_SPEC §4)
__global__ void sbm_pair_chunks(SbmArgs A, int q, int32_t *nch, int8_t *qp) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= A.npairs) return;
    int32_t r, s;
    pair_of(p, A.K, r, s);
    PairView v;
    v.diag = r == s;
    v.nr = A.boff[r + 1] - A.boff[r];
    v.ns = A.boff[s + 1] - A.boff[s];
    v.Cr = A.mem + A.boff[r];
    v.Cs = A.mem + A.boff[s];
    v.Tr = A.thm + A.boff[r];
    v.Pr = A.P + A.boff[r] + r;
    v.Ps = A.P + A.boff[s] + s;
    v.Qr = A.Q + A.boff[r] + r;
    v.omega = A.omega[(int64_t)r * A.K + s];
    const int64_t T = v.diag ? v.nr * (v.nr - 1) / 2 : v.nr * v.ns;
    if (v.omega == 0.0 || T <= 0) {
        nch[p] = 0;
        qp[p] = 4;
        return;
    }
    int64_t a0, b0;
    cell_ab(v, 0, a0, b0);   // the first cell: (0, 0), or (0, 1) on the diagonal
    const double Rp = range_sum(A, v, a0, b0, T - 1);
    int qq = 4;
    for (int t = q; t >= 4; --t)
        if (scalbn(Rp, t) <= 8.0 * (double)T) {
            qq = t;
            break;
        }
    qp[p] = (int8_t)qq;
    nch[p] = (int32_t)((T + ((int64_t)1 << qq) - 1) >> qq);
}

__global__ void sbm_bip_edges(const int32_t *c, int64_t n, int32_t *src, int32_t *dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        src[i] = (int32_t)i;
        dst[i] = (int32_t)(n + c[i]);
    }
}

__global__ void sbm_validate(const int32_t *c, const double *theta, int64_t n, const double *omega, int32_t K,
                             int32_t *err) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n && (c[t] < 0 || c[t] >= K || !(theta[t] > 0.0))) atomicExch(err, 1);
    if (t < (int64_t)K * K) {
        const int64_t r = t / K, s = t % K;
        const double w = omega[t];
        if (!(w >= 0.0) || w != omega[s * K + r]) atomicExch(err, 1);
    }
}

// Member lists (block r's nodes in ascending id) by a stable counting sort, for K <= kMemMaxK: one warp per tile
// of kMemTile consecutive nodes counts its blocks in shared memory (bucket-major counts, no global atomics); a
// scan gives every (block, tile) its offset; the same warp then places its nodes in id order, ranking equal
// blocks within each 32-node round with __match_any_sync (stable). Larger K: the CSR build of (i, N + c_i).
constexpr int kMemTile = 2048;
constexpr int kMemWarps = 4;
constexpr int kMemMaxK = 4096;

__global__ void __launch_bounds__(kMemWarps * 32) sbm_member_count(const int32_t *__restrict__ c, int64_t n, int K,
                                                                  int64_t ntiles, int32_t *__restrict__ cnt) {
    extern __shared__ int32_t mcs[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *h = mcs + (size_t)w * K;
    for (int64_t tile = (int64_t)blockIdx.x * kMemWarps + w; tile < ntiles; tile += (int64_t)gridDim.x * kMemWarps) {
        for (int b = lane; b < K; b += 32) h[b] = 0;
        __syncwarp();
        const int64_t t0 = tile * kMemTile, t1 = min(n, t0 + kMemTile);
        for (int64_t i = t0 + lane; i < t1; i += 32) atomicAdd(&h[__ldg(c + i)], 1);
        __syncwarp();
        for (int b = lane; b < K; b += 32) cnt[(int64_t)b * ntiles + tile] = h[b];
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kMemWarps * 32) sbm_member_scatter(const int32_t *__restrict__ c, int64_t n, int K,
                                                                    int64_t ntiles, const int64_t *__restrict__ base,
                                                                    int32_t *__restrict__ mem) {
    extern __shared__ long long mss[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long *h = mss + (size_t)w * K;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t tile = (int64_t)blockIdx.x * kMemWarps + w; tile < ntiles; tile += (int64_t)gridDim.x * kMemWarps) {
        for (int b = lane; b < K; b += 32) h[b] = base[(int64_t)b * ntiles + tile];
        __syncwarp();
        const int64_t t0 = tile * kMemTile, t1 = min(n, t0 + kMemTile);
        for (int64_t r0 = t0; r0 < t1; r0 += 8 * 32) {
            int32_t bb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t i = r0 + j * 32 + lane;
                bb[j] = i < t1 ? __ldg(c + i) : -1;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t i = r0 + j * 32 + lane;
                const int32_t b = bb[j];
                const unsigned peers = __match_any_sync(0xffffffffu, b);
                if (b >= 0) mem[h[b] + __popc(peers & lt)] = (int32_t)i;
                __syncwarp();
                if (b >= 0 && lane == __ffs(peers) - 1) h[b] += __popc(peers);
                __syncwarp();
            }
        }
    }
}

__global__ void sbm_member_boff(const int64_t *base, int K, int64_t ntiles, int64_t n, int64_t *boff) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b <= K) boff[b] = b < K ? base[(int64_t)b * ntiles] : n;
}

inline unsigned grid1(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, ceil_div(n, t)); }

}  // namespace

raftgp_status sbm_sample(raftgp_ctx ctx, int64_t n, int32_t K, const int32_t *c, const double *theta,
                         const double *omega, uint64_t seed, int32_t q, int32_t *src, int32_t *dst, int64_t cap,
                         int64_t *m_out) {
    cudaStream_t st = ctx->stream;
    int32_t *err = nullptr;
    RG_TRY(dalloc_t(ctx, &err, 1));
    RG_TRY(dzero(ctx, err, sizeof(int32_t), st));
    {
        LaunchScope LS(ctx, K_SBM);
        sbm_validate<<<grid1(std::max<int64_t>(n, (int64_t)K * K), 256), 256, 0, st>>>(c, theta, n, omega, K, err);
    }
    RG_CHECK_LAUNCH(ctx);
    int32_t herr = 0;
    RG_TRY(dread(ctx, &herr, err, sizeof(int32_t), st));
    dfree(ctx, err);
    if (herr) return fail(RAFTGP_ERR_PARAM, "raftgp_sbm_sample: label outside [0,K), theta <= 0, or Omega negative / "
                                            "not symmetric");
    // members per block (ascending id)
    raftgp_graph_s members;
    members.ctx = ctx;
    int64_t *mboff = nullptr;
    int32_t *mmem = nullptr;
    auto drop_members = [&]() {
        dfree(ctx, members.row_ptr); dfree(ctx, members.col); dfree(ctx, members.deg_local); dfree(ctx, members.order);
        dfree(ctx, members.deg_all); dfree(ctx, members.s_all); dfree(ctx, members.sh_all); drop_slots(&members);
        dfree(ctx, mboff); dfree(ctx, mmem);
    };
    if (K <= kMemMaxK) {   // stable counting sort
        const int64_t ntiles = std::max<int64_t>(1, ceil_div(n, kMemTile));
        int32_t *mcnt = nullptr;
        int64_t *mbase = nullptr;
        raftgp_status rs = dalloc_t(ctx, &mcnt, (size_t)K * ntiles);
        if (rs == RAFTGP_OK) rs = dalloc_t(ctx, &mbase, (size_t)K * ntiles + 1);
        if (rs == RAFTGP_OK) rs = dalloc_t(ctx, &mboff, (size_t)K + 1);
        if (rs == RAFTGP_OK) rs = dalloc_t(ctx, &mmem, (size_t)std::max<int64_t>(n, 1));
        static const char attrs_key = 0;
        if (rs == RAFTGP_OK)
            rs = per_device(ctx->device, &attrs_key, nullptr, [&](int *) -> raftgp_status {
                RG_CUDA(cudaFuncSetAttribute(sbm_member_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMemWarps * kMemMaxK * 4));
                RG_CUDA(cudaFuncSetAttribute(sbm_member_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMemWarps * kMemMaxK * 8));
                return RAFTGP_OK;
            });
        const unsigned mg = (unsigned)ceil_div(ntiles, kMemWarps);
        if (rs == RAFTGP_OK) {
            LaunchScope LS(ctx, K_SBM);
            sbm_member_count<<<mg, kMemWarps * 32, (size_t)kMemWarps * K * 4, st>>>(c, n, K, ntiles, mcnt);
        }
        if (rs == RAFTGP_OK) rs = scan_i32_to_i64(ctx, mcnt, mbase, (int64_t)K * ntiles);
        if (rs == RAFTGP_OK) {
            LaunchScope LS(ctx, K_SBM);
            sbm_member_scatter<<<mg, kMemWarps * 32, (size_t)kMemWarps * K * 8, st>>>(c, n, K, ntiles, mbase, mmem);
            sbm_member_boff<<<grid1(K + 1, 256), 256, 0, st>>>(mbase, K, ntiles, n, mboff);
        }
        if (rs == RAFTGP_OK) {
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rs = cuda_fail(e, "sbm member lists");
        }
        dfree(ctx, mcnt);
        dfree(ctx, mbase);
        if (rs != RAFTGP_OK) {
            drop_members();
            return rs;
        }
    } else {   // CSR rows N..N+K-1 of the bipartite edges (i, N + c_i)
        int32_t *bsrc = nullptr;
        RG_TRY(dalloc_t(ctx, &bsrc, 2 * (size_t)std::max<int64_t>(n, 1)));
        {
            LaunchScope LS(ctx, K_SBM);
            sbm_bip_edges<<<grid1(n, 256), 256, 0, st>>>(c, n, bsrc, bsrc + n);
        }
        RG_CHECK_LAUNCH(ctx);
        raftgp_status rs = csr_build(ctx, n + K, n, bsrc, bsrc + n, n, n + K, &members);
        dfree(ctx, bsrc);
        if (rs != RAFTGP_OK) {
            drop_members();
            return rs;
        }
    }
    SbmArgs A{};
    A.K = K;
    A.boff = mboff ? mboff : members.row_ptr;
    A.mem = mmem ? mmem : members.col;
    A.omega = omega;
    A.seed = seed;
    A.q = q;
    A.npairs = (int64_t)K * (K + 1) / 2;
    double *P = nullptr, *Q = nullptr, *thm = nullptr;
    int32_t *nch = nullptr, *cnt = nullptr;
    int8_t *qp = nullptr;
    int64_t *choff = nullptr, *off = nullptr;
    unsigned long long *next = nullptr;
    uint32_t *slots = nullptr;
    int64_t *ovf = nullptr;
    LogEnt *logb = nullptr;
    raftgp_status s2 = dalloc_t(ctx, &P, (size_t)(n + K + 1));
    if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &Q, (size_t)(n + K + 1));
    if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &thm, (size_t)std::max<int64_t>(n, 1));
    if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &nch, (size_t)A.npairs);
    if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &choff, (size_t)A.npairs + 1);
    if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &qp, (size_t)A.npairs);
    A.P = P;
    A.Q = Q;
    A.thm = thm;
    A.qp = qp;
    if (s2 == RAFTGP_OK) {
        {
            LaunchScope LS(ctx, K_SBM);
            sbm_gather_theta<<<grid1(n, 256), 256, 0, st>>>(A.mem, theta, n, thm);
        }
        {
            LaunchScope LS(ctx, K_SBM);
            sbm_tables<<<std::max<int32_t>(K, 1), 32, 0, st>>>(K, A.boff, thm, P, Q);
        }
        {
            LaunchScope LS(ctx, K_SBM);
            sbm_pair_chunks<<<grid1(A.npairs, 128), 128, 0, st>>>(A, q, nch, qp);
        }
        s2 = scan_i32_to_i64(ctx, nch, choff, A.npairs);
    }
    int64_t nchunks = 0;
    if (s2 == RAFTGP_OK) {
        s2 = dread(ctx, &nchunks, choff + A.npairs, sizeof(int64_t), st);
    }
    A.choff = choff;
    A.nchunks = nchunks;
    int64_t total = 0;
    if (s2 == RAFTGP_OK && nchunks > 0) {
        s2 = dalloc_t(ctx, &cnt, (size_t)nchunks);
        if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &off, (size_t)nchunks + 1);
        if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &next, 4);
        if (s2 == RAFTGP_OK) RG_TRY(dzero(ctx, next, 4 * sizeof(unsigned long long), st));
        // recorded event cells (nslot per chunk; RAFTGP_SBM_SLOTS overrides, 0 = none) and the log of the
        // events past them; without room for the cells both passes walk, without room for the log the write
        // pass re-walks the chunks with more than nslot events
        static const int nslot_env = [] {
            const char *e = getenv("RAFTGP_SBM_SLOTS");
            return e ? std::max(0, std::min(64, atoi(e))) : kSlots;
        }();
        A.nslot = nslot_env;
        if (s2 == RAFTGP_OK && A.nslot > 0 && dalloc_t(ctx, &slots, (size_t)nchunks * A.nslot) != RAFTGP_OK)
            slots = nullptr;
        if (s2 == RAFTGP_OK && slots && dalloc_t(ctx, &ovf, (size_t)nchunks) != RAFTGP_OK) {
            dfree(ctx, slots);
            slots = nullptr;
        }
        if (!slots) A.nslot = 0;
        static const int64_t log_env = [] {   // RAFTGP_SBM_LOG: log capacity override (0 = no log)
            const char *e = getenv("RAFTGP_SBM_LOG");
            return e ? std::max<int64_t>(0, atoll(e)) : (int64_t)-1;
        }();
        const int64_t log_cap = !slots ? 0 : log_env >= 0 ? log_env : std::max<int64_t>(1 << 20, nchunks);
        if (s2 == RAFTGP_OK && log_cap > 0 && dalloc(ctx, reinterpret_cast<void **>(&logb), (size_t)log_cap * sizeof(LogEnt)) != RAFTGP_OK)
            logb = nullptr;
        static const char walk_key = 0;
        int walk_blocks = 1;
        if (s2 == RAFTGP_OK)
            s2 = per_device(ctx->device, &walk_key, &walk_blocks, [&](int *v) -> raftgp_status {
                int b = 0;
                RG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sbm_walk<false>, 128, 0));
                *v = std::max(1, b);
                return RAFTGP_OK;
            });
        auto wgrid = [&](int64_t items) {
            return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 128), (int64_t)ctx->sm_count * walk_blocks));
        };
        if (s2 == RAFTGP_OK) {
            LaunchScope LS(ctx, K_SBM_WALK);
            sbm_walk<false><<<wgrid(nchunks), 128, 0, st>>>(A, next, cnt, nullptr, nullptr, nullptr, slots, ovf, next + 2,
                                                           logb, next + 3, log_cap, nullptr, nchunks);
        }
        if (s2 == RAFTGP_OK) s2 = scan_i32_to_i64(ctx, cnt, off, nchunks);
        int64_t novf = 0, nlogged = 0;
        if (s2 == RAFTGP_OK) {
            s2 = dread(ctx, &total, off + nchunks, sizeof(int64_t), st);
            if (s2 == RAFTGP_OK) s2 = dread(ctx, &novf, next + 2, sizeof(int64_t), st);
            if (s2 == RAFTGP_OK) s2 = dread(ctx, &nlogged, next + 3, sizeof(int64_t), st);
        }
        if (s2 == RAFTGP_OK && total <= cap && total > 0) {
            LaunchScope LS(ctx, K_SBM_WALK);
            if (slots) {
                const bool with_log = logb && nlogged <= log_cap;
                sbm_emit<<<wgrid(nchunks), 128, 0, st>>>(A, cnt, off, slots, with_log, src, dst);
                if (with_log && nlogged > 0)
                    sbm_emit_log<<<grid1(nlogged, 128), 128, 0, st>>>(A, logb, nlogged, off, src, dst);
                if (!with_log && novf > 0)
                    sbm_walk<true><<<wgrid(novf), 128, 0, st>>>(A, next + 1, nullptr, off, src, dst, nullptr, nullptr,
                                                                nullptr, nullptr, nullptr, 0, ovf, novf);
            } else {
                sbm_walk<true><<<wgrid(nchunks), 128, 0, st>>>(A, next + 1, nullptr, off, src, dst, nullptr, nullptr,
                                                               nullptr, nullptr, nullptr, 0, nullptr, nchunks);
            }
        }
    }
    if (s2 == RAFTGP_OK) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) s2 = cuda_fail(e, "sbm kernels");
    }
    dfree(ctx, P); dfree(ctx, Q); dfree(ctx, thm); dfree(ctx, qp); dfree(ctx, nch); dfree(ctx, choff); dfree(ctx, cnt); dfree(ctx, off); dfree(ctx, next);
    dfree(ctx, slots); dfree(ctx, ovf); dfree(ctx, logb);
    drop_members();
    if (s2 == RAFTGP_OK) *m_out = total;
    return s2;
}

}  // namespace raftgp
