// sbm.cu — NEXT-3: Alg. 2 (§IV), the exact degree-corrected SBM sampler, per
// docs/SBM_SPEC.md. The walk of every block pair is cut into fixed chunks of 2^q cells (independent Poisson
// events, so the distribution is the exact SBM one), and every chunk is one GPU thread:
//   members   block member lists in ascending id: the CSR build (csr.cu) of the bipartite edge list
//             (i, N + c_i), keeping only the block rows N..N+K-1
//   tables    P_r (theta prefix sums) and Q_r (upper-triangle row-sum prefixes), one thread per block,
//             sequential fp64 in the spec's order
//   chunks    per pair (r <= s): T_rs cells -> ceil(T / 2^q) chunks; exclusive scan -> chunk ids
//   count     thread per chunk: the spec's walk (draw u, E = -ln_spec64(u), binary search of the first cell
//             whose RangeSum exceeds E), counting edges
//   write     scan of the counts, then the same walk writing (src, dst) at its offset
// Every floating-point value that decides an integer (RangeSum bits, E) is computed with the spec's operation
// sequence (explicit round-to-nearest intrinsics, no contraction), so the edge list is bit-identical to the
// oracle's, in (pair, chunk, cell) order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

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

// One chunk's walk (SBM_SPEC §4). WRITE = false counts, true writes at out offset.
template <bool WRITE>
__device__ int64_t walk_chunk(const SbmArgs &A, int64_t chunk, int32_t *src, int32_t *dst, int64_t off) {
    // pair of this chunk: largest p with choff[p] <= chunk
    int64_t lo = 0, hi = A.npairs - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (A.choff[mid] <= chunk) lo = mid;
        else hi = mid - 1;
    }
    const int64_t p = lo, k = chunk - A.choff[p];
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
    const int q = A.qp[p];
    const int64_t x0 = k << q, x1 = min(T, (k + 1) << q);
    int64_t mm = x0, cnt = 0;
    uint32_t d = 0;
    int64_t a1, b1;
    cell_ab(v, mm, a1, b1);
    for (;;) {
        const double u = sbm_uniform(A.seed, (uint32_t)p, (uint32_t)k, d++);
        const double E = -ln_spec64(u);
        if (!(range_sum(A, v, a1, b1, x1 - 1) > E)) break;
        int64_t l = mm, h = x1 - 1;
        while (l < h) {
            const int64_t mid = l + (h - l) / 2;
            if (range_sum(A, v, a1, b1, mid) > E) h = mid;
            else l = mid + 1;
        }
        if (WRITE) {
            int64_t a, b;
            cell_ab(v, l, a, b);
            src[off + cnt] = v.Cr[a];
            dst[off + cnt] = v.diag ? v.Cr[b] : v.Cs[b];
        }
        ++cnt;
        mm = l + 1;
        if (mm >= x1) break;
        cell_ab(v, mm, a1, b1);
    }
    return cnt;
}

__global__ void sbm_count(SbmArgs A, int32_t *cnt) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < A.nchunks; c += (int64_t)gridDim.x * blockDim.x)
        cnt[c] = (int32_t)walk_chunk<false>(A, c, nullptr, nullptr, 0);
}

__global__ void sbm_write(SbmArgs A, const int64_t *off, int32_t *src, int32_t *dst) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < A.nchunks; c += (int64_t)gridDim.x * blockDim.x)
        walk_chunk<true>(A, c, src, dst, off[c]);
}

__global__ void sbm_gather_theta(const int32_t *mem, const double *theta, int64_t n, double *thm) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) thm[t] = theta[mem[t]];
}

// SBM_SPEC §2: one thread per block, sequential fp64 sums in member order (over the contiguous member thetas)
__global__ void sbm_tables(int32_t K, const int64_t *boff, const double *thm, double *P, double *Q) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= K) return;
    const int64_t b0 = boff[r], nr = boff[r + 1] - b0, o = b0 + r;
    // sequential in a (the spec's order); operands are loaded 8 ahead so the add chain is the only dependency
    double acc = 0.0;
    P[o] = 0.0;
    for (int64_t a0 = 0; a0 < nr; a0 += 8) {
        double t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = a0 + j < nr ? thm[b0 + a0 + j] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (a0 + j < nr) {
                acc = __dadd_rn(acc, t[j]);
                P[o + a0 + j + 1] = acc;
            }
    }
    const double tot = acc;
    double q = 0.0;
    Q[o] = 0.0;
    for (int64_t a0 = 0; a0 < nr; a0 += 8) {
        double t[8], pp[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            t[j] = a0 + j < nr ? thm[b0 + a0 + j] : 0.0;
            pp[j] = a0 + j < nr ? P[o + a0 + j + 1] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (a0 + j < nr) {
                q = __dadd_rn(q, __dmul_rn(t[j], __dsub_rn(tot, pp[j])));
                Q[o + a0 + j + 1] = q;
            }
    }
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

inline unsigned grid1(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, ceil_div(n, t)); }

}  // namespace

raftgp_status sbm_sample(raftgp_ctx ctx, int64_t n, int32_t K, const int32_t *c, const double *theta,
                         const double *omega, uint64_t seed, int32_t q, int32_t *src, int32_t *dst, int64_t cap,
                         int64_t *m_out) {
    cudaStream_t st = ctx->stream;
    int32_t *err = nullptr;
    RG_TRY(dalloc_t(ctx, &err, 1));
    RG_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    {
        LaunchScope LS(ctx, K_SBM);
        sbm_validate<<<grid1(std::max<int64_t>(n, (int64_t)K * K), 256), 256, 0, st>>>(c, theta, n, omega, K, err);
    }
    RG_CHECK_LAUNCH(ctx);
    int32_t herr = 0;
    RG_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    dfree(ctx, err);
    if (herr) return fail(RAFTGP_ERR_PARAM, "raftgp_sbm_sample: label outside [0,K), theta <= 0, or Omega negative / "
                                            "not symmetric");
    // members per block (ascending id): CSR rows N..N+K-1 of the bipartite edges (i, N + c_i)
    int32_t *bsrc = nullptr;
    RG_TRY(dalloc_t(ctx, &bsrc, 2 * (size_t)std::max<int64_t>(n, 1)));
    {
        LaunchScope LS(ctx, K_SBM);
        sbm_bip_edges<<<grid1(n, 256), 256, 0, st>>>(c, n, bsrc, bsrc + n);
    }
    RG_CHECK_LAUNCH(ctx);
    raftgp_graph_s members;
    members.ctx = ctx;
    raftgp_status rs = csr_build(ctx, n + K, n, bsrc, bsrc + n, n, n + K, &members);
    dfree(ctx, bsrc);
    auto drop_members = [&]() {
        dfree(ctx, members.row_ptr); dfree(ctx, members.col); dfree(ctx, members.deg_local); dfree(ctx, members.order);
        dfree(ctx, members.deg_all); dfree(ctx, members.s_all); dfree(ctx, members.sh_all);
    };
    if (rs != RAFTGP_OK) {
        drop_members();
        return rs;
    }
    SbmArgs A{};
    A.K = K;
    A.boff = members.row_ptr;
    A.mem = members.col;
    A.omega = omega;
    A.seed = seed;
    A.q = q;
    A.npairs = (int64_t)K * (K + 1) / 2;
    double *P = nullptr, *Q = nullptr, *thm = nullptr;
    int32_t *nch = nullptr, *cnt = nullptr;
    int8_t *qp = nullptr;
    int64_t *choff = nullptr, *off = nullptr;
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
            sbm_tables<<<grid1(K, 32), 32, 0, st>>>(K, A.boff, thm, P, Q);
        }
        {
            LaunchScope LS(ctx, K_SBM);
            sbm_pair_chunks<<<grid1(A.npairs, 128), 128, 0, st>>>(A, q, nch, qp);
        }
        s2 = scan_i32_to_i64(ctx, nch, choff, A.npairs);
    }
    int64_t nchunks = 0;
    if (s2 == RAFTGP_OK) {
        RG_CUDA(cudaMemcpyAsync(&nchunks, choff + A.npairs, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RG_CUDA(cudaStreamSynchronize(st));
    }
    A.choff = choff;
    A.nchunks = nchunks;
    int64_t total = 0;
    if (s2 == RAFTGP_OK && nchunks > 0) {
        s2 = dalloc_t(ctx, &cnt, (size_t)nchunks);
        if (s2 == RAFTGP_OK) s2 = dalloc_t(ctx, &off, (size_t)nchunks + 1);
        const unsigned g = (unsigned)std::min<int64_t>(ceil_div(nchunks, 128), (int64_t)ctx->sm_count * 64);
        if (s2 == RAFTGP_OK) {
            LaunchScope LS(ctx, K_SBM_WALK);
            sbm_count<<<g, 128, 0, st>>>(A, cnt);
        }
        if (s2 == RAFTGP_OK) s2 = scan_i32_to_i64(ctx, cnt, off, nchunks);
        if (s2 == RAFTGP_OK) {
            RG_CUDA(cudaMemcpyAsync(&total, off + nchunks, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            RG_CUDA(cudaStreamSynchronize(st));
        }
        if (s2 == RAFTGP_OK && total <= cap && total > 0) {
            LaunchScope LS(ctx, K_SBM_WALK);
            sbm_write<<<g, 128, 0, st>>>(A, off, src, dst);
        }
    }
    if (s2 == RAFTGP_OK) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) s2 = cuda_fail(e, "sbm kernels");
    }
    dfree(ctx, P); dfree(ctx, Q); dfree(ctx, thm); dfree(ctx, qp); dfree(ctx, nch); dfree(ctx, choff); dfree(ctx, cnt); dfree(ctx, off);
    drop_members();
    if (s2 == RAFTGP_OK) *m_out = total;
    return s2;
}

}  // namespace raftgp
