// stream.cu — NEXT-4: streaming updates (§III-D "Extension to Streaming Graphs").
//
// A stream keeps the graph and the embedding state of one feature operator: Theta' = Theta W^(1) (fixed:
// Theta is counter-based per node), the hop operands T_1..T_L and Z. Adding edges E':
//   1. merge E' into the CSR (the new entries of each row are merged into its sorted list; duplicates of
//      existing edges and self-loops drop out), degrees / s / s^ / 2e recomputed;
//   2. V' = the nodes whose degree changed; R_1 = V' u N(V'), R_{k+1} = R_k u N(R_k) on the new graph
//      ("only the multi-hop neighbors of V' (denoted by V'') will participate");
//   3. the feature hop recomputes the rows of R_1, GCN hop k the rows of R_{k+1} (their operands' changed
//      rows are exactly the previous set), with the same kernels as a full embedding.
// Every row's arithmetic is a function of its neighbour list and its inputs only, so the streamed embedding
// is BIT-IDENTICAL to a full recompute on G u E'. This holds for X = M (NCut): Q and Q~ depend on 2e,
// which changes every row when an edge is added, so their exact update is the full recompute (the paper's
// O(|E'|) update of Q~ ignores that change).
// Delta mode (raftgp_stream_set_mode): every GCN hop is updated from its stored pre-activation sums plus the changed
// rows of its input (last_hop_delta below) — equal up to fp32 re-association instead of bit-identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"


namespace raftgp {

namespace {

// per row: new entries of the delta row not already in the old row (both sorted ascending)
__global__ void merge_count(int64_t n, const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                            const int64_t *__restrict__ drp, const int32_t *__restrict__ dcol,
                            const int32_t *__restrict__ odeg, int32_t *__restrict__ ndeg, int32_t *__restrict__ changed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t db = drp[i], de = drp[i + 1];
    int32_t add = 0;
    if (de > db) {
        const int64_t ob = orp[i], oe = orp[i + 1];
        for (int64_t p = db; p < de; ++p) {
            const int32_t j = dcol[p];
            int64_t lo = ob, hi = oe;   // lower_bound of j in the old row
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (ocol[mid] < j) lo = mid + 1;
                else hi = mid;
            }
            add += (lo == oe || ocol[lo] != j);
        }
    }
    ndeg[i] = odeg[i] + add;
    changed[i] = add > 0;
}

// write the merged rows: warp per row; rows without new entries are copied (coalesced), the others merged
__global__ void merge_write(int64_t n, const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                            const int64_t *__restrict__ drp, const int32_t *__restrict__ dcol,
                            const int32_t *__restrict__ changed, const int64_t *__restrict__ nrp,
                            int32_t *__restrict__ ncol) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t ob = orp[i], oe = orp[i + 1], nb = nrp[i];
    if (!changed[i]) {
        for (int64_t p = ob + lane; p < oe; p += 32) ncol[nb + (p - ob)] = ocol[p];
        return;
    }
    if (lane != 0) return;
    int64_t a = ob, b = drp[i], be = drp[i + 1], o = nb;
    while (a < oe || b < be) {
        if (b >= be || (a < oe && ocol[a] < dcol[b])) ncol[o++] = ocol[a++];
        else if (a < oe && ocol[a] == dcol[b]) { ncol[o++] = ocol[a++]; ++b; }
        else ncol[o++] = dcol[b++];
    }
}

// ---- affected sets as frontier lists. level[i] = hop distance from V' (127 = farther than L + 1). The rows of
// level k are appended to one list right after those of level k - 1, so R_k = V' u ... u N^k(V') is a PREFIX of
// the list and the hops of step 3 read prefixes. Only frontier rows are visited (the round-1 version scanned all n
// rows per level with a thread per row, so a hub's neighbour loop ran serially in one thread).
__global__ void fill_value(int64_t n, int32_t *a, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}
__global__ void fill_level(int64_t n, int32_t *level) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        level[i] = 127;
}

// V' from the changed flags (large-delta path): level 0 and the list head
__global__ void seed_changed(int64_t n, const int32_t *__restrict__ changed, int32_t *level, int32_t *rows,
                             int32_t *cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {   // whole warps iterate together
        const int64_t i = i0 + threadIdx.x;
        const bool c = i < n && changed[i];
        if (c) level[i] = 0;
        const unsigned bal = __ballot_sync(0xffffffffu, c);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(cnt, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (c) rows[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)i;
    }
}

// warp per frontier row (rows[f0 .. f0 + fc)): every neighbour j first reached at level k (atomicMin saw a larger
// level) is appended exactly once at the end of the list
__global__ void expand_frontier(const int64_t *__restrict__ rp, const int32_t *__restrict__ col, int32_t *level,
                                int32_t *rows, int64_t f0, int64_t fc, int k, int32_t *cnt) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w; t < fc; t += nw) {
        const int32_t i = rows[f0 + t];
        const int64_t b = rp[i], e = rp[i + 1];
        for (int64_t p0 = b; p0 < e; p0 += 32) {
            const int64_t p = p0 + lane;
            const int32_t j = p < e ? col[p] : 0;
            const bool fresh = p < e && atomicMin(&level[j], k) > k;
            // warp-aggregated append (one atomic per warp and chunk, not per row: the list counter is one address)
            const unsigned bal = __ballot_sync(0xffffffffu, fresh);
            int base = 0;
            if (lane == 0 && bal) base = atomicAdd(cnt, __popc(bal));   // cnt = the list's length
            base = __shfl_sync(0xffffffffu, base, 0);
            if (fresh) rows[base + __popc(bal & ((1u << lane) - 1u))] = j;
        }
    }
}

// ---- small deltas (m <= kSmallPairs pairs): ONE CTA sorts both orientations of the pairs by (row, col) in shared
// memory and drops self-loops and duplicates, instead of the full-graph CSR build of the delta (which visits all
// n rows: bucket sort, visiting order, degrees)
constexpr int kSmallPairs = 2048;   // 4096 keys x 8 B in static shared memory
constexpr int kSmallKeys = 2 * kSmallPairs;

__global__ void __launch_bounds__(1024) delta_sort_small(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                                         int64_t m, int64_t n, unsigned long long *__restrict__ keys,
                                                         int32_t *__restrict__ nkeys, int *__restrict__ err) {
    __shared__ unsigned long long k[kSmallKeys];
    __shared__ int32_t wsum[32];
    const int t = threadIdx.x;
    int P = 2;
    while (P < 2 * m) P <<= 1;
    for (int e = t; e < P; e += blockDim.x) {
        unsigned long long v = ~0ull;
        if (e < 2 * m) {
            const int64_t pi = e >> 1;
            const int32_t u = src[pi], w = dst[pi];
            if (u < 0 || w < 0 || u >= n || w >= n) atomicOr(err, 1);
            else if (u != w) {
                const uint32_t a = (e & 1) ? (uint32_t)w : (uint32_t)u, b = (e & 1) ? (uint32_t)u : (uint32_t)w;
                v = ((unsigned long long)a << 32) | b;
            }
        }
        k[e] = v;
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int e = t; e < P; e += blockDim.x) {
                const int o = e ^ stride;
                if (o > e) {
                    const bool up = (e & size) == 0;
                    const unsigned long long a = k[e], b = k[o];
                    if ((a > b) == up) {
                        k[e] = b;
                        k[o] = a;
                    }
                }
            }
            __syncthreads();
        }
    // unique, valid keys keep their order: per-thread segment counts, block scan, write
    const int per = (P + blockDim.x - 1) / blockDim.x;
    const int e0 = t * per, e1 = min(P, e0 + per);
    int c = 0;
    for (int e = e0; e < e1; ++e) c += k[e] != ~0ull && (e == 0 || k[e] != k[e - 1]);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((t & 31) >= o) incl += y;
    }
    if ((t & 31) == 31) wsum[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        int x = t < (int)(blockDim.x >> 5) ? wsum[t] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (t >= o) x += y;
        }
        wsum[t] = x;
    }
    __syncthreads();
    int pos = incl - c + ((t >> 5) ? wsum[(t >> 5) - 1] : 0);
    for (int e = e0; e < e1; ++e)
        if (k[e] != ~0ull && (e == 0 || k[e] != k[e - 1])) keys[pos++] = k[e];
    if (t == blockDim.x - 1) *nkeys = pos;
}

// per sorted delta entry (row u, col v): is v new in u's old row? count per row; the first new entry of a row puts
// the row on the list (V') at level 0
__global__ void delta_new(const unsigned long long *__restrict__ keys, const int32_t *__restrict__ nkeys,
                          const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol, int32_t *__restrict__ add,
                          uint8_t *__restrict__ isnew, int32_t *level, int32_t *rows, int32_t *cnt) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= *nkeys) return;
    const int32_t u = (int32_t)(keys[e] >> 32), v = (int32_t)(keys[e] & 0xffffffffu);
    int64_t lo = orp[u], hi = orp[u + 1];
    const int64_t oe = hi;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ocol[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    const bool nw = lo == oe || ocol[lo] != v;
    isnew[e] = nw;
    if (nw && atomicAdd(add + u, 1) == 0) {
        level[u] = 0;
        rows[atomicAdd(cnt, 1)] = u;
    }
}

// V' (rows[0 .. nc), any order, nc <= kSmallKeys) sorted ascending by one CTA; ends[t] = old end of the t-th changed
// row, shift[t] = new entries of the changed rows before it (so an old entry p after t changed rows moves by shift[t])
__global__ void __launch_bounds__(1024) changed_table(const int32_t *__restrict__ rows, int nc,
                                                      const int64_t *__restrict__ orp, const int32_t *__restrict__ add,
                                                      int32_t *__restrict__ sorted, int64_t *__restrict__ ends,
                                                      int64_t *__restrict__ shift) {
    __shared__ int32_t k[kSmallKeys];
    const int t = threadIdx.x;
    int P = 1;
    while (P < nc) P <<= 1;
    for (int e = t; e < P; e += blockDim.x) k[e] = e < nc ? rows[e] : 0x7fffffff;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int e = t; e < P; e += blockDim.x) {
                const int o = e ^ stride;
                if (o > e) {
                    const bool up = (e & size) == 0;
                    const int32_t a = k[e], b = k[o];
                    if ((a > b) == up) {
                        k[e] = b;
                        k[o] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (t == 0) {   // serial prefix over <= 4096 entries
        int64_t acc = 0;
        for (int e = 0; e < nc; ++e) {
            sorted[e] = k[e];
            ends[e] = orp[k[e] + 1];
            shift[e] = acc;
            acc += add[k[e]];
        }
        shift[nc] = acc;
    }
}

// the unchanged rows of the merged CSR: every old entry p outside the changed rows moves by the new entries of the
// changed rows before it (a streaming, coalesced copy; the changed rows are written by merge_changed)
__global__ void merge_copy(int64_t nnz, const int32_t *__restrict__ ocol, const int32_t *__restrict__ sorted,
                           const int64_t *__restrict__ orp, const int64_t *__restrict__ ends,
                           const int64_t *__restrict__ shift, int nc, int32_t *__restrict__ ncol) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nc;   // t = changed rows that end at or before p
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ends[mid] <= p) lo = mid + 1;
            else hi = mid;
        }
        if (lo < nc && orp[sorted[lo]] <= p) continue;   // inside a changed row
        ncol[p + shift[lo]] = ocol[p];
    }
}

// the same copy by chunks: a warp takes 32 x kMcVec consecutive entries, one lane locates the chunk start among the
// changed rows (binary search, once per chunk instead of per entry), and a chunk that lies inside one unchanged
// segment (all but ~2 per changed row) is moved with 16-byte loads and a constant shift; the others go entry by entry
constexpr int kMcVec = 8;   // entries per lane and chunk (two int4 loads)
__global__ void merge_copy_chunks(int64_t nnz, const int32_t *__restrict__ ocol, const int32_t *__restrict__ sorted,
                                  const int64_t *__restrict__ orp, const int64_t *__restrict__ ends,
                                  const int64_t *__restrict__ shift, int nc, int32_t *__restrict__ ncol) {
    const int lane = threadIdx.x & 31;
    constexpr int64_t CH = 32 * kMcVec;
    const int64_t nch = (nnz + CH - 1) / CH;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = wid; c < nch; c += nw) {
        const int64_t p0 = c * CH, p1 = min(nnz, p0 + CH);
        int seg = 0;
        bool clean = false;
        if (lane == 0) {
            int lo = 0, hi = nc;   // changed rows ending at or before p0
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ends[mid] <= p0) lo = mid + 1;
                else hi = mid;
            }
            seg = lo;
            // clean: the chunk ends before the next changed row starts (and does not start inside one)
            clean = lo >= nc || orp[sorted[lo]] >= p1;
        }
        seg = __shfl_sync(0xffffffffu, seg, 0);
        clean = __shfl_sync(0xffffffffu, clean, 0);
        if (clean && p1 - p0 == CH) {
            const int64_t sh = shift[seg];
            const int4 *src = reinterpret_cast<const int4 *>(ocol + p0);
#pragma unroll
            for (int h = 0; h < kMcVec / 4; ++h) {
                const int4 v = __ldcs(src + h * 32 + lane);
                int32_t *d = ncol + p0 + sh + (int64_t)(h * 32 + lane) * 4;
                d[0] = v.x;
                d[1] = v.y;
                d[2] = v.z;
                d[3] = v.w;
            }
        } else {
            for (int64_t p = p0 + lane; p < p1; p += 32) {
                int lo = 0, hi = nc;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (ends[mid] <= p) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < nc && orp[sorted[lo]] <= p) continue;   // inside a changed row
                ncol[p + shift[lo]] = ocol[p];
            }
        }
    }
}

// the changed rows: warp per row. The row's new entries d_0 < d_1 < ... are a contiguous run of the sorted keys
// (flagged new); every old entry moves by the number of new entries below it and every new entry lands after the old
// entries below it (binary searches, all lanes in parallel: a hub row is not merged by one lane)
__global__ void merge_changed(const int32_t *__restrict__ sorted, int nc, const int64_t *__restrict__ orp,
                              const int32_t *__restrict__ ocol, const unsigned long long *__restrict__ keys,
                              const int32_t *__restrict__ nkeys, const uint8_t *__restrict__ isnew,
                              const int64_t *__restrict__ nrp, int32_t *__restrict__ ncol) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nc) return;
    const int64_t i = sorted[w];
    const int64_t ob = orp[i], oe = orp[i + 1], nb = nrp[i];
    int lo = 0, hi = *nkeys;
    const unsigned long long first = (unsigned long long)i << 32;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < first) lo = mid + 1;
        else hi = mid;
    }
    int kb = lo, ke = lo;
    while (ke < *nkeys && (int64_t)(keys[ke] >> 32) == i) ++ke;   // the row's delta run [kb, ke), few entries
    // new entries: rank among the new ones (prefix count of isnew) + old entries below
    for (int q = kb + lane; q < ke; q += 32) {
        if (!isnew[q]) continue;
        int r = 0;
        for (int u = kb; u < q; ++u) r += isnew[u];
        const int32_t d = (int32_t)(keys[q] & 0xffffffffu);
        int64_t a = ob, b = oe;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (ocol[mid] < d) a = mid + 1;
            else b = mid;
        }
        ncol[nb + (a - ob) + r] = d;
    }
    // old entries: index + new entries below
    for (int64_t p = ob + lane; p < oe; p += 32) {
        const int32_t v = ocol[p];
        int r = 0;
        for (int u = kb; u < ke; ++u) r += isnew[u] && (int32_t)(keys[u] & 0xffffffffu) < v;
        ncol[nb + (p - ob) + r] = v;
    }
}

// merged rows, warp per row (many changed rows): unchanged rows copied, changed rows left to merge_changed
__global__ void merge_rows_copy(int64_t n, const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                                const int32_t *__restrict__ add, const int64_t *__restrict__ nrp,
                                int32_t *__restrict__ ncol) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n || add[i] != 0) return;
    const int64_t ob = orp[i], oe = orp[i + 1], nb = nrp[i];
    for (int64_t p = ob + lane; p < oe; p += 32) ncol[nb + (p - ob)] = ocol[p];
}

__global__ void new_degrees(int64_t n, const int32_t *__restrict__ odeg, const int32_t *__restrict__ add,
                            int32_t *__restrict__ ndeg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ndeg[i] = odeg[i] + add[i];
}

// sum of the degrees of the frontier rows rows[f0 .. f0 + fc) (how many entries the next expansion would visit)
__global__ void frontier_degsum(const int32_t *__restrict__ rows, int64_t f0, int64_t fc, const int32_t *__restrict__ deg,
                                unsigned long long *__restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < fc; i += (int64_t)gridDim.x * blockDim.x)
        s += (unsigned long long)deg[rows[f0 + i]];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// R_k in natural row order (for large sets: the hop then streams row_ptr / col_idx like a full pass)
__global__ void level_flags(int64_t n, const int32_t *__restrict__ level, int k, int32_t *__restrict__ flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = level[i] <= k;
}

__global__ void compact_rows(int64_t n, const int32_t *__restrict__ flag, const int64_t *__restrict__ pos,
                             int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = (int32_t)i;
}

// ---- delta mode (raftgp_stream_set_mode(RAFTGP_STREAM_DELTA)): the last GCN hop updated incrementally.
// Eq. 6 as the hop kernels compute it: H_i = s^_i A_i with A_i = T_i + sum_{j in N(i)} T_j
// (T = s^ (.) (Z W), T_j already carries s^_j). After a batch only the T_L rows of R_L changed (listed), and only
// the rows of V' changed their neighbour list or s^_i. So for i outside V'
//     A_i(new) = A_i(old) + sum_{j in (N(i) u {i}) n R_L} (T_j(new) - T_j(old)),
// and the rows of V' are summed in full. The stream keeps A (n x d_L); the dT rows of R_L are tiny (L2-resident) and
// a row gathers only its neighbours in R_L, found through pos[] (row -> dT index, -1 elsewhere). The last hop then
// reads col_idx once instead of gathering one operand row per entry. Exact up to fp32 rounding order (the sums are
// re-associated), not bit-identical: the exact mode stays the default.
__global__ void delta_save(const int32_t *__restrict__ rows, int64_t cnt, const float4 *__restrict__ T, int lpn,
                           int32_t *__restrict__ pos, float4 *__restrict__ dT) {
    const int64_t tot = cnt * lpn;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = t / lpn;
        const int c = (int)(t - idx * lpn);
        const int64_t r = rows[idx];
        dT[t] = T[r * lpn + c];
        if (c == 0) pos[r] = (int32_t)idx;
    }
}

__global__ void delta_finish(const int32_t *__restrict__ rows, int64_t cnt, const float4 *__restrict__ T, int lpn,
                             float4 *__restrict__ dT) {
    const int64_t tot = cnt * lpn;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = t / lpn;
        const float4 nw = T[(int64_t)rows[idx] * lpn + (t - idx * lpn)], od = dT[t];
        dT[t] = make_float4(nw.x - od.x, nw.y - od.y, nw.z - od.z, nw.w - od.w);
    }
}

__global__ void delta_clear(const int32_t *__restrict__ rows, int64_t cnt, int32_t *__restrict__ pos) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
        pos[rows[t]] = -1;
}

__device__ __forceinline__ void add4s(float4 &a, const float4 &v) {
    a.x += v.x;
    a.y += v.y;
    a.z += v.z;
    a.w += v.w;
}

// warp per row, rows claimed kDeltaRows at a time in the graph's visiting order. all_full = 1: every row summed in full
// (state build / resync); otherwise the rows of V' (level 0) in full and the rest by their changed neighbours. Rows
// with no changed neighbour (and an unchanged own T row) are not written.
constexpr int kDeltaRows = 4;
#ifndef RG_HIT_SLOTS
#define RG_HIT_SLOTS 4
#endif
constexpr int kHitSlots = RG_HIT_SLOTS;   // dT loads in flight per lane in the delta pass
template <int W>
__global__ void __launch_bounds__(256, 8) last_hop_delta(int64_t n, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ col, const int32_t *__restrict__ order,
                                                      const float *__restrict__ T, const int32_t *__restrict__ pos,
                                                      const float *__restrict__ dT, const int32_t *__restrict__ level,
                                                      const float *__restrict__ sh, float *__restrict__ A,
                                                      float *__restrict__ Z, int all_full,
                                                      unsigned long long *__restrict__ ctr,
                                                      unsigned long long *__restrict__ touched) {
    constexpr int LPN = W / 4, NB = 32 / LPN;
    const unsigned FULLM = 0xffffffffu;
    __shared__ int32_t hitq[8][32];   // per warp: the dT indices of a chunk's changed neighbours, compacted
    const int lane = threadIdx.x & 31, sub = lane / LPN, cl = lane % LPN;
    int32_t *q = hitq[threadIdx.x >> 5];
    const float4 *T4 = reinterpret_cast<const float4 *>(T);
    const float4 *D4 = reinterpret_cast<const float4 *>(dT);
    unsigned long long mine = 0;
    for (;;) {
        unsigned long long g0 = 0;
        if (lane == 0) g0 = atomicAdd(ctr, (unsigned long long)kDeltaRows);
        const int64_t q0 = (int64_t)__shfl_sync(FULLM, g0, 0);
        if (q0 >= n) break;
        const int64_t q1 = min(n, q0 + kDeltaRows);
        for (int64_t qq = q0; qq < q1; ++qq) {
            const int64_t i = order ? (int64_t)order[qq] : qq;
            const bool full = all_full || level[i] == 0;
            const int64_t b = rp[i], e = rp[i + 1];
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), ao = acc;
            bool any = full;
            if (full) {
                for (int64_t p0 = b; p0 < e; p0 += 32) {
                    const int cnt = (int)(e - p0 < 32 ? e - p0 : 32);
                    const int32_t c = lane < cnt ? __ldg(col + p0 + lane) : 0;
#pragma unroll 4
                    for (int t = 0; t < 32; t += NB) {
                        if (t >= cnt) break;
                        const int k = t + sub;
                        const int32_t j = __shfl_sync(FULLM, c, k);
                        if (k < cnt) add4s(acc, __ldg(T4 + (int64_t)j * LPN + cl));
                    }
                }
            } else {
                ao = reinterpret_cast<const float4 *>(A)[i * LPN + cl];   // issued before the neighbour walk
                for (int64_t p0 = b; p0 < e; p0 += 32) {
                    const int64_t p = p0 + lane;
                    const int32_t pj = p < e ? __ldg(pos + __ldg(col + p)) : -1;
                    const unsigned hits = __ballot_sync(FULLM, pj >= 0);
                    if (!hits) continue;
                    any = true;
                    if (pj >= 0) q[__popc(hits & ((1u << lane) - 1u))] = pj;
                    __syncwarp();
                    const int nh = __popc(hits);
                    for (int t = 0; t < nh; t += kHitSlots * NB) {   // kHitSlots loads in flight per lane
                        float4 v[kHitSlots];
#pragma unroll
                        for (int h = 0; h < kHitSlots; ++h) {
                            const int x = t + h * NB + sub;
                            v[h] = x < nh ? __ldg(D4 + (int64_t)q[x] * LPN + cl) : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int h = 0; h < kHitSlots; ++h) add4s(acc, v[h]);
                    }
                    __syncwarp();
                }
            }
#pragma unroll
            for (int o = LPN; o < 32; o <<= 1) {
                acc.x += __shfl_xor_sync(FULLM, acc.x, o);
                acc.y += __shfl_xor_sync(FULLM, acc.y, o);
                acc.z += __shfl_xor_sync(FULLM, acc.z, o);
                acc.w += __shfl_xor_sync(FULLM, acc.w, o);
            }
            if (full) {
                add4s(acc, __ldg(T4 + i * LPN + cl));   // the self term (A + I)
            } else {
                const int32_t pi = __ldg(pos + i);
                if (pi >= 0) {
                    add4s(acc, __ldg(D4 + (int64_t)pi * LPN + cl));
                    any = true;
                }
                if (!any) continue;
                acc = make_float4(ao.x + acc.x, ao.y + acc.y, ao.z + acc.z, ao.w + acc.w);
            }
            const float s = __ldg(sh + i);
            if constexpr (NB == 1) {
                float4 y = make_float4(tanhf(s * acc.x), tanhf(s * acc.y), tanhf(s * acc.z), tanhf(s * acc.w));
                float ss = y.x * y.x + y.y * y.y + y.z * y.z + y.w * y.w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) ss += __shfl_xor_sync(FULLM, ss, o);
                if (ss > 0.f) {   // one reciprocal square root (this mode is not bit-identical to the hop kernels anyway)
                    const float inv = rsqrtf(ss);
                    y = make_float4(y.x * inv, y.y * inv, y.z * inv, y.w * inv);
                }
                reinterpret_cast<float4 *>(A)[i * LPN + cl] = acc;
                if (Z) reinterpret_cast<float4 *>(Z)[i * LPN + cl] = y;
            } else {
                // every sub-slot holds the whole row sum after the butterfly: sub-slot s finishes columns
                // 4 cl + s CPL .. + CPL - 1 only, so the tanh / norm work is not repeated NB times
                constexpr int CPL = 4 / NB;
                const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
                float v[CPL], y[CPL], ss = 0.f;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    float x = a4[c];
#pragma unroll
                    for (int q2 = 1; q2 < NB; ++q2)
                        if (sub == q2) x = a4[q2 * CPL + c];
                    v[c] = x;
                    y[c] = tanhf(s * x);
                    ss += y[c] * y[c];
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) ss += __shfl_xor_sync(FULLM, ss, o);
                if (ss > 0.f) {
                    const float inv = rsqrtf(ss);
#pragma unroll
                    for (int c = 0; c < CPL; ++c) y[c] *= inv;
                }
                const int64_t f0 = i * W + cl * 4 + sub * CPL;   // this lane's first column
                if constexpr (CPL == 2) {
                    reinterpret_cast<float2 *>(A + f0)[0] = make_float2(v[0], v[1]);
                    if (Z) reinterpret_cast<float2 *>(Z + f0)[0] = make_float2(y[0], y[1]);
                } else {
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        A[f0 + c] = v[c];
                        if (Z) Z[f0 + c] = y[c];
                    }
                }
            }
            ++mine;
        }
    }
    if (lane == 0 && mine) atomicAdd(touched, mine);
}

inline unsigned g256(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }

bool fast_width(int32_t w) { return w == 32 || w == 64 || w == 128; }

// GCN hop h of a delta-mode stream (A[h] updated, Zout = rownorm(tanh(s^ A)) or null) over the listed rows, or over
// every row in the graph's visiting order (rows = null, count = n); all_full = 1: every row summed in full (state
// build / resync, or when the changed rows of T_h are too many for dT); touched_out: rows rewritten
raftgp_status launch_hop_delta(raftgp_stream s, raftgp_graph g, int h, const int32_t *rows, int64_t count,
                               const int32_t *level, const float *dT, int all_full, float *Zout, int64_t *touched_out) {
    raftgp_ctx ctx = g->ctx;
    if (count == 0) {
        if (touched_out) *touched_out = 0;
        return RAFTGP_OK;
    }
    const int d = s->dims[h];
    unsigned long long *ctr = nullptr;
    RG_TRY(dalloc_t(ctx, &ctr, 2));
    raftgp_status rc = dzero(ctx, ctr, 2 * sizeof(unsigned long long));
    if (rc == RAFTGP_OK) {
        const unsigned grid = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(ceil_div(count, kDeltaRows), 8), (int64_t)ctx->sm_count * 8));
        LaunchScope LS(ctx, h == s->layers ? K_STREAM_LAST : K_STREAM);
        const int32_t *order = rows ? rows : g->order;
        auto go = [&](auto kern) {
            kern<<<grid, 256, 0, ctx->stream>>>(count, g->row_ptr, g->col, order, s->T[h], s->pos, dT, level, g->sh_all,
                                                s->A[h], Zout, all_full, ctr, ctr + 1);
        };
        if (d == 32) go(last_hop_delta<32>);
        else if (d == 64) go(last_hop_delta<64>);
        else go(last_hop_delta<128>);
    }
    if (rc == RAFTGP_OK) {
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
    }
    unsigned long long t = 0;
    if (rc == RAFTGP_OK && touched_out) rc = dread(ctx, &t, ctr + 1, sizeof(t), ctx->stream);
    if (touched_out) *touched_out = (int64_t)t;
    dfree(ctx, ctr);
    return rc;
}

// the exact chain over every row (stream_create's state build; EXACT / DELTA mode switches restore it)
raftgp_status exact_chain(raftgp_stream s) {
    raftgp_graph g = s->g;
    const auto &dims = s->dims;
    const int L = s->layers;
    RG_TRY(feature_hop_pre(g, RAFTGP_NCUT, dims[1], s->thw, nullptr, s->T[1], nullptr));
    for (int k = 1; k <= L; ++k) {
        const bool last = k == L;
        RG_TRY(gcn_hop(g, s->T[k], dims[k], last ? s->Z : nullptr, last ? nullptr : s->W[k + 1], last ? 0 : dims[k + 1],
                       last ? nullptr : s->T[k + 1]));
    }
    return RAFTGP_OK;
}

}  // namespace

raftgp_status stream_create(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed, raftgp_stream *out) {
    raftgp_ctx ctx = g->ctx;
    if (!sketch_w_supported(dims[0], dims[1])) return fail(RAFTGP_ERR_PARAM, "stream: r and dims[1] must be 32, 64 or 128");
    for (int k = 1; k <= layers; ++k)
        if (!fast_width(dims[k])) return fail(RAFTGP_ERR_PARAM, "stream: layer widths must be 32, 64 or 128");
    raftgp_stream s = new raftgp_stream_s();
    s->ctx = ctx;
    ctx_retain(ctx);
    s->g = g;
    s->layers = layers;
    s->dims.assign(dims, dims + layers + 1);
    s->seed = seed;
    s->T.assign(layers + 2, nullptr);
    s->W.assign(layers + 2, nullptr);
    const int64_t n = g->n;
    raftgp_status st = dalloc_t(ctx, &s->thw, (size_t)n * dims[1]);
    float *W1 = nullptr;
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &W1, (size_t)dims[0] * dims[1]);
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, dims[0], dims[1], dims[0], W1);
    if (st == RAFTGP_OK) st = sketch_w_any(ctx, seed, n, dims[0], W1, dims[1], s->thw);
    dfree(ctx, W1);
    for (int k = 1; k <= layers && st == RAFTGP_OK; ++k) st = dalloc_t(ctx, &s->T[k], (size_t)n * dims[k]);
    for (int k = 2; k <= layers && st == RAFTGP_OK; ++k) {
        st = dalloc_t(ctx, &s->W[k], (size_t)dims[k - 1] * dims[k]);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, (uint32_t)k, 0, dims[k - 1], dims[k], dims[k - 1], s->W[k]);
    }
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &s->Z, (size_t)n * dims[layers]);
    if (st == RAFTGP_OK) st = feature_hop_pre(g, RAFTGP_NCUT, dims[1], s->thw, nullptr, s->T[1], nullptr);
    for (int k = 1; k <= layers && st == RAFTGP_OK; ++k) {
        const bool last = k == layers;
        st = gcn_hop(g, s->T[k], dims[k], last ? s->Z : nullptr, last ? nullptr : s->W[k + 1], last ? 0 : dims[k + 1],
                     last ? nullptr : s->T[k + 1]);
    }
    if (st != RAFTGP_OK) {
        s->g = nullptr;   // the caller keeps the graph on failure
        stream_destroy(s);
        return st;
    }
    *out = s;
    return RAFTGP_OK;
}

raftgp_status stream_add(raftgp_stream s, int64_t m, const int32_t *src, const int32_t *dst, int64_t *stats) {
    if (s->stale)
        return fail(RAFTGP_ERR_STATE, "stream: a failed batch left the state partly updated; call raftgp_stream_set_mode");
    raftgp_graph g = s->g;
    raftgp_ctx ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t n = g->n;
    const int L = s->layers;
    const bool small = m <= kSmallPairs;
    raftgp_graph ng = new raftgp_graph_s();
    ng->ctx = ctx;
    ng->n = n;
    ng->row_begin = 0;
    ng->row_end = n;
    ng->nl = n;
    auto drop = [&](raftgp_graph_s &x) {
        dfree(ctx, x.row_ptr); dfree(ctx, x.col); dfree(ctx, x.deg_local); dfree(ctx, x.order); dfree(ctx, x.deg_all);
        dfree(ctx, x.s_all); dfree(ctx, x.sh_all); drop_slots(&x);
    };
    int32_t *add = nullptr, *level = nullptr, *rows = nullptr, *cnt = nullptr, *nkeys = nullptr;
    int *err = nullptr;
    unsigned long long *keys = nullptr;
    uint8_t *isnew = nullptr;
    raftgp_graph_s delta;
    delta.ctx = ctx;
    bool have_delta = false;
    raftgp_status rc = dalloc_t(ctx, &ng->deg_local, (size_t)std::max<int64_t>(1, n));
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->row_ptr, (size_t)n + 1);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &add, (size_t)std::max<int64_t>(1, n));
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &level, (size_t)std::max<int64_t>(1, n));
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &rows, (size_t)std::max<int64_t>(1, n));
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &cnt, 4);   // [0] list length, [1] nkeys, [2] data error
    if (rc == RAFTGP_OK) rc = dzero(ctx, cnt, 4 * sizeof(int32_t));
    if (rc == RAFTGP_OK && n > 0) {
        LaunchScope LS(ctx, K_STREAM);
        fill_level<<<(unsigned)std::min<int64_t>(g256(n), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(n, level);
    }
    nkeys = cnt + 1;
    err = cnt + 2;
    // ---- 1. the new entries of every row, V' (rows with new entries) at level 0, new degrees
    if (rc == RAFTGP_OK && small) {
        rc = dalloc_t(ctx, &keys, (size_t)kSmallKeys);
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &isnew, (size_t)kSmallKeys);
        if (rc == RAFTGP_OK) rc = dzero(ctx, add, sizeof(int32_t) * (size_t)std::max<int64_t>(1, n));
        if (rc == RAFTGP_OK && m > 0) {
            {
                LaunchScope LS(ctx, K_STREAM);
                delta_sort_small<<<1, 1024, 0, st>>>(src, dst, m, n, keys, nkeys, err);
            }
            {
                LaunchScope LS(ctx, K_STREAM);
                delta_new<<<kSmallKeys / 256, 256, 0, st>>>(keys, nkeys, g->row_ptr, g->col, add, isnew, level, rows, cnt);
            }
            RG_CHECK_LAUNCH(ctx);
        }
    } else if (rc == RAFTGP_OK) {   // large delta: canonical CSR of E' (both orientations, sorted, deduplicated)
        rc = csr_build(ctx, n, m, src, dst, 0, n, &delta);
        have_delta = rc == RAFTGP_OK || delta.row_ptr != nullptr;
        int32_t *changed = nullptr;
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &changed, (size_t)std::max<int64_t>(1, n));
        if (rc == RAFTGP_OK && n > 0) {
            {
                LaunchScope LS(ctx, K_STREAM);
                merge_count<<<g256(n), 256, 0, st>>>(n, g->row_ptr, g->col, delta.row_ptr, delta.col, g->deg_local,
                                                     ng->deg_local, changed);
            }
            {
                LaunchScope LS(ctx, K_STREAM);
                seed_changed<<<(unsigned)std::min<int64_t>(g256(n), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(
                    n, changed, level, rows, cnt);
            }
            RG_CHECK_LAUNCH(ctx);
        }
        if (rc == RAFTGP_OK) rc = dcopy(ctx, add, changed, sizeof(int32_t) * (size_t)std::max<int64_t>(1, n));   // add > 0 <=> changed
        dfree(ctx, changed);
    }
    int32_t head[3] = {0, 0, 0};
    if (rc == RAFTGP_OK) rc = dread(ctx, head, cnt, sizeof(head), st);   // |V'|, delta keys, data error
    if (rc == RAFTGP_OK && head[2]) rc = fail(RAFTGP_ERR_DATA, "stream: node id outside [0, n)");
    // ---- merged CSR (new row pointers from the new degrees; changed rows merged, the others copied)
    if (rc == RAFTGP_OK && small && n > 0) {
        LaunchScope LS(ctx, K_STREAM);
        new_degrees<<<(unsigned)std::min<int64_t>(g256(n), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(n, g->deg_local, add,
                                                                                                  ng->deg_local);
    }
    if (rc == RAFTGP_OK) rc = scan_i32_to_i64(ctx, ng->deg_local, ng->row_ptr, n);
    if (rc == RAFTGP_OK) rc = dread(ctx, &ng->nnz_local, ng->row_ptr + n, sizeof(int64_t), st);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->col, (size_t)std::max<int64_t>(1, ng->nnz_local));
    if (rc == RAFTGP_OK && n > 0 && small) {   // coalesced copy of the unchanged rows + merge of the |V'| changed rows
        const int nc = head[0];
        int32_t *sorted = nullptr;
        int64_t *ends = nullptr, *shift = nullptr;
        rc = dalloc_t(ctx, &sorted, (size_t)nc + 1);
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ends, (size_t)nc + 1);
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &shift, (size_t)nc + 1);
        if (rc == RAFTGP_OK) {
            {
                LaunchScope LS(ctx, K_STREAM);
                changed_table<<<1, 1024, 0, st>>>(rows, nc, g->row_ptr, add, sorted, ends, shift);
            }
            if (g->nnz_local > 0 && nc <= 64 && aligned16(g->col)) {   // few changed rows: a streaming chunked copy
                LaunchScope LS(ctx, K_STREAM);
                merge_copy_chunks<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(g->nnz_local, 256 * kMcVec * 8),
                                                                                   (int64_t)ctx->sm_count * 16)),
                                    256, 0, st>>>(g->nnz_local, g->col, sorted, g->row_ptr, ends, shift, nc, ng->col);
            } else if (g->nnz_local > 0 && nc <= 64) {
                LaunchScope LS(ctx, K_STREAM);
                merge_copy<<<(unsigned)std::min<int64_t>(ceil_div(g->nnz_local, 256), (int64_t)ctx->sm_count * 16), 256, 0,
                             st>>>(g->nnz_local, g->col, sorted, g->row_ptr, ends, shift, nc, ng->col);
            } else if (g->nnz_local > 0) {        // many: warp per row (the element-wise search would cost more)
                LaunchScope LS(ctx, K_STREAM);
                merge_rows_copy<<<g256(n * 32), 256, 0, st>>>(n, g->row_ptr, g->col, add, ng->row_ptr, ng->col);
            }
            if (nc > 0) {
                LaunchScope LS(ctx, K_STREAM);
                merge_changed<<<(unsigned)ceil_div((int64_t)nc * 32, 256), 256, 0, st>>>(sorted, nc, g->row_ptr, g->col, keys,
                                                                                      nkeys, isnew, ng->row_ptr, ng->col);
            }
            RG_CHECK_LAUNCH(ctx);
        }
        dfree(ctx, sorted);
        dfree(ctx, ends);
        dfree(ctx, shift);
    } else if (rc == RAFTGP_OK && n > 0) {
        LaunchScope LS(ctx, K_STREAM);
        merge_write<<<g256(n * 32), 256, 0, st>>>(n, g->row_ptr, g->col, delta.row_ptr, delta.col, add, ng->row_ptr,
                                                  ng->col);
    }
    if (rc == RAFTGP_OK) {
        RG_CHECK_LAUNCH(ctx);
        rc = dalloc_t(ctx, &ng->deg_all, (size_t)std::max<int64_t>(1, n));
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->s_all, (size_t)std::max<int64_t>(1, n));
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->sh_all, (size_t)std::max<int64_t>(1, n));
    }
    if (rc == RAFTGP_OK) {
        if (n > 0) rc = dcopy(ctx, ng->deg_all, ng->deg_local, sizeof(int32_t) * n, st);
        if (rc == RAFTGP_OK) rc = degrees_finalize(ng);
    }
    if (have_delta) drop(delta);
    dfree(ctx, keys);
    dfree(ctx, isnew);
    // ---- 2 + 3. level by level: the frontier of level k - 1 marks level k; then the rows of R_k (a prefix of the
    // list) are recomputed: the feature hop for k = 1, GCN hop k - 1 for k >= 2
    std::vector<int64_t> counts(L + 2, 0);
    counts[0] = head[0];
    int32_t *hop_rows = nullptr, *nat_rows = nullptr;
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &hop_rows, (size_t)std::max<int64_t>(1, n));
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &nat_rows, (size_t)std::max<int64_t>(1, n));
    int64_t f0 = 0, fc = head[0];
    // The last level: when the frontier's entries reach most of the graph (sum of its degrees >= 1.5 n: a random
    // reach of 1 - e^-1.5 = 78 % or more), the last hop runs over every row with the full-graph kernel instead of
    // expanding the closure and listing it (rows outside the closure have unchanged inputs and come out bit-identical;
    // |R_{L+1}| is then reported as n). RAFTGP_STREAM_FULL_LAST=0 / 1 forces the listed / full last hop (tests).
    static const int full_last_env = [] {
        const char *e = getenv("RAFTGP_STREAM_FULL_LAST");
        return e ? atoi(e) : -1;
    }();
    const bool hops_started = rc == RAFTGP_OK;   // from here on the embedding state is being rewritten
    const bool delta_mode = s->mode == RAFTGP_STREAM_DELTA;
    // delta mode: dT[k] = T_k(new) - T_k(old) for the rows of R_k (list order; pos[] indexes it), or null when R_k is
    // too large for the changed-row gathers to pay (RAFTGP_STREAM_DELTA_FRAC = f: none when |R_k| f >= n, default 8;
    // 0: always kept) — the hop reading T_k then sums its rows in full
    std::vector<float *> dT(L + 2, nullptr);
    const char *fe = getenv("RAFTGP_STREAM_DELTA_FRAC");
    const int64_t frac = fe ? atoll(fe) : 8;
    float *Zs = s->Zs;     // delta mode: Z_h of the listed rows (full size, indexed by row), input of the transform
    auto clear_pos = [&](int k) {
        if (!dT[k] || counts[k] == 0) return;
        LaunchScope LS(ctx, K_STREAM);
        delta_clear<<<(unsigned)std::min<int64_t>(g256(counts[k]), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(rows, counts[k],
                                                                                                        s->pos);
    };
    for (int k = 1; k <= L + 1 && rc == RAFTGP_OK; ++k) {
        if (k == L + 1 && delta_mode) {   // the last hop by its changed inputs only (no level L + 1 expansion)
            if (counts[0] > 0) {
                int32_t *own = ng->order;
                if (!own && g->nl == ng->nl) ng->order = g->order;
                int64_t touched = 0;
                rc = launch_hop_delta(s, ng, L, nullptr, n, level, dT[L], dT[L] ? 0 : 1, s->Z, &touched);
                ng->order = own;
                counts[k] = touched;   // rows whose Z was rewritten
                if (rc == RAFTGP_OK) clear_pos(L);
            }
            break;
        }
        if (k == L + 1 && fc > 0 && full_last_env != 0) {
            bool full = full_last_env == 1;
            if (!full) {
                unsigned long long *ds = nullptr, hs = 0;
                rc = dalloc_t(ctx, &ds, 1);
                if (rc == RAFTGP_OK) rc = dzero(ctx, ds, sizeof(unsigned long long), st);
                if (rc == RAFTGP_OK) {
                    LaunchScope LS(ctx, K_STREAM);
                    const unsigned eg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(g256(fc), (int64_t)ctx->sm_count * 8));
                    frontier_degsum<<<eg, 256, 0, st>>>(rows, f0, fc, ng->deg_local, ds);
                }
                if (rc == RAFTGP_OK) rc = dread(ctx, &hs, ds, sizeof(hs), st);
                dfree(ctx, ds);
                if (rc != RAFTGP_OK) break;
                full = (double)hs >= 1.5 * (double)n;
            }
            if (full) {
                counts[k] = n;
                const auto &d = s->dims;
                int32_t *own = ng->order;   // the old graph's visiting order, borrowed for this launch
                if (!own && g->nl == ng->nl) ng->order = g->order;
                rc = gcn_hop(ng, s->T[L], d[L], s->Z, nullptr, 0, nullptr, 0, nullptr);
                ng->order = own;
                break;
            }
        }
        if (fc > 0) {
            LaunchScope LS(ctx, K_STREAM);
            const unsigned eg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(fc, 8), (int64_t)ctx->sm_count * 16));
            expand_frontier<<<eg, 256, 0, st>>>(ng->row_ptr, ng->col, level, rows, f0, fc, k, cnt);
        }
        RG_CHECK_LAUNCH(ctx);
        int32_t total = 0;
        rc = dread(ctx, &total, cnt, sizeof(int32_t), st);
        if (rc != RAFTGP_OK) break;
        f0 += fc;
        fc = total - f0;
        counts[k] = total;   // |R_k|: the list prefix
        const auto &d = s->dims;
        // the hop visits R_k with its heavy rows spread from the front (one per dynamic claim where possible), so no
        // hub is left for the end of the launch; a separate list: the frontier positions of `rows` stay intact
        // (a set covering much of the graph is first put in natural row order: row_ptr / col_idx then stream)
        const int32_t *list = rows;
        if (counts[k] * 8 >= n) {
            int32_t *flag = nullptr;
            int64_t *pos = nullptr;
            rc = dalloc_t(ctx, &flag, (size_t)n);
            if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &pos, (size_t)n + 1);
            if (rc == RAFTGP_OK) {
                const unsigned gg = (unsigned)std::min<int64_t>(g256(n), (int64_t)ctx->sm_count * 8);
                {
                    LaunchScope LS(ctx, K_STREAM);
                    level_flags<<<gg, 256, 0, st>>>(n, level, k, flag);
                }
                rc = scan_i32_to_i64(ctx, flag, pos, n);
                if (rc == RAFTGP_OK) {
                    LaunchScope LS(ctx, K_STREAM);
                    compact_rows<<<gg, 256, 0, st>>>(n, flag, pos, nat_rows);
                }
                list = nat_rows;
            }
            dfree(ctx, flag);
            dfree(ctx, pos);
        }
        if (rc == RAFTGP_OK) rc = spread_heavy_list(ctx, list, counts[k], ng->deg_local, hop_rows);
        if (rc == RAFTGP_OK && delta_mode && k >= 2) {   // GCN hop h = k - 1 over R_k from A_h and T_h's changed rows
            const int h = k - 1;
            if (rc == RAFTGP_OK) rc = launch_hop_delta(s, ng, h, hop_rows, counts[k], level, dT[h], dT[h] ? 0 : 1, Zs, nullptr);
            if (rc == RAFTGP_OK) clear_pos(h);
        }
        const int lpn = s->dims[k <= L ? k : L] / 4;
        if (rc == RAFTGP_OK && delta_mode && counts[k] > 0 && (frac <= 0 || counts[k] * frac < n)) {   // keep T_k(old)
            rc = dalloc_t(ctx, &dT[k], (size_t)counts[k] * s->dims[k]);
            if (rc == RAFTGP_OK) {
                LaunchScope LS(ctx, K_STREAM);
                delta_save<<<(unsigned)std::min<int64_t>(g256(counts[k] * lpn), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(
                    rows, counts[k], reinterpret_cast<const float4 *>(s->T[k]), lpn, s->pos, reinterpret_cast<float4 *>(dT[k]));
            }
        }
        if (rc != RAFTGP_OK) break;
        if (k == 1) {
            rc = feature_hop_pre_rows(ng, RAFTGP_NCUT, d[1], s->thw, nullptr, s->T[1], hop_rows, counts[1]);
        } else if (delta_mode) {   // T_k = s^ (.) (Z_{k-1} W_k) for the rows of R_k
            rc = gcn_transform_rows(ng, Zs, d[k - 1], s->W[k], d[k], s->T[k], hop_rows, counts[k]);
        } else {
            const int h = k - 1;   // GCN hop h reads T_h, writes T_{h+1} (or Z after the last layer)
            const bool last = h == L;
            rc = gcn_hop_rows(ng, s->T[h], d[h], last ? s->Z : nullptr, last ? nullptr : s->W[h + 1],
                              last ? 0 : d[h + 1], last ? nullptr : s->T[h + 1], hop_rows, counts[k]);
        }
        if (rc == RAFTGP_OK && dT[k]) {
            LaunchScope LS(ctx, K_STREAM);
            delta_finish<<<(unsigned)std::min<int64_t>(g256(counts[k] * lpn), (int64_t)ctx->sm_count * 8), 256, 0, st>>>(
                rows, counts[k], reinterpret_cast<const float4 *>(s->T[k]), lpn, reinterpret_cast<float4 *>(dT[k]));
        }
    }
    for (float *p : dT) dfree(ctx, p);
    dfree(ctx, add); dfree(ctx, level); dfree(ctx, rows); dfree(ctx, cnt); dfree(ctx, hop_rows); dfree(ctx, nat_rows);
    if (rc != RAFTGP_OK) {
        drop(*ng);
        delete ng;
        // the stream keeps its previous graph; once the hops ran, some rows (and the delta state) belong to the new
        // graph: further batches are refused until raftgp_stream_set_mode recomputes the state on the kept graph
        if (hops_started) s->stale = true;
        return rc;
    }
    // the stream now owns the merged graph; it inherits the visiting order (any permutation gives bit-identical
    // rows; this one spreads the old graph's heavy rows, which are still the heavy rows)
    if (!ng->order && g->order && g->nl == ng->nl) {
        ng->order = g->order;
        g->order = nullptr;
    }
    drop(*g);
    delete g;
    s->g = ng;
    if (stats) {
        for (int k = 0; k <= L + 1; ++k) stats[k] = counts[k];
        stats[L + 2] = ng->nnz_local;
    }
    return RAFTGP_OK;
}

void stream_destroy(raftgp_stream s) {
    if (!s) return;
    raftgp_ctx ctx = s->ctx;
    dfree(ctx, s->thw);
    for (auto t : s->T) dfree(ctx, t);
    for (auto w : s->W) dfree(ctx, w);
    dfree(ctx, s->Z);
    for (float *a : s->A) dfree(ctx, a);
    dfree(ctx, s->pos);
    dfree(ctx, s->Zs);
    if (s->g) {
        raftgp_graph_s &x = *s->g;
        dfree(ctx, x.row_ptr); dfree(ctx, x.col); dfree(ctx, x.deg_local); dfree(ctx, x.order); dfree(ctx, x.deg_all);
        dfree(ctx, x.s_all); dfree(ctx, x.sh_all); drop_slots(&x);
        delete s->g;
        ctx_release(ctx);
    }
    delete s;
    ctx_release(ctx);
}

// Both modes first recompute the exact chain over every row (so a switch, or setting DELTA again, removes any drift);
// RAFTGP_STREAM_DELTA then builds A[h] for every GCN hop by a full pass (Z keeps the exact values) and pos = -1.
raftgp_status stream_set_mode(raftgp_stream s, int32_t mode) {
    raftgp_graph g = s->g;
    raftgp_ctx ctx = s->ctx;
    const int64_t n = g->n;
    const int L = s->layers;
    RG_TRY(exact_chain(s));
    s->stale = false;
    if (mode == RAFTGP_STREAM_DELTA) {
        s->A.resize(L + 1, nullptr);
        for (int h = 1; h <= L; ++h)
            if (!s->A[h]) RG_TRY(dalloc_t(ctx, &s->A[h], (size_t)std::max<int64_t>(1, n) * s->dims[h]));
        if (!s->pos) RG_TRY(dalloc_t(ctx, &s->pos, (size_t)std::max<int64_t>(1, n)));
        int32_t maxd = 0;
        for (int q = 1; q < L; ++q) maxd = std::max(maxd, s->dims[q]);
        if (!s->Zs && maxd > 0) RG_TRY(dalloc_t(ctx, &s->Zs, (size_t)std::max<int64_t>(1, n) * maxd));
        if (n > 0) {
            LaunchScope LS(ctx, K_STREAM);
            fill_value<<<(unsigned)std::min<int64_t>(g256(n), (int64_t)ctx->sm_count * 8), 256, 0, ctx->stream>>>(n, s->pos,
                                                                                                                -1);
        }
        RG_CHECK_LAUNCH(ctx);
        for (int h = 1; h <= L; ++h) RG_TRY(launch_hop_delta(s, g, h, nullptr, n, nullptr, nullptr, 1, nullptr, nullptr));
        s->mode = mode;
        return RAFTGP_OK;
    }
    for (float *&a : s->A) {
        dfree(ctx, a);
        a = nullptr;
    }
    dfree(ctx, s->pos);
    dfree(ctx, s->Zs);
    s->pos = nullptr;
    s->Zs = nullptr;
    s->mode = RAFTGP_STREAM_EXACT;
    return RAFTGP_OK;
}

}  // namespace raftgp
