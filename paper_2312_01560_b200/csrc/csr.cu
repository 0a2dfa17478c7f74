// csr.cu — a1/a2 of the hot path: canonical CSR build of the simple undirected graph
// and the degree / normalisation pass (deg, 2e, s = D^-1/2 for M, s^ = (D+I)^-1/2 for
// Eq. 6's propagation matrix).
//
// Build pipeline (all on the ctx stream; csr_build, the default path for every graph whose buckets fit):
//   count        : CTA c (2 per SM) histograms its contiguous range of raw pairs into shared memory by COARSE bucket
//                  (2^cs consecutive local rows, <= kMaxCoarse buckets; both orientations of every u != v pair whose row
//                  is local) and writes per-(bucket, CTA) counts; ids outside [0, n) raise a device data-error flag.
//   scan         : exclusive scan of the counts -> every CTA's private region of every coarse bucket.
//   level 1      : csr_coarse_part, the same ranges: per tile, warp-private counts, a scan over the buckets, ranks into a
//                  shared-memory stage in bucket order, runs copied out with coalesced stores into the CTA's regions.
//   level 2      : csr_fine_count + scan + csr_fine_part split each coarse bucket into its fine buckets (2^shift rows,
//                  the bucket sort's unit) the same staged way; entries 32-bit packed when log2(B) + id bits <= 32.
//   bucket sort  : one CTA per fine bucket (persistent): counts its own rows, writes the raw row pointers, places the
//                  entries into rows in shared memory, sorts each row (one warp in registers up to 128 entries,
//                  groups of 4 warps by value sub-ranges beyond) and removes duplicates; the unique count is the
//                  degree. Buckets larger than shared memory are processed window by window; single rows longer
//                  than a window fall back to global placement + csr_sort_warp / csr_sort_block.
//   scan         : exclusive int64 scan of the degrees -> row_ptr; one host read-back (nnz, raw entry count,
//                  data-error flag).
//   compact      : copies each row's unique prefix into the final col array (skipped when no duplicate was
//                  dropped: the raw layout is then the CSR).
//   order        : degree-aware visiting order of the rows for the hop kernels (order.cu; one read-back).
//   degrees      : deg -> 2e, s, s^ and a degree histogram (whole-graph builds; one read-back).
// RAFTGP_CSR_TWO_LEVEL=0 (or > 2^32 raw entries) takes round 1's one-level partition instead (count by fine bucket,
// csr_partition: shared-memory ranks straight into bucket fronts claimed per tile). Graphs whose rows cannot be
// bucketed take the older per-row path: count (global atomics) -> scan -> scatter -> per-row warp / block sorts.
// The result is canonical (sorted, unique), hence independent of atomic ordering: bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace raftgp {

namespace {

constexpr int kScanBlock = 1024;
constexpr int kScanItems = 8;   // elements per thread per tile
constexpr int kWarpSortCap = 512;
constexpr int kBlockSortSmemCap = 24576;   // ints (96 KB)

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide inclusive scan of one int64 per thread (blockDim = kScanBlock)
__device__ __forceinline__ int64_t block_incl_scan(int64_t v, int64_t *sh_warp, int64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_incl_scan(v, lane);
    if (lane == 31) sh_warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < (kScanBlock / 32) ? sh_warp[lane] : 0;
        w = warp_incl_scan(w, lane);
        sh_warp[lane] = w;
    }
    __syncthreads();
    if (wid > 0) v += sh_warp[wid - 1];
    total = sh_warp[kScanBlock / 32 - 1];
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kScanBlock) scan_tile_sums(const int32_t *__restrict__ in, int64_t n,
                                                            int64_t *__restrict__ tile_sums) {
    __shared__ int64_t sh[32];
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * (int64_t)kScanBlock * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t idx = base + (int64_t)k * kScanBlock + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    int64_t total;
    block_incl_scan(s, sh, total);
    if (threadIdx.x == 0) tile_sums[tile] = total;
}

// single block: exclusive scan of the tile sums in place, total written to tile_sums[ntiles]
__global__ void __launch_bounds__(kScanBlock) scan_tile_offsets(int64_t *__restrict__ tile_sums, int64_t ntiles) {
    __shared__ int64_t sh[32];
    int64_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += kScanBlock) {
        int64_t idx = base + threadIdx.x;
        int64_t v = idx < ntiles ? tile_sums[idx] : 0;
        int64_t total;
        int64_t incl = block_incl_scan(v, sh, total);
        if (idx < ntiles) tile_sums[idx] = carry + incl - v;
        carry += total;
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

__global__ void __launch_bounds__(kScanBlock) scan_apply(const int32_t *__restrict__ in, int64_t n,
                                                        const int64_t *__restrict__ tile_off,
                                                        int64_t *__restrict__ out) {
    __shared__ int64_t sh[32];
    const int64_t tile = blockIdx.x;
    // each thread owns kScanItems CONSECUTIVE elements so the scan is in order
    const int64_t base = tile * (int64_t)kScanBlock * kScanItems + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        s += v[k];
    }
    int64_t total;
    int64_t incl = block_incl_scan(s, sh, total);
    int64_t run = tile_off[tile] + incl - s;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (tile == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_off[gridDim.x];
}

// ---------------------------------------------------------------- count / scatter
__global__ void csr_count(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t m, int64_t n,
                          int64_t rb, int64_t re, int32_t *__restrict__ cnt, int *__restrict__ err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const int32_t u = __ldg(src + e), v = __ldg(dst + e);
        if (u < 0 || v < 0 || u >= n || v >= n) {
            atomicOr(err, 1);
            continue;
        }
        if (u == v) continue;
        if (u >= rb && u < re) atomicAdd(cnt + (u - rb), 1);
        if (v >= rb && v < re) atomicAdd(cnt + (v - rb), 1);
    }
}

// cnt counts down to 0 again while slots are claimed
__global__ void csr_scatter(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t m, int64_t n,
                            int64_t rb, int64_t re, const int64_t *__restrict__ raw_ptr, int32_t *__restrict__ cnt,
                            int32_t *__restrict__ col_raw) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const int32_t u = __ldg(src + e), v = __ldg(dst + e);
        if (u < 0 || v < 0 || u >= n || v >= n || u == v) continue;
        if (u >= rb && u < re) {
            const int32_t k = atomicSub(cnt + (u - rb), 1) - 1;
            col_raw[raw_ptr[u - rb] + k] = v;
        }
        if (v >= rb && v < re) {
            const int32_t k = atomicSub(cnt + (v - rb), 1) - 1;
            col_raw[raw_ptr[v - rb] + k] = u;
        }
    }
}

// ---------------------------------------------------------------- sort + dedup
// In-place ascending bitonic sort of a[0..len) for ANY len, all stages ascending ("flip" form):
// virtual +inf padding beyond len never moves, so no padding storage is needed.
// Work is split over `nthr` threads with index t; `sync` is the barrier between stages.
template <typename Sync>
__device__ __forceinline__ void bitonic_any(int32_t *a, int len, int t, int nthr, Sync sync) {
    int lg = 0;
    while ((1 << lg) < len) ++lg;
    const int half = (1 << lg) >> 1;      // compare-exchange pairs per stage
    for (int lk = 1; lk <= lg; ++lk) {
        // flip stage of block size k = 2^lk: i in the lower half of its k-block, partner = its mirror
        const int lh = lk - 1;
        for (int x = t; x < half; x += nthr) {
            const int i = ((x >> lh) << lk) | (x & ((1 << lh) - 1));
            const int j = i ^ ((1 << lk) - 1);
            if (j < len) {
                const int32_t ai = a[i], aj = a[j];
                if (ai > aj) { a[i] = aj; a[j] = ai; }
            }
        }
        sync();
        for (int lj = lk - 2; lj >= 0; --lj) {
            for (int x = t; x < half; x += nthr) {
                const int i = ((x >> lj) << (lj + 1)) | (x & ((1 << lj) - 1));
                const int j = i + (1 << lj);
                if (j < len) {
                    const int32_t ai = a[i], aj = a[j];
                    if (ai > aj) { a[i] = aj; a[j] = ai; }
                }
            }
            sync();
        }
    }
}

struct WarpSync {
    __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct BlockSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// barrier over a group of `nthreads` threads (named barrier `id`, 1..15)
struct GroupSync {
    int id, nthreads;
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
    }
};

// warp register bitonic sort of 32 values (ascending by lane)
// ascending bitonic sort of the first N lanes' values (N = 8, 16, 32; the other lanes hold INT_MAX padding)
template <int N = 32>
__device__ __forceinline__ int32_t warp_sort32(int32_t v, int lane) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j >= 1; j >>= 1) {
            const int32_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = ((lane & k) == 0);
            const bool lower = ((lane & j) == 0);
            // lower partner keeps min when ascending block, max when descending
            const int32_t mn = min(v, o), mx = max(v, o);
            v = (lower == up) ? mn : mx;
        }
    }
    return v;
}

// one warp per row; rows longer than kWarpSortCap are pushed to big_rows
__global__ void __launch_bounds__(256) csr_sort_warp(int64_t nl, const int64_t *__restrict__ rows_list,
                                                     const int32_t *__restrict__ rows_count,
                                                     const int64_t *__restrict__ raw_ptr,
                                                     int32_t *__restrict__ col_raw, int32_t *__restrict__ deg,
                                                     int64_t *__restrict__ big_rows, int32_t *__restrict__ big_count) {
    __shared__ int32_t sh[8][kWarpSortCap];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps = (int64_t)gridDim.x * 8;
    const int64_t nrows = rows_list ? *rows_count : nl;
    for (int64_t it = (int64_t)blockIdx.x * 8 + wib; it < nrows; it += warps) {
        const int64_t row = rows_list ? rows_list[it] : it;
        const int64_t beg = raw_ptr[row];
        const int len = static_cast<int>(raw_ptr[row + 1] - beg);
        int32_t *a = col_raw + beg;
        if (len <= 32) {
            int32_t v = lane < len ? a[lane] : INT_MAX;
            v = warp_sort32(v, lane);
            const int32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
            const bool keep = lane < len && (lane == 0 || v != prev);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) a[__popc(bal & ((1u << lane) - 1u))] = v;
            if (lane == 0) deg[row] = __popc(bal);
        } else if (len <= kWarpSortCap) {
            int32_t *s = sh[wib];
            for (int x = lane; x < len; x += 32) s[x] = a[x];
            __syncwarp();
            bitonic_any(s, len, lane, 32, WarpSync());
            int written = 0;
            for (int base = 0; base < len; base += 32) {
                const int x = base + lane;
                const int32_t v = x < len ? s[x] : INT_MAX;
                const bool keep = x < len && (x == 0 || v != s[x - 1]);
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep) a[written + __popc(bal & ((1u << lane) - 1u))] = v;
                written += __popc(bal);
            }
            if (lane == 0) deg[row] = written;
            __syncwarp();
        } else if (lane == 0) {
            big_rows[atomicAdd(big_count, 1)] = row;
        }
    }
}

// one block (1024 threads) per long row
__global__ void __launch_bounds__(1024) csr_sort_block(const int64_t *__restrict__ big_rows,
                                                       const int32_t *__restrict__ big_count,
                                                       const int64_t *__restrict__ raw_ptr,
                                                       int32_t *__restrict__ col_raw, int32_t *__restrict__ deg) {
    extern __shared__ int32_t smem[];
    __shared__ int32_t wsum[32];
    const int nb = *big_count;
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t row = big_rows[b];
        const int64_t beg = raw_ptr[row];
        const int len = static_cast<int>(raw_ptr[row + 1] - beg);
        int32_t *a = col_raw + beg;
        int32_t *s = len <= kBlockSortSmemCap ? smem : a;
        if (s == smem) {
            for (int x = threadIdx.x; x < len; x += blockDim.x) s[x] = a[x];
        }
        __syncthreads();
        bitonic_any(s, len, (int)threadIdx.x, (int)blockDim.x, BlockSync());
        // dedup with a block scan over chunks of blockDim, writing in place (writes never pass reads)
        int written = 0;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int base = 0; base < len; base += blockDim.x) {
            const int x = base + threadIdx.x;
            const int32_t v = x < len ? s[x] : INT_MAX;
            const bool keep = x < len && (x == 0 || v != s[x - 1]);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) wsum[wid] = __popc(bal);
            __syncthreads();
            int before = 0, total = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                if (w < wid) before += wsum[w];
                total += wsum[w];
            }
            __syncthreads();   // all reads of s[x-1] in this chunk done before anyone writes
            if (keep) a[written + before + __popc(bal & ((1u << lane) - 1u))] = v;
            written += total;
            __syncthreads();
        }
        if (threadIdx.x == 0) deg[row] = written;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- bucketed build (main path)
// Rows are grouped in buckets of B = 2^shift consecutive rows. Pass "partition" moves every directed entry
// (local row, neighbour) into its bucket's region of `pairs` (the bucket's rows' raw segments, back to
// back): per tile a shared-memory histogram, ONE global atomic per (tile, bucket) to reserve space, then
// shared-memory ranks — no per-entry global atomics. Pass "bucket_sort" gives each bucket to one CTA, which
// places the entries into their rows in shared memory, sorts and dedups every row (one warp per row) and
// writes the unique prefix of each row to col_raw. Buckets that do not fit shared memory are placed into
// col_raw in global memory and their rows handed to the warp / block sort kernels above.
#ifndef RG_PART_TILE
#define RG_PART_TILE 16384
#endif
constexpr int kPartTile = RG_PART_TILE;   // raw pairs per partition tile
#ifndef RG_PART_UNROLL
#define RG_PART_UNROLL 16
#endif
constexpr int kPartUnroll = RG_PART_UNROLL;   // edge loads in flight per thread
constexpr int kMaxBuckets = 12288;      // partition smem with 64-bit bucket cursors: 12 B per bucket
constexpr int kMaxBuckets32 = 24576;    // with 32-bit cursors (raw entry count < 2^32): 8 B per bucket
constexpr int kMaxBucketRows = 4096;    // bucket_sort smem for row cursors/offsets
constexpr int kBucketCap = 44032;       // entries of one bucket held in shared memory (172 KB)
#ifndef RG_GROUP_ROW
#define RG_GROUP_ROW 128
#endif
constexpr int kGroupRow = RG_GROUP_ROW;   // rows longer than this are sorted by a group of 4 warps

// Bucket entries: (row within the bucket, neighbour id). PACKED = one 32-bit word (row << vbits | id) when
// log2(B) + vbits <= 32 (C4: 9 + 23 bits), else an int2.
template <bool PACKED>
struct Entry;
template <>
struct Entry<true> {
    using T = uint32_t;
    __device__ __forceinline__ static T make(int lr, int32_t v, int vbits) {
        return (static_cast<uint32_t>(lr) << vbits) | static_cast<uint32_t>(v);
    }
    __device__ __forceinline__ static int row(T e, int vbits) { return static_cast<int>(e >> vbits); }
    __device__ __forceinline__ static int32_t col(T e, int vbits) {
        return static_cast<int32_t>(e & ((vbits < 32 ? (1u << vbits) : 0u) - 1u));
    }
    __device__ __forceinline__ static T invalid() { return 0xffffffffu; }
    __device__ __forceinline__ static bool valid(T e) { return e != 0xffffffffu; }
};
template <>
struct Entry<false> {
    using T = int2;
    __device__ __forceinline__ static T make(int lr, int32_t v, int) { return make_int2(lr, v); }
    __device__ __forceinline__ static int row(T e, int) { return e.x; }
    __device__ __forceinline__ static int32_t col(T e, int) { return e.y; }
    __device__ __forceinline__ static T invalid() { return make_int2(-1, 0); }
    __device__ __forceinline__ static bool valid(T e) { return e.x >= 0; }
};

// Radix-style bucket partition of the raw entries (both orientations of every valid pair, local rows only)
// into buckets of 2^shift consecutive local rows. csr_bucket_count: CTA c histograms its contiguous edge range
// into shared memory and writes the counts bucket-major (cnt[b * G + c], no global atomics); an exclusive scan
// gives the bucket starts base[b * G] (and the bucket sizes the bucket sort needs). The order of the entries
// inside a bucket is irrelevant: the bucket sort sorts every row. The count pass also checks the node ids.
__device__ __forceinline__ void cta_range(int64_t m, int64_t &e0, int64_t &e1) {
    const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
    e0 = min(m, (int64_t)blockIdx.x * chunk);
    e1 = min(m, e0 + chunk);
}

__global__ void __launch_bounds__(1024) csr_bucket_count(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                                         int64_t m, int64_t n, int64_t rb, int64_t re, int shift,
                                                         int nb, int32_t *__restrict__ cnt, int *__restrict__ err) {
    extern __shared__ unsigned int hsm[];
    int64_t e0, e1;
    cta_range(m, e0, e1);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) hsm[b] = 0u;
    __syncthreads();
    bool bad = false;
    for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += kPartUnroll * (int64_t)blockDim.x) {
        int32_t us[kPartUnroll], vs[kPartUnroll];
#pragma unroll
        for (int k = 0; k < kPartUnroll; ++k) {
            const int64_t e = eb + (int64_t)k * blockDim.x;
            us[k] = e < e1 ? __ldg(src + e) : 0;
            vs[k] = e < e1 ? __ldg(dst + e) : 0;
        }
#pragma unroll
        for (int k = 0; k < kPartUnroll; ++k) {
            const int32_t u = us[k], v = vs[k];
            if (u < 0 || v < 0 || u >= n || v >= n) {
                bad = true;
                continue;
            }
            if (u == v) continue;
            if (u >= rb && u < re) atomicAdd(&hsm[(u - rb) >> shift], 1u);
            if (v >= rb && v < re) atomicAdd(&hsm[(v - rb) >> shift], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[(int64_t)b * gridDim.x + blockIdx.x] = (int32_t)hsm[b];
    if (bad) atomicOr(err, 1);
}

// The scatter pass runs over tiles of kPartTile edges claimed round robin: each tile histograms its entries
// in shared memory, claims one contiguous slot range per bucket with a global atomic on the bucket cursor
// (initialised to the bucket start), then writes. Concurrent tiles thus fill neighbouring slots of every
// bucket, which keeps the scattered writes sector-local in L2 (per-CTA fixed offsets, i.e. an atomic-free
// scatter, measured 2x slower: DESIGN.md "tried and rejected").
__global__ void csr_bucket_cursor(const int64_t *__restrict__ base, int pgrid, int nb,
                                  unsigned long long *__restrict__ bcur) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb) bcur[b] = (unsigned long long)base[(int64_t)b * pgrid];
}

template <bool PACKED, typename BT>
__global__ void __launch_bounds__(1024) csr_partition(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                                      int64_t m, int64_t n, int64_t rb, int64_t re, int shift, int nb,
                                                      int vbits, int64_t ptile, unsigned long long *__restrict__ bcur,
                                                      typename Entry<PACKED>::T *__restrict__ pairs) {
    using E = Entry<PACKED>;
    extern __shared__ __align__(8) unsigned char psm_raw[];
    BT *base = reinterpret_cast<BT *>(psm_raw);                                       // nb slot bases
    unsigned int *hist = reinterpret_cast<unsigned int *>(psm_raw + sizeof(BT) * nb);  // nb
    const int bmask = (1 << shift) - 1;
    const int64_t ntiles = (m + ptile - 1) / ptile;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t e0 = tile * ptile;
        const int64_t e1 = min(m, e0 + ptile);
        for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0u;
        __syncthreads();
        for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += kPartUnroll * (int64_t)blockDim.x) {
            int32_t us[kPartUnroll], vs[kPartUnroll];
#pragma unroll
            for (int k = 0; k < kPartUnroll; ++k) {
                const int64_t e = eb + (int64_t)k * blockDim.x;
                us[k] = e < e1 ? __ldg(src + e) : -1;
                vs[k] = e < e1 ? __ldg(dst + e) : -1;
            }
#pragma unroll
            for (int k = 0; k < kPartUnroll; ++k) {
                const int32_t u = us[k], v = vs[k];
                if (u < 0 || v < 0 || u >= n || v >= n || u == v) continue;
                if (u >= rb && u < re) atomicAdd(&hist[(u - rb) >> shift], 1u);
                if (v >= rb && v < re) atomicAdd(&hist[(v - rb) >> shift], 1u);
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const unsigned int h = hist[b];
            if (h) base[b] = (BT)atomicAdd(&bcur[b], (unsigned long long)h);
            hist[b] = 0u;
        }
        __syncthreads();
        for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += kPartUnroll * (int64_t)blockDim.x) {
            int32_t us[kPartUnroll], vs[kPartUnroll];
#pragma unroll
            for (int k = 0; k < kPartUnroll; ++k) {
                const int64_t e = eb + (int64_t)k * blockDim.x;
                us[k] = e < e1 ? __ldg(src + e) : -1;
                vs[k] = e < e1 ? __ldg(dst + e) : -1;
            }
#pragma unroll
            for (int k = 0; k < kPartUnroll; ++k) {
                const int32_t u = us[k], v = vs[k];
                if (u < 0 || v < 0 || u >= n || v >= n || u == v) continue;
                if (u >= rb && u < re) {
                    const int b = static_cast<int>((u - rb) >> shift);
                    pairs[base[b] + atomicAdd(&hist[b], 1u)] = E::make(static_cast<int>(u - rb) & bmask, v, vbits);
                }
                if (v >= rb && v < re) {
                    const int b = static_cast<int>((v - rb) >> shift);
                    pairs[base[b] + atomicAdd(&hist[b], 1u)] = E::make(static_cast<int>(v - rb) & bmask, u, vbits);
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- two-level partition (default)
// The one-level partition above writes every entry straight to its bucket front: with ~10^4 buckets shared by all
// SMs each warp store touches 32 different sectors that other SMs are writing too, and the stores bound it
// (microbenchmark, 10^8 pairs: ranks alone 0.6 ms, with the scattered stores 5 ms). The two-level path stages
// every tile in shared memory in bucket order and writes each bucket's run of the tile with coalesced stores
// into a region no other CTA writes:
//   level 1 (csr_coarse_part): CTA c takes the same contiguous range of raw pairs as in the count pass, whose
//            per-(coarse bucket, CTA) counts give it a private region of every coarse bucket (2^cs rows, <=
//            kMaxCoarse buckets); per tile of kCT pairs: warp-private counts -> scan over buckets -> ranks into
//            the stage (shared-memory atomics on the warp's own counters) -> runs copied out. Entries are
//            (row in coarse bucket, neighbour) int2.
//   level 2 (csr_fine_part): one CTA per coarse bucket counts its F = 2^(cs - shift) fine buckets (2^shift rows,
//            the bucket sort's unit), writes their starts, then splits the coarse bucket tile by tile the same
//            way into Entry<PACKED> form.
// Both are deterministic (no global atomics); the bucket sort makes the result canonical anyway.
constexpr int kPT = 512;           // threads of the level-1 / level-2 CTAs (2 CTAs per SM: one stages while the other loads)
constexpr int kPW = kPT / 32;
constexpr int kCT = 4096;          // level-1 tile: pairs (8 per thread)
constexpr int kFT = 4096;          // level-2 tile: entries (8 per thread)
constexpr int kMaxCoarse = 512;    // level-1 buckets (kPW warp-private counters each: 32 KB)
constexpr int kMaxFine = 256;      // fine buckets per coarse bucket

// bins <= kPT bucket counters held per warp in cnt[kPW][nb]: totals -> tot, exclusive scan over the buckets ->
// ls, and every warp's counter becomes its first slot (ls + the counts of the lower warps). kPT threads; the
// caller syncs before (counts complete) and after.
__device__ __forceinline__ void bins_scan(unsigned *cnt, int nbins, unsigned *ls, unsigned *tot, unsigned *wsum) {
    const int b = threadIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned t = 0u;
    if (b < nbins)
#pragma unroll 8
        for (int w = 0; w < kPW; ++w) t += cnt[w * nbins + b];
    unsigned x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const unsigned y = lane < kPW ? wsum[lane] : 0u;
        unsigned z = y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned q = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += q;
        }
        if (lane < kPW) wsum[lane] = z - y;
    }
    __syncthreads();
    if (b < nbins) {
        unsigned p = wsum[wid] + x - t;
        ls[b] = p;
        tot[b] = t;
#pragma unroll 8
        for (int w = 0; w < kPW; ++w) {
            const unsigned c = cnt[w * nbins + b];
            cnt[w * nbins + b] = p;
            p += c;
        }
    }
}

__host__ __device__ constexpr size_t coarse_smem(int nc) { return (size_t)2 * kCT * 8 + ((size_t)(kPW + 3) * nc) * 4; }
__host__ __device__ constexpr size_t fine_smem(int F) { return (size_t)kFT * 8 + ((size_t)(kPW + 3) * F) * 4; }

__global__ void __launch_bounds__(kPT) csr_coarse_part(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                                        int64_t m, int64_t n, int64_t rb, int64_t re, int cs, int nc,
                                                        const int64_t *__restrict__ bstart, int2 *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char cp_raw[];
    int2 *stage = reinterpret_cast<int2 *>(cp_raw);              // 2 kCT entries in coarse-bucket order
    unsigned *cnt = reinterpret_cast<unsigned *>(stage + 2 * kCT);   // [kPW][nc] warp-private counters
    unsigned *ls = cnt + kPW * nc, *tot = ls + nc, *gcur = tot + nc;  // tile run starts / lengths, region cursors
    __shared__ unsigned wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned *my = cnt + wid * nc;
    const int cmask = (1 << cs) - 1;
    int64_t e0, e1;
    cta_range(m, e0, e1);
    for (int b = threadIdx.x; b < nc; b += blockDim.x) gcur[b] = (unsigned)bstart[(int64_t)b * gridDim.x + blockIdx.x];
    for (int64_t t0 = e0; t0 < e1; t0 += kCT) {
        const int64_t w0 = min(e1, t0 + (int64_t)wid * (kCT / kPW)), w1 = min(e1, w0 + kCT / kPW);
        for (int b = lane; b < nc; b += 32) my[b] = 0u;
        __syncwarp();
        int32_t lu[kCT / kPT], lv[kCT / kPT];   // local rows (or -1: no entry for this orientation)
        int32_t us[kCT / kPT], vs[kCT / kPT];
#pragma unroll
        for (int k = 0; k < kCT / kPT; ++k) {
            const int64_t e = w0 + lane + 32 * k;
            us[k] = e < w1 ? __ldg(src + e) : -1;
            vs[k] = e < w1 ? __ldg(dst + e) : -1;
        }
#pragma unroll
        for (int k = 0; k < kCT / kPT; ++k) {
            const int32_t u = us[k], v = vs[k];
            const bool valid = u >= 0 && v >= 0 && u < n && v < n && u != v;
            lu[k] = (valid && u >= rb && u < re) ? static_cast<int32_t>(u - rb) : -1;
            lv[k] = (valid && v >= rb && v < re) ? static_cast<int32_t>(v - rb) : -1;
            if (lu[k] >= 0) atomicAdd(&my[lu[k] >> cs], 1u);
            if (lv[k] >= 0) atomicAdd(&my[lv[k] >> cs], 1u);
        }
        __syncthreads();
        bins_scan(cnt, nc, ls, tot, wsum);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kCT / kPT; ++k) {
            if (lu[k] >= 0) stage[atomicAdd(&my[lu[k] >> cs], 1u)] = make_int2(lu[k], vs[k]);
            if (lv[k] >= 0) stage[atomicAdd(&my[lv[k] >> cs], 1u)] = make_int2(lv[k], us[k]);
        }
        __syncthreads();
        const unsigned ntile = ls[nc - 1] + tot[nc - 1];
        for (unsigned i = threadIdx.x; i < ntile; i += blockDim.x) {
            const int2 e = stage[i];
            const int b = e.x >> cs;
            out[gcur[b] + (i - ls[b])] = make_int2(e.x & cmask, e.y);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nc; b += blockDim.x) gcur[b] += tot[b];
    }
}

#ifndef RG_FINE_SLOTS
#define RG_FINE_SLOTS 8
#endif
constexpr int kFineSlots = RG_FINE_SLOTS;   // CTAs per coarse bucket in level 2 (blockIdx.x), tiles dealt round robin

// Level 2a: fine bucket sizes. CTA (j, c) counts the tiles j, j + J, ... of coarse bucket c into its warp-private
// counters and adds the CTA totals to fcnt[c * F + f] (one global atomic per fine bucket and CTA).
__global__ void __launch_bounds__(kPT) csr_fine_count(const int2 *__restrict__ in, const int64_t *__restrict__ cstart,
                                                       int pgrid, int shift, int fbits, int nb,
                                                       int32_t *__restrict__ fcnt) {
    __shared__ unsigned cnt[kPW][kMaxFine];
    const int F = 1 << fbits, c = blockIdx.y;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t cb = cstart[(int64_t)c * pgrid], ce = cstart[(int64_t)(c + 1) * pgrid];
    for (int f = lane; f < F; f += 32) cnt[wid][f] = 0u;
    __syncwarp();
    constexpr int kPer = kFT / kPT;
    for (int64_t t0 = cb + (int64_t)blockIdx.x * kFT; t0 < ce; t0 += (int64_t)gridDim.x * kFT) {
        const int64_t t1 = min(ce, t0 + kFT);
        int2 p[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t e = t0 + threadIdx.x + (int64_t)k * kPT;
            p[k] = e < t1 ? __ldg(in + e) : make_int2(-1, 0);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (p[k].x >= 0) atomicAdd(&cnt[wid][p[k].x >> shift], 1u);
    }
    __syncthreads();
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        unsigned t = 0u;
        for (int w = 0; w < kPW; ++w) t += cnt[w][f];
        const int64_t gf = (int64_t)c * F + f;
        if (t && gf < nb) atomicAdd(&fcnt[gf], (int32_t)t);
    }
}

// Level 2b: CTA (j, c) splits the tiles j, j + J, ... of coarse bucket c: per tile warp-private counts, a scan over
// the F fine buckets, one global claim per fine bucket on its cursor, ranks into the stage, runs copied out.
template <bool PACKED>
__global__ void __launch_bounds__(kPT) csr_fine_part(const int2 *__restrict__ in, const int64_t *__restrict__ cstart,
                                                      int pgrid, int shift, int fbits, int vbits,
                                                      unsigned long long *__restrict__ fcur,
                                                      typename Entry<PACKED>::T *__restrict__ out) {
    using E = Entry<PACKED>;
    extern __shared__ __align__(16) unsigned char fp_raw[];
    const int F = 1 << fbits, fmask = (1 << shift) - 1, c = blockIdx.y;
    int2 *stage = reinterpret_cast<int2 *>(fp_raw);               // kFT entries in fine-bucket order
    unsigned *cnt = reinterpret_cast<unsigned *>(stage + kFT);    // [kPW][F]
    unsigned *ls = cnt + kPW * F, *tot = ls + F, *gcur = tot + F;
    __shared__ unsigned wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned *my = cnt + wid * F;
    constexpr int kPer = kFT / kPT;
    const int64_t cb = cstart[(int64_t)c * pgrid], ce = cstart[(int64_t)(c + 1) * pgrid];
    for (int64_t t0 = cb + (int64_t)blockIdx.x * kFT; t0 < ce; t0 += (int64_t)gridDim.x * kFT) {
        const int64_t t1 = min(ce, t0 + kFT);
        for (int f = lane; f < F; f += 32) my[f] = 0u;
        __syncwarp();
        int2 p[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t e = t0 + wid * (kFT / kPW) + lane + 32 * k;
            p[k] = e < t1 ? __ldg(in + e) : make_int2(-1, 0);
            if (p[k].x >= 0) atomicAdd(&my[p[k].x >> shift], 1u);
        }
        __syncthreads();
        bins_scan(cnt, F, ls, tot, wsum);
        for (int f = threadIdx.x; f < F; f += blockDim.x)
            if (tot[f]) gcur[f] = (unsigned)atomicAdd(&fcur[(int64_t)c * F + f], (unsigned long long)tot[f]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (p[k].x >= 0) stage[atomicAdd(&my[p[k].x >> shift], 1u)] = p[k];
        __syncthreads();
        const unsigned ntile = static_cast<unsigned>(t1 - t0);
        for (unsigned i = threadIdx.x; i < ntile; i += blockDim.x) {
            const int2 e = stage[i];
            const int f = e.x >> shift;
            out[gcur[f] + (i - ls[f])] = E::make(e.x & fmask, e.y, vbits);
        }
        __syncthreads();
    }
}

// Register bitonic sort of up to 32*E values per warp: element e of lane l has index e*32 + l; stages with
// j >= 32 swap inside a lane, the others exchange by shuffle. Then dedup and write the unique prefix.
template <int E>
__device__ __forceinline__ int warp_sort_dedup_reg(const int32_t *a, int len, int32_t *outp, int lane) {
    int32_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = (e * 32 + lane < len) ? a[e * 32 + lane] : INT_MAX;
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j >= 1; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int e2 = e ^ (j >> 5);
                    if (e2 > e) {
                        const bool up = (((e * 32 + lane) & k) == 0);
                        const int32_t lo = min(v[e], v[e2]), hi = max(v[e], v[e2]);
                        v[e] = up ? lo : hi;
                        v[e2] = up ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int32_t o = __shfl_xor_sync(0xffffffffu, v[e], j);
                    const bool up = (((e * 32 + lane) & k) == 0);
                    const bool lower = ((lane & j) == 0);
                    v[e] = (lower == up) ? min(v[e], o) : max(v[e], o);
                }
            }
        }
    }
    int written = 0;
    int32_t last_prev = INT_MIN;   // last element of the previous 32-chunk (lane 31's value)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int32_t prev = __shfl_up_sync(0xffffffffu, v[e], 1);
        if (lane == 0) prev = last_prev;
        const int idx = e * 32 + lane;
        const bool keep = idx < len && (idx == 0 || v[e] != prev);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) outp[written + __popc(bal & ((1u << lane) - 1u))] = v[e];
        written += __popc(bal);
        last_prev = __shfl_sync(0xffffffffu, v[e], 31);
    }
    return written;
}

// warp sort + dedup of one row held in shared memory; writes the unique prefix to outp, returns its length
// SHORT: rows of <= 8 / 16 entries take the 6- / 10-stage networks (the packed-entry kernel, C4's: bucket sort
// 3.48 -> 3.29 ms); the unpacked kernel (C5's) keeps the single network — with the extra branches the compiler
// gave it 32 registers and spills instead of 55 (bucket sort 36.5 -> 39.8 ms at C5)
template <bool SHORT>
__device__ __forceinline__ int warp_sort_dedup(int32_t *a, int len, int32_t *outp, int lane) {
    if (len <= 32) {   // rows of <= 8 / 16 entries (a third of C4's rows) take the shorter networks
        int32_t v = lane < len ? a[lane] : INT_MAX;
        if constexpr (SHORT)
            v = len <= 8 ? warp_sort32<8>(v, lane) : len <= 16 ? warp_sort32<16>(v, lane) : warp_sort32<32>(v, lane);
        else
            v = warp_sort32<32>(v, lane);
        const int32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
        const bool keep = lane < len && (lane == 0 || v != prev);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) outp[__popc(bal & ((1u << lane) - 1u))] = v;
        return __popc(bal);
    }
    if (len <= 64) return warp_sort_dedup_reg<2>(a, len, outp, lane);
    if (len <= 128) return warp_sort_dedup_reg<4>(a, len, outp, lane);
    bitonic_any(a, len, lane, 32, WarpSync());
    int written = 0;
    for (int base = 0; base < len; base += 32) {
        const int x = base + lane;
        const int32_t v = x < len ? a[x] : INT_MAX;
        const bool keep = x < len && (x == 0 || v != a[x - 1]);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) outp[written + __popc(bal & ((1u << lane) - 1u))] = v;
        written += __popc(bal);
    }
    return written;
}

// in-place ascending warp sort of a[0..len) (registers up to 128 values, shared-memory bitonic beyond)
template <int E>
__device__ __forceinline__ void warp_sort_reg_inplace(int32_t *a, int len, int lane) {
    int32_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = (e * 32 + lane < len) ? a[e * 32 + lane] : INT_MAX;
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j >= 1; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int e2 = e ^ (j >> 5);
                    if (e2 > e) {
                        const bool up = (((e * 32 + lane) & k) == 0);
                        const int32_t lo = min(v[e], v[e2]), hi = max(v[e], v[e2]);
                        v[e] = up ? lo : hi;
                        v[e2] = up ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int32_t o = __shfl_xor_sync(0xffffffffu, v[e], j);
                    const bool up = (((e * 32 + lane) & k) == 0);
                    const bool lower = ((lane & j) == 0);
                    v[e] = (lower == up) ? min(v[e], o) : max(v[e], o);
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (e * 32 + lane < len) a[e * 32 + lane] = v[e];
    __syncwarp();
}

template <bool SHORT>
__device__ __forceinline__ void warp_sort_inplace(int32_t *a, int len, int lane) {
    if (len <= 1) return;
    if (len <= 32) {
        int32_t v = lane < len ? a[lane] : INT_MAX;
        if constexpr (SHORT)
            v = len <= 8 ? warp_sort32<8>(v, lane) : len <= 16 ? warp_sort32<16>(v, lane) : warp_sort32<32>(v, lane);
        else
            v = warp_sort32<32>(v, lane);
        __syncwarp();
        if (lane < len) a[lane] = v;
        __syncwarp();
    } else if (len <= 64) {
        warp_sort_reg_inplace<2>(a, len, lane);
    } else if (len <= 128) {
        warp_sort_reg_inplace<4>(a, len, lane);
    } else {
        bitonic_any(a, len, lane, 32, WarpSync());
    }
}

#ifndef RG_SUB_AVG
#define RG_SUB_AVG 32
#endif
constexpr int kSubAvg = RG_SUB_AVG;   // mean entries per value sub-range when a long row is split for sorting

// 4 group-shared counters per 4-warp group for the dedup of long rows. The row cursors `cur` of the rows
// being sorted are still needed when a bucket is processed window by window, so the counters live at the
// top of the cursor array (kMaxBucketRows slots; a bucket has at most kMaxBucketRows rows, and the window
// path only runs for buckets of that size... so they use a separate small shared array instead).
__device__ __forceinline__ int32_t *gtmp_cnt(int32_t *cur, int nr, int grp) {
    __shared__ int32_t wcnt[8][4];
    (void)cur;
    (void)nr;
    return wcnt[grp];
}

template <bool PACKED>
__global__ void __launch_bounds__(1024) csr_bucket_sort(const typename Entry<PACKED>::T *__restrict__ pairs,
                                                        const int64_t *__restrict__ base, int pgrid,
                                                        int64_t *__restrict__ raw_ptr,
                                                        int64_t nl, int shift, int nb, int vbits,
                                                        int32_t *__restrict__ col_raw, int32_t *__restrict__ deg,
                                                        int64_t *__restrict__ fb_rows, int32_t *__restrict__ fb_count,
                                                        unsigned int *__restrict__ bnext, int cap) {
    extern __shared__ int32_t bsm[];
    int32_t *s = bsm;                                   // cap (<= kBucketCap) values
    int32_t *cur = bsm + kBucketCap;                    // B cursors (first: the row counts)
    int32_t *off = cur + kMaxBucketRows;                // B + 1 offsets (relative to the bucket start)
    int32_t *big = off + kMaxBucketRows + 1;            // rows longer than kGroupRow
    __shared__ int nbig, qnext, tail, wend;
    __shared__ int gtmp[8];
    __shared__ int64_t scan_sh[32];
    const int lane = threadIdx.x & 31;
    constexpr int kLoadBatch = 8;
    constexpr int kRowsPerThread = kMaxBucketRows / 1024;
    __shared__ int bclaim;
    for (;;) {   // buckets claimed dynamically (their sizes and hub rows vary)
        if (threadIdx.x == 0) bclaim = (int)atomicAdd(bnext, 1u);
        __syncthreads();
        const int b = bclaim;
        if (b >= nb) break;
        const int64_t r0 = (int64_t)b << shift;
        const int nr = static_cast<int>(min(nl, r0 + ((int64_t)1 << shift)) - r0);
        const int64_t e0 = base[(int64_t)b * pgrid];            // bucket b starts at its first CTA's offset
        const int64_t E = base[(int64_t)(b + 1) * pgrid] - e0;
        for (int t = threadIdx.x; t < nr; t += blockDim.x) cur[t] = 0;
        __syncthreads();
        // row lengths of this bucket (the bucket is its own count pass: no global per-row counters)
        for (int64_t i0 = (int64_t)threadIdx.x * kLoadBatch; i0 < E; i0 += (int64_t)blockDim.x * kLoadBatch) {
            typename Entry<PACKED>::T p[kLoadBatch];
#pragma unroll
            for (int k = 0; k < kLoadBatch; ++k)
                p[k] = (i0 + k < E) ? pairs[e0 + i0 + k] : Entry<PACKED>::invalid();
#pragma unroll
            for (int k = 0; k < kLoadBatch; ++k)
                if (Entry<PACKED>::valid(p[k])) atomicAdd(&cur[Entry<PACKED>::row(p[k], vbits)], 1);
        }
        __syncthreads();
        {   // exclusive scan of the row lengths: thread t owns rows [kRowsPerThread t, +kRowsPerThread)
            int32_t v[kRowsPerThread];
            int64_t sum = 0;
#pragma unroll
            for (int j = 0; j < kRowsPerThread; ++j) {
                const int t = threadIdx.x * kRowsPerThread + j;
                v[j] = t < nr ? cur[t] : 0;
                sum += v[j];
            }
            int64_t total;
            int64_t run = block_incl_scan(sum, scan_sh, total) - sum;
#pragma unroll
            for (int j = 0; j < kRowsPerThread; ++j) {
                const int t = threadIdx.x * kRowsPerThread + j;
                if (t < nr) off[t] = static_cast<int32_t>(run);
                run += v[j];
            }
            if (threadIdx.x == 0) off[nr] = static_cast<int32_t>(total);
        }
        __syncthreads();
        for (int t = threadIdx.x; t <= nr; t += blockDim.x) {
            if (t < nr || r0 + nr == nl) raw_ptr[r0 + t] = e0 + off[t];
            if (t < nr) cur[t] = 0;
        }
        __syncthreads();
        // windows of consecutive rows [ws, we) whose entries fit shared memory (the whole bucket when it
        // fits; a bucket too large is sorted window by window, each window re-reading the bucket's entries).
        // A single row longer than `cap` goes to the global fallback (warp / block sort kernels).
        for (int ws = 0; ws < nr;) {
            if (threadIdx.x == 0) {
                int lo = ws, hi = nr;   // largest we with off[we] - off[ws] <= cap
                while (lo < hi) {
                    const int mid = (lo + hi + 1) / 2;
                    if (off[mid] - off[ws] <= cap) lo = mid;
                    else hi = mid - 1;
                }
                wend = lo;
                nbig = 0;
                qnext = ws;
            }
            __syncthreads();
            const int we = wend;
            if (we == ws) {   // one oversized row: place it in col_raw (global) for the fallback kernels
                const int t = ws;
                for (int64_t idx = threadIdx.x; idx < E; idx += blockDim.x) {
                    const typename Entry<PACKED>::T p = pairs[e0 + idx];
                    if (Entry<PACKED>::valid(p) && Entry<PACKED>::row(p, vbits) == t) {
                        const int64_t k = atomicAdd(&cur[t], 1);
                        col_raw[e0 + off[t] + k] = Entry<PACKED>::col(p, vbits);
                    }
                }
                if (threadIdx.x == 0) fb_rows[atomicAdd(fb_count, 1)] = r0 + t;
                __syncthreads();
                ws = we + 1;
                continue;
            }
            const int wbase = off[ws];
            if (threadIdx.x == 0) tail = off[we] - wbase;   // free shared memory after the window's entries
            for (int t = ws + threadIdx.x; t < we; t += blockDim.x)
                if (off[t + 1] - off[t] > kGroupRow) big[atomicAdd(&nbig, 1)] = t;
            // placement: batched loads for memory-level parallelism
            for (int64_t i0 = (int64_t)threadIdx.x * kLoadBatch; i0 < E; i0 += (int64_t)blockDim.x * kLoadBatch) {
                typename Entry<PACKED>::T p[kLoadBatch];
#pragma unroll
                for (int k = 0; k < kLoadBatch; ++k)
                    p[k] = (i0 + k < E) ? pairs[e0 + i0 + k] : Entry<PACKED>::invalid();
#pragma unroll
                for (int k = 0; k < kLoadBatch; ++k) {
                    if (Entry<PACKED>::valid(p[k])) {
                        const int lr = Entry<PACKED>::row(p[k], vbits);
                        if (lr >= ws && lr < we)
                            s[off[lr] - wbase + atomicAdd(&cur[lr], 1)] = Entry<PACKED>::col(p[k], vbits);
                    }
                }
            }
            __syncthreads();
            // long rows (> kGroupRow, the hubs): 8 groups of 4 warps, one row per group at a time
            const int nbr = nbig;
            const int wid = threadIdx.x >> 5, grp = wid >> 2, gt = threadIdx.x & 127;
            const GroupSync gsync{1 + grp, 128};
            for (int q = grp; q < nbr; q += 8) {
                const int t = big[q];
                int32_t *a = s + off[t] - wbase;
                const int len = off[t + 1] - off[t];
                // split by value into ~len/kSubAvg sub-ranges (ids are spread over [0, 2^vbits)), then one warp
                // sorts each sub-range in registers; the free shared memory holds the counts and a copy.
                // Equal values share a sub-range, so the row ends up fully sorted. No room: plain bitonic.
                const int nsub = (len + kSubAvg - 1) / kSubAvg;
                if (gt == 0) gtmp[grp] = atomicAdd(&tail, nsub + len);
                gsync();
                const int tb = gtmp[grp];
                if (tb + nsub + len <= kBucketCap) {
                    int32_t *cnt = s + tb, *tmp = cnt + nsub;
                    const int gw = gt >> 5;
                    auto sub_of = [&](int32_t v) {
                        return (int)(((uint64_t)(uint32_t)v * (uint64_t)nsub) >> vbits);
                    };
                    for (int k = gt; k < nsub; k += 128) cnt[k] = 0;
                    gsync();
                    for (int i = gt; i < len; i += 128) atomicAdd(&cnt[sub_of(a[i])], 1);
                    gsync();
                    if (gw == 0) {   // exclusive scan of the counts (one warp)
                        int run = 0;
                        for (int k0 = 0; k0 < nsub; k0 += 32) {
                            const int k = k0 + lane;
                            const int c = k < nsub ? cnt[k] : 0;
                            int x = c;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const int y = __shfl_up_sync(0xffffffffu, x, o);
                                if (lane >= o) x += y;
                            }
                            if (k < nsub) cnt[k] = run + x - c;
                            run += __shfl_sync(0xffffffffu, x, 31);
                        }
                    }
                    gsync();
                    for (int i = gt; i < len; i += 128) {
                        const int32_t v = a[i];
                        tmp[atomicAdd(&cnt[sub_of(v)], 1)] = v;
                    }
                    gsync();
                    // cnt[k] now ends sub-range k; sort each range into place
                    for (int k = gw; k < nsub; k += 4) {
                        const int b0 = k ? cnt[k - 1] : 0, b1 = cnt[k];
                        warp_sort_inplace<PACKED>(tmp + b0, b1 - b0, lane);
                        for (int i = b0 + lane; i < b1; i += 32) a[i] = tmp[i];
                    }
                    gsync();
                } else {
                    bitonic_any(a, len, gt, 128, gsync);
                }
                // dedup: running count over 128-wide chunks (group-shared partial counts in `cur`)
                int written = 0;
                for (int base0 = 0; base0 < len; base0 += 128) {
                    const int x = base0 + gt;
                    const int32_t v = x < len ? a[x] : INT_MAX;
                    const bool keep = x < len && (x == 0 || v != a[x - 1]);
                    const unsigned bal = __ballot_sync(0xffffffffu, keep);
                    const int lw = gt >> 5;
                    int32_t *wc = gtmp_cnt(cur, nr, grp);
                    if (lane == 0) wc[lw] = __popc(bal);
                    gsync();
                    int before = 0, total = 0;
                    for (int w = 0; w < 4; ++w) {
                        if (w < lw) before += wc[w];
                        total += wc[w];
                    }
                    if (keep) col_raw[e0 + off[t] + written + before + __popc(bal & ((1u << lane) - 1u))] = v;
                    written += total;
                    gsync();
                }
                if (gt == 0) deg[r0 + t] = written;
            }
            // all other rows of the window: one warp per row, fetched dynamically
            for (;;) {
                int t = 0;
                if (lane == 0) t = atomicAdd(&qnext, 1);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= we) break;
                const int len = off[t + 1] - off[t];
                if (len > kGroupRow) continue;
                const int w = warp_sort_dedup<PACKED>(s + off[t] - wbase, len, col_raw + e0 + off[t], lane);
                if (lane == 0) deg[r0 + t] = w;
            }
            __syncthreads();
            ws = we;
        }
        __syncthreads();
    }
}

__global__ void csr_compact(int64_t nl, const int64_t *__restrict__ raw_ptr, const int32_t *__restrict__ col_raw,
                            const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col) {
    // a warp takes 32 consecutive rows (offsets loaded once, coalesced, lane = row) and copies their unique prefixes as
    // ONE flat range of entries, 32 x 4 at a time: entry x belongs to the row whose prefix sum of lengths brackets it
    // (a 5-step search over the lanes' sums), so every lane moves an entry on every step and the stores, whose
    // destination range is contiguous, are fully coalesced
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < nl; r0 += warps * 32) {
        const int64_t row = r0 + lane;
        int64_t src = 0;
        int len = 0;
        if (row < nl) {
            src = raw_ptr[row];
            len = static_cast<int>(row_ptr[row + 1] - row_ptr[row]);
        }
        int incl = len;   // inclusive prefix of the lengths over the lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t dst0 = row_ptr[min(r0, nl - 1)];   // the 32 rows' unique entries are contiguous from here
        const int64_t sb = src - (incl - len);            // raw start minus the row's flat offset
        for (int x0 = 0; x0 < total; x0 += 32 * 4) {
            int32_t v[4];
            int xs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int x = x0 + u * 32 + lane;
                int k = 0;   // the first lane whose inclusive prefix exceeds x
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const int p = __shfl_sync(0xffffffffu, incl, k + st - 1);
                    if (p <= x) k += st;
                }
                const int64_t base = __shfl_sync(0xffffffffu, sb, k & 31);
                xs[u] = x;
                v[u] = x < total ? col_raw[base + x] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (xs[u] < total) col[dst0 + xs[u]] = v[u];
        }
    }
}

// deg_all -> s, s^ ; two_e = sum deg (int64) via one atomic per block; degree histogram (capped bins)
// out[0] = nnz (row_ptr[nl]), out[1] = raw entries (raw_ptr[nl], 0 without rows), out[2] = data-error flag
__global__ void gather_scalars(const int64_t *nnz, const int64_t *raw_total, const int *err, bool has_rows,
                               int64_t *out) {
    if (threadIdx.x == 0) {
        out[0] = *nnz;
        out[1] = has_rows ? *raw_total : 0;
        out[2] = *err;
    }
}

__global__ void degree_scalars(const int32_t *__restrict__ deg, int64_t n, float *__restrict__ s,
                               float *__restrict__ sh, unsigned long long *__restrict__ two_e,
                               unsigned long long *__restrict__ hist) {
    __shared__ unsigned long long part;
    __shared__ unsigned int hsh[kDegHistBins];
    if (threadIdx.x == 0) part = 0;
    for (int b = threadIdx.x; b < kDegHistBins; b += blockDim.x) hsh[b] = 0;
    __syncthreads();
    unsigned long long local = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t d = deg[i];
        local += static_cast<unsigned long long>(d);
        s[i] = d > 0 ? __frsqrt_rn(static_cast<float>(d)) : 0.0f;
        sh[i] = __frsqrt_rn(static_cast<float>(d) + 1.0f);
        atomicAdd(&hsh[d < kDegHistBins - 1 ? d : kDegHistBins - 1], 1u);
    }
    atomicAdd(&part, local);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(two_e, part);
    for (int b = threadIdx.x; b < kDegHistBins; b += blockDim.x)
        if (hsh[b]) atomicAdd(&hist[b], static_cast<unsigned long long>(hsh[b]));
}

}  // namespace

raftgp_status scan_i32_to_i64(raftgp_ctx ctx, const int32_t *in, int64_t *out, int64_t n) {
    const int64_t per_tile = (int64_t)kScanBlock * kScanItems;
    const int64_t ntiles = n > 0 ? ceil_div(n, per_tile) : 0;
    if (ntiles == 0) {
        RG_TRY(dzero(ctx, out, sizeof(int64_t), ctx->stream));
        return RAFTGP_OK;
    }
    int64_t *tiles = nullptr;
    RG_TRY(dalloc_t(ctx, &tiles, ntiles + 1));
    {
        LaunchScope L(ctx, K_SCAN);
        scan_tile_sums<<<(unsigned)ntiles, kScanBlock, 0, ctx->stream>>>(in, n, tiles);
    }
    RG_CHECK_LAUNCH(ctx);
    {
        LaunchScope L(ctx, K_SCAN);
        scan_tile_offsets<<<1, kScanBlock, 0, ctx->stream>>>(tiles, ntiles);
    }
    RG_CHECK_LAUNCH(ctx);
    {
        LaunchScope L(ctx, K_SCAN);
        scan_apply<<<(unsigned)ntiles, kScanBlock, 0, ctx->stream>>>(in, n, tiles, out);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, tiles);
    return RAFTGP_OK;
}

// known_2e >= 0: the caller knows 2e (a whole-graph build: 2e = nnz of the symmetric CSR), so the scalars are
// launched without the host read-back of the degree sum (no host sync; the histogram is not kept then)
raftgp_status degrees_finalize(raftgp_graph g, int64_t known_2e) {
    raftgp_ctx ctx = g->ctx;
    drop_slots(g);   // the slot layout follows the degrees
    unsigned long long *d_buf = nullptr;   // [0] = 2e, [1..] = degree histogram
    RG_TRY(dalloc_t(ctx, &d_buf, 1 + kDegHistBins));
    RG_TRY(dzero(ctx, d_buf, sizeof(unsigned long long) * (1 + kDegHistBins), ctx->stream));
    if (g->n > 0) {
        const int grid = static_cast<int>(std::min<int64_t>(ceil_div(g->n, 256), (int64_t)ctx->sm_count * 4));
        LaunchScope L(ctx, K_DEGREES);
        degree_scalars<<<grid, 256, 0, ctx->stream>>>(g->deg_all, g->n, g->s_all, g->sh_all, d_buf, d_buf + 1);
    }
    RG_CHECK_LAUNCH(ctx);
    if (known_2e >= 0) {
        dfree(ctx, d_buf);   // stream-ordered: the kernel's scratch returns to the pool after it
        g->two_e = known_2e;
        g->deg_hist.clear();
        return RAFTGP_OK;
    }
    std::vector<unsigned long long> h(1 + kDegHistBins, 0);
    RG_TRY(dread(ctx, h.data(), d_buf, sizeof(unsigned long long) * h.size()));
    dfree(ctx, d_buf);
    g->two_e = static_cast<int64_t>(h[0]);
    g->deg_hist.assign(h.begin() + 1, h.end());
    return RAFTGP_OK;
}

// Two-level partition + bucket sort (see csr_coarse_part / csr_fine_part): bucket count by COARSE bucket ->
// scan -> level 1 -> level 2 (skipped when one coarse bucket is one fine bucket) -> csr_bucket_sort on the fine
// buckets -> warp-sort fallback for rows longer than a shared-memory window. Leaves raw_ptr / col_raw / deg as
// the one-level path does; *fb_rows / *fb_count are allocated here and freed by the caller.
raftgp_status csr_partition_two_level(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                      int64_t rb, int64_t re, int shift, int fbits, int nb, int vbits, int64_t cap,
                                      int64_t *raw_ptr, int32_t *col_raw, int32_t *deg, int *err, int64_t **fb_rows_out,
                                      int32_t **fb_count_out) {
    cudaStream_t st = ctx->stream;
    const int64_t nl = re - rb;
    const int cs = shift + fbits;
    const int nc = static_cast<int>(ceil_div(nl, (int64_t)1 << cs));
    static const bool force_unpacked = [] {   // RAFTGP_CSR_UNPACKED=1: int2 fine entries even when packing fits (tests)
        const char *e = getenv("RAFTGP_CSR_UNPACKED");
        return e && e[0] == '1';
    }();
    const bool packed = fbits > 0 && shift + vbits <= 32 && !force_unpacked;
    // level-1 CTAs (2 per SM) and the count pass share the raw-pair ranges
    const int pgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 32768), 2 * (int64_t)ctx->sm_count)));
    int2 *p1 = nullptr;
    void *p2 = nullptr;
    int32_t *bcnt = nullptr;
    int64_t *bstart = nullptr, *fst = nullptr, *fb_rows = nullptr;
    int32_t *fb_count = nullptr;
    unsigned int *bnext = nullptr;
    RG_TRY(dalloc_t(ctx, &bnext, 1));
    RG_TRY(dzero(ctx, bnext, sizeof(unsigned int), st));
    RG_TRY(dalloc_t(ctx, &bcnt, (size_t)nc * pgrid));
    RG_TRY(dalloc_t(ctx, &bstart, (size_t)nc * pgrid + 1));
    RG_TRY(dalloc_t(ctx, &p1, (size_t)std::max<int64_t>(cap, 1)));
    int32_t *fcnt = nullptr;
    unsigned long long *fcur = nullptr;
    if (fbits > 0) {
        RG_TRY(dalloc(ctx, &p2, (size_t)std::max<int64_t>(cap, 1) * (packed ? 4 : 8)));
        RG_TRY(dalloc_t(ctx, &fst, (size_t)nb + 1));
        RG_TRY(dalloc_t(ctx, &fcnt, (size_t)nb));
        RG_TRY(dalloc_t(ctx, &fcur, (size_t)nb));
        RG_TRY(dzero(ctx, fcnt, sizeof(int32_t) * nb, st));
    }
    RG_TRY(dalloc_t(ctx, &fb_rows, (size_t)nl));
    RG_TRY(dalloc_t(ctx, &fb_count, 1));
    RG_TRY(dzero(ctx, fb_count, sizeof(int32_t), st));
    *fb_rows_out = fb_rows;
    *fb_count_out = fb_count;
    const size_t bsmem = (size_t)(kBucketCap + 3 * kMaxBucketRows + 1) * 4;
    const size_t cpsmem = coarse_smem(nc), fpsmem = fine_smem(1 << fbits);
    static const char attrs_key = 0;
    RG_TRY(per_device(ctx->device, &attrs_key, nullptr, [&](int *) -> raftgp_status {
        RG_CUDA(cudaFuncSetAttribute(csr_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets32 * 4));
        RG_CUDA(cudaFuncSetAttribute(csr_coarse_part, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coarse_smem(kMaxCoarse)));
        RG_CUDA(cudaFuncSetAttribute(csr_fine_part<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fine_smem(kMaxFine)));
        RG_CUDA(cudaFuncSetAttribute(csr_fine_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
        RG_CUDA(cudaFuncSetAttribute(csr_fine_part<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fine_smem(kMaxFine)));
        RG_CUDA(cudaFuncSetAttribute(csr_bucket_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
        RG_CUDA(cudaFuncSetAttribute(csr_bucket_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
        return RAFTGP_OK;
    }));
    {
        LaunchScope L(ctx, K_CSR_COUNT);
        csr_bucket_count<<<pgrid, 1024, (size_t)nc * 4, st>>>(src, dst, m, n, rb, re, cs, nc, bcnt, err);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(scan_i32_to_i64(ctx, bcnt, bstart, (int64_t)nc * pgrid));
    if (m > 0) {
        LaunchScope L(ctx, K_CSR_PARTITION);
        csr_coarse_part<<<pgrid, kPT, cpsmem, st>>>(src, dst, m, n, rb, re, cs, nc, bstart, p1);
    }
    RG_CHECK_LAUNCH(ctx);
    if (fbits > 0) {
        const dim3 fgrid(kFineSlots, nc);
        {
            LaunchScope L(ctx, K_CSR_FINE);
            csr_fine_count<<<fgrid, kPT, 0, st>>>(p1, bstart, pgrid, shift, fbits, nb, fcnt);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, fcnt, fst, nb));
        LaunchScope L(ctx, K_CSR_FINE);
        csr_bucket_cursor<<<(nb + 255) / 256, 256, 0, st>>>(fst, 1, nb, fcur);
        if (packed)
            csr_fine_part<true><<<fgrid, kPT, fpsmem, st>>>(p1, bstart, pgrid, shift, fbits, vbits, fcur,
                                                             static_cast<uint32_t *>(p2));
        else
            csr_fine_part<false><<<fgrid, kPT, fpsmem, st>>>(p1, bstart, pgrid, shift, fbits, vbits, fcur,
                                                              static_cast<int2 *>(p2));
    }
    RG_CHECK_LAUNCH(ctx);
    static const int bcap = [] {   // RAFTGP_BUCKET_CAP: smaller shared-memory windows (tests)
        const char *e = getenv("RAFTGP_BUCKET_CAP");
        return e ? std::max(256, std::min(kBucketCap, atoi(e))) : kBucketCap;
    }();
    {
        LaunchScope L(ctx, K_CSR_BUCKET);
        const int bgrid = std::min(nb, ctx->sm_count);
        if (fbits == 0)
            csr_bucket_sort<false><<<bgrid, 1024, bsmem, st>>>(p1, bstart, pgrid, raw_ptr, nl, shift, nb, vbits, col_raw,
                                                               deg, fb_rows, fb_count, bnext, bcap);
        else if (packed)
            csr_bucket_sort<true><<<bgrid, 1024, bsmem, st>>>(static_cast<const uint32_t *>(p2), fst, 1, raw_ptr, nl,
                                                              shift, nb, vbits, col_raw, deg, fb_rows, fb_count, bnext,
                                                              bcap);
        else
            csr_bucket_sort<false><<<bgrid, 1024, bsmem, st>>>(static_cast<const int2 *>(p2), fst, 1, raw_ptr, nl,
                                                               shift, nb, vbits, col_raw, deg, fb_rows, fb_count, bnext,
                                                               bcap);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, bcnt);
    dfree(ctx, bstart);
    dfree(ctx, bnext);
    dfree(ctx, p1);
    if (p2) dfree(ctx, p2);
    if (fst) dfree(ctx, fst);
    if (fcnt) dfree(ctx, fcnt);
    if (fcur) dfree(ctx, fcur);
    return RAFTGP_OK;
}

raftgp_status csr_build(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int64_t rb,
                        int64_t re, raftgp_graph g) {
    cudaStream_t st = ctx->stream;
    const int64_t nl = re - rb;
    g->n = n;
    g->row_begin = rb;
    g->row_end = re;
    g->nl = nl;
    const int64_t cap = 2 * m;   // upper bound of raw entries in any row range
    int32_t *cnt = nullptr, *col_raw = nullptr, *big_count = nullptr, *err = nullptr;
    int64_t *raw_ptr = nullptr, *big_rows = nullptr;
    RG_TRY(dalloc_t(ctx, &cnt, nl));
    RG_TRY(dalloc_t(ctx, &raw_ptr, nl + 4));
    RG_TRY(dalloc_t(ctx, &col_raw, cap));
    RG_TRY(dalloc_t(ctx, &big_rows, nl));
    RG_TRY(dalloc_t(ctx, &big_count, 2));
    err = big_count + 1;
    RG_TRY(dalloc_t(ctx, &g->row_ptr, nl + 1));
    RG_TRY(dalloc_t(ctx, &g->deg_local, nl));
    RG_TRY(dalloc_t(ctx, &g->deg_all, n));
    RG_TRY(dalloc_t(ctx, &g->s_all, n));
    RG_TRY(dalloc_t(ctx, &g->sh_all, n));
    RG_TRY(dzero(ctx, big_count, sizeof(int32_t) * 2, st));
    const int egrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->sm_count * 16)));
    // 32-bit partition cursors when every raw entry position fits: twice the buckets in the same shared memory,
    // so huge graphs (C5) get buckets half as large; then buckets grow while a typical one still fits a window
    const bool b32 = cap < ((int64_t)1 << 32);
    static const bool two_level_env = [] {   // RAFTGP_CSR_TWO_LEVEL=0: the one-level partition (A/B runs, tests)
        const char *e = getenv("RAFTGP_CSR_TWO_LEVEL");
        return !e || atoi(e) != 0;
    }();
    // two-level partition: needs 32-bit positions and at most kMaxCoarse x kMaxFine buckets of 512 rows
    const bool two_level = two_level_env && b32 && nl > 0 && ceil_div(nl, (int64_t)512) <= (int64_t)kMaxCoarse * kMaxFine;
    const int kMaxB = two_level ? INT_MAX : b32 ? kMaxBuckets32 : kMaxBuckets;
    int shift = 0;
    while (shift < 31 && ceil_div(nl, (int64_t)1 << shift) > kMaxB) ++shift;
    while (nl > 0 && shift < 12 && (cap / nl + 1) * ((int64_t)2 << shift) <= kBucketCap / 2 &&
           ceil_div(nl, (int64_t)2 << shift) >= 4 * (int64_t)ctx->sm_count)
        ++shift;
    const bool bucketed = nl > 0 && ((int64_t)1 << shift) <= kMaxBucketRows;
    if (!bucketed) {   // per-row counts (the bucketed path lets every bucket count its own rows)
        RG_TRY(dzero(ctx, cnt, sizeof(int32_t) * (nl ? nl : 1), st));
        if (m > 0) {
            LaunchScope L(ctx, K_CSR_COUNT);
            csr_count<<<egrid, 256, 0, st>>>(src, dst, m, n, rb, re, cnt, err);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, cnt, raw_ptr, nl));
    }
    const int rgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nl, 8), (int64_t)ctx->sm_count * 8)));
    int64_t *fb_rows = nullptr;
    int32_t *fb_count = nullptr;
    if (bucketed) {
        const int nb = static_cast<int>(ceil_div(nl, (int64_t)1 << shift));
        int vbits = 1;
        while (vbits < 31 && ((int64_t)1 << vbits) < n) ++vbits;
        // two-level: fine buckets = the bucket sort's buckets (2^shift rows), coarse = 2^fbits fine buckets
        static const int64_t max_coarse = [] {   // RAFTGP_CSR_COARSE: fewer coarse buckets (tests force level 2)
            const char *e = getenv("RAFTGP_CSR_COARSE");
            return e ? std::max<int64_t>(1, std::min<int64_t>(kMaxCoarse, atoll(e))) : (int64_t)kMaxCoarse;
        }();
        int fbits = 0;
        if (two_level)
            while (fbits < 8 && ceil_div((int64_t)nb, (int64_t)1 << fbits) > max_coarse) ++fbits;
        const bool use2 = two_level && ceil_div((int64_t)nb, (int64_t)1 << fbits) <= max_coarse;
        if (use2) {
            RG_TRY(csr_partition_two_level(ctx, n, m, src, dst, rb, re, shift, fbits, nb, vbits, cap, raw_ptr, col_raw,
                                           g->deg_local, err, &fb_rows, &fb_count));
            LaunchScope L(ctx, K_CSR_SORT_WARP);
            csr_sort_warp<<<rgrid, 256, 0, st>>>(nl, fb_rows, fb_count, raw_ptr, col_raw, g->deg_local, big_rows, big_count);
        } else {
        const bool packed = shift + vbits <= 32;
        const int pgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 65536), ctx->sm_count)));
        void *pairs = nullptr;
        int32_t *bcnt = nullptr;
        int64_t *bstart = nullptr;
        unsigned long long *bcur = nullptr;
        unsigned int *bnext = nullptr;
        RG_TRY(dalloc_t(ctx, &bcur, (size_t)nb));
        RG_TRY(dalloc_t(ctx, &bnext, 1));
        RG_TRY(dzero(ctx, bnext, sizeof(unsigned int), st));
        RG_TRY(dalloc_t(ctx, &bcnt, (size_t)nb * pgrid));
        RG_TRY(dalloc_t(ctx, &bstart, (size_t)nb * pgrid + 1));
        RG_TRY(dalloc(ctx, &pairs, (size_t)cap * (packed ? 4 : 8)));
        RG_TRY(dalloc_t(ctx, &fb_rows, (size_t)nl));
        RG_TRY(dalloc_t(ctx, &fb_count, 1));
        RG_TRY(dzero(ctx, fb_count, sizeof(int32_t), st));
        const size_t bsmem = (size_t)(kBucketCap + 3 * kMaxBucketRows + 1) * 4;
        static const char attrs_key = 0;   // per-(device, instantiation) key
        RG_TRY(per_device(ctx->device, &attrs_key, nullptr, [&](int *) -> raftgp_status {
            RG_CUDA(cudaFuncSetAttribute(csr_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets32 * 4));
            RG_CUDA(cudaFuncSetAttribute(csr_partition<true, long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 12));
            RG_CUDA(cudaFuncSetAttribute(csr_partition<false, long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 12));
            RG_CUDA(cudaFuncSetAttribute(csr_partition<true, unsigned int>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets32 * 8));
            RG_CUDA(cudaFuncSetAttribute(csr_partition<false, unsigned int>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets32 * 8));
            RG_CUDA(cudaFuncSetAttribute(csr_bucket_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
            RG_CUDA(cudaFuncSetAttribute(csr_bucket_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
            return RAFTGP_OK;
        }));
        {
            LaunchScope L(ctx, K_CSR_COUNT);
            csr_bucket_count<<<pgrid, 1024, (size_t)nb * 4, st>>>(src, dst, m, n, rb, re, shift, nb, bcnt, err);
        }
        RG_CHECK_LAUNCH(ctx);
        RG_TRY(scan_i32_to_i64(ctx, bcnt, bstart, (int64_t)nb * pgrid));
        if (m > 0) {
            LaunchScope L(ctx, K_CSR_PARTITION);
            csr_bucket_cursor<<<(nb + 255) / 256, 256, 0, st>>>(bstart, pgrid, nb, bcur);
            static const int64_t ptile = [] {
                const char *e = getenv("RAFTGP_PART_TILE");
                return e ? std::max<int64_t>(1024, atoll(e)) : (int64_t)kPartTile;
            }();
            const int tgrid = static_cast<int>(std::min<int64_t>(ceil_div(m, ptile), ctx->sm_count));
            const size_t psmem = (size_t)nb * (b32 ? 8 : 12);
            if (packed && b32)
                csr_partition<true, unsigned int><<<tgrid, 1024, psmem, st>>>(src, dst, m, n, rb, re, shift, nb, vbits, ptile,
                                                                               bcur, static_cast<uint32_t *>(pairs));
            else if (packed)
                csr_partition<true, long long><<<tgrid, 1024, psmem, st>>>(src, dst, m, n, rb, re, shift, nb, vbits, ptile,
                                                                            bcur, static_cast<uint32_t *>(pairs));
            else if (b32)
                csr_partition<false, unsigned int><<<tgrid, 1024, psmem, st>>>(src, dst, m, n, rb, re, shift, nb, vbits, ptile,
                                                                                bcur, static_cast<int2 *>(pairs));
            else
                csr_partition<false, long long><<<tgrid, 1024, psmem, st>>>(src, dst, m, n, rb, re, shift, nb, vbits, ptile,
                                                                             bcur, static_cast<int2 *>(pairs));
        }
        RG_CHECK_LAUNCH(ctx);
        static const int bcap = [] {   // RAFTGP_BUCKET_CAP: smaller shared-memory windows (tests)
            const char *e = getenv("RAFTGP_BUCKET_CAP");
            return e ? std::max(256, std::min(kBucketCap, atoi(e))) : kBucketCap;
        }();
        {
            LaunchScope L(ctx, K_CSR_BUCKET);
            const int bgrid = std::min(nb, ctx->sm_count);
            if (packed)
                csr_bucket_sort<true><<<bgrid, 1024, bsmem, st>>>(static_cast<const uint32_t *>(pairs), bstart, pgrid, raw_ptr,
                                                                  nl, shift, nb, vbits, col_raw, g->deg_local, fb_rows,
                                                                  fb_count, bnext, bcap);
            else
                csr_bucket_sort<false><<<bgrid, 1024, bsmem, st>>>(static_cast<const int2 *>(pairs), bstart, pgrid, raw_ptr,
                                                                   nl, shift, nb, vbits, col_raw, g->deg_local, fb_rows,
                                                                   fb_count, bnext, bcap);
        }
        RG_CHECK_LAUNCH(ctx);
        {
            LaunchScope L(ctx, K_CSR_SORT_WARP);
            csr_sort_warp<<<rgrid, 256, 0, st>>>(nl, fb_rows, fb_count, raw_ptr, col_raw, g->deg_local, big_rows, big_count);
        }
        RG_CHECK_LAUNCH(ctx);
        dfree(ctx, bcnt);
        dfree(ctx, bstart);
        dfree(ctx, bcur);
        dfree(ctx, bnext);
        dfree(ctx, pairs);
        }
    } else {
        if (m > 0) {
            LaunchScope L(ctx, K_CSR_SCATTER);
            csr_scatter<<<egrid, 256, 0, st>>>(src, dst, m, n, rb, re, raw_ptr, cnt, col_raw);
        }
        RG_CHECK_LAUNCH(ctx);
        if (nl > 0) {
            LaunchScope L(ctx, K_CSR_SORT_WARP);
            csr_sort_warp<<<rgrid, 256, 0, st>>>(nl, nullptr, nullptr, raw_ptr, col_raw, g->deg_local, big_rows, big_count);
        }
        RG_CHECK_LAUNCH(ctx);
    }
    if (nl > 0) {
        static const char attr_set_key = 0;   // per-(device, instantiation) key
        RG_TRY(per_device(ctx->device, &attr_set_key, nullptr, [&](int *) -> raftgp_status {
            RG_CUDA(cudaFuncSetAttribute(csr_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kBlockSortSmemCap * (int)sizeof(int32_t)));
            return RAFTGP_OK;
        }));
        LaunchScope L(ctx, K_CSR_SORT_BLOCK);
        csr_sort_block<<<ctx->sm_count, 1024, kBlockSortSmemCap * sizeof(int32_t), st>>>(big_rows, big_count, raw_ptr,
                                                                                         col_raw, g->deg_local);
    }
    RG_CHECK_LAUNCH(ctx);
    dfree(ctx, fb_rows);
    dfree(ctx, fb_count);
    RG_TRY(scan_i32_to_i64(ctx, g->deg_local, g->row_ptr, nl));
    // one host read-back for the three scalars (nnz, raw entry count, data-error flag): gather them into
    // raw_ptr's spare slots [nl + 1 .. nl + 3] (allocated nl + 4 long) with one tiny kernel, then read them together
    int64_t hv[3] = {0, 0, 0};
    {
        LaunchScope L(ctx, K_MISC);
        gather_scalars<<<1, 32, 0, st>>>(g->row_ptr + nl, raw_ptr + nl, err, nl > 0, raw_ptr + nl + 1);
    }
    RG_CHECK_LAUNCH(ctx);
    RG_TRY(dread(ctx, hv, raw_ptr + nl + 1, sizeof(hv), st));
    const int64_t nnz = hv[0];
    const int herr = (int)hv[2];
    if (herr) {
        dfree(ctx, cnt); dfree(ctx, raw_ptr); dfree(ctx, col_raw); dfree(ctx, big_rows); dfree(ctx, big_count);
        return fail(RAFTGP_ERR_DATA, "build_csr: node id outside [0, n)");
    }
    g->nnz_local = nnz;
    // without duplicate pairs every row kept all its raw entries: the raw layout IS the CSR (no compaction)
    const int64_t raw_total = hv[1];
    const bool no_dups = raw_total == nnz;
    if (no_dups) {
        g->col = col_raw;
        col_raw = nullptr;
    } else {
        RG_TRY(dalloc_t(ctx, &g->col, nnz));
        if (nl > 0 && nnz > 0) {
            LaunchScope L(ctx, K_CSR_COMPACT);
            const int cgrid = static_cast<int>(std::min<int64_t>(ceil_div(nl, 256), (int64_t)ctx->sm_count * 16));
            csr_compact<<<cgrid, 256, 0, st>>>(nl, raw_ptr, col_raw, g->row_ptr, g->col);
        }
        RG_CHECK_LAUNCH(ctx);
    }
    dfree(ctx, cnt);
    dfree(ctx, raw_ptr);
    dfree(ctx, col_raw);
    dfree(ctx, big_rows);
    dfree(ctx, big_count);
    RG_TRY(compute_order(g));
    if (rb == 0 && re == n) {
        if (n > 0) RG_TRY(dcopy(ctx, g->deg_all, g->deg_local, sizeof(int32_t) * n, st));
        RG_TRY(degrees_finalize(g, g->nnz_local));   // whole graph: 2e = nnz (no second read-back)
    }
    return RAFTGP_OK;
}

}  // namespace raftgp
