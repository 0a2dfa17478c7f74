// capi.cu — the extern "C" boundary of libraftgp (include/raftgp.h): contexts, graph handles, argument
// checks, orchestration of the kernels in csr.cu / sketch.cu / spmm.cu, per-launch profiling, and the
// host-side scoring functions (a7: Eq. 1, 3, 7).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "gauss.cuh"
#include "internal.cuh"

namespace raftgp {

const char *const kKernelNames[K_NUM] = {
    "csr_count", "scan", "csr_scatter", "csr_sort_warp", "csr_sort_block", "csr_compact", "degree_scalars",
    "sketch", "g_partials", "g_final", "feature_hop", "transform", "gcn_hop", "hop_generic", "misc", "csr_partition", "csr_bucket_sort", "row_order", "model_select", "select_seed", "select_lloyd", "select_split", "gemm_tf32x3", "gemm_tile", "wide_hop", "sbm_setup", "sbm_walk", "stream_update", "exchange", "push_copy", "csr_fine_part", "stream_last_hop"};

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

raftgp_status fail(raftgp_status st, const std::string &msg) {
    set_error(msg);
    return st;
}

raftgp_status cuda_fail(cudaError_t e, const char *what) {
    std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    set_error(m);
    return e == cudaErrorMemoryAllocation ? RAFTGP_ERR_NOMEM : RAFTGP_ERR_CUDA;
}

static cudaEvent_t take_event(raftgp_ctx ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

LaunchScope::LaunchScope(raftgp_ctx c, int k, bool count) : ctx(c), kid(k) {
    if (count) ctx->launches += 1;
    if (ctx->prof) {
        a = take_event(ctx);
        b = take_event(ctx);
        cudaEventRecord(a, ctx->stream);
    }
}

LaunchScope::~LaunchScope() {
    if (ctx->prof && a && b) {
        cudaEventRecord(b, ctx->stream);
        ctx->recs.push_back({kid, a, b});
    }
}

static size_t round_block(size_t bytes) {
    const size_t mb = size_t(1) << 20;
    if (bytes >= mb) return (bytes + 2 * mb - 1) / (2 * mb) * (2 * mb);
    return (bytes + 511) / 512 * 512;
}

// Stream-ordered workspace: every user of a block runs on ctx->stream, so a block released by dfree may
// be handed out again immediately — the next user is ordered after the previous one on the stream.
namespace {
__global__ void zero_bytes(uint4 *p16, size_t n16, unsigned char *tail, size_t ntail) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (size_t i = t; i < n16; i += (size_t)gridDim.x * blockDim.x) p16[i] = make_uint4(0u, 0u, 0u, 0u);
    if (t < ntail) tail[t] = 0;
}
}  // namespace

raftgp_status dzero(raftgp_ctx ctx, void *p, size_t bytes, cudaStream_t st) {
    if (!p || bytes == 0) return RAFTGP_OK;
    if (!st) st = ctx->stream;
    unsigned char *b = static_cast<unsigned char *>(p);
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(b) & 15)) & 15;   // bytes before 16-B alignment
    const size_t pre = std::min(head, bytes);
    const size_t n16 = (bytes - pre) / 16;
    const size_t ntail = bytes - pre - n16 * 16;
    if (pre) zero_bytes<<<1, 32, 0, st>>>(nullptr, 0, b, pre);
    if (n16 || ntail) {
        const size_t blocks = std::min<size_t>(std::max<size_t>(1, (n16 + 255) / 256), (size_t)ctx->sm_count * 8);
        zero_bytes<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<uint4 *>(b + pre), n16, b + pre + n16 * 16, ntail);
    }
    RG_CUDA(cudaGetLastError());
    return RAFTGP_OK;
}

namespace {
__global__ void copy_16(const uint4 *s, uint4 *d, size_t n16) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}
__global__ void copy_u8(const unsigned char *s, unsigned char *d, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}
constexpr size_t kMbox = 64 << 10;
}  // namespace

raftgp_status dcopy(raftgp_ctx ctx, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return RAFTGP_OK;
    if (!st) st = ctx->stream;
    const unsigned char *s = static_cast<const unsigned char *>(src);
    unsigned char *d = static_cast<unsigned char *>(dst);
    const bool al = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    const size_t n16 = al ? bytes / 16 : 0;
    const size_t rest = bytes - n16 * 16;
    const size_t cap = (size_t)ctx->sm_count * 8;
    if (n16)
        copy_16<<<(unsigned)std::min<size_t>((n16 + 255) / 256, cap), 256, 0, st>>>(
            reinterpret_cast<const uint4 *>(s), reinterpret_cast<uint4 *>(d), n16);
    if (rest)
        copy_u8<<<(unsigned)std::min<size_t>((rest + 255) / 256, cap), 256, 0, st>>>(s + n16 * 16, d + n16 * 16, rest);
    RG_CUDA(cudaGetLastError());
    return RAFTGP_OK;
}

raftgp_status dread(raftgp_ctx ctx, void *host, const void *dev, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return RAFTGP_OK;
    if (!st) st = ctx->stream;
    if (!ctx->mbox_h && bytes <= kMbox) {
        if (cudaHostAlloc(&ctx->mbox_h, kMbox, cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer(&ctx->mbox_d, ctx->mbox_h, 0) != cudaSuccess) {
            cudaGetLastError();
            if (ctx->mbox_h) cudaFreeHost(ctx->mbox_h);
            ctx->mbox_h = ctx->mbox_d = nullptr;
        }
    }
    if (ctx->mbox_d && bytes <= kMbox) {
        RG_TRY(dcopy(ctx, ctx->mbox_d, dev, bytes, st));
        RG_CUDA(cudaStreamSynchronize(st));
        std::memcpy(host, ctx->mbox_h, bytes);
        return RAFTGP_OK;
    }
    RG_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    return RAFTGP_OK;
}

raftgp_status dalloc(raftgp_ctx ctx, void **p, size_t bytes) {
    const size_t want = round_block(bytes ? bytes : 16);
    auto it = ctx->free_blocks.lower_bound(want);
    if (it != ctx->free_blocks.end() && it->first <= want + want / 4 + (size_t(2) << 20)) {
        *p = it->second;
        ctx->live_blocks[it->second] = it->first;
        ctx->cached_bytes -= it->first;
        ctx->free_blocks.erase(it);
        return RAFTGP_OK;
    }
    cudaError_t e = cudaMallocFromPoolAsync(p, want, ctx->pool, ctx->stream);
    if (e == cudaErrorMemoryAllocation && !ctx->free_blocks.empty()) {   // give the cache back, retry once
        cudaGetLastError();
        for (auto &kv : ctx->free_blocks) cudaFreeAsync(kv.second, ctx->stream);
        ctx->free_blocks.clear();
        ctx->cached_bytes = 0;
        cudaStreamSynchronize(ctx->stream);
        cudaMemPoolTrimTo(ctx->pool, 0);
        e = cudaMallocFromPoolAsync(p, want, ctx->pool, ctx->stream);
    }
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return cuda_fail(e, "cudaMallocAsync");
    }
    ctx->live_blocks[*p] = want;
    return RAFTGP_OK;
}

void dfree(raftgp_ctx ctx, void *p) {
    if (!p) return;
    auto it = ctx->live_blocks.find(p);
    if (it == ctx->live_blocks.end()) {
        cudaFreeAsync(p, ctx->stream);
        return;
    }
    ctx->free_blocks.emplace(it->second, p);
    ctx->cached_bytes += it->second;
    ctx->live_blocks.erase(it);
}

void release_cache(raftgp_ctx ctx) {
    for (auto &kv : ctx->free_blocks) cudaFreeAsync(kv.second, ctx->stream);
    ctx->free_blocks.clear();
    ctx->cached_bytes = 0;
}

raftgp_status per_device(int device, const void *key, int *value, const std::function<raftgp_status(int *)> &init) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> done;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({device, key});
    if (it == done.end()) {
        int v = 0;
        const raftgp_status st = init(&v);
        if (st != RAFTGP_OK) return st;
        it = done.emplace(std::make_pair(device, key), v).first;
    }
    if (value) *value = it->second;
    return RAFTGP_OK;
}

}  // namespace raftgp

using namespace raftgp;

#define RG_GUARD_BEGIN try {
#define RG_GUARD_END                                                      \
    }                                                                     \
    catch (const std::bad_alloc &) {                                      \
        return fail(RAFTGP_ERR_NOMEM, "host allocation failed");          \
    }                                                                     \
    catch (...) {                                                         \
        return fail(RAFTGP_ERR_INTERNAL, "unexpected C++ exception");    \
    }

static raftgp_status set_device(raftgp_ctx ctx) {
    RG_CUDA(cudaSetDevice(ctx->device));
    return RAFTGP_OK;
}

static raftgp_status need_ready(raftgp_graph g) {
    if (!g) return fail(RAFTGP_ERR_PARAM, "null graph");
    if (g->two_e < 0) return fail(RAFTGP_ERR_STATE, "partial graph: call raftgp_graph_set_degrees first");
    return RAFTGP_OK;
}

namespace raftgp {

void dist_comm_destroy(raftgp_ctx ctx);   // dist.cu

static void ctx_teardown(raftgp_ctx ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    dist_comm_destroy(ctx);
    for (auto &r : ctx->recs) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    release_cache(ctx);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);   // blocks still live (caller never freed them) are released too
    if (ctx->hip) {
        cudaStreamSynchronize(ctx->hip);
        cudaStreamDestroy(ctx->hip);
        ctx->hip = nullptr;
    }
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->mbox_h) cudaFreeHost(ctx->mbox_h);
    delete ctx;
}


void ctx_retain(raftgp_ctx ctx) { ctx->refs.fetch_add(1); }

void ctx_release(raftgp_ctx ctx) {
    if (ctx->refs.fetch_sub(1) == 1) ctx_teardown(ctx);
}

}  // namespace raftgp

extern "C" {

const char *raftgp_last_error(void) { return g_last_error.c_str(); }

const char *raftgp_version(void) { return "raftgp-b200 0.1 (sm_100a)"; }

raftgp_status raftgp_ctx_create(int device, void *cuda_stream, raftgp_ctx *out) {
    RG_GUARD_BEGIN
    if (!out) return fail(RAFTGP_ERR_PARAM, "null out");
    *out = nullptr;
    int ndev = 0;
    RG_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(RAFTGP_ERR_PARAM, "device ordinal out of range");
    RG_CUDA(cudaSetDevice(device));
    raftgp_ctx c = new raftgp_ctx_s();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);   // NULL = the legacy default stream
    c->own_stream = false;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    // the context's own stream-ordered pool: freed blocks stay reserved in it (hot calls never reach the driver
    // allocator) without changing the device's default pool, which other cudaMallocAsync users share
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaError_t pe = cudaMemPoolCreate(&c->pool, &props);
    if (pe != cudaSuccess) {
        delete c;
        return cuda_fail(pe, "cudaMemPoolCreate");
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    *out = c;
    return RAFTGP_OK;
    RG_GUARD_END
}

raftgp_status raftgp_ctx_destroy(raftgp_ctx ctx) {
    if (ctx) ctx_release(ctx);
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_trim(raftgp_ctx ctx, int64_t *bytes_released) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    RG_TRY(set_device(ctx));
    const int64_t b = (int64_t)ctx->cached_bytes;
    release_cache(ctx);
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    RG_CUDA(cudaMemPoolTrimTo(ctx->pool, 0));   // the pool's unused memory goes back to the device
    if (bytes_released) *bytes_released = b;
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_sync(raftgp_ctx ctx) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_stream(raftgp_ctx ctx, void **s) {
    if (!ctx || !s) return fail(RAFTGP_ERR_PARAM, "null argument");
    *s = ctx->stream;
    return RAFTGP_OK;
}

raftgp_status raftgp_ctx_set_profiling(raftgp_ctx ctx, int enable) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    ctx->prof = enable != 0;
    return RAFTGP_OK;
}

int raftgp_prof_kernels(void) { return K_NUM; }

const char *raftgp_prof_name(int kid) { return (kid >= 0 && kid < K_NUM) ? kKernelNames[kid] : "?"; }

raftgp_status raftgp_prof_read(raftgp_ctx ctx, int kid, double *total_ms, int64_t *launches) {
    if (!ctx || kid < 0 || kid >= K_NUM) return fail(RAFTGP_ERR_PARAM, "bad ctx or kernel id");
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    double t = 0;
    int64_t c = 0;
    for (auto &r : ctx->recs) {
        if (r.kid != kid) continue;
        float ms = 0;
        RG_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
        t += ms;
        c += 1;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = c;
    return RAFTGP_OK;
}

raftgp_status raftgp_prof_reset(raftgp_ctx ctx) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto &r : ctx->recs) {
        ctx->event_pool.push_back(r.start);
        ctx->event_pool.push_back(r.stop);
    }
    ctx->recs.clear();
    return RAFTGP_OK;
}

raftgp_status raftgp_launch_count(raftgp_ctx ctx, int64_t *out, int reset) {
    if (!ctx || !out) return fail(RAFTGP_ERR_PARAM, "null argument");
    *out = ctx->launches;
    if (reset) ctx->launches = 0;
    return RAFTGP_OK;
}

// ---------------------------------------------------------------- graph
raftgp_status raftgp_build_csr(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                               int64_t row_begin, int64_t row_end, uint32_t flags, raftgp_graph *out) {
    RG_GUARD_BEGIN
    if (!ctx || !out) return fail(RAFTGP_ERR_PARAM, "null argument");
    *out = nullptr;
    if (n < 0 || n >= (int64_t)INT32_MAX || m < 0) return fail(RAFTGP_ERR_PARAM, "n must be in [0, 2^31-1), m >= 0");
    if (row_begin < 0 || row_end < row_begin || row_end > n) return fail(RAFTGP_ERR_PARAM, "bad row range");
    if (m > 0 && (!src || !dst)) return fail(RAFTGP_ERR_PARAM, "null edge arrays");
    if (flags > 1u) return fail(RAFTGP_ERR_PARAM, "bad flags");
    RG_TRY(set_device(ctx));
    const int32_t *dsrc = src, *ddst = dst;
    int32_t *tmp = nullptr;
    if (flags == RAFTGP_HOST_PTRS && m > 0) {
        RG_TRY(dalloc_t(ctx, &tmp, 2 * (size_t)m));
        RG_CUDA(cudaMemcpyAsync(tmp, src, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(tmp + m, dst, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        dsrc = tmp;
        ddst = tmp + m;
    }
    raftgp_graph g = new raftgp_graph_s();
    g->ctx = ctx;
    ctx_retain(ctx);
    raftgp_status st = csr_build(ctx, n, m, dsrc, ddst, row_begin, row_end, g);
    dfree(ctx, tmp);
    if (st != RAFTGP_OK) {
        std::string msg = g_last_error;
        raftgp_graph_destroy(g);
        set_error(msg);
        return st;
    }
    *out = g;
    return RAFTGP_OK;
    RG_GUARD_END
}

raftgp_status raftgp_graph_info(raftgp_graph g, int64_t *n, int64_t *row_begin, int64_t *row_end, int64_t *nnz_local,
                                int64_t *two_e) {
    if (!g) return fail(RAFTGP_ERR_PARAM, "null graph");
    if (n) *n = g->n;
    if (row_begin) *row_begin = g->row_begin;
    if (row_end) *row_end = g->row_end;
    if (nnz_local) *nnz_local = g->nnz_local;
    if (two_e) *two_e = g->two_e;
    return RAFTGP_OK;
}

raftgp_status raftgp_graph_export(raftgp_graph g, int64_t *row_ptr, int32_t *col_idx, int32_t *deg, uint32_t flags) {
    if (!g) return fail(RAFTGP_ERR_PARAM, "null graph");
    if (flags > 1u) return fail(RAFTGP_ERR_PARAM, "bad flags");
    RG_TRY(set_device(g->ctx));
    const cudaMemcpyKind k = flags == RAFTGP_HOST_PTRS ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    cudaStream_t st = g->ctx->stream;
    if (row_ptr) RG_CUDA(cudaMemcpyAsync(row_ptr, g->row_ptr, sizeof(int64_t) * (g->nl + 1), k, st));
    if (col_idx && g->nnz_local) RG_CUDA(cudaMemcpyAsync(col_idx, g->col, sizeof(int32_t) * g->nnz_local, k, st));
    if (deg && g->nl) RG_CUDA(cudaMemcpyAsync(deg, g->deg_local, sizeof(int32_t) * g->nl, k, st));
    if (flags == RAFTGP_HOST_PTRS) RG_CUDA(cudaStreamSynchronize(st));
    return RAFTGP_OK;
}

raftgp_status raftgp_graph_local_degrees(raftgp_graph g, int32_t *deg_dev) {
    if (!g || (!deg_dev && g->nl)) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(set_device(g->ctx));
    if (g->nl)
        RG_TRY(dcopy(g->ctx, deg_dev, g->deg_local, sizeof(int32_t) * g->nl));
    return RAFTGP_OK;
}

raftgp_status raftgp_graph_set_degrees(raftgp_graph g, const int32_t *deg_all_dev) {
    RG_GUARD_BEGIN
    if (!g || (!deg_all_dev && g->n)) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(set_device(g->ctx));
    if (g->n)
        RG_TRY(dcopy(g->ctx, g->deg_all, deg_all_dev, sizeof(int32_t) * g->n));
    return degrees_finalize(g);
    RG_GUARD_END
}

raftgp_status raftgp_graph_set_order(raftgp_graph g, const int32_t *order_dev) {
    if (!g) return fail(RAFTGP_ERR_PARAM, "null graph");
    RG_TRY(set_device(g->ctx));
    if (!order_dev) {   // natural order
        dfree(g->ctx, g->order);
        g->order = nullptr;
        return RAFTGP_OK;
    }
    bool ok = true;
    RG_TRY(order_is_permutation(g->ctx, order_dev, g->nl, &ok));
    if (!ok) return fail(RAFTGP_ERR_PARAM, "order is not a permutation of the local rows 0..rows-1");
    if (g->order == nullptr && g->nl > 0) RG_TRY(dalloc_t(g->ctx, &g->order, (size_t)g->nl));
    if (g->nl > 0)
        RG_TRY(dcopy(g->ctx, g->order, order_dev, sizeof(int32_t) * g->nl));
    return RAFTGP_OK;
}

raftgp_status raftgp_graph_destroy(raftgp_graph g) {
    if (!g) return RAFTGP_OK;
    raftgp_ctx ctx = g->ctx;
    cudaSetDevice(ctx->device);
    dfree(ctx, g->row_ptr);
    dfree(ctx, g->col);
    dfree(ctx, g->deg_local);
    dfree(ctx, g->order);
    dfree(ctx, g->deg_all);
    dfree(ctx, g->s_all);
    dfree(ctx, g->sh_all);
    drop_slots(g);
    delete g;
    ctx_release(ctx);
    return RAFTGP_OK;
}

// ---------------------------------------------------------------- sketch / weights
raftgp_status raftgp_sketch(raftgp_ctx ctx, uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows, int32_t cols,
                            int32_t den, float *out_dev) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    if (rows < 0 || cols <= 0 || den <= 0 || row_begin < 0) return fail(RAFTGP_ERR_PARAM, "bad sketch shape");
    if (rows > 0 && !out_dev) return fail(RAFTGP_ERR_PARAM, "null output");
    RG_TRY(set_device(ctx));
    return sketch_fill(ctx, seed, tag, row_begin, rows, cols, den, out_dev);
}

raftgp_status raftgp_weights(raftgp_ctx ctx, uint64_t seed, int32_t k, int32_t fan_in, int32_t fan_out, float *W_dev) {
    if (k < 1) return fail(RAFTGP_ERR_PARAM, "layer index k must be >= 1");
    if (fan_in <= 0 || fan_out <= 0) return fail(RAFTGP_ERR_PARAM, "layer widths must be > 0");
    return raftgp_sketch(ctx, seed, static_cast<uint32_t>(k), 0, fan_in, fan_out, fan_in, W_dev);
}

raftgp_status raftgp_sketch_transform(raftgp_ctx ctx, uint64_t seed, int64_t rows, int32_t r, const float *W_dev,
                                      int32_t l1, float *out_dev) {
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    if (rows < 0 || !sketch_w_supported(r, l1)) return fail(RAFTGP_ERR_PARAM, "r and l1 must be 32, 64 or 128");
    if (rows > 0 && (!W_dev || !out_dev || !aligned16(W_dev) || !aligned16(out_dev)))
        return fail(RAFTGP_ERR_PARAM, "null or unaligned buffer");
    RG_TRY(set_device(ctx));
    return sketch_w_any(ctx, seed, rows, r, W_dev, l1, out_dev);
}

// ---------------------------------------------------------------- project / gcn
static raftgp_status check_variant(raftgp_graph g, int variant, int32_t r) {
    if (variant < 0 || variant > 2) return fail(RAFTGP_ERR_PARAM, "bad variant");
    if (r <= 0) return fail(RAFTGP_ERR_PARAM, "r must be > 0");
    if (variant != RAFTGP_NCUT && g->two_e == 0)
        return fail(RAFTGP_ERR_DATA, "modularity operator needs at least one edge (2e = 0)");
    return RAFTGP_OK;
}

// Theta (+ g for MOD) into pool workspace; caller frees
static raftgp_status make_theta(raftgp_graph g, int variant, int32_t r, uint64_t seed, float **theta, double **gvec) {
    raftgp_ctx ctx = g->ctx;
    *theta = nullptr;
    *gvec = nullptr;
    RG_TRY(dalloc_t(ctx, theta, (size_t)g->n * r));
    if (variant == RAFTGP_MOD) RG_TRY(dalloc_t(ctx, gvec, (size_t)r));
    return sketch_theta(g, seed, r, *theta, *gvec);
}

raftgp_status raftgp_project(raftgp_graph g, raftgp_variant variant, int32_t r, uint64_t seed, float *Y_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    RG_TRY(check_variant(g, variant, r));
    if (g->nl > 0 && !Y_dev) return fail(RAFTGP_ERR_PARAM, "null Y");
    RG_TRY(set_device(g->ctx));
    float *theta = nullptr;
    double *gvec = nullptr;
    raftgp_status st = make_theta(g, variant, r, seed, &theta, &gvec);
    if (st == RAFTGP_OK) st = feature_hop(g, variant, r, theta, gvec, Y_dev, nullptr, 0, nullptr);
    dfree(g->ctx, theta);
    dfree(g->ctx, gvec);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_gcn_transform(raftgp_graph g, const float *Z_dev, int32_t lin, const float *W_dev, int32_t lout,
                                   float *T_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    if (lin <= 0 || lout <= 0) return fail(RAFTGP_ERR_PARAM, "widths must be > 0");
    if (g->nl > 0 && (!Z_dev || !W_dev || !T_dev)) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(set_device(g->ctx));
    return gcn_transform(g, Z_dev, lin, W_dev, lout, T_dev);
    RG_GUARD_END
}

raftgp_status raftgp_gcn_hop(raftgp_graph g, const float *T_full_dev, int32_t w, float *Z_out_dev,
                             const float *W_next_dev, int32_t w_next, float *T_next_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    if (w <= 0) return fail(RAFTGP_ERR_PARAM, "width must be > 0");
    if (W_next_dev && (w_next <= 0 || !T_next_dev)) return fail(RAFTGP_ERR_PARAM, "W_next needs w_next > 0 and T_next");
    if (g->nl > 0 && !T_full_dev) return fail(RAFTGP_ERR_PARAM, "null T_full");
    RG_TRY(set_device(g->ctx));
    return gcn_hop(g, T_full_dev, w, Z_out_dev, W_next_dev, W_next_dev ? w_next : 0, W_next_dev ? T_next_dev : nullptr);
    RG_GUARD_END
}

static raftgp_status check_dims(int32_t layers, const int32_t *dims) {
    if (layers < 1 || !dims) return fail(RAFTGP_ERR_PARAM, "layers must be >= 1");
    for (int k = 0; k <= layers; ++k)
        if (dims[k] <= 0) return fail(RAFTGP_ERR_PARAM, "every layer width must be > 0");
    return RAFTGP_OK;
}

// GCN layers 1..L given T1 = s^ (.) (Y W1) already computed.
static raftgp_status gcn_stack(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed, float *T1,
                               float *Z_dev, float *const *Zk_dev) {
    raftgp_ctx ctx = g->ctx;
    std::vector<float *> Ws(layers + 1, nullptr);
    raftgp_status st = RAFTGP_OK;
    for (int k = 2; k <= layers && st == RAFTGP_OK; ++k) {
        st = dalloc_t(ctx, &Ws[k], (size_t)dims[k - 1] * dims[k]);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, (uint32_t)k, 0, dims[k - 1], dims[k], dims[k - 1], Ws[k]);
    }
    float *Tcur = T1;
    for (int k = 1; k <= layers && st == RAFTGP_OK; ++k) {
        float *Zout = (k == layers) ? Z_dev : (Zk_dev ? Zk_dev[k - 1] : nullptr);
        float *Tnext = nullptr;
        if (k < layers) st = dalloc_t(ctx, &Tnext, (size_t)g->n * dims[k + 1]);
        if (st == RAFTGP_OK)
            st = gcn_hop(g, Tcur, dims[k], Zout, k < layers ? Ws[k + 1] : nullptr, k < layers ? dims[k + 1] : 0, Tnext);
        if (Tcur != T1) dfree(ctx, Tcur);
        Tcur = Tnext;
    }
    if (Tcur != T1) dfree(ctx, Tcur);
    for (auto w : Ws) dfree(ctx, w);
    return st;
}

// GCN stacks of two variants; their last hop runs as ONE pair hop over the interleaved operand
// [T_a | T_b] written by the previous hops' epilogues (512-B instead of 256-B rows per gather at d = 64).
static raftgp_status gcn_stack_pair(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed, float *T1a,
                                    float *T1b, float *Za, float *Zb) {
    const int32_t d = dims[layers];
    if (layers < 2 || !gcn_pair_supported(d)) {
        RG_TRY(gcn_stack(g, layers, dims, seed, T1a, Za, nullptr));
        return gcn_stack(g, layers, dims, seed, T1b, Zb, nullptr);
    }
    raftgp_ctx ctx = g->ctx;
    std::vector<float *> Ws(layers + 1, nullptr);
    raftgp_status st = RAFTGP_OK;
    for (int k = 2; k <= layers && st == RAFTGP_OK; ++k) {
        st = dalloc_t(ctx, &Ws[k], (size_t)dims[k - 1] * dims[k]);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, (uint32_t)k, 0, dims[k - 1], dims[k], dims[k - 1], Ws[k]);
    }
    float *Tboth = nullptr;
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &Tboth, (size_t)g->n * 2 * d);
    float *cur[2] = {T1a, T1b};
    for (int k = 1; k < layers && st == RAFTGP_OK; ++k) {
        for (int v = 0; v < 2 && st == RAFTGP_OK; ++v) {
            float *Tnext = nullptr;
            int32_t ld = 0;
            if (k + 1 == layers) {
                Tnext = Tboth + v * d;
                ld = 2 * d;
            } else {
                st = dalloc_t(ctx, &Tnext, (size_t)g->n * dims[k + 1]);
            }
            if (st == RAFTGP_OK) st = gcn_hop(g, cur[v], dims[k], nullptr, Ws[k + 1], dims[k + 1], Tnext, ld);
            if (cur[v] != T1a && cur[v] != T1b) dfree(ctx, cur[v]);
            cur[v] = (k + 1 == layers) ? nullptr : Tnext;
        }
    }
    if (st == RAFTGP_OK) st = gcn_final_pair(g, Tboth, d, Za, Zb);
    dfree(ctx, Tboth);
    for (auto w : Ws) dfree(ctx, w);
    return st;
}

static raftgp_status whole_graph(raftgp_graph g) {
    if (g->row_begin != 0 || g->row_end != g->n)
        return fail(RAFTGP_ERR_PARAM, "this call needs a whole-graph handle (use raftgp_gcn_hop per rank)");
    return RAFTGP_OK;
}

raftgp_status raftgp_gnn_embed(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed, const float *Y_dev,
                               float *Z_dev, float *const *Zk_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    RG_TRY(whole_graph(g));
    RG_TRY(check_dims(layers, dims));
    if (g->n > 0 && (!Y_dev || !Z_dev)) return fail(RAFTGP_ERR_PARAM, "null Y or Z");
    RG_TRY(set_device(g->ctx));
    raftgp_ctx ctx = g->ctx;
    float *W1 = nullptr, *T1 = nullptr;
    raftgp_status st = dalloc_t(ctx, &W1, (size_t)dims[0] * dims[1]);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &T1, (size_t)g->n * dims[1]);
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, dims[0], dims[1], dims[0], W1);
    if (st == RAFTGP_OK) st = gcn_transform(g, Y_dev, dims[0], W1, dims[1], T1);
    if (st == RAFTGP_OK) st = gcn_stack(g, layers, dims, seed, T1, Z_dev, Zk_dev);
    dfree(ctx, W1);
    dfree(ctx, T1);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_embed(raftgp_graph g, raftgp_variant variant, int32_t layers, const int32_t *dims, uint64_t seed,
                           float *Y_dev, float *Z_dev, float *const *Zk_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    RG_TRY(whole_graph(g));
    RG_TRY(check_dims(layers, dims));
    RG_TRY(check_variant(g, variant, dims[0]));
    if (g->n > 0 && !Z_dev) return fail(RAFTGP_ERR_PARAM, "null Z");
    RG_TRY(set_device(g->ctx));
    raftgp_ctx ctx = g->ctx;
    const int32_t r = dims[0];
    float *theta = nullptr, *W1 = nullptr, *T1 = nullptr;
    double *gvec = nullptr;
    raftgp_status st = make_theta(g, variant, r, seed, &theta, &gvec);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &W1, (size_t)dims[0] * dims[1]);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &T1, (size_t)g->n * dims[1]);
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, dims[0], dims[1], dims[0], W1);
    if (st == RAFTGP_OK) st = feature_hop(g, variant, r, theta, gvec, Y_dev, W1, dims[1], T1);
    dfree(ctx, theta);
    dfree(ctx, gvec);
    if (st == RAFTGP_OK) st = gcn_stack(g, layers, dims, seed, T1, Z_dev, Zk_dev);
    dfree(ctx, W1);
    dfree(ctx, T1);
    return st;
    RG_GUARD_END
}

// project + GCN without materialising Y: Theta' = Theta W1 is generated once (Theta on chip), every
// variant's first operand T1 = s^ (.) (X Theta') comes from a GEMM-free feature hop (NCUT and MOD share
// one gather), then the GCN stacks. Same results as the Y path up to fp32 rounding order (reading #13).
// T1 = s^ (.) (X Theta W1) of the local rows for every listed variant (Theta' = Theta W1 on chip, one
// shared gather for NCUT + MOD). T1[v]: local_rows x l1 device buffers.
// T1 of every variant from Theta' = Theta W1 (thw_pre: already computed, e.g. on a side stream; else here)
static raftgp_status first_transform_pre(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t r,
                                         int32_t l1, uint64_t seed, float *const *T1, const int where[3],
                                         const float *thw_pre = nullptr, float *const *rep = nullptr,
                                         int32_t nrep = 0) {
    raftgp_ctx ctx = g->ctx;
    float *W1 = nullptr, *thw = nullptr;
    double *gw = nullptr;
    raftgp_status st = RAFTGP_OK;
    if (!thw_pre) {
        st = dalloc_t(ctx, &W1, (size_t)r * l1);
        if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, r, l1, r, W1);
        if (st == RAFTGP_OK) st = dalloc_t(ctx, &thw, (size_t)g->n * l1);
        if (st == RAFTGP_OK && g->slots_active)   // Theta' rows written into the slot layout (relabel.cu)
            st = sketch_w_tc_rows(ctx, seed, 0, g->n, r, W1, l1, &thw, 1, g->slot);
        else if (st == RAFTGP_OK)
            st = sketch_w_any(ctx, seed, g->n, r, W1, l1, thw);
    }
    const float *tw = thw_pre ? thw_pre : thw;
    if (st == RAFTGP_OK && where[RAFTGP_MOD] >= 0) st = dalloc_t(ctx, &gw, (size_t)l1);
    if (st == RAFTGP_OK && gw) st = g_reduce(g, tw, l1, gw);
    const bool dual = where[RAFTGP_NCUT] >= 0 && where[RAFTGP_MOD] >= 0;
    // rep (push mode): variant v's replicas are rep[v * nrep .. v * nrep + nrep)
    auto spec = [&](int va, int vb) {
        PushSpec p{};
        p.nrep = nrep;
        p.row0 = g->row_begin;
        for (int q = 0; q < nrep; ++q) {
            p.rep[q] = rep[(size_t)va * nrep + q];
            p.rep2[q] = vb >= 0 ? rep[(size_t)vb * nrep + q] : nullptr;
        }
        return p;
    };
    if (st == RAFTGP_OK && dual) {
        const int a = where[RAFTGP_NCUT], b = where[RAFTGP_MOD];
        const PushSpec p = rep ? spec(a, b) : PushSpec{};
        st = feature_hop_pre(g, -1, l1, tw, gw, T1 ? T1[a] : nullptr, T1 ? T1[b] : p.rep2[0], rep ? &p : nullptr);
    }
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
        if (dual && (variants[v] == RAFTGP_NCUT || variants[v] == RAFTGP_MOD)) continue;
        const PushSpec p = rep ? spec(v, -1) : PushSpec{};
        st = feature_hop_pre(g, variants[v], l1, tw, gw, T1 ? T1[v] : nullptr, nullptr, rep ? &p : nullptr);
    }
    dfree(ctx, thw);
    dfree(ctx, gw);
    dfree(ctx, W1);
    return st;
}

// the slot layout applies to whole-graph embeddings with the tcgen05 Theta' kernel (it writes the slots)
static bool slots_usable(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                         const int32_t *dims) {
    for (int v = 0; v < nvariants; ++v)
        if (variants[v] != RAFTGP_NCUT && variants[v] != RAFTGP_MOD) return false;   // MOD_REDUCED gathers by node id
    for (int k = 1; k <= layers; ++k)   // every hop on the fast kernels (the generic one gathers by node id)
        if (dims[k] != 32 && dims[k] != 64 && dims[k] != 128) return false;
    return slots_enabled() && sketch_tc_enabled() && g->row_begin == 0 && g->row_end == g->n && g->n > 0 &&
           g->nnz_local > 0;
}

static raftgp_status embed_pre(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                               const int32_t *dims, uint64_t seed, float *const *Z_dev, const int where[3],
                               const float *thw_pre = nullptr) {
    raftgp_ctx ctx = g->ctx;
    const int32_t r = dims[0], l1 = dims[1];
    std::vector<float *> T1(nvariants, nullptr);
    raftgp_status st = RAFTGP_OK;
    // slot layout of the operands (relabel.cu): the hub rows first, so the hops keep them in L2. Theta' must then be
    // generated here (in slots), not handed in
    if (!thw_pre && slots_usable(g, nvariants, variants, layers, dims)) {
        st = ensure_slots(g);
        g->slots_active = st == RAFTGP_OK;
    }
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) st = dalloc_t(ctx, &T1[v], (size_t)g->n * l1);
    if (st == RAFTGP_OK) st = first_transform_pre(g, nvariants, variants, r, l1, seed, T1.data(), where, thw_pre);
    const bool dual = where[RAFTGP_NCUT] >= 0 && where[RAFTGP_MOD] >= 0;
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
        if (dual && variants[v] == RAFTGP_MOD) continue;    // computed with its NCUT partner below
        if (dual && variants[v] == RAFTGP_NCUT) {
            const int a = where[RAFTGP_NCUT], b = where[RAFTGP_MOD];
            st = gcn_stack_pair(g, layers, dims, seed, T1[a], T1[b], Z_dev[a], Z_dev[b]);
        } else {
            st = gcn_stack(g, layers, dims, seed, T1[v], Z_dev[v], nullptr);
        }
    }
    for (auto t : T1) dfree(ctx, t);
    g->slots_active = false;
    return st;
}

raftgp_status raftgp_embed_multi(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                                 const int32_t *dims, uint64_t seed, float *const *Y_dev, float *const *Z_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    RG_TRY(whole_graph(g));
    RG_TRY(check_dims(layers, dims));
    if (nvariants < 1 || !variants || !Z_dev) return fail(RAFTGP_ERR_PARAM, "need >= 1 variant and Z outputs");
    int where[3] = {-1, -1, -1};
    for (int v = 0; v < nvariants; ++v) {
        RG_TRY(check_variant(g, variants[v], dims[0]));
        if (where[variants[v]] >= 0) return fail(RAFTGP_ERR_PARAM, "variant listed twice");
        where[variants[v]] = v;
        if (g->n > 0 && !Z_dev[v]) return fail(RAFTGP_ERR_PARAM, "null Z");
    }
    RG_TRY(set_device(g->ctx));
    raftgp_ctx ctx = g->ctx;
    const int32_t r = dims[0];
    if (Y_dev == nullptr && wide_supported(layers, dims))
        return embed_wide(g, nvariants, variants, layers, dims, seed, Z_dev, where);
    if (Y_dev == nullptr && sketch_w_supported(r, dims[1]))
        return embed_pre(g, nvariants, variants, layers, dims, seed, Z_dev, where);
    float *theta = nullptr, *W1 = nullptr;
    double *gvec = nullptr;
    std::vector<float *> T1(nvariants, nullptr);
    raftgp_status st = dalloc_t(ctx, &theta, (size_t)g->n * r);
    if (st == RAFTGP_OK && where[RAFTGP_MOD] >= 0) st = dalloc_t(ctx, &gvec, (size_t)r);
    if (st == RAFTGP_OK) st = sketch_theta(g, seed, r, theta, gvec);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &W1, (size_t)dims[0] * dims[1]);
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, dims[0], dims[1], dims[0], W1);
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) st = dalloc_t(ctx, &T1[v], (size_t)g->n * dims[1]);
    auto Yp = [&](int v) { return Y_dev ? Y_dev[v] : nullptr; };
    const bool dual = where[RAFTGP_NCUT] >= 0 && where[RAFTGP_MOD] >= 0;
    if (st == RAFTGP_OK && dual) {
        const int a = where[RAFTGP_NCUT], b = where[RAFTGP_MOD];
        st = feature_hop_dual(g, r, theta, gvec, Yp(a), Yp(b), W1, dims[1], T1[a], T1[b]);
    }
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
        if (dual && (variants[v] == RAFTGP_NCUT || variants[v] == RAFTGP_MOD)) continue;
        st = feature_hop(g, variants[v], r, theta, gvec, Yp(v), W1, dims[1], T1[v]);
    }
    dfree(ctx, theta);
    dfree(ctx, gvec);
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) st = gcn_stack(g, layers, dims, seed, T1[v], Z_dev[v], nullptr);
    dfree(ctx, W1);
    for (auto t : T1) dfree(ctx, t);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_feature_transform(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t r,
                                       int32_t l1, uint64_t seed, float *const *T1_dev) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    if (nvariants < 1 || !variants || !T1_dev) return fail(RAFTGP_ERR_PARAM, "need >= 1 variant and outputs");
    if (l1 <= 0) return fail(RAFTGP_ERR_PARAM, "l1 must be > 0");
    int where[3] = {-1, -1, -1};
    for (int v = 0; v < nvariants; ++v) {
        RG_TRY(check_variant(g, variants[v], r));
        if (where[variants[v]] >= 0) return fail(RAFTGP_ERR_PARAM, "variant listed twice");
        where[variants[v]] = v;
        if (g->nl > 0 && !T1_dev[v]) return fail(RAFTGP_ERR_PARAM, "null T1");
    }
    RG_TRY(set_device(g->ctx));
    if (sketch_w_supported(r, l1)) {
        bool al = true;
        for (int v = 0; v < nvariants; ++v) al = al && aligned16(T1_dev[v]);
        if (al) return first_transform_pre(g, nvariants, variants, r, l1, seed, T1_dev, where);
    }
    // any other shape: Theta materialised, feature hop then transform per variant
    raftgp_ctx ctx = g->ctx;
    float *theta = nullptr, *W1 = nullptr, *Y = nullptr;
    double *gvec = nullptr;
    raftgp_status st = dalloc_t(ctx, &theta, (size_t)g->n * r);
    if (st == RAFTGP_OK && where[RAFTGP_MOD] >= 0) st = dalloc_t(ctx, &gvec, (size_t)r);
    if (st == RAFTGP_OK) st = sketch_theta(g, seed, r, theta, gvec);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &W1, (size_t)r * l1);
    if (st == RAFTGP_OK) st = sketch_fill(ctx, seed, 1u, 0, r, l1, r, W1);
    if (st == RAFTGP_OK) st = dalloc_t(ctx, &Y, (size_t)g->nl * r);
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
        st = feature_hop(g, variants[v], r, theta, gvec, Y, nullptr, 0, nullptr);
        if (st == RAFTGP_OK) st = gcn_transform(g, Y, r, W1, l1, T1_dev[v]);
    }
    dfree(ctx, theta);
    dfree(ctx, gvec);
    dfree(ctx, W1);
    dfree(ctx, Y);
    return st;
    RG_GUARD_END
}

// ---------------------------------------------------------------- a7: host scoring
static raftgp_status host_mirror(raftgp_graph g) {
    RG_TRY(whole_graph(g));
    if (g->host_valid) return RAFTGP_OK;
    g->h_row_ptr.resize(g->nl + 1);
    g->h_col.resize(g->nnz_local);
    RG_TRY(raftgp_graph_export(g, g->h_row_ptr.data(), g->h_col.data(), nullptr, RAFTGP_HOST_PTRS));
    g->host_valid = true;
    return RAFTGP_OK;
}

static raftgp_status check_labels(const int32_t *assign, int64_t n, int32_t k) {
    if (k <= 0) return fail(RAFTGP_ERR_PARAM, "k must be > 0");
    if (n > 0 && !assign) return fail(RAFTGP_ERR_PARAM, "null labels");
    for (int64_t i = 0; i < n; ++i)
        if (assign[i] < 0 || assign[i] >= k) return fail(RAFTGP_ERR_PARAM, "label outside [0, k)");
    return RAFTGP_OK;
}

raftgp_status raftgp_modularity(raftgp_graph g, const int32_t *assign, int32_t k, double *out) {
    RG_GUARD_BEGIN
    if (!g || !out) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(host_mirror(g));
    RG_TRY(check_labels(assign, g->n, k));
    const int64_t two_e = g->h_row_ptr[g->n];
    if (two_e == 0) return fail(RAFTGP_ERR_DATA, "modularity of a graph without edges");
    // per-block intra (directed) edge counts and volumes, Eq. 3 regrouped by block
    std::vector<int64_t> intra(k, 0), vol(k, 0);
    for (int64_t i = 0; i < g->n; ++i) {
        const int32_t bi = assign[i];
        vol[bi] += g->h_row_ptr[i + 1] - g->h_row_ptr[i];
        for (int64_t p = g->h_row_ptr[i]; p < g->h_row_ptr[i + 1]; ++p) intra[bi] += (assign[g->h_col[p]] == bi);
    }
    const double e2 = static_cast<double>(two_e);
    double q = 0.0;
    for (int32_t b = 0; b < k; ++b) {
        const double f = static_cast<double>(vol[b]) / e2;
        q += static_cast<double>(intra[b]) / e2 - f * f;
    }
    *out = q;
    return RAFTGP_OK;
    RG_GUARD_END
}

raftgp_status raftgp_ncut(raftgp_graph g, const int32_t *assign, int32_t k, double *out) {
    RG_GUARD_BEGIN
    if (!g || !out) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(host_mirror(g));
    RG_TRY(check_labels(assign, g->n, k));
    std::vector<int64_t> cut(k, 0), vol(k, 0);
    for (int64_t i = 0; i < g->n; ++i) {
        const int32_t bi = assign[i];
        vol[bi] += g->h_row_ptr[i + 1] - g->h_row_ptr[i];
        for (int64_t p = g->h_row_ptr[i]; p < g->h_row_ptr[i + 1]; ++p) cut[bi] += (assign[g->h_col[p]] != bi);
    }
    double s = 0.0;
    for (int32_t b = 0; b < k; ++b)
        if (vol[b] > 0) s += static_cast<double>(cut[b]) / static_cast<double>(vol[b]);
    *out = 0.5 * s;
    return RAFTGP_OK;
    RG_GUARD_END
}

raftgp_status raftgp_local_modularity(raftgp_graph g, const int64_t *nodes, int64_t count, const int32_t *block_of_node,
                                      int32_t k, double *out) {
    RG_GUARD_BEGIN
    if (!g || !out || count < 0 || (count > 0 && (!nodes || !block_of_node))) return fail(RAFTGP_ERR_PARAM, "bad argument");
    if (k <= 0) return fail(RAFTGP_ERR_PARAM, "k must be > 0");
    RG_TRY(host_mirror(g));
    std::vector<int32_t> blk(g->n, -1);
    for (int64_t t = 0; t < count; ++t) {
        const int64_t v = nodes[t];
        if (v < 0 || v >= g->n) return fail(RAFTGP_ERR_PARAM, "node outside [0, n)");
        if (block_of_node[t] < 0 || block_of_node[t] >= k) return fail(RAFTGP_ERR_PARAM, "label outside [0, k)");
        if (blk[v] >= 0) return fail(RAFTGP_ERR_PARAM, "node listed twice");
        blk[v] = block_of_node[t];
    }
    std::vector<int64_t> intra(k, 0), mbar(k, 0);
    for (int64_t t = 0; t < count; ++t) {
        const int64_t v = nodes[t];
        const int32_t b = blk[v];
        mbar[b] += g->h_row_ptr[v + 1] - g->h_row_ptr[v];
        for (int64_t p = g->h_row_ptr[v]; p < g->h_row_ptr[v + 1]; ++p) intra[b] += (blk[g->h_col[p]] == b);
    }
    int64_t two_e = 0;
    for (int32_t b = 0; b < k; ++b) two_e += mbar[b];
    if (two_e == 0) return fail(RAFTGP_ERR_DATA, "local modularity with zero total degree");
    // Eq. 7: sum_r m_r / e - (mbar_r / 2e)^2 with m_r = intra_r / 2 (each intra edge seen from both ends)
    const double e2 = static_cast<double>(two_e);
    double q = 0.0;
    for (int32_t b = 0; b < k; ++b) {
        const double f = static_cast<double>(mbar[b]) / e2;
        q += static_cast<double>(intra[b]) / e2 - f * f;
    }
    *out = q;
    return RAFTGP_OK;
    RG_GUARD_END
}

// ---------------------------------------------------------------- NEXT-1: Alg. 1 model selection
raftgp_status raftgp_model_select(raftgp_graph g, const float *Z_dev, int32_t L, int32_t eps, int32_t max_iter,
                                  int32_t rule, int32_t *labels_dev, int32_t *num_blocks, int64_t *stats) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    RG_TRY(whole_graph(g));
    if (!num_blocks) return fail(RAFTGP_ERR_PARAM, "null num_blocks");
    if (eps < 0 || max_iter < 1) return fail(RAFTGP_ERR_PARAM, "eps must be >= 0 and max_iter >= 1");
    if (rule != RAFTGP_LMOD_GLOBAL && rule != RAFTGP_LMOD_LOCAL) return fail(RAFTGP_ERR_PARAM, "bad LMod rule");
    if (g->n > 0 && (!Z_dev || !labels_dev)) return fail(RAFTGP_ERR_PARAM, "null Z or labels");
    if (g->n > 0 && !aligned16(Z_dev)) return fail(RAFTGP_ERR_PARAM, "Z must be 16-byte aligned");
    RG_TRY(set_device(g->ctx));
    if (g->n == 0) {
        *num_blocks = 0;
        if (stats) for (int i = 0; i < 7; ++i) stats[i] = 0;
        return RAFTGP_OK;
    }
    return model_select(g, Z_dev, L, eps, max_iter, rule, labels_dev, num_blocks, stats);
    RG_GUARD_END
}

// ---------------------------------------------------------------- NEXT-2: tensor-core GEMM
raftgp_status raftgp_gemm_tf32x3(raftgp_ctx ctx, int64_t M, int32_t K, int32_t N, const float *A_dev, const float *B_dev,
                                 const float *row_scale_dev, float *C_dev) {
    RG_GUARD_BEGIN
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null context");
    if (M < 0 || K <= 0 || N <= 0) return fail(RAFTGP_ERR_PARAM, "M must be >= 0, K and N > 0");
    if (M > 0 && (!A_dev || !B_dev || !C_dev)) return fail(RAFTGP_ERR_PARAM, "null A, B or C");
    RG_TRY(set_device(ctx));
    return gemm_rowmajor(ctx, A_dev, M, K, B_dev, N, row_scale_dev, C_dev);
    RG_GUARD_END
}

// ---------------------------------------------------------------- NEXT-3: Alg. 2 SBM sampler
raftgp_status raftgp_sbm_sample(raftgp_ctx ctx, int64_t n, int32_t K, const int32_t *c_dev, const double *theta_dev,
                                const double *omega_dev, uint64_t seed, int32_t q, int32_t *src_dev, int32_t *dst_dev,
                                int64_t cap, int64_t *m_out) {
    RG_GUARD_BEGIN
    if (!ctx || !m_out) return fail(RAFTGP_ERR_PARAM, "null argument");
    if (n < 0 || n + K >= (int64_t)INT32_MAX || K <= 0 || q < 4 || q > 30 || cap < 0)
        return fail(RAFTGP_ERR_PARAM, "need 0 <= n, n + K < 2^31 - 1, K > 0, 4 <= q <= 30, cap >= 0");
    if (n > 0 && (!c_dev || !theta_dev)) return fail(RAFTGP_ERR_PARAM, "null c or theta");
    if (!omega_dev) return fail(RAFTGP_ERR_PARAM, "null omega");
    if (cap > 0 && (!src_dev || !dst_dev)) return fail(RAFTGP_ERR_PARAM, "null edge outputs");
    RG_TRY(set_device(ctx));
    return sbm_sample(ctx, n, K, c_dev, theta_dev, omega_dev, seed, q, src_dev, dst_dev, cap, m_out);
    RG_GUARD_END
}

// ---------------------------------------------------------------- NEXT-4: streaming updates
raftgp_status raftgp_stream_create(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed,
                                   raftgp_stream *out) {
    RG_GUARD_BEGIN
    if (!out) return fail(RAFTGP_ERR_PARAM, "null out");
    *out = nullptr;
    RG_TRY(need_ready(g));
    RG_TRY(whole_graph(g));
    RG_TRY(check_dims(layers, dims));
    RG_TRY(set_device(g->ctx));
    return stream_create(g, layers, dims, seed, out);
    RG_GUARD_END
}

raftgp_status raftgp_stream_add_edges(raftgp_stream s, int64_t m, const int32_t *src, const int32_t *dst,
                                      uint32_t flags, int64_t *stats) {
    RG_GUARD_BEGIN
    if (!s) return fail(RAFTGP_ERR_PARAM, "null stream");
    if (m < 0 || (m > 0 && (!src || !dst)) || flags > 1u) return fail(RAFTGP_ERR_PARAM, "bad edge arguments");
    raftgp_ctx ctx = s->ctx;
    RG_TRY(set_device(ctx));
    const int32_t *dsrc = src, *ddst = dst;
    int32_t *tmp = nullptr;
    if (flags == RAFTGP_HOST_PTRS && m > 0) {
        RG_TRY(dalloc_t(ctx, &tmp, 2 * (size_t)m));
        RG_CUDA(cudaMemcpyAsync(tmp, src, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(tmp + m, dst, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        dsrc = tmp;
        ddst = tmp + m;
    }
    raftgp_status st = stream_add(s, m, dsrc, ddst, stats);
    dfree(ctx, tmp);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_stream_embedding(raftgp_stream s, float *Z_dev) {
    if (!s || (!Z_dev && s->g->n > 0)) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(set_device(s->ctx));
    if (s->g->n > 0) RG_TRY(dcopy(s->ctx, Z_dev, s->Z, sizeof(float) * (size_t)s->g->n * s->dims[s->layers]));
    return RAFTGP_OK;
}

raftgp_status raftgp_stream_graph(raftgp_stream s, raftgp_graph *g_out) {
    if (!s || !g_out) return fail(RAFTGP_ERR_PARAM, "null argument");
    *g_out = s->g;
    return RAFTGP_OK;
}

raftgp_status raftgp_stream_set_mode(raftgp_stream s, int32_t mode) {
    RG_GUARD_BEGIN
    if (!s) return fail(RAFTGP_ERR_PARAM, "null stream");
    if (mode != RAFTGP_STREAM_EXACT && mode != RAFTGP_STREAM_DELTA) return fail(RAFTGP_ERR_PARAM, "unknown stream mode");
    RG_TRY(set_device(s->ctx));
    return stream_set_mode(s, mode);
    RG_GUARD_END
}

raftgp_status raftgp_stream_destroy(raftgp_stream s) {
    if (!s) return RAFTGP_OK;
    cudaSetDevice(s->ctx->device);
    stream_destroy(s);
    return RAFTGP_OK;
}

// ---------------------------------------------------------------- row-partitioned build + embed (dist.cu)
static raftgp_status build_embed_partitioned(raftgp_ctx ctx, int32_t P, bool loopback, int64_t n, int64_t m,
                                             const int32_t *src, const int32_t *dst, uint32_t flags, int32_t nvariants,
                                             const int32_t *variants, int32_t layers, const int32_t *dims, uint64_t seed,
                                             float *const *Z_dev) {
    int seen[3] = {0, 0, 0};
    for (int v = 0; v < nvariants; ++v) {
        if (variants[v] < 0 || variants[v] > 2) return fail(RAFTGP_ERR_PARAM, "bad variant");
        if (seen[variants[v]]++) return fail(RAFTGP_ERR_PARAM, "variant listed twice");
        if (n > 0 && !Z_dev[v]) return fail(RAFTGP_ERR_PARAM, "null Z");
        if (Z_dev[v] && !aligned16(Z_dev[v])) return fail(RAFTGP_ERR_PARAM, "Z must be 16-byte aligned");
    }
    const int32_t *dsrc = src, *ddst = dst;
    int32_t *tmp = nullptr;
    if (flags == RAFTGP_HOST_PTRS && m > 0) {
        RG_TRY(dalloc_t(ctx, &tmp, 2 * (size_t)m));
        RG_CUDA(cudaMemcpyAsync(tmp, src, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(tmp + m, dst, sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        dsrc = tmp;
        ddst = tmp + m;
    }
    raftgp_status st = dist_build_embed(ctx, P, loopback, n, m, dsrc, ddst, nvariants, variants, layers, dims, seed, Z_dev);
    dfree(ctx, tmp);
    return st;
}

// ---------------------------------------------------------------- build + embed with overlap
// raftgp_build_csr + raftgp_embed_multi in one call. Theta' = Theta W^(1) depends only on the seed, so it is
// generated on a side stream (tensor cores / ALUs) while the CSR build (atomics / HBM) runs on the context
// stream; the results are those of the two separate calls.
// How Theta' overlaps the CSR build (RAFTGP_OVERLAP_MODE):
//   split (default): Theta' as persistent CTAs on RAFTGP_OVERLAP_CTAS SMs (default half), the CSR build beside it;
//   prio:            the CSR build runs on a high-priority library stream, Theta' on the (default-priority) side stream
//                    as many short CTAs (16 tiles each): the block scheduler gives every SM that frees up to the CSR
//                    kernels first, and Theta' fills the gaps (host read-backs, small kernels, kernel tails);
//   serial:          Theta' on every SM, then the CSR build (also RAFTGP_BUILD_OVERLAP=0).
// All three measured within 0.4 ms of each other at C4 (72.8-73.2 ms) and C5 (780 ms): the two phases' work adds up
// whatever the arrangement (profiles/r02/overlap_modes.txt).
enum class OverlapMode { prio, split, serial };
static OverlapMode overlap_mode() {
    static const OverlapMode m = [] {
        const char *b = getenv("RAFTGP_BUILD_OVERLAP");
        if (b && b[0] == '0') return OverlapMode::serial;
        const char *e = getenv("RAFTGP_OVERLAP_MODE");
        if (e && !strcmp(e, "prio")) return OverlapMode::prio;
        if (e && !strcmp(e, "serial")) return OverlapMode::serial;
        return OverlapMode::split;
    }();
    return m;
}
static int build_overlap_ctas(raftgp_ctx ctx, int64_t n) {
    static const int env = [] {
        const char *e = getenv("RAFTGP_OVERLAP_CTAS");
        return e ? atoi(e) : -1;
    }();
    if (env >= 0) return env;
    switch (overlap_mode()) {
        case OverlapMode::prio: return (int)std::max<int64_t>(ctx->sm_count, ceil_div(n, (int64_t)128 * 16));
        case OverlapMode::split: return std::max(1, ctx->sm_count / 2);
        default: return ctx->sm_count;
    }
}

raftgp_status raftgp_build_embed(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                 uint32_t flags, int32_t nvariants, const int32_t *variants, int32_t layers,
                                 const int32_t *dims, uint64_t seed, float *const *Z_dev, raftgp_graph *g_out) {
    RG_GUARD_BEGIN
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    if (g_out) *g_out = nullptr;
    RG_TRY(check_dims(layers, dims));
    if (nvariants < 1 || !variants || !Z_dev) return fail(RAFTGP_ERR_PARAM, "need >= 1 variant and Z outputs");
    if (n < 0 || n >= (int64_t)INT32_MAX || m < 0 || flags > 1u || (m > 0 && (!src || !dst)))
        return fail(RAFTGP_ERR_PARAM, "bad graph arguments");
    RG_TRY(set_device(ctx));
    if (ctx->nccl) {   // distributed context: the row-partitioned step (dist.cu)
        if (g_out) return fail(RAFTGP_ERR_PARAM, "distributed build_embed returns no graph handle (g_out must be NULL)");
        return build_embed_partitioned(ctx, ctx->world, false, n, m, src, dst, flags, nvariants, variants, layers, dims,
                                       seed, Z_dev);
    }
    const int32_t r = dims[0], l1 = dims[1];
    // with the slot layout Theta' is generated after the CSR build (its rows go to slots that need the degrees);
    // the arrangements measured the same step time
    const bool overlap = sketch_w_supported(r, l1) && !wide_supported(layers, dims) && n > 0 &&
                         !(slots_enabled() && sketch_tc_enabled());
    float *W1 = nullptr, *thw = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    raftgp_status st = RAFTGP_OK;
    if (overlap) {
        if (!ctx->side) RG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        RG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        RG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        st = dalloc_t(ctx, &W1, (size_t)r * l1);
        if (st == RAFTGP_OK) st = dalloc_t(ctx, &thw, (size_t)n * l1);
        if (st == RAFTGP_OK) {
            RG_CUDA(cudaEventRecord(ev_fork, ctx->stream));
            RG_CUDA(cudaStreamWaitEvent(ctx->side, ev_fork, 0));
            const bool serial = overlap_mode() == OverlapMode::serial;
            cudaStream_t main = ctx->stream;
            if (!serial) ctx->stream = ctx->side;   // the sketch kernels enqueue on the side stream
            ctx->sketch_ctas = build_overlap_ctas(ctx, n);
            st = sketch_fill(ctx, seed, 1u, 0, r, l1, r, W1);
            if (st == RAFTGP_OK) st = sketch_w_any(ctx, seed, n, r, W1, l1, thw);
            ctx->sketch_ctas = 0;
            ctx->stream = main;
            RG_CUDA(cudaEventRecord(ev_join, ctx->side));
        }
    }
    raftgp_graph g = nullptr;
    if (st == RAFTGP_OK && overlap && overlap_mode() == OverlapMode::prio) {
        // the CSR build on the high-priority stream, forked from and joined back into the caller's stream
        if (!ctx->hip) {
            int lo = 0, hi = 0;
            RG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            RG_CUDA(cudaStreamCreateWithPriority(&ctx->hip, cudaStreamNonBlocking, hi));
        }
        cudaEvent_t ev_b = nullptr;
        RG_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
        RG_CUDA(cudaStreamWaitEvent(ctx->hip, ev_fork, 0));
        cudaStream_t main = ctx->stream;
        ctx->stream = ctx->hip;
        st = raftgp_build_csr(ctx, n, m, src, dst, 0, n, flags, &g);
        ctx->stream = main;
        cudaEventRecord(ev_b, ctx->hip);
        cudaStreamWaitEvent(main, ev_b, 0);
        cudaEventDestroy(ev_b);
    } else if (st == RAFTGP_OK) {
        st = raftgp_build_csr(ctx, n, m, src, dst, 0, n, flags, &g);
    }
    if (overlap && ev_join) cudaStreamWaitEvent(ctx->stream, ev_join, 0);   // Theta' ready (also on failure)
    if (st == RAFTGP_OK) {
        int where[3] = {-1, -1, -1};
        for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) {
            st = check_variant(g, variants[v], r);
            if (st == RAFTGP_OK && where[variants[v]] >= 0) st = fail(RAFTGP_ERR_PARAM, "variant listed twice");
            if (st == RAFTGP_OK) where[variants[v]] = v;
            if (st == RAFTGP_OK && !Z_dev[v] && g->nl > 0) st = fail(RAFTGP_ERR_PARAM, "null Z");
        }
        if (st == RAFTGP_OK) {
            if (overlap) st = embed_pre(g, nvariants, variants, layers, dims, seed, Z_dev, where, thw);
            else st = raftgp_embed_multi(g, nvariants, variants, layers, dims, seed, nullptr, Z_dev);
        }
    }
    dfree(ctx, W1);
    dfree(ctx, thw);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (st == RAFTGP_OK && g_out) *g_out = g;
    else if (g) raftgp_graph_destroy(g);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_build_embed_loopback(raftgp_ctx ctx, int32_t P, int64_t n, int64_t m, const int32_t *src,
                                          const int32_t *dst, uint32_t flags, int32_t nvariants, const int32_t *variants,
                                          int32_t layers, const int32_t *dims, uint64_t seed, float *const *Z_dev) {
    RG_GUARD_BEGIN
    if (!ctx) return fail(RAFTGP_ERR_PARAM, "null ctx");
    RG_TRY(check_dims(layers, dims));
    if (P < 1 || P > kMaxPush) return fail(RAFTGP_ERR_PARAM, "P must be in [1, 8]");
    if (nvariants < 1 || !variants || !Z_dev) return fail(RAFTGP_ERR_PARAM, "need >= 1 variant and Z outputs");
    if (n < 0 || n >= (int64_t)INT32_MAX || m < 0 || flags > 1u || (m > 0 && (!src || !dst)))
        return fail(RAFTGP_ERR_PARAM, "bad graph arguments");
    RG_TRY(set_device(ctx));
    return build_embed_partitioned(ctx, P, true, n, m, src, dst, flags, nvariants, variants, layers, dims, seed, Z_dev);
    RG_GUARD_END
}

// ---------------------------------------------------------------- fused exchange (a6): push replicas + CUDA IPC
static raftgp_status check_reps(float *const *rep, int32_t nrep, int32_t nvariants) {
    if (!rep || nrep < 1 || nrep > kMaxPush) return fail(RAFTGP_ERR_PARAM, "push: need 1..8 replicas");
    for (int64_t i = 0; i < (int64_t)nrep * nvariants; ++i)
        if (!rep[i]) return fail(RAFTGP_ERR_PARAM, "push: null replica");
    return RAFTGP_OK;
}

raftgp_status raftgp_feature_transform_push(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t r,
                                            int32_t l1, uint64_t seed, float *const *rep, int32_t nrep) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    if (nvariants < 1 || !variants) return fail(RAFTGP_ERR_PARAM, "need >= 1 variant");
    if (l1 <= 0) return fail(RAFTGP_ERR_PARAM, "l1 must be > 0");
    RG_TRY(check_reps(rep, nrep, nvariants));
    int where[3] = {-1, -1, -1};
    for (int v = 0; v < nvariants; ++v) {
        RG_TRY(check_variant(g, variants[v], r));
        if (where[variants[v]] >= 0) return fail(RAFTGP_ERR_PARAM, "variant listed twice");
        where[variants[v]] = v;
    }
    RG_TRY(set_device(g->ctx));
    if (g->nl == 0) return RAFTGP_OK;
    bool al = sketch_w_supported(r, l1) && push_fusable(l1, 0);
    for (int64_t i = 0; i < (int64_t)nrep * nvariants; ++i) al = al && aligned16(rep[i]);
    if (al) return first_transform_pre(g, nvariants, variants, r, l1, seed, nullptr, where, nullptr, rep, nrep);
    // other shapes: local T1, then copied into every replica (not overlapped)
    raftgp_ctx ctx = g->ctx;
    std::vector<float *> T(nvariants, nullptr);
    raftgp_status st = RAFTGP_OK;
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v) st = dalloc_t(ctx, &T[v], (size_t)g->nl * l1);
    if (st == RAFTGP_OK) st = raftgp_feature_transform(g, nvariants, variants, r, l1, seed, T.data());
    for (int v = 0; v < nvariants && st == RAFTGP_OK; ++v)
        for (int q = 0; q < nrep && st == RAFTGP_OK; ++q)
            st = dcopy(ctx, rep[(size_t)v * nrep + q] + (size_t)g->row_begin * l1, T[v], sizeof(float) * g->nl * l1);
    for (auto t : T) dfree(ctx, t);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_gcn_hop_push(raftgp_graph g, const float *T_full_dev, int32_t w, float *Z_out_dev,
                                  const float *W_next_dev, int32_t w_next, float *const *rep, int32_t nrep) {
    RG_GUARD_BEGIN
    RG_TRY(need_ready(g));
    if (w <= 0 || w_next <= 0 || !W_next_dev) return fail(RAFTGP_ERR_PARAM, "push hop needs w > 0 and W_next");
    if (g->nl > 0 && !T_full_dev) return fail(RAFTGP_ERR_PARAM, "null T_full");
    RG_TRY(check_reps(rep, nrep, 1));
    RG_TRY(set_device(g->ctx));
    if (g->nl == 0) return RAFTGP_OK;
    PushSpec p{};
    p.nrep = nrep;
    p.row0 = g->row_begin;
    for (int q = 0; q < nrep; ++q) p.rep[q] = rep[q];
    bool al = push_fusable(w, w_next) && aligned16(T_full_dev) && aligned16(W_next_dev) &&
              (!Z_out_dev || aligned16(Z_out_dev));
    for (int q = 0; q < nrep; ++q) al = al && aligned16(rep[q]);
    if (al) return gcn_hop(g, T_full_dev, w, Z_out_dev, W_next_dev, w_next, nullptr, 0, &p);
    raftgp_ctx ctx = g->ctx;
    float *T = nullptr;
    raftgp_status st = dalloc_t(ctx, &T, (size_t)g->nl * w_next);
    if (st == RAFTGP_OK) st = gcn_hop(g, T_full_dev, w, Z_out_dev, W_next_dev, w_next, T);
    for (int q = 0; q < nrep && st == RAFTGP_OK; ++q)
        st = dcopy(ctx, rep[q] + (size_t)g->row_begin * w_next, T, sizeof(float) * g->nl * w_next);
    dfree(ctx, T);
    return st;
    RG_GUARD_END
}

raftgp_status raftgp_ipc_alloc(raftgp_ctx ctx, size_t bytes, void **dev_ptr, void *handle64) {
    if (!ctx || !dev_ptr || !handle64) return fail(RAFTGP_ERR_PARAM, "null argument");
    *dev_ptr = nullptr;
    RG_TRY(set_device(ctx));
    cudaError_t e = cudaMalloc(dev_ptr, bytes ? bytes : 16);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dev_ptr = nullptr;
        return cuda_fail(e, "raftgp_ipc_alloc");
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(handle64), *dev_ptr);
    if (e != cudaSuccess) {
        cudaFree(*dev_ptr);
        *dev_ptr = nullptr;
        cudaGetLastError();
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    return RAFTGP_OK;
}

raftgp_status raftgp_ipc_free(raftgp_ctx ctx, void *dev_ptr) {
    if (!ctx || !dev_ptr) return RAFTGP_OK;
    RG_TRY(set_device(ctx));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    RG_CUDA(cudaFree(dev_ptr));
    return RAFTGP_OK;
}

raftgp_status raftgp_ipc_open(raftgp_ctx ctx, const void *handle64, void **dev_ptr) {
    if (!ctx || !handle64 || !dev_ptr) return fail(RAFTGP_ERR_PARAM, "null argument");
    *dev_ptr = nullptr;
    RG_TRY(set_device(ctx));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dev_ptr = nullptr;
        return cuda_fail(e, "cudaIpcOpenMemHandle");
    }
    return RAFTGP_OK;
}

raftgp_status raftgp_ipc_close(raftgp_ctx ctx, void *dev_ptr) {
    if (!ctx || !dev_ptr) return RAFTGP_OK;
    RG_TRY(set_device(ctx));
    RG_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return RAFTGP_OK;
}

raftgp_status raftgp_copy(raftgp_ctx ctx, void *dst_dev, const void *src_dev, size_t bytes) {
    if (!ctx || (bytes && (!dst_dev || !src_dev))) return fail(RAFTGP_ERR_PARAM, "null argument");
    RG_TRY(set_device(ctx));
    return dcopy(ctx, dst_dev, src_dev, bytes);
}

}  // extern "C"
