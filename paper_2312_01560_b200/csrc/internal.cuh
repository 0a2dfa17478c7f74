// internal.cuh — shared internals of libraftgp (context/graph structs, errors, launch accounting).
// Product code only: nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <unordered_map>
#include <atomic>
#include <functional>
#include <vector>

#include "../../include/raftgp.h"

namespace raftgp {

// ---------------------------------------------------------------- kernel ids (profiling)
enum KernelId : int {
    K_CSR_COUNT = 0,
    K_SCAN,
    K_CSR_SCATTER,
    K_CSR_SORT_WARP,
    K_CSR_SORT_BLOCK,
    K_CSR_COMPACT,
    K_DEGREES,
    K_SKETCH,
    K_SKETCH_G,
    K_G_FINAL,
    K_FEATURE_HOP,
    K_TRANSFORM,
    K_GCN_HOP,
    K_GENERIC,
    K_MISC,
    K_CSR_PARTITION,
    K_CSR_BUCKET,
    K_ORDER,
    K_SELECT,
    K_SEL_SEED,
    K_SEL_LLOYD,
    K_SEL_SPLIT,
    K_GEMM,
    K_GEMM_TILE,
    K_WIDE_HOP,
    K_SBM,
    K_SBM_WALK,
    K_STREAM,
    K_EXCHANGE,     // NCCL collectives of the row-partitioned path (barrier, all-gathers; not counted as our launches)
    K_PUSH_COPY,    // deferred push of a finished operand block into the peers' copies (dist.cu)
    K_CSR_FINE,     // second level of the two-level CSR partition (csr.cu)
    K_STREAM_LAST,  // the incrementally updated last GCN hop of a delta-mode stream (stream.cu)
    K_NUM
};
extern const char *const kKernelNames[K_NUM];

struct ProfRec {
    int kid;
    cudaEvent_t start, stop;
};

// Operand copies of the row-partitioned path (dist.cu), cached in the context across steps: for every slot (Theta'
// and the GCN operands T_k) an n_pad x width buffer on this GPU plus the peers' buffers mapped through CUDA IPC.
struct DistBufs {
    int64_t rows = 0;                       // P * R (padded: ncclAllGather in place needs equal blocks)
    std::vector<int32_t> widths;            // per slot
    std::vector<float *> own;               // per slot: this rank's copy (cudaMalloc: IPC-exportable)
    std::vector<std::vector<float *>> rep;  // per slot: [q] = rank q's copy (rep[s][rank] == own[s])
    bool mapped = false;                    // peers' copies mapped: pushes fused into the producing kernels;
                                            // else every rank holds its own copy only, completed by all-gathers
};

}  // namespace raftgp

struct raftgp_ctx_s {
    // references: the caller's (dropped by raftgp_ctx_destroy) + one per live graph / stream, so a graph or
    // stream destroyed after its context (e.g. by a garbage collector) still finds the context alive
    std::atomic<int> refs{1};
    int device = 0;
    void *mbox_h = nullptr;        // mapped pinned host mailbox for scalar readbacks (dread), and its device alias
    void *mbox_d = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;   // library-owned side stream (overlapped work inside one call)
    cudaStream_t hip = nullptr;    // library-owned high-priority stream (the CSR build beside the Theta' kernel)
    cudaMemPool_t pool = nullptr;  // this context's own stream-ordered pool (release threshold: keep everything)
    bool own_stream = false;
    int sm_count = 148;
    int sketch_ctas = 0;           // CTAs of the tcgen05 Theta' kernel (0 = every SM); set while it shares the GPU
    int64_t launches = 0;
    bool prof = false;
    std::vector<raftgp::ProfRec> recs;
    std::vector<cudaEvent_t> event_pool;
    // workspace cache: blocks freed by the library are kept (keyed by size) and reused in stream order,
    // so steady-state calls make no allocator calls at all
    std::multimap<size_t, void *> free_blocks;
    std::unordered_map<void *, size_t> live_blocks;
    size_t cached_bytes = 0;
    // row-partitioned contexts (raftgp_ctx_create_dist): NCCL communicator over `world` ranks, one per GPU
    void *nccl = nullptr;          // ncclComm_t
    int rank = 0, world = 1;
    float *dist_flag = nullptr;    // 1-element operand of the stream-ordered barrier (all-reduce)
    raftgp::DistBufs dist;         // cached operand copies (dist.cu)
};

struct raftgp_graph_s {
    raftgp_ctx ctx = nullptr;
    int64_t n = 0, row_begin = 0, row_end = 0, nl = 0;
    int64_t nnz_local = 0;
    int64_t two_e = -1;            // global 2e; -1 until degrees are global
    int64_t *row_ptr = nullptr;    // device int64[nl+1], local offsets
    int32_t *col = nullptr;        // device int32[nnz_local], global ids (canonical CSR)
    int32_t *deg_local = nullptr;  // device int32[nl]
    int32_t *order = nullptr;      // device int32[nl]: locality-aware visiting order of the local rows (order.cu)
    int32_t *deg_all = nullptr;    // device int32[n] (global degrees)
    float *s_all = nullptr;        // device fp32[n]: deg^-1/2, 0 for isolated nodes
    float *sh_all = nullptr;       // device fp32[n]: (deg+1)^-1/2
    // slot layout of the hop operands (relabel.cu, whole-graph embeddings): node i's operand row lives at slot[i], the
    // highest-degree rows (the hubs, up to a byte budget) in the first slots, so the hop gathers can keep them in L2
    // (gathers of slots >= *hubk are loaded evict-first); built lazily, dropped when the degrees change
    int32_t *slot = nullptr;       // device int32[n]
    int32_t *colx = nullptr;       // device int32[nnz_local]: slot[col[p]]
    float *s_slot = nullptr;       // device fp32[n]: s by slot (the NCut weight of a gathered row)
    int32_t *hubk = nullptr;       // device int32[1]: number of hub slots
    bool slots_active = false;     // set while embed_pre runs the hops on the slot layout
    std::vector<int64_t> deg_hist;   // host: #nodes per degree (last bin = degree >= kDegHistBins-1)
    // host mirror (scoring), filled lazily
    bool host_valid = false;
    std::vector<int64_t> h_row_ptr;
    std::vector<int32_t> h_col;
};

// NEXT-4 (stream.cu): a graph + the state of its NCut embedding
struct raftgp_stream_s {
    raftgp_ctx ctx = nullptr;
    raftgp_graph g = nullptr;
    int32_t layers = 0;
    std::vector<int32_t> dims;
    uint64_t seed = 0;
    float *thw = nullptr;               // Theta' (n x dims[1])
    std::vector<float *> T;             // T[k], k = 1..layers (n x dims[k])
    std::vector<float *> W;             // W[k], k = 2..layers (dims[k-1] x dims[k])
    float *Z = nullptr;                 // n x dims[layers]
    int32_t mode = 0;                   // RAFTGP_STREAM_EXACT / RAFTGP_STREAM_DELTA
    bool stale = false;                 // a failed batch rewrote part of the state: add_edges refused until set_mode
    std::vector<float *> A;             // delta mode: A[h] = GCN hop h's pre-activation sums T_i + sum_j T_j (n x dims[h])
    int32_t *pos = nullptr;             // delta mode: row -> index into the current dT (-1: row unchanged)
    float *Zs = nullptr;                // delta mode: Z_h rows of a hop h < L (n x max dims[1..L-1]), transform input
};

namespace raftgp {

// ---------------------------------------------------------------- context lifetime (capi.cu)
void ctx_retain(raftgp_ctx ctx);
void ctx_release(raftgp_ctx ctx);   // tears the context down when the last reference goes

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
raftgp_status fail(raftgp_status st, const std::string &msg);
raftgp_status cuda_fail(cudaError_t e, const char *what);

#define RG_CUDA(call)                                               \
    do {                                                            \
        cudaError_t _e = (call);                                    \
        if (_e != cudaSuccess) return ::raftgp::cuda_fail(_e, #call); \
    } while (0)

#define RG_CHECK_LAUNCH(ctx)                                                     \
    do {                                                                         \
        cudaError_t _e = cudaGetLastError();                                     \
        if (_e != cudaSuccess) return ::raftgp::cuda_fail(_e, "kernel launch"); \
    } while (0)

#define RG_TRY(expr)                             \
    do {                                         \
        raftgp_status _s = (expr);               \
        if (_s != RAFTGP_OK) return _s;          \
    } while (0)

// ---------------------------------------------------------------- per-device one-time setup
// Kernel attributes (dynamic shared-memory limits) and occupancy results belong to a device context, so they are
// set / computed once per (device, kernel): a process with contexts on several GPUs gets them on each device.
// Thread-safe. `init` runs at most once per (device, key) (again if it failed) and may store an int (e.g. CTAs
// per SM) that later calls receive in *value.
raftgp_status per_device(int device, const void *key, int *value, const std::function<raftgp_status(int *)> &init);

// ---------------------------------------------------------------- launch accounting
// Scope object placed around ONE kernel launch: counts it, and when profiling is on records CUDA
// events before/after it on the context stream.
struct LaunchScope {
    raftgp_ctx ctx;
    int kid;
    cudaEvent_t a = nullptr, b = nullptr;
    // count = false: a library call that is not one of our kernels (NCCL), timed but not counted as a launch
    LaunchScope(raftgp_ctx c, int k, bool count = true);
    ~LaunchScope();
};

// ---------------------------------------------------------------- memory (stream-ordered pool)
raftgp_status dalloc(raftgp_ctx ctx, void **p, size_t bytes);
// Zero `bytes` of device memory with a kernel on `st` (default: the context stream). cudaMemsetAsync is not
// used on the hot paths: it can queue behind host<->device copies in flight on other streams, which
// serialised the pipelined end-to-end steps.
raftgp_status dzero(raftgp_ctx ctx, void *p, size_t bytes, cudaStream_t st = nullptr);
// Device-to-device copy with a kernel (same reason as dzero).
raftgp_status dcopy(raftgp_ctx ctx, void *dst, const void *src, size_t bytes, cudaStream_t st = nullptr);
// Synchronous device-to-host read of a few bytes: a kernel stores them into a mapped pinned mailbox, then the
// stream is synchronised. Keeps the library's readbacks off the copy engines, where they would wait behind
// large transfers of other streams. Falls back to cudaMemcpyAsync above the mailbox size.
raftgp_status dread(raftgp_ctx ctx, void *host, const void *dev, size_t bytes, cudaStream_t st = nullptr);
void dfree(raftgp_ctx ctx, void *p);
void release_cache(raftgp_ctx ctx);

template <typename T>
raftgp_status dalloc_t(raftgp_ctx ctx, T **p, size_t count) {
    return dalloc(ctx, reinterpret_cast<void **>(p), sizeof(T) * (count ? count : 1));
}

constexpr int kDegHistBins = 4096;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- components (csr.cu, sketch.cu, spmm.cu)
raftgp_status scan_i32_to_i64(raftgp_ctx ctx, const int32_t *in, int64_t *out, int64_t n);
raftgp_status csr_build(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int64_t rb,
                        int64_t re, raftgp_graph g);
raftgp_status degrees_finalize(raftgp_graph g, int64_t known_2e = -1);
raftgp_status ensure_slots(raftgp_graph g);   // relabel.cu: g->slot / colx / s_slot / hubk for a whole graph
// relabel.cu: the smallest degree t with #(deg >= t) <= kmax (device int32[1]) for L2 hints on hub rows
raftgp_status hub_degree_threshold(raftgp_ctx ctx, const int32_t *deg, int64_t n, int64_t kmax, int32_t *thr_dev);
void drop_slots(raftgp_graph g);
bool slots_enabled();                          // RAFTGP_RELABEL (default 1)
int64_t slot_hub_bytes();                      // operand bytes of hub slots (RAFTGP_HUB_MB, default 64 MB)
bool sketch_tc_enabled();                      // RAFTGP_TC (default 1; sketch.cu)
raftgp_status compute_order(raftgp_graph g);
// a row list reordered for the hop kernels: heavy rows spread from the front (order.cu)
raftgp_status spread_heavy_list(raftgp_ctx ctx, const int32_t *rows, int64_t count, const int32_t *deg, int32_t *out);
// whether order[0..nl) is a permutation of 0..nl-1 (device check, synchronous)
raftgp_status order_is_permutation(raftgp_ctx ctx, const int32_t *order, int64_t nl, bool *ok);      // g->order (label propagation + counting sort)   // deg_all -> two_e, s_all, sh_all, deg_hist

raftgp_status sketch_fill(raftgp_ctx ctx, uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows, int32_t cols,
                          int32_t den, float *out);
// Theta for all n rows + g = sum_j d_j Theta_j (fp64) when g_out != nullptr.
raftgp_status sketch_theta(raftgp_graph g, uint64_t seed, int32_t r, float *theta, double *g_out);
// g = d^T X over all n rows (fp64, fixed chunk order); X is n x r
raftgp_status g_reduce(raftgp_graph g, const float *X, int32_t r, double *g_out);
// the same in two steps (row-partitioned path): per-chunk partial sums of the global chunks chunk0 .. chunk0+count-1
// (partial[chunk * r + c]; X holds all n rows), then the sum over all chunks in chunk order
int64_t g_chunks(int64_t n);
int64_t g_chunk_rows();
raftgp_status g_partials_range(raftgp_graph g, const float *X, int32_t r, int64_t chunk0, int64_t count, double *partial);
raftgp_status g_final_chunks(raftgp_ctx ctx, const double *partial, int64_t nchunks, int32_t r, double *g_out);
// Theta' = Theta W1 (Theta generated on chip, n x l1 written) and optionally g' = d^T Theta'
bool sketch_w_supported(int32_t r, int32_t l1);
// Theta' = Theta W1 on tcgen05 tensor cores (3xTF32, fp32-accurate), Theta generated on chip
raftgp_status sketch_w_tc(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, const float *W1, int32_t l1, float *out);
// rows row0 .. row0 + rows - 1 of Theta', each stored at its global row into all nout copies (row-partitioned path)
raftgp_status sketch_w_tc_rows(raftgp_ctx ctx, uint64_t seed, int64_t row0, int64_t rows, int32_t r, const float *W1,
                               int32_t l1, float *const *outs, int nout, const int32_t *slot = nullptr);
raftgp_status sketch_w_any(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, const float *W1, int32_t l1, float *out);
raftgp_status sketch_theta_w(raftgp_graph g, uint64_t seed, int32_t r, const float *W1, int32_t l1, float *out,
                             double *g_out);

raftgp_status feature_hop(raftgp_graph g, int variant, int32_t r, const float *theta, const double *gvec, float *Y,
                          const float *W1, int32_t l1, float *T1);
// NCut and full-modularity feature hops from ONE gather of Theta (+ both first transforms).
raftgp_status feature_hop_dual(raftgp_graph g, int32_t r, const float *theta, const double *gvec, float *Y_ncut,
                               float *Y_mod, const float *W1, int32_t l1, float *T_ncut, float *T_mod);
// Fused exchange (a6 without a separate all-gather): a producing hop's epilogue stores each of its rows of
// the next operand T straight into every rank's full n-row copy of T (`rep`: the ranks' buffers, peer
// pointers opened through CUDA IPC over NVLink; `rep2`: the second variant's, for the dual kernels), at
// global row row0 + local row. The kernel ends with a system-scope fence so the peers see the rows once the
// producing kernels of all ranks have completed (the caller then runs a stream-ordered barrier).
constexpr int kMaxPush = 8;
struct PushSpec {
    float *rep[kMaxPush];
    float *rep2[kMaxPush];
    int nrep;
    int nrep2;      // replicas of the second variant's rows (dual kernels); 0 = nrep. 1 = this rank's copy only (its
                    // push to the peers is deferred to a copy kernel on another stream, dist.cu)
    int64_t row0;
    int32_t ld;     // row stride of the replicas in floats (0 = the row width); > width for interleaved operands
};
// Feature hop on a pre-transformed operand Theta' = Theta W1 (no epilogue GEMM): writes
// T1 = s^ (.) (X Theta') for NCUT (T_ncut) and/or MOD (T_mod), or MOD_REDUCED (T_ncut slot, variant 2).
raftgp_status feature_hop_pre(raftgp_graph g, int variant_or_dual, int32_t l1, const float *theta_w,
                              const double *gvec_w, float *T_a, float *T_b, const PushSpec *push = nullptr);
raftgp_status gcn_transform(raftgp_graph g, const float *Z, int32_t lin, const float *W, int32_t lout, float *T);
raftgp_status gcn_hop(raftgp_graph g, const float *Tfull, int32_t w, float *Zout, const float *Wn, int32_t wn,
                      float *Tnext, int32_t tn_ld = 0, const PushSpec *push = nullptr);
// whether gcn_hop / feature_hop_pre can fuse the push into their epilogue for these widths
bool push_fusable(int32_t w, int32_t wn);
// the same hops over a list of local rows (NEXT-4 streaming)
raftgp_status feature_hop_pre_rows(raftgp_graph g, int variant, int32_t l1, const float *theta_w, const double *gvec_w,
                                   float *T, const int32_t *rows, int64_t count);
// T_next rows = s^ (.) (Z rows W) for the listed local rows (Z and T_next full-size, indexed by row)
raftgp_status gcn_transform_rows(raftgp_graph g, const float *Z, int32_t lin, const float *W, int32_t lout, float *T,
                                 const int32_t *rows, int64_t count);
raftgp_status gcn_hop_rows(raftgp_graph g, const float *Tfull, int32_t w, float *Zout, const float *Wn, int32_t wn,
                           float *Tnext, const int32_t *rows, int64_t count);
// last GCN hop of two variants over the interleaved operand [T_a | T_b] (n x 2d); d in {32, 64}
bool gcn_pair_supported(int32_t d);
raftgp_status gcn_final_pair(raftgp_graph g, const float *Tboth, int32_t d, float *Za, float *Zb, int half = 0);
// NEXT-2: tensor-core 3xTF32 GEMM on pre-split, pre-tiled operands (wide.cu)
int gemm_nt(int N);
int64_t gemm_pad_rows(int64_t M);
int gemm_pad_k(int K);
raftgp_status gemm_tile_a(raftgp_ctx ctx, const float *X, int64_t M, int K, int64_t ldx, float *hi, float *lo);
raftgp_status gemm_tile_b(raftgp_ctx ctx, const float *W, int K, int N, float *hi, float *lo);
raftgp_status gemm_theta_tiles(raftgp_ctx ctx, uint64_t seed, int64_t n, int32_t r, float *hi, float *lo);
raftgp_status gemm_tiled(raftgp_ctx ctx, const float *Ahi, const float *Alo, const float *Bhi, const float *Blo,
                         int64_t M, int K, int N, const float *row_scale, float *C, int64_t ldc);
raftgp_status gemm_rowmajor(raftgp_ctx ctx, const float *A, int64_t M, int K, const float *B, int N,
                            const float *row_scale, float *C);
// Table I widths: the whole embedding with tensor-core transforms and wide hops (Y not materialised)
bool wide_supported(int32_t layers, const int32_t *dims);
raftgp_status embed_wide(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                         const int32_t *dims, uint64_t seed, float *const *Z_dev, const int where[3]);
// NEXT-4: streaming updates (stream.cu)
raftgp_status stream_create(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed, raftgp_stream *out);
raftgp_status stream_add(raftgp_stream s, int64_t m, const int32_t *src, const int32_t *dst, int64_t *stats);
void stream_destroy(raftgp_stream s);
raftgp_status stream_set_mode(raftgp_stream s, int32_t mode);
// NEXT-3: Alg. 2 exact SBM sampler (sbm.cu)
raftgp_status sbm_sample(raftgp_ctx ctx, int64_t n, int32_t K, const int32_t *c, const double *theta,
                         const double *omega, uint64_t seed, int32_t q, int32_t *src, int32_t *dst, int64_t cap,
                         int64_t *m_out);
// Row-partitioned path (dist.cu). P ranks; `loopback`: all P ranks are simulated in this process on this ctx's GPU
// (one stream, lockstep stages; tests), else this ctx is rank ctx->rank of an NCCL communicator.
raftgp_status dist_build_embed(raftgp_ctx ctx, int P, bool loopback, int64_t n, int64_t m, const int32_t *src,
                               const int32_t *dst, int32_t nvariants, const int32_t *variants, int32_t layers,
                               const int32_t *dims, uint64_t seed, float *const *Z_dev);
void dist_release(raftgp_ctx ctx);   // drop the cached operand copies (collective on NCCL contexts)
// NEXT-1: Alg. 1 hierarchical model selection (select.cu)
raftgp_status model_select(raftgp_graph g, const float *Z, int32_t L, int32_t eps, int32_t max_iter, int32_t rule,
                           int32_t *labels, int32_t *num_blocks, int64_t *stats);

}  // namespace raftgp
