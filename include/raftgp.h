/*
 * raftgp.h — C-ABI of the B200-native RaftGP embedding hot path (arxiv 2312.01560).
 *
 * The path: canonical CSR build (a1) -> degree/normalisation pass (a2) ->
 * Gaussian sketch (a3) -> feature hop Y = X Theta (a4, Eq. 5) -> untrained GCN hops with fused
 * tanh / row-l2 / next-layer transform (a5, Eq. 6) -> [per-hop all-gather when row-partitioned (a6)]
 * -> host scoring (a7, Eq. 1/3/7). Every compute step runs in this library's sm_100a kernels.
 *
 * Conventions for every entry point
 *  - Plain C types only. "dev" pointers are CUDA device pointers on the context's device; "host"
 *    pointers are ordinary host memory. Dense matrices are fp32, row-major, contiguous (row stride =
 *    width). Fast kernels are used when a matrix pointer is 16-byte aligned and its width is 32, 64 or
 *    128; other widths/alignments take a slower generic kernel with the same results up to rounding.
 *  - Asynchrony: calls enqueue work on the context's stream and return; outputs are valid after the
 *    caller synchronises that stream (raftgp_ctx_sync). Exceptions are noted ("synchronous").
 *  - Ownership: the library owns raftgp_ctx and raftgp_graph handles and the graph's device CSR. The
 *    caller owns every array passed in. Device inputs must stay valid until the stream work completes.
 *  - Errors: every function returns raftgp_status; on non-OK, raftgp_last_error() holds a message for
 *    the calling thread. No C++ exception crosses this ABI. Handles are not thread-safe.
 *  - Multi-GPU: one process and one context per GPU. raftgp_ctx_create_dist gives the
 *    contexts of a job an NCCL communicator (the unique id comes from raftgp_nccl_unique_id on rank 0 and
 *    reaches the other ranks by any out-of-band means). On such a context raftgp_build_embed runs the whole
 *    row-partitioned step inside the library (rank p owns rows [p R, min((p+1) R, n)), R = ceil(n / P);
 *    exchanges fused into the producing kernels, see "a6" below) and returns the local rows of Z. The
 *    building blocks stay public too: a graph may hold only the rows [row_begin, row_end) of the global CSR
 *    (column ids always global; row-indexed outputs hold the local rows), and raftgp_barrier /
 *    raftgp_allgather run the job's collectives on the context stream.
 */
#ifndef RAFTGP_H
#define RAFTGP_H

#include <stdint.h>

#if defined(__GNUC__)
#define RAFTGP_API __attribute__((visibility("default")))
#else
#define RAFTGP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct raftgp_ctx_s *raftgp_ctx;     /* device + stream + profiling state; library-owned */
typedef struct raftgp_graph_s *raftgp_graph; /* device CSR (local rows) + degree scalars; library-owned */
typedef struct raftgp_stream_s *raftgp_stream; /* a graph + its NCut embedding state, updated by edge additions */

typedef enum {
    RAFTGP_OK = 0,
    RAFTGP_ERR_PARAM = 2,    /* bad argument: r <= 0, dims <= 0, bad variant, label out of [0,k), ... */
    RAFTGP_ERR_DATA = 3,     /* bad data: node id outside [0,n), 2e = 0 for MOD variants, zero degree sum */
    RAFTGP_ERR_INTERNAL = 4,
    RAFTGP_ERR_CUDA = 5,     /* a CUDA runtime call or kernel launch failed */
    RAFTGP_ERR_NOMEM = 6,    /* device allocation failed */
    RAFTGP_ERR_COMM = 7,     /* an NCCL call of a distributed context failed (raftgp_ctx_create_dist) */
    RAFTGP_ERR_STATE = 8     /* handle not ready (e.g. partial graph without raftgp_graph_set_degrees) */
} raftgp_status;

/* The feature operator X of Eq. 5 ("X in {M, Q~}"; PAPER.md:289 RaftGP-C / RaftGP-M). */
typedef enum {
    RAFTGP_NCUT = 0,         /* X = M = D^-1/2 A D^-1/2; isolated rows give zero rows */
    RAFTGP_MOD = 1,          /* X = Q = A - d d^T / 2e (Eq. 4), applied as A Theta minus the
                                fused rank-1 term d (d^T Theta) / 2e; never materialised */
    RAFTGP_MOD_REDUCED = 2   /* X = Q~ = Q on the edges of A, 0 elsewhere */
} raftgp_variant;

#define RAFTGP_HOST_PTRS 0u    /* edge arrays are host memory: copied to the device inside the call */
#define RAFTGP_DEVICE_PTRS 1u  /* edge arrays are device memory on the context's device */

/* ---------------------------------------------------------------- context */
RAFTGP_API const char *raftgp_last_error(void);          /* thread-local message of the last non-OK status */
RAFTGP_API const char *raftgp_version(void);

/* device: CUDA ordinal. cuda_stream: the cudaStream_t every call of this context enqueues on (NULL =
 * the legacy default stream). The stream stays owned by the caller and must outlive the context. */
RAFTGP_API raftgp_status raftgp_ctx_create(int device, void *cuda_stream, raftgp_ctx *out);
/* Drops the caller's reference. Graphs and streams hold their own reference, so they may be destroyed
 * before or after their context; the context (its side stream, events and cached workspace) is torn down
 * when the last of them goes. NULL is a no-op. Always RAFTGP_OK. */
RAFTGP_API raftgp_status raftgp_ctx_destroy(raftgp_ctx ctx);
RAFTGP_API raftgp_status raftgp_ctx_sync(raftgp_ctx ctx);                     /* synchronous */
RAFTGP_API raftgp_status raftgp_ctx_stream(raftgp_ctx ctx, void **cuda_stream_out);
/* Workspace: every context allocates from its OWN stream-ordered memory pool (the device's default pool and its
 * release threshold are left untouched) and keeps freed blocks cached for reuse. raftgp_ctx_trim returns the
 * cached blocks to the pool and the pool's unused memory to the device (cudaMemPoolTrimTo), so it is visible to
 * other allocators (e.g. PyTorch's) afterwards. Synchronous. bytes_released: host out or NULL. */
RAFTGP_API raftgp_status raftgp_ctx_trim(raftgp_ctx ctx, int64_t *bytes_released);

/* Per-kernel device timing with CUDA events recorded around every launch on the ctx stream.
 * raftgp_prof_read is synchronous; kernel ids are 0..raftgp_prof_kernels()-1. */
RAFTGP_API raftgp_status raftgp_ctx_set_profiling(raftgp_ctx ctx, int enable);
RAFTGP_API int raftgp_prof_kernels(void);
RAFTGP_API const char *raftgp_prof_name(int kernel_id);
RAFTGP_API raftgp_status raftgp_prof_read(raftgp_ctx ctx, int kernel_id, double *total_ms, int64_t *launches);
RAFTGP_API raftgp_status raftgp_prof_reset(raftgp_ctx ctx);
/* number of kernels this context has launched since creation (or since the last reset) */
RAFTGP_API raftgp_status raftgp_launch_count(raftgp_ctx ctx, int64_t *out, int reset);

/* ---------------------------------------------------------------- multi-GPU contexts
 * raftgp_nccl_unique_id: a new NCCL unique id (128 bytes, host out), created by ONE rank (rank 0) and passed to all.
 * raftgp_ctx_create_dist: like raftgp_ctx_create, plus membership `rank` of a `world`-rank NCCL communicator
 *   (1 <= world <= 8, one rank per GPU of one node; collective: every rank calls it with the same id).
 *   raftgp_ctx_destroy of such a context is collective too (the cached operand copies are unmapped and freed
 *   behind a barrier, then the communicator is destroyed).
 * raftgp_ctx_rank: rank and world of a context (0 and 1 for raftgp_ctx_create).
 * raftgp_barrier: stream-ordered barrier (a 1-element ncclAllReduce on the context stream): work enqueued after it
 *   on any rank runs after the work every rank enqueued before it. No-op on a one-rank context.
 * raftgp_allgather: ncclAllGather of bytes_per_rank bytes per rank on the context stream (device buffers; recv
 *   holds world * bytes_per_rank; send may alias recv + rank * bytes_per_rank). A copy on non-dist contexts.
 * Errors: PARAM, COMM (NCCL failure; raftgp_last_error has NCCL's message), CUDA, NOMEM. */
RAFTGP_API raftgp_status raftgp_nccl_unique_id(void *out128);
RAFTGP_API raftgp_status raftgp_ctx_create_dist(int device, void *cuda_stream, int rank, int world, const void *id128,
                                                raftgp_ctx *out);
RAFTGP_API raftgp_status raftgp_ctx_rank(raftgp_ctx ctx, int *rank, int *world);
RAFTGP_API raftgp_status raftgp_barrier(raftgp_ctx ctx);
RAFTGP_API raftgp_status raftgp_allgather(raftgp_ctx ctx, const void *send_dev, void *recv_dev, size_t bytes_per_rank);

/* ---------------------------------------------------------------- a1 + a2: CSR build, degrees
 * Canonical CSR of the simple undirected graph given by m raw pairs (src[e], dst[e]) over n nodes
 * (§II: A_ij = A_ji in {0,1}): pairs with u == v are dropped, both orientations are
 * added, rows are sorted ascending and duplicates removed. Only the rows
 * [row_begin, row_end) are kept (pass 0, n for the whole graph).
 *   n: node count (ids in [0, n)), 0 <= n < 2^31.  m: pair count >= 0.
 *   src, dst: int32[m], host or device per flags (RAFTGP_HOST_PTRS / RAFTGP_DEVICE_PTRS).
 * Errors: PARAM (n, m or the range invalid), DATA (an id outside [0, n)), NOMEM, CUDA.
 * Synchronous at its end (reads the local nnz and the data-error flag back).
 * When the range is the whole graph the degree pass (a2) runs too: deg, 2e, s = deg^-1/2 (0 if
 * deg = 0), s^ = (deg+1)^-1/2 over all n nodes. A partial graph is not usable by the compute calls
 * until raftgp_graph_set_degrees has supplied the global degree vector. */
RAFTGP_API raftgp_status raftgp_build_csr(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                               int64_t row_begin, int64_t row_end, uint32_t flags, raftgp_graph *out);

/* n, local rows, local nnz (entries of A in the local rows = sum of their degrees), 2e (global; -1
 * while a partial graph has no global degrees yet). */
RAFTGP_API raftgp_status raftgp_graph_info(raftgp_graph g, int64_t *n, int64_t *row_begin, int64_t *row_end,
                                int64_t *nnz_local, int64_t *two_e);

/* Copy the local CSR out (parity checks / host use). row_ptr: int64[rows+1] (local offsets from 0);
 * col_idx: int32[nnz_local] (global ids); deg: int32[rows] local degrees. Any pointer may be NULL.
 * flags: RAFTGP_HOST_PTRS (synchronous) or RAFTGP_DEVICE_PTRS (async, device buffers). */
RAFTGP_API raftgp_status raftgp_graph_export(raftgp_graph g, int64_t *row_ptr, int32_t *col_idx, int32_t *deg, uint32_t flags);

/* Local degrees of the rows [row_begin, row_end) into a device int32 buffer (async). */
RAFTGP_API raftgp_status raftgp_graph_local_degrees(raftgp_graph g, int32_t *deg_dev);

/* Multi-GPU degree pass (a2): deg_all_dev = device int32[n], the degrees of ALL n nodes (the
 * concatenation of every rank's raftgp_graph_local_degrees). Computes 2e, s and s^ over all nodes. */
RAFTGP_API raftgp_status raftgp_graph_set_degrees(raftgp_graph g, const int32_t *deg_all_dev);

/* Visiting order of the local rows used by the hop kernels (a permutation of 0..rows-1, device int32;
 * NULL = natural order). Performance only: every row's arithmetic, and so every output bit, is the same
 * for any order. With RAFTGP_ORDER_ROUNDS=k > 0 in the environment build_csr installs an order from k rounds
 * of label propagation (paper_2312_01560_b200/csrc/order.cu); by default build_csr installs the degree-aware
 * order (hub rows spread one per claim). Synchronous: the array is checked on the device and rejected with
 * RAFTGP_ERR_PARAM unless it is a permutation of 0..rows-1 (out-of-range or repeated entries). */
RAFTGP_API raftgp_status raftgp_graph_set_order(raftgp_graph g, const int32_t *order_dev);

RAFTGP_API raftgp_status raftgp_graph_destroy(raftgp_graph g);

/* ---------------------------------------------------------------- a3: Gaussian sketch
 * rows x cols block (global rows row_begin..) of the generator of docs/SKETCH_SPEC.md: element (i,c)
 * = z(seed, tag, i, c) * fp32(1/sqrt(den)), z a standard normal from Philox4x32-10 + Box-Muller.
 * Theta of Eq. 5 is tag 0, den = r (variance 1/r, reading #2); W^(k) of
 * Eq. 6 is tag k, den = fan-in (reading #4). out: device fp32 rows x cols. Bit-exact with the oracle. */
RAFTGP_API raftgp_status raftgp_sketch(raftgp_ctx ctx, uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows,
                            int32_t cols, int32_t den, float *out_dev);

/* Theta' = Theta W for the global rows 0..rows-1: Theta (tag 0, den r) is generated on chip and multiplied
 * by W (device, r x l1 row-major) on the tcgen05 tensor cores with a 3xTF32 split (fp32-accurate); only
 * Theta' (rows x l1, device) is written. r, l1 in {32, 64, 128}; 16-byte aligned buffers. */
RAFTGP_API raftgp_status raftgp_sketch_transform(raftgp_ctx ctx, uint64_t seed, int64_t rows, int32_t r,
                                                 const float *W_dev, int32_t l1, float *out_dev);

/* W^(k) of Eq. 6, untrained: fan_in x fan_out, tag k, den fan_in. */
RAFTGP_API raftgp_status raftgp_weights(raftgp_ctx ctx, uint64_t seed, int32_t k, int32_t fan_in, int32_t fan_out,
                             float *W_dev);

/* ---------------------------------------------------------------- a4: feature hop (Eq. 5)
 * Y = X Theta for the graph's local rows, Theta = raftgp_sketch(seed, tag 0, den r)
 * over all n rows (generated inside the call; no exchange is needed across ranks).
 *   NCUT:        Y_i = s_i sum_j s_j Theta_j
 *   MOD:         Y_i = sum_j Theta_j - d_i g / 2e,  g = sum_{all j} d_j Theta_j (fp64, fixed order)
 *   MOD_REDUCED: Y_i = sum_j (1 - d_i d_j / 2e) Theta_j
 * Y_dev: device fp32 local_rows x r. Errors: PARAM (r <= 0, bad variant), DATA (2e = 0 and variant
 * != NCUT), STATE (partial graph without degrees). Workspace: Theta (n x r fp32) is allocated from
 * the stream-ordered pool and released at the end of the call. */
RAFTGP_API raftgp_status raftgp_project(raftgp_graph g, raftgp_variant variant, int32_t r, uint64_t seed, float *Y_dev);

/* ---------------------------------------------------------------- a5: GCN (Eq. 6 + l2 norm)
 * Transform: T = s^ (.) (Z W) for the local rows: Z local_rows x lin, W lin x lout (device), T
 * local_rows x lout. This is the "GEMM-first" half of Eq. 6: P Z W = s^ (.) ((A + I)(s^ (.) Z W)). */
RAFTGP_API raftgp_status raftgp_gcn_transform(raftgp_graph g, const float *Z_dev, int32_t lin, const float *W_dev,
                                   int32_t lout, float *T_dev);

/* One GCN hop on the local rows: H_i = s^_i (T_i + sum_{j in N(i)} T_j) = (P Z W)_i,
 * Z'_i = tanh(H_i) / ||tanh(H_i)||_2 (a zero row stays zero), then optionally the next transform
 * T'_i = s^_i (Z'_i W_next).
 *   T_full_dev: fp32 n x w, the operand for ALL n rows (on P > 1 ranks: the all-gathered block).
 *   Z_out_dev: local_rows x w, or NULL.  W_next_dev: w x w_next, or NULL (w_next = 0).
 *   T_next_dev: local_rows x w_next, or NULL. */
RAFTGP_API raftgp_status raftgp_gcn_hop(raftgp_graph g, const float *T_full_dev, int32_t w, float *Z_out_dev,
                             const float *W_next_dev, int32_t w_next, float *T_next_dev);

/* The whole untrained GCN on one GPU (whole-graph handle): Z^(k) = rownorm(tanh(P Z^(k-1) W^(k))),
 * Z^(0) = Y, k = 1..layers, W^(k) = raftgp_weights(seed, k, dims[k-1], dims[k]).
 *   dims: host int32[layers+1], dims[0] = width of Y.  Y_dev: n x dims[0].  Z_dev: n x dims[layers].
 *   Zk_dev: NULL, or host array of layers-1 device pointers receiving Z^(1..layers-1) (NULL entries
 *   skipped). Workspace (T buffers) comes from the stream-ordered pool. */
RAFTGP_API raftgp_status raftgp_gnn_embed(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed,
                               const float *Y_dev, float *Z_dev, float *const *Zk_dev);

/* project + gnn_embed in one call with the first transform fused into the feature-hop epilogue.
 * Y_dev may be NULL (Y is then not written). Same arguments and errors as the two calls. */
RAFTGP_API raftgp_status raftgp_embed(raftgp_graph g, raftgp_variant variant, int32_t layers, const int32_t *dims,
                           uint64_t seed, float *Y_dev, float *Z_dev, float *const *Zk_dev);

/* Several feature operators of the same graph in one call (the RaftGP-C and RaftGP-M embeddings of
 * PAPER.md:289 side by side): Theta is generated once, and when both NCUT and MOD are requested their
 * feature hops share ONE gather of Theta (Y_ncut and Y_mod come out of the same pass; their arithmetic
 * per row is identical to raftgp_embed's). variants: host int32[nvariants] (distinct raftgp_variant
 * values). Y_dev: NULL or host array of nvariants device pointers (NULL entries skipped). Z_dev: host
 * array of nvariants device pointers (n x dims[layers]). Same errors as raftgp_embed. */
RAFTGP_API raftgp_status raftgp_embed_multi(raftgp_graph g, int32_t nvariants, const int32_t *variants, int32_t layers,
                                            const int32_t *dims, uint64_t seed, float *const *Y_dev,
                                            float *const *Z_dev);

/* raftgp_build_csr (whole graph) + raftgp_embed_multi (Y not written) in one call: Theta' = Theta W^(1)
 * depends only on the seed, so it is generated on a library-owned side stream while the CSR build runs on the
 * context stream (tensor cores / ALUs against atomics / HBM); outputs are those of the two calls. Edge arrays
 * host or device per flags. g_out: NULL, or receives the graph handle (caller destroys it). Synchronous like
 * raftgp_build_csr; the embedding is enqueued on the context stream. Errors: those of the two calls.
 * On a distributed context (raftgp_ctx_create_dist; collective: every rank calls it with the same graph, all m
 * pairs, and the same arguments) this is the row-partitioned step: rank p builds the CSR of its
 * rows, degrees are all-gathered, Theta' rows are generated by their owner and pushed into every rank's copy
 * during the CSR build, and every feature / GCN hop stores its output rows into all ranks' copies of the next
 * operand (NVLink peer stores, CUDA IPC mappings cached in the context across calls; a stream-ordered barrier
 * between producing and consuming hops). Z_dev[v] then receives the LOCAL rows (row_end - row_begin) x dims[L];
 * the results are bit-identical to one GPU. Needs r and every width in {32, 64, 128}; g_out must be NULL. */
RAFTGP_API raftgp_status raftgp_build_embed(raftgp_ctx ctx, int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                            uint32_t flags, int32_t nvariants, const int32_t *variants, int32_t layers,
                                            const int32_t *dims, uint64_t seed, float *const *Z_dev,
                                            raftgp_graph *g_out);

/* The row-partitioned step of raftgp_build_embed with P logical ranks simulated on this context's GPU (P CSR shards,
 * P full copies of every operand, each shard's hops storing into all P copies, lockstep stages on one stream): the
 * single-GPU double of a P-GPU job, used to check that the partitioned schedule is bit-identical to one GPU.
 * Z_dev[v]: n x dims[L] (all rows, shard p's rows at [p R, ...)). 1 <= P <= 8. Errors: those of raftgp_build_embed. */
RAFTGP_API raftgp_status raftgp_build_embed_loopback(raftgp_ctx ctx, int32_t P, int64_t n, int64_t m, const int32_t *src,
                                                     const int32_t *dst, uint32_t flags, int32_t nvariants,
                                                     const int32_t *variants, int32_t layers, const int32_t *dims,
                                                     uint64_t seed, float *const *Z_dev);

/* First GCN operand of every listed variant for the LOCAL rows (works on row-partitioned graphs):
 * T1 = s^ (.) (X Theta W^(1)) = s^ (.) (Y W^(1)), X the variant's feature operator, Theta and W^(1) as in
 * raftgp_embed. Theta' = Theta W^(1) is generated on chip (Theta never written) and NCUT + MOD share one
 * gather of Theta' (GEMM before aggregation, reading #13). r = Theta width, l1 = W^(1) width.
 * T1_dev: host array of nvariants device pointers (local_rows x l1). Same errors as raftgp_project. */
RAFTGP_API raftgp_status raftgp_feature_transform(raftgp_graph g, int32_t nvariants, const int32_t *variants,
                                                  int32_t r, int32_t l1, uint64_t seed, float *const *T1_dev);

/* ---------------------------------------------------------------- a7: scoring (host, synchronous)
 * On a whole-graph handle. assign: host int32[n] labels in [0, k).
 * Modularity, Eq. 3. Errors: PARAM (label outside [0,k), k <= 0), DATA (2e = 0). */
RAFTGP_API raftgp_status raftgp_modularity(raftgp_graph g, const int32_t *assign, int32_t k, double *out);
/* NCut, Eq. 1; a block with vol = 0 contributes 0 (reading #17). */
RAFTGP_API raftgp_status raftgp_ncut(raftgp_graph g, const int32_t *assign, int32_t k, double *out);
/* Local modularity, Eq. 7 of the blocks U_1..U_k of U = nodes[0..count): node
 * nodes[t] is in block block_of_node[t]; degrees are full-graph degrees, 2e = their sum over U.
 * Errors: PARAM (duplicate or out-of-range node, label outside [0,k)), DATA (zero degree sum). */
RAFTGP_API raftgp_status raftgp_local_modularity(raftgp_graph g, const int64_t *nodes, int64_t count,
                                      const int32_t *block_of_node, int32_t k, double *out);

/* ---------------------------------------------------------------- NEXT-1: hierarchical model selection
 * Alg. 1 (§III-C) from U = V on the embedding Z, with KMeans(K = 2) and the split test of
 * docs/SELECT_SPEC.md (deterministic farthest-first seeding, Lloyd iterations with exact fixed-point centroid
 * sums, exact integer form of "m_1 > m_2" for the local modularity of Eq. 7). The tree is processed level by
 * level on the GPU; the partition equals the depth-first recursion's.
 *   Z_dev: device fp32 n x L, row-major, 16-byte aligned, every |z| <= 1 (rows of the l2-normalised
 *          embedding). L in {8, 16, 32, 64, 128}.
 *   eps: the size threshold epsilon (PAPER.md:200 uses 5), >= 0. max_iter: Lloyd cap (>= 1; 100 suggested).
 *   rule: RAFTGP_LMOD_GLOBAL (2e = 2|E|: m_1 > m_2 iff splitting U lowers the modularity of G, PAPER.md:203;
 *         DESIGN.md reading #28) or RAFTGP_LMOD_LOCAL (2e = total degree of U, PAPER.md:167 as printed).
 *   labels_dev: device int32[n] out: block of every node, blocks numbered 0..K-1 by their smallest member.
 *   num_blocks: host out, K.  stats: host int64[9] out or NULL: {blocks, splits, Lloyd iterations summed
 *          over levels (lock-step), levels, rows visited by Lloyd passes (rows of unconverged segments),
 *          rows per seeding pass summed over levels, Z rows read by Lloyd passes (the others are skipped
 *          by exact distance bounds), segments whose Lloyd iterations stopped at max_iter without converging
 *          (summed over levels; the convergence diagnostic), their rows}.
 * Whole-graph handle only. Synchronous (the host drives the levels). Workspace from the context pool.
 * Errors: PARAM (L, eps, max_iter, rule, null/misaligned pointers, partial graph), DATA (|z| > 1 or NaN),
 * STATE, NOMEM, CUDA. */
typedef enum { RAFTGP_LMOD_GLOBAL = 0, RAFTGP_LMOD_LOCAL = 1 } raftgp_lmod_rule;
RAFTGP_API raftgp_status raftgp_model_select(raftgp_graph g, const float *Z_dev, int32_t L, int32_t eps,
                                             int32_t max_iter, int32_t rule, int32_t *labels_dev, int32_t *num_blocks,
                                             int64_t *stats);

/* ---------------------------------------------------------------- NEXT-2: tensor-core GEMM
 * C = diag(row_scale) A B on the tcgen05 tensor cores, fp32-accurate by the 3xTF32 split (error ~2^-20
 * relative): the dense transforms of Eq. 6 at the paper's Table I widths and Theta W^(1).
 *   A_dev: device fp32 M x K row-major; B_dev: device fp32 K x N row-major; row_scale_dev: device fp32[M] or
 *   NULL (= 1); C_dev: device fp32 M x N row-major (rows 16-byte aligned for the vectorised epilogue).
 * Workspace (hi / lo tiles of A and B) from the context pool. Errors: PARAM (sizes, null pointers). */
RAFTGP_API raftgp_status raftgp_gemm_tf32x3(raftgp_ctx ctx, int64_t M, int32_t K, int32_t N, const float *A_dev,
                                            const float *B_dev, const float *row_scale_dev, float *C_dev);

/* ---------------------------------------------------------------- NEXT-3: exact SBM sampler
 * Alg. 2 for the degree-corrected SBM of Def. 5: every node pair
 * (i, j), i != j, is an edge with probability 1 - exp(-theta_i theta_j Omega[c_i][c_j]), independently; the
 * walk over each block pair's virtual table jumps to the next cell with a Poisson event by binary search over
 * prefix sums. Stream, fp64 evaluation and the chunking of the walk are fixed by docs/SBM_SPEC.md, so the edge
 * list is identical to the oracle's, in (block pair, chunk, cell) order; src is the member of the lower block.
 *   c_dev: device int32[n] block labels in [0, K); theta_dev: device fp64[n] > 0; omega_dev: device fp64[K*K]
 *   symmetric, >= 0; q: chunks of 2^q cells (4..30; 20 suggested); src_dev/dst_dev: device int32[cap].
 *   m_out: host, the number of edges. If it exceeds cap nothing is written: call again with cap >= *m_out.
 * Synchronous. Errors: PARAM (sizes, null pointers, invalid labels / theta / Omega). */
RAFTGP_API raftgp_status raftgp_sbm_sample(raftgp_ctx ctx, int64_t n, int32_t K, const int32_t *c_dev,
                                           const double *theta_dev, const double *omega_dev, uint64_t seed, int32_t q,
                                           int32_t *src_dev, int32_t *dst_dev, int64_t cap, int64_t *m_out);

/* ---------------------------------------------------------------- NEXT-4: streaming updates
 * PAPER.md:207-214 (§III-D): after edges E' are added only the multi-hop neighbourhood of the nodes V' whose
 * degree changed is re-embedded. A stream holds the graph and the state of the X = M (NCut) embedding of
 * raftgp_embed (Theta' = Theta W^(1), the GCN operands T_1..T_L and Z). raftgp_stream_add_edges merges E' into
 * the CSR (duplicates and self-loops drop out), recomputes the feature-hop rows of R_1 = V' u N(V') and the
 * GCN hop-k rows of R_{k+1} = R_k u N(R_k) (new graph) with the same kernels as raftgp_embed, so Z is
 * bit-identical to raftgp_embed(NCUT) on the whole new graph. (Q and Q~ depend on 2e, which changes every row
 * when an edge is added: their exact update is the full recompute, so streams are NCut only.)
 *   raftgp_stream_create: g = whole-graph handle, ownership passes to the stream (do not destroy it);
 *     dims[0] = r and every width in {32, 64, 128}. Synchronous state build.
 *   raftgp_stream_add_edges: m pairs (host or device per flags). stats: host int64[layers + 3] or NULL:
 *     {|V'|, |R_1|, ..., |R_{layers+1}|, nnz of the new graph}. Synchronous.
 *   raftgp_stream_embedding: copies Z (n x dims[layers], device) out (async on the context stream).
 *   raftgp_stream_graph: borrowed handle of the current graph (export / scoring), valid until the next add.
 * Errors: PARAM (widths, arguments), DATA (node id outside [0, n); nothing is changed), STATE (a previous batch failed
 * after its hops started: the state is partly updated and raftgp_stream_set_mode must recompute it first), NOMEM, CUDA. */
RAFTGP_API raftgp_status raftgp_stream_create(raftgp_graph g, int32_t layers, const int32_t *dims, uint64_t seed,
                                              raftgp_stream *out);
RAFTGP_API raftgp_status raftgp_stream_add_edges(raftgp_stream s, int64_t m, const int32_t *src, const int32_t *dst,
                                                 uint32_t flags, int64_t *stats);
RAFTGP_API raftgp_status raftgp_stream_embedding(raftgp_stream s, float *Z_dev);
RAFTGP_API raftgp_status raftgp_stream_graph(raftgp_stream s, raftgp_graph *g_out);
RAFTGP_API raftgp_status raftgp_stream_destroy(raftgp_stream s);
/* raftgp_stream_set_mode: how raftgp_stream_add_edges updates the GCN hops (Eq. 6).
 *   RAFTGP_STREAM_EXACT (the default): the hops are recomputed over R_{k} (or every row) with the hop kernels, so Z
 *     stays bit-identical to raftgp_embed(NCUT) on the new graph.
 *   RAFTGP_STREAM_DELTA: the stream keeps every GCN hop's pre-activation sums A^h_i = T^h_i + sum_{j in N(i)} T^h_j
 *     (n x dims[h] fp32 each, device, library-owned, plus an n x max(dims[1..L-1]) scratch and an int32[n] index);
 *     after a batch, rows outside V' add the changes
 *     T^h_j(new) - T^h_j(old) of their neighbours in R_h only, and the rows of V' are summed in full. Hop h < L visits
 *     the rows of R_{h+1}, the last hop every row, each reading col_idx once instead of one operand row per CSR
 *     entry. Z equals the full recompute up to fp32 rounding order (re-associated sums; the error grows slowly with
 *     the number of batches), not bit-identically.
 *   Setting either mode (again) first recomputes the exact chain over every row (Z bit-identical to raftgp_embed:
 *   a resync); DELTA then builds the sums by a full pass.
 *   stats[layers + 1] of raftgp_stream_add_edges is then the number of rows whose Z was rewritten.
 * Errors: PARAM (null stream, unknown mode), NOMEM, CUDA. Asynchronous on the context stream. */
#define RAFTGP_STREAM_EXACT 0
#define RAFTGP_STREAM_DELTA 1
RAFTGP_API raftgp_status raftgp_stream_set_mode(raftgp_stream s, int32_t mode);

/* ---------------------------------------------------------------- a6 fused: exchange inside the producing hop
 * SURVEY §8(e) / north_star "per-hop all-gather": on P ranks every GCN hop needs the next operand T for ALL n
 * rows. Instead of computing local rows and then all-gathering them, the producing kernel's epilogue stores
 * each finished row of T straight into every rank's full n-row copy (peer memory over NVLink, opened with the
 * IPC calls below), so the transfer overlaps the hop's gathers row by row. After the producing calls of all
 * ranks, the caller runs one stream-ordered barrier (e.g. a 1-element NCCL all-reduce) before the next hop
 * reads its copy. Results are bit-identical to raftgp_feature_transform / raftgp_gcn_hop + all-gather.
 *   raftgp_feature_transform_push: as raftgp_feature_transform; rep = host array [nvariants][nrep] of device
 *     pointers, rep[v][q] = rank q's n x l1 copy of variant v's T1 (this rank's rows land at rows
 *     [row_begin, row_end)). nrep in [1, 8].
 *   raftgp_gcn_hop_push: as raftgp_gcn_hop with W_next (required); T_next goes to rep[0..nrep) (n x w_next each)
 *     instead of a local buffer. Z_out_dev may be NULL.
 *   Widths in {32, 64, 128} and 16-B aligned pointers fuse the stores into the hop kernels; other shapes compute
 *   locally and then copy into the replicas (same result).
 *   raftgp_ipc_alloc: cudaMalloc'd buffer (library-owned until raftgp_ipc_free) and its 64-byte IPC handle.
 *   raftgp_ipc_open / raftgp_ipc_close: map / unmap another process's buffer on this context's device (peer
 *     access enabled lazily). raftgp_copy: device-to-device copy by a kernel on the context stream.
 * Errors: PARAM (replica count / null pointers / widths), CUDA (IPC failures), NOMEM. */
RAFTGP_API raftgp_status raftgp_feature_transform_push(raftgp_graph g, int32_t nvariants, const int32_t *variants,
                                                       int32_t r, int32_t l1, uint64_t seed, float *const *rep,
                                                       int32_t nrep);
RAFTGP_API raftgp_status raftgp_gcn_hop_push(raftgp_graph g, const float *T_full_dev, int32_t w, float *Z_out_dev,
                                             const float *W_next_dev, int32_t w_next, float *const *rep, int32_t nrep);
RAFTGP_API raftgp_status raftgp_ipc_alloc(raftgp_ctx ctx, size_t bytes, void **dev_ptr, void *handle64);
RAFTGP_API raftgp_status raftgp_ipc_free(raftgp_ctx ctx, void *dev_ptr);
RAFTGP_API raftgp_status raftgp_ipc_open(raftgp_ctx ctx, const void *handle64, void **dev_ptr);
RAFTGP_API raftgp_status raftgp_ipc_close(raftgp_ctx ctx, void *dev_ptr);
RAFTGP_API raftgp_status raftgp_copy(raftgp_ctx ctx, void *dst_dev, const void *src_dev, size_t bytes);


#ifdef __cplusplus
}
#endif
#endif /* RAFTGP_H */
