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
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
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

// frontier expansion: nodes at level k - 1 mark their unmarked neighbours with level k
__global__ void expand_level(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col, int8_t *level,
                             int k) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || level[i] != k - 1) return;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = col[p];
        if (level[j] > k) level[j] = (int8_t)k;   // idempotent: every writer stores k
    }
}

__global__ void init_level(int64_t n, const int32_t *__restrict__ changed, int8_t *level) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) level[i] = changed[i] ? 0 : 127;
}

__global__ void level_flags(int64_t n, const int8_t *__restrict__ level, int k, int32_t *__restrict__ flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = level[i] <= k;
}

__global__ void compact_rows(int64_t n, const int32_t *__restrict__ flag, const int64_t *__restrict__ pos,
                             int32_t *__restrict__ rows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) rows[pos[i]] = (int32_t)i;
}

inline unsigned g256(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }

bool fast_width(int32_t w) { return w == 32 || w == 64 || w == 128; }

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
    raftgp_graph g = s->g;
    raftgp_ctx ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t n = g->n;
    const int L = s->layers;
    // ---- 1. delta CSR of E' (canonical: both orientations, sorted, deduplicated, no self-loops)
    raftgp_graph_s delta;
    delta.ctx = ctx;
    RG_TRY(csr_build(ctx, n, m, src, dst, 0, n, &delta));
    auto drop = [&](raftgp_graph_s &x) {
        dfree(ctx, x.row_ptr); dfree(ctx, x.col); dfree(ctx, x.deg_local); dfree(ctx, x.order); dfree(ctx, x.deg_all);
        dfree(ctx, x.s_all); dfree(ctx, x.sh_all);
    };
    // ---- merged CSR
    raftgp_graph ng = new raftgp_graph_s();
    ng->ctx = ctx;
    ng->n = n;
    ng->row_begin = 0;
    ng->row_end = n;
    ng->nl = n;
    int32_t *changed = nullptr, *flag = nullptr, *rows = nullptr;
    int64_t *pos = nullptr;
    int8_t *level = nullptr;
    raftgp_status rc = dalloc_t(ctx, &ng->deg_local, (size_t)n);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->row_ptr, (size_t)n + 1);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &changed, (size_t)n);
    if (rc == RAFTGP_OK) {
        {
            LaunchScope LS(ctx, K_STREAM);
            merge_count<<<g256(n), 256, 0, st>>>(n, g->row_ptr, g->col, delta.row_ptr, delta.col, g->deg_local,
                                                 ng->deg_local, changed);
        }
        rc = scan_i32_to_i64(ctx, ng->deg_local, ng->row_ptr, n);
    }
    if (rc == RAFTGP_OK) {
        RG_TRY(dread(ctx, &ng->nnz_local, ng->row_ptr + n, sizeof(int64_t), st));
        rc = dalloc_t(ctx, &ng->col, (size_t)std::max<int64_t>(1, ng->nnz_local));
    }
    if (rc == RAFTGP_OK) {
        {
            LaunchScope LS(ctx, K_STREAM);
            merge_write<<<g256(n * 32), 256, 0, st>>>(n, g->row_ptr, g->col, delta.row_ptr, delta.col, changed,
                                                      ng->row_ptr, ng->col);
        }
        RG_CHECK_LAUNCH(ctx);
        rc = dalloc_t(ctx, &ng->deg_all, (size_t)n);
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->s_all, (size_t)n);
        if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &ng->sh_all, (size_t)n);
    }
    if (rc == RAFTGP_OK) {
        if (n > 0) RG_TRY(dcopy(ctx, ng->deg_all, ng->deg_local, sizeof(int32_t) * n, st));
        rc = degrees_finalize(ng);
    }
    drop(delta);
    // ---- 2. affected sets R_1..R_{L+1} (levels 0..L+1 from V')
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &level, (size_t)n);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &flag, (size_t)n);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &pos, (size_t)n + 1);
    if (rc == RAFTGP_OK) rc = dalloc_t(ctx, &rows, (size_t)std::max<int64_t>(1, n));
    std::vector<int64_t> counts(L + 2, 0);
    if (rc == RAFTGP_OK) {
        LaunchScope LS(ctx, K_STREAM);
        init_level<<<g256(n), 256, 0, st>>>(n, changed, level);
    }
    for (int k = 1; k <= L + 1 && rc == RAFTGP_OK; ++k) {
        LaunchScope LS(ctx, K_STREAM);
        expand_level<<<g256(n), 256, 0, st>>>(n, ng->row_ptr, ng->col, level, k);
    }
    // |V'| and the sizes of R_k (synchronous reads: the row lists are built per set below)
    for (int k = 0; k <= L + 1 && rc == RAFTGP_OK; ++k) {
        {
            LaunchScope LS(ctx, K_STREAM);
            level_flags<<<g256(n), 256, 0, st>>>(n, level, k, flag);
        }
        rc = scan_i32_to_i64(ctx, flag, pos, n);
        if (rc == RAFTGP_OK) {
            RG_TRY(dread(ctx, &counts[k], pos + n, sizeof(int64_t), st));
        }
        if (rc != RAFTGP_OK || k == 0) continue;
        // ---- 3. recompute the rows of R_k: the feature hop for k = 1, GCN hop k - 1 for k >= 2
        {
            LaunchScope LS(ctx, K_STREAM);
            compact_rows<<<g256(n), 256, 0, st>>>(n, flag, pos, rows);
        }
        const auto &d = s->dims;
        if (k == 1) {
            rc = feature_hop_pre_rows(ng, RAFTGP_NCUT, d[1], s->thw, nullptr, s->T[1], rows, counts[1]);
        } else {
            const int h = k - 1;   // GCN hop h reads T_h, writes T_{h+1} (or Z after the last layer)
            const bool last = h == L;
            rc = gcn_hop_rows(ng, s->T[h], d[h], last ? s->Z : nullptr, last ? nullptr : s->W[h + 1],
                              last ? 0 : d[h + 1], last ? nullptr : s->T[h + 1], rows, counts[k]);
        }
    }
    dfree(ctx, changed); dfree(ctx, flag); dfree(ctx, pos); dfree(ctx, rows); dfree(ctx, level);
    if (rc != RAFTGP_OK) {
        drop(*ng);
        delete ng;
        return rc;   // the stream keeps its previous graph; rows already recomputed for the new graph are stale
    }
    // the stream now owns the merged graph
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
    if (s->g) {
        raftgp_graph_s &x = *s->g;
        dfree(ctx, x.row_ptr); dfree(ctx, x.col); dfree(ctx, x.deg_local); dfree(ctx, x.order); dfree(ctx, x.deg_all);
        dfree(ctx, x.s_all); dfree(ctx, x.sh_all);
        delete s->g;
        ctx_release(ctx);
    }
    delete s;
    ctx_release(ctx);
}

}  // namespace raftgp
