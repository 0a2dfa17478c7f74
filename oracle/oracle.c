/*
 * oracle/oracle.c — plain, slow, obviously-correct CPU ORACLE of the RaftGP embedding path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2312_01560_b200/) never
 * imports, links or executes it, and shares no code, header, constant or table with it.
 *
 * Precision: fp64 for all method arithmetic, except the Gaussian generator, whose fp32 values are
 * defined bit-exactly by docs/SKETCH_SPEC.md (the paper fixes no generator).
 * Compile with -ffp-contract=off (no silent FMA contraction); fmaf() is the C99 fused multiply-add.
 *
 * Threads ("OpenMP over rows allowed because per-row sums are sequential"): the loops
 * over OUTPUT ROWS (operator rows, GEMM rows, generator rows, per-row CSR sorts) run under OpenMP. Every
 * row is still computed by one thread, sequentially, in the order written below, so every output bit is
 * independent of the thread count (pinned: tests/test_oracle_graph_ops.py::test_thread_count_invariance).
 * Reductions across rows (g = d^T Theta, scores) stay sequential. oracle_set_threads(k) fixes the count.
 *
 * What each function follows:
 *   oracle_philox4x32_10   SKETCH_SPEC §1 (pinned against curand's host Philox)
 *   oracle_ln_spec_batch,
 *   oracle_sincos_spec_batch,
 *   oracle_gaussian        SKETCH_SPEC §2-§5; Eq. 5 Theta_ir ~ N(0, 1/L) (reading #2)
 *   oracle_build_csr       PAPER.md:56 (§II: undirected, unweighted, A_ij = A_ji in {0,1})
 *   oracle_apply           X in {M, Q (Eq. 4), Q~,
 *                          P = D^-1/2 (A+I) D^-1/2 (Eq. 6)} times a dense block
 *   oracle_project         Eq. 5: Y = X Theta
 *   oracle_gcn             Eq. 6 + row l2 normalisation
 *   oracle_embed_rows      the same, for selected output rows only (receptive field)
 *   oracle_modularity      Eq. 3
 *   oracle_ncut            Eq. 1
 *   oracle_local_modularity Eq. 7
 *   oracle_kmeans2,
 *   oracle_model_select    Alg. 1 with the 2-means of docs/SELECT_SPEC.md (NEXT-1)
 *   oracle_sbm_sample      Alg. 2 per docs/SBM_SPEC.md (NEXT-3)
 *
 * Status codes: 0 ok, 2 parameter error, 3 data error (same numbering as include/raftgp.h, which
 * is NOT included here).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* thread count of the row loops (0 = the OpenMP default); results never depend on it (see header) */
static int g_threads = 0;
void oracle_set_threads(int k) { g_threads = k > 0 ? k : 0; }
int oracle_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}
#define ORACLE_ROWS_PARALLEL _Pragma("omp parallel for schedule(dynamic, 256) num_threads(oracle_get_threads())")

/* ---------------------------------------------------------------- Philox4x32-10 (SKETCH_SPEC §1) */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* ---------------------------------------------------------------- ln_spec (SKETCH_SPEC §3) */
static float ln_spec(float u) {
    uint32_t bits;
    memcpy(&bits, &u, 4);
    int e = (int)((bits >> 23) & 0xFFu) - 127;
    uint32_t mbits = (bits & 0x7FFFFFu) | 0x3F800000u;
    float m;
    memcpy(&m, &mbits, 4);
    if (m > 0x1.6a09e6p+0f) { m = m * 0.5f; e = e + 1; }
    float t = (m - 1.0f) / (m + 1.0f);
    float t2 = t * t;
    float p = fmaf(t2, 0x1.745d18p-3f, 0x1.c71c72p-3f);
    p = fmaf(t2, p, 0x1.24924ap-2f);
    p = fmaf(t2, p, 0x1.99999ap-2f);
    p = fmaf(t2, p, 0x1.555556p-1f);
    p = fmaf(t2, p, 0x1.000000p+1f);
    float lnm = t * p;
    return fmaf((float)e, 0x1.62e430p-1f, lnm);
}

/* ---------------------------------------------------------------- sincos2pi_spec (SKETCH_SPEC §3) */
static void sincos2pi_spec(uint32_t k2, float *c, float *s) {
    uint32_t q = k2 >> 22;
    float f = (float)(k2 & 0x3FFFFFu) * 0x1p-22f;
    float phi = f * 0x1.921fb6p+0f;
    float p2 = phi * phi;
    float sp = fmaf(p2, -0x1.ae6456p-26f, 0x1.71de3ap-19f);
    sp = fmaf(p2, sp, -0x1.a01a02p-13f);
    sp = fmaf(p2, sp, 0x1.111112p-7f);
    sp = fmaf(p2, sp, -0x1.555556p-3f);
    float phi3 = phi * p2;
    float sn = fmaf(phi3, sp, phi);
    float cp = fmaf(p2, 0x1.1eed8ep-29f, -0x1.27e4fcp-22f);
    cp = fmaf(p2, cp, 0x1.a01a02p-16f);
    cp = fmaf(p2, cp, -0x1.6c16c2p-10f);
    cp = fmaf(p2, cp, 0x1.555556p-5f);
    cp = fmaf(p2, cp, -0x1.000000p-1f);
    float cs = fmaf(p2, cp, 1.0f);
    switch (q) {
        case 0: *c = cs; *s = sn; break;
        case 1: *c = -sn; *s = cs; break;
        case 2: *c = -cs; *s = -sn; break;
        default: *c = sn; *s = -cs; break;
    }
}

void oracle_ln_spec_batch(const float *u, float *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = ln_spec(u[i]);
}

void oracle_sincos_spec_batch(const uint32_t *k2, float *c, float *s, int64_t n) {
    for (int64_t i = 0; i < n; ++i) sincos2pi_spec(k2[i], &c[i], &s[i]);
}

/* The four consecutive elements (i, 4q..4q+3) of SKETCH_SPEC §1-§4, from one Philox call. */
static void gaussian_quad(uint64_t seed, uint32_t tag, uint64_t i, uint32_t q, float sigma, float out[4]) {
    uint32_t ctr[4] = {q, (uint32_t)(i & 0xFFFFFFFFu), (uint32_t)(i >> 32), tag};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    for (int pair = 0; pair < 2; ++pair) {
        uint32_t xa = x[2 * pair], xb = x[2 * pair + 1];
        float u1 = (float)((xa >> 8) + 1u) * 0x1p-24f;
        uint32_t k2 = xb >> 8;
        float R = sqrtf(-2.0f * ln_spec(u1));
        float c, s;
        sincos2pi_spec(k2, &c, &s);
        float za = R * c, zb = R * s;
        out[2 * pair] = za * sigma;
        out[2 * pair + 1] = zb * sigma;
    }
}

static float sigma_of(int32_t den) { return 1.0f / sqrtf((float)den); }

/* rows x cols block of the generator matrix, global rows row_begin.. (SKETCH_SPEC §5) */
int oracle_gaussian(uint64_t seed, uint32_t tag, int64_t row_begin, int64_t rows, int32_t cols, int32_t den,
                    float *out) {
    if (rows < 0 || cols <= 0 || den <= 0 || row_begin < 0) return 2;
    float sigma = sigma_of(den);
    ORACLE_ROWS_PARALLEL
    for (int64_t i = 0; i < rows; ++i)
        for (int32_t q = 0; 4 * q < cols; ++q) {
            float v[4];
            gaussian_quad(seed, tag, (uint64_t)(row_begin + i), (uint32_t)q, sigma, v);
            for (int32_t c = 4 * q; c < cols && c < 4 * q + 4; ++c) out[i * (int64_t)cols + c] = v[c - 4 * q];
        }
    return 0;
}

/* ---------------------------------------------------------------- CSR build */
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * Canonical CSR of the simple undirected graph of the raw pairs (src[e], dst[e]):
 * drop u == v, add (u,v) and (v,u), sort lexicographically, drop duplicates.
 * The lexicographic sort of (row, col) keys is done as "group by row, then sort each row by col":
 *   1. count the entries of every row (both orientations, self pairs dropped);
 *   2. place each entry's col into its row's segment of col[] (raw offsets = prefix sum of the counts);
 *   3. sort every row segment ascending and drop consecutive duplicates;
 *   4. row_ptr = prefix sum of the deduplicated lengths; move the rows left into place (in row order,
 *      never overwriting a row not yet moved, since every destination is at or before its source).
 * row_ptr: int64[n+1]; col: int32[capacity >= 2m] (also the workspace); *nnz_out = row_ptr[n] = 2e.
 */
int oracle_build_csr(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int64_t *row_ptr, int32_t *col,
                     int64_t *nnz_out) {
    if (n < 0 || m < 0) return 2;
    for (int64_t e = 0; e < m; ++e)
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) return 3;
    int64_t *raw = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));   /* raw row offsets, then cursors */
    int64_t *len = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!raw || !len) { free(raw); free(len); return 4; }
    /* 1. */
    for (int64_t e = 0; e < m; ++e) {
        if (src[e] == dst[e]) continue;
        raw[src[e] + 1] += 1;
        raw[dst[e] + 1] += 1;
    }
    for (int64_t i = 0; i < n; ++i) raw[i + 1] += raw[i];
    /* 2. (len[] doubles as the fill cursor) */
    for (int64_t i = 0; i < n; ++i) len[i] = raw[i];
    for (int64_t e = 0; e < m; ++e) {
        int32_t u = src[e], v = dst[e];
        if (u == v) continue;
        col[len[u]++] = v;
        col[len[v]++] = u;
    }
    /* 3. */
    ORACLE_ROWS_PARALLEL
    for (int64_t i = 0; i < n; ++i) {
        int32_t *r = col + raw[i];
        int64_t cnt = raw[i + 1] - raw[i], k = 0;
        qsort(r, (size_t)cnt, sizeof(int32_t), cmp_i32);
        for (int64_t t = 0; t < cnt; ++t)
            if (t == 0 || r[t] != r[t - 1]) r[k++] = r[t];
        len[i] = k;
    }
    /* 4. */
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + len[i];
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i] != raw[i]) memmove(col + row_ptr[i], col + raw[i], sizeof(int32_t) * (size_t)len[i]);
    *nnz_out = row_ptr[n];
    free(raw);
    free(len);
    return 0;
}

/* ---------------------------------------------------------------- operators */
enum { OP_NCUT = 0, OP_MOD = 1, OP_MOD_REDUCED = 2, OP_PROP = 3 };

static int64_t deg_of(const int64_t *row_ptr, int64_t i) { return row_ptr[i + 1] - row_ptr[i]; }

/* out[i, :] = (X_op @ X)[i, :] for the rows i in rows[0..S) (all rows if rows == NULL, S = n).
 *   NCUT:        M_ij = A_ij / sqrt(d_i d_j), 0 row if d_i = 0
 *   MOD:         Q X = A X - d (d^T X) / 2e             (Q_ij = A_ij - d_i d_j / 2e)
 *   MOD_REDUCED: Q~_ij = A_ij (1 - d_i d_j / 2e)        (Q restricted to edges)
 *   PROP:        P_ij = Ahat_ij / sqrt(dhat_i dhat_j), Ahat = A + I, dhat = d + 1 (Eq. 6)
 * X is addressed through xslot: row j of X is X[xslot ? xslot[j] : j]; dTX (length w) is required for MOD.
 * Each output row is summed sequentially in CSR order (self term first for PROP). */
static void apply_rows(int64_t n, const int64_t *row_ptr, const int32_t *col, int op, int32_t w, const double *X,
                       const int32_t *xslot, const double *dTX, double two_e, const int64_t *rows, int64_t S,
                       double *out) {
    ORACLE_ROWS_PARALLEL
    for (int64_t s = 0; s < S; ++s) {
        int64_t i = rows ? rows[s] : s;
        double *o = out + s * (int64_t)w;
        for (int32_t c = 0; c < w; ++c) o[c] = 0.0;
        double di = (double)deg_of(row_ptr, i);
        if (op == OP_PROP) {
            double shi = 1.0 / sqrt(di + 1.0);
            const double *xi = X + (int64_t)(xslot ? xslot[i] : i) * w;
            double wii = shi * shi;
            for (int32_t c = 0; c < w; ++c) o[c] += wii * xi[c];
        }
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            int64_t j = col[p];
            double dj = (double)deg_of(row_ptr, j);
            double wij;
            switch (op) {
                case OP_NCUT: wij = (1.0 / sqrt(di)) * (1.0 / sqrt(dj)); break;
                case OP_MOD: wij = 1.0; break;
                case OP_MOD_REDUCED: wij = 1.0 - di * dj / two_e; break;
                default: wij = (1.0 / sqrt(di + 1.0)) * (1.0 / sqrt(dj + 1.0)); break;
            }
            const double *xj = X + (int64_t)(xslot ? xslot[j] : j) * w;
            for (int32_t c = 0; c < w; ++c) o[c] += wij * xj[c];
        }
        if (op == OP_MOD)
            for (int32_t c = 0; c < w; ++c) o[c] -= di * dTX[c] / two_e;
    }
}

int oracle_apply(int64_t n, const int64_t *row_ptr, const int32_t *col, int op, int32_t w, const double *X,
                 double *out) {
    if (n < 0 || w <= 0 || op < 0 || op > 3) return 2;
    double two_e = (double)row_ptr[n];
    if ((op == OP_MOD || op == OP_MOD_REDUCED) && two_e == 0.0) return 3;
    double *dTX = NULL;
    if (op == OP_MOD) {
        dTX = (double *)calloc((size_t)w, sizeof(double));
        for (int64_t j = 0; j < n; ++j) {
            double dj = (double)deg_of(row_ptr, j);
            for (int32_t c = 0; c < w; ++c) dTX[c] += dj * X[j * (int64_t)w + c];
        }
    }
    apply_rows(n, row_ptr, col, op, w, X, NULL, dTX, two_e, NULL, n, out);
    free(dTX);
    return 0;
}

/* Eq. 5: Y = X Theta, Theta from the spec generator (seed, tag 0, den r), promoted to fp64. */
int oracle_project(int64_t n, const int64_t *row_ptr, const int32_t *col, int variant, int32_t r, uint64_t seed,
                   double *Y) {
    if (r <= 0 || variant < 0 || variant > 2) return 2;
    if (variant != OP_NCUT && row_ptr[n] == 0) return 3;
    float *th = (float *)malloc(sizeof(float) * (size_t)(n * (int64_t)r + 1));
    double *X = (double *)malloc(sizeof(double) * (size_t)(n * (int64_t)r + 1));
    oracle_gaussian(seed, 0u, 0, n, r, r, th);
    ORACLE_ROWS_PARALLEL
    for (int64_t k = 0; k < n * (int64_t)r; ++k) X[k] = (double)th[k];
    int rc = oracle_apply(n, row_ptr, col, variant, r, X, Y);
    free(th);
    free(X);
    return rc;
}

/* tanh then row l2 normalisation of one row; a zero row stays zero. */
static void act_normalize(double *h, int32_t w) {
    double ss = 0.0;
    for (int32_t c = 0; c < w; ++c) { h[c] = tanh(h[c]); ss += h[c] * h[c]; }
    if (ss > 0.0) {
        double nrm = sqrt(ss);
        for (int32_t c = 0; c < w; ++c) h[c] = h[c] / nrm;
    }
}

/* h[c] = sum_{t = 0..a-1} z[t] W[t][c], each h[c] summed sequentially in t starting from 0.0 (the loops are
 * nested t-outer so W is read row by row; the sequence of additions into every h[c] is unchanged). */
static void row_times_w(const double *z, const double *W, int32_t a, int32_t b, double *h) {
    for (int32_t c = 0; c < b; ++c) h[c] = 0.0;
    for (int32_t t = 0; t < a; ++t) {
        const double zt = z[t];
        const double *w = W + (int64_t)t * b;
        for (int32_t c = 0; c < b; ++c) h[c] += zt * w[c];
    }
}

static double *weights_f64(uint64_t seed, int k, int32_t fan_in, int32_t fan_out) {
    float *wf = (float *)malloc(sizeof(float) * (size_t)fan_in * fan_out);
    double *wd = (double *)malloc(sizeof(double) * (size_t)fan_in * fan_out);
    oracle_gaussian(seed, (uint32_t)k, 0, fan_in, fan_out, fan_in, wf);
    for (int64_t q = 0; q < (int64_t)fan_in * fan_out; ++q) wd[q] = (double)wf[q];
    free(wf);
    return wd;
}

/* Eq. 6 with l2 normalisation: Z^(k) = rownorm(tanh((P Z^(k-1)) W^(k))), Z^(0) = Y.
 * Zcat receives Z^(1), ..., Z^(K) back to back (block k is n x dims[k]). */
int oracle_gcn(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t layers, const int32_t *dims,
               uint64_t seed, const double *Y, double *Zcat) {
    if (layers < 1) return 2;
    for (int k = 0; k <= layers; ++k) if (dims[k] <= 0) return 2;
    const double *Zin = Y;
    double *Zout = Zcat;
    for (int k = 1; k <= layers; ++k) {
        int32_t a = dims[k - 1], b = dims[k];
        double *Wk = weights_f64(seed, k, a, b);
        double *AZ = (double *)malloc(sizeof(double) * (size_t)(n * (int64_t)a + 1));
        oracle_apply(n, row_ptr, col, OP_PROP, a, Zin, AZ);
        ORACLE_ROWS_PARALLEL
        for (int64_t i = 0; i < n; ++i) {
            double *h = Zout + i * (int64_t)b;
            row_times_w(AZ + i * (int64_t)a, Wk, a, b, h);
            act_normalize(h, b);
        }
        free(AZ);
        free(Wk);
        Zin = Zout;
        Zout += n * (int64_t)b;
    }
    return 0;
}

/* ---------------------------------------------------------------- selected rows (receptive field) */
typedef struct { int64_t *v; int64_t len, cap; } vec64;
static void vpush(vec64 *a, int64_t x) {
    if (a->len == a->cap) { a->cap = a->cap ? 2 * a->cap : 1024; a->v = (int64_t *)realloc(a->v, sizeof(int64_t) * a->cap); }
    a->v[a->len++] = x;
}

/* closure: set out = in  U  N(in); mark[] must be all -1 on entry for the ids in question and is
 * left holding the slot (position in out) of each member. */
static void closure(const int64_t *row_ptr, const int32_t *col, const vec64 *in, vec64 *out, int32_t *mark) {
    for (int64_t s = 0; s < in->len; ++s) {
        int64_t i = in->v[s];
        if (mark[i] < 0) { mark[i] = (int32_t)out->len; vpush(out, i); }
    }
    for (int64_t s = 0; s < in->len; ++s) {
        int64_t i = in->v[s];
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            int64_t j = col[p];
            if (mark[j] < 0) { mark[j] = (int32_t)out->len; vpush(out, j); }
        }
    }
}

/*
 * Y and Z^(1..K) for the rows rows[0..S) only, by walking the receptive field: Z^(K) rows need
 * Z^(K-1) on rows U N(rows), ..., Y on the (K)-hop closure, Theta on the (K+1)-hop closure.
 * Same arithmetic, same order per row as oracle_project + oracle_gcn, so the results are identical.
 * MOD needs g = d^T Theta over all n rows: one streaming pass regenerating Theta row by row.
 * Yrows: S x r. Zrows: layer-major, block k is S x dims[k]. layers may be 0 (Y only).
 */
int oracle_embed_rows(int64_t n, const int64_t *row_ptr, const int32_t *col, int variant, int32_t r,
                      int32_t layers, const int32_t *dims, uint64_t seed, const int64_t *rows, int64_t S,
                      double *Yrows, double *Zrows) {
    if (r <= 0 || variant < 0 || variant > 2 || layers < 0) return 2;
    if (layers > 0 && dims[0] != r) return 2;
    for (int64_t s = 0; s < S; ++s) if (rows[s] < 0 || rows[s] >= n) return 2;
    double two_e = (double)row_ptr[n];
    if (variant != OP_NCUT && two_e == 0.0) return 3;
    int L = layers;
    /* chain[0] = output rows; chain[t+1] = chain[t] U N(chain[t]). chain[L-k] holds the rows of Z^(k)
     * that are needed (Z^(0) = Y), chain[L+1] the Theta rows. cslot[t][i] = position of i in chain[t]. */
    vec64 *chain = (vec64 *)calloc((size_t)L + 2, sizeof(vec64));
    int32_t **cslot = (int32_t **)calloc((size_t)L + 2, sizeof(int32_t *));
    for (int k = 0; k <= L + 1; ++k) {
        cslot[k] = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
        for (int64_t i = 0; i < n; ++i) cslot[k][i] = -1;
    }
    for (int64_t s = 0; s < S; ++s)
        if (cslot[0][rows[s]] < 0) { cslot[0][rows[s]] = (int32_t)chain[0].len; vpush(&chain[0], rows[s]); }
    for (int t = 0; t < L + 1; ++t) closure(row_ptr, col, &chain[t], &chain[t + 1], cslot[t + 1]);
    /* chain[L - k] holds the rows of Z^(k) needed (Z^(0) = Y); chain[L + 1] the Theta rows. */
    const vec64 *thr = &chain[L + 1];
    double *TH = (double *)malloc(sizeof(double) * (size_t)(thr->len * (int64_t)r + 1));
    ORACLE_ROWS_PARALLEL
    for (int64_t q = 0; q < thr->len; ++q) {
        float tmp[4];
        for (int32_t c0 = 0; c0 < r; c0 += 4) {
            int32_t w4 = r - c0 < 4 ? r - c0 : 4;
            /* columns c0..c0+3 of row thr->v[q]: the generator's quad q = c0/4 */
            float sigma = sigma_of(r);
            gaussian_quad(seed, 0u, (uint64_t)thr->v[q], (uint32_t)(c0 / 4), sigma, tmp);
            for (int32_t c = 0; c < w4; ++c) TH[q * r + c0 + c] = (double)tmp[c];
        }
    }
    double *dTX = NULL;
    if (variant == OP_MOD) {
        /* g = d^T Theta over ALL n rows, summed sequentially in j (Theta regenerated chunk by chunk; the chunk
         * generation is parallel over rows, the accumulation is not) */
        dTX = (double *)calloc((size_t)r, sizeof(double));
        const int64_t CH = 1 << 16;
        float *buf = (float *)malloc(sizeof(float) * (size_t)(CH * (int64_t)r));
        for (int64_t j0 = 0; j0 < n; j0 += CH) {
            int64_t cnt = n - j0 < CH ? n - j0 : CH;
            oracle_gaussian(seed, 0u, j0, cnt, r, r, buf);
            for (int64_t j = j0; j < j0 + cnt; ++j) {
                double dj = (double)deg_of(row_ptr, j);
                for (int32_t c = 0; c < r; ++c) dTX[c] += dj * (double)buf[(j - j0) * (int64_t)r + c];
            }
        }
        free(buf);
    }
    /* Y on chain[L] */
    const vec64 *yr = &chain[L];
    double *Zprev = (double *)malloc(sizeof(double) * (size_t)(yr->len * (int64_t)r + 1));
    apply_rows(n, row_ptr, col, variant, r, TH, cslot[L + 1], dTX, two_e, yr->v, yr->len, Zprev);
    free(TH);
    free(dTX);
    for (int64_t s = 0; s < S; ++s)
        memcpy(Yrows + s * (int64_t)r, Zprev + (int64_t)cslot[L][rows[s]] * r, sizeof(double) * (size_t)r);
    double *zout = Zrows;
    for (int k = 1; k <= L; ++k) {
        int32_t a = dims[k - 1], b = dims[k];
        const vec64 *zr = &chain[L - k];
        double *Wk = weights_f64(seed, k, a, b);
        double *AZ = (double *)malloc(sizeof(double) * (size_t)(zr->len * (int64_t)a + 1));
        apply_rows(n, row_ptr, col, OP_PROP, a, Zprev, cslot[L - k + 1], NULL, two_e, zr->v, zr->len, AZ);
        double *Zk = (double *)malloc(sizeof(double) * (size_t)(zr->len * (int64_t)b + 1));
        ORACLE_ROWS_PARALLEL
        for (int64_t q = 0; q < zr->len; ++q) {
            double *h = Zk + q * (int64_t)b;
            row_times_w(AZ + q * (int64_t)a, Wk, a, b, h);
            act_normalize(h, b);
        }
        for (int64_t s = 0; s < S; ++s)
            memcpy(zout + s * (int64_t)b, Zk + (int64_t)cslot[L - k][rows[s]] * b, sizeof(double) * (size_t)b);
        zout += S * (int64_t)b;
        free(AZ);
        free(Wk);
        free(Zprev);
        Zprev = Zk;
    }
    free(Zprev);
    for (int k = 0; k <= L + 1; ++k) { free(chain[k].v); free(cslot[k]); }
    free(chain);
    free(cslot);
    return 0;
}

/* ---------------------------------------------------------------- scoring */
/* Eq. 3: Mod = (1/2e) sum_r sum_{i,j in C_r} [A_ij - d_i d_j / 2e]
 *            = sum_r [ (sum_{i,j in C_r} A_ij) / 2e - (sum_{i in C_r} d_i)^2 / (2e)^2 ]. */
int oracle_modularity(int64_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *assign, int32_t k,
                      double *out) {
    if (k <= 0) return 2;
    for (int64_t i = 0; i < n; ++i) if (assign[i] < 0 || assign[i] >= k) return 2;
    double two_e = (double)row_ptr[n];
    if (two_e == 0.0) return 3;
    double *in_sum = (double *)calloc((size_t)k, sizeof(double)), *vol = (double *)calloc((size_t)k, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        vol[assign[i]] += (double)deg_of(row_ptr, i);
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            if (assign[col[p]] == assign[i]) in_sum[assign[i]] += 1.0;
    }
    double q = 0.0;
    for (int32_t c = 0; c < k; ++c) q += in_sum[c] / two_e - (vol[c] / two_e) * (vol[c] / two_e);
    free(in_sum);
    free(vol);
    *out = q;
    return 0;
}

/* Eq. 1: NCut = 1/2 sum_r cut(C_r, V - C_r) / vol(C_r); a block with vol = 0 contributes 0 (reading #17). */
int oracle_ncut(int64_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *assign, int32_t k,
                double *out) {
    if (k <= 0) return 2;
    for (int64_t i = 0; i < n; ++i) if (assign[i] < 0 || assign[i] >= k) return 2;
    double *cut = (double *)calloc((size_t)k, sizeof(double)), *vol = (double *)calloc((size_t)k, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        vol[assign[i]] += (double)deg_of(row_ptr, i);
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            if (assign[col[p]] != assign[i]) cut[assign[i]] += 1.0;
    }
    double s = 0.0;
    for (int32_t c = 0; c < k; ++c) if (vol[c] > 0.0) s += cut[c] / vol[c];
    free(cut);
    free(vol);
    *out = 0.5 * s;
    return 0;
}

/* Eq. 7: LMod(U_1..U_K; G) = sum_r [ m_r / e - (mbar_r / 2e)^2 ], m_r = #edges of G inside U_r,
 * mbar_r = sum_{v in U_r} deg_G(v) (full-graph degree), 2e = sum_r mbar_r. */
int oracle_local_modularity(int64_t n, const int64_t *row_ptr, const int32_t *col, const int64_t *nodes,
                            int64_t count, const int32_t *block_of_node, int32_t k, double *out) {
    if (k <= 0 || count < 0) return 2;
    int32_t *blk = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) blk[i] = -1;
    for (int64_t t = 0; t < count; ++t) {
        if (nodes[t] < 0 || nodes[t] >= n || block_of_node[t] < 0 || block_of_node[t] >= k || blk[nodes[t]] >= 0) {
            free(blk);
            return 2;
        }
        blk[nodes[t]] = block_of_node[t];
    }
    double *m2 = (double *)calloc((size_t)k, sizeof(double)), *mbar = (double *)calloc((size_t)k, sizeof(double));
    for (int64_t t = 0; t < count; ++t) {
        int64_t i = nodes[t];
        mbar[blk[i]] += (double)deg_of(row_ptr, i);
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            if (blk[col[p]] == blk[i]) m2[blk[i]] += 1.0;   /* counts each intra edge twice */
    }
    double two_e = 0.0;
    for (int32_t c = 0; c < k; ++c) two_e += mbar[c];
    int rc = 0;
    if (two_e == 0.0) rc = 3;
    else {
        double e = two_e / 2.0, q = 0.0;
        for (int32_t c = 0; c < k; ++c) q += (m2[c] / 2.0) / e - (mbar[c] / two_e) * (mbar[c] / two_e);
        *out = q;
    }
    free(blk);
    free(m2);
    free(mbar);
    return rc;
}

/* ---------------------------------------------------------------- Alg. 1: hierarchical model selection
 * (§III-C) with the deterministic 2-means of docs/SELECT_SPEC.md. Plain recursion in the
 * paper's (depth-first) order; every step cites the spec section it follows. */

/* SELECT_SPEC §2: q(z) = round_half_even(double(z) * 2^32) */
static int64_t sel_fixq(float z) { return (int64_t)llrint((double)z * 4294967296.0); }

/* SELECT_SPEC §2: centroid of the members U[t] with (side == NULL or side[t] == want); returns the count */
static int64_t sel_centroid(const float *Z, int32_t L, const int32_t *U, int64_t cnt, const uint8_t *side, int want,
                            double *mu) {
    int64_t *S = (int64_t *)calloc((size_t)L, sizeof(int64_t));
    int64_t c = 0;
    for (int64_t t = 0; t < cnt; ++t) {
        if (side && side[t] != want) continue;
        const float *z = Z + (int64_t)U[t] * L;
        for (int32_t l = 0; l < L; ++l) S[l] += sel_fixq(z[l]);
        c++;
    }
    if (c > 0)
        for (int32_t l = 0; l < L; ++l) mu[l] = ((double)S[l] * 0x1p-32) / (double)c;
    free(S);
    return c;
}

/* SELECT_SPEC §2: d = sum_l (double(x_l) - mu_l)^2, sequential in l, no contraction (-ffp-contract=off) */
static double sel_sqdist(const float *x, const double *mu, int32_t L) {
    double d = 0.0;
    for (int32_t l = 0; l < L; ++l) {
        double t = (double)x[l] - mu[l];
        d = d + t * t;
    }
    return d;
}

/* SELECT_SPEC §3.1: the member farthest from ref (ties: smallest node id) */
static int32_t sel_farthest(const float *Z, int32_t L, const int32_t *U, int64_t cnt, const double *ref) {
    int32_t best = -1;
    double bd = -1.0;
    for (int64_t t = 0; t < cnt; ++t) {
        double d = sel_sqdist(Z + (int64_t)U[t] * L, ref, L);
        if (d > bd || (d == bd && U[t] < best)) { bd = d; best = U[t]; }
    }
    return best;
}

/* SELECT_SPEC §3: KMeans with K = 2 on U (Alg. 1 line 3). side[t] in {0,1} for member U[t]; returns the
 * number of Lloyd iterations t. */
int32_t oracle_kmeans2(const float *Z, int32_t L, const int32_t *U, int64_t cnt, int32_t max_iter, uint8_t *side) {
    double *mu0 = (double *)malloc(sizeof(double) * (size_t)L), *mu1 = (double *)malloc(sizeof(double) * (size_t)L);
    double *mbar = (double *)malloc(sizeof(double) * (size_t)L);
    uint8_t *prev = (uint8_t *)malloc((size_t)cnt + 1);
    int32_t it = 0;
    if (cnt > 0) {
        /* §3.1 seeding */
        sel_centroid(Z, L, U, cnt, NULL, 0, mbar);
        int32_t a = sel_farthest(Z, L, U, cnt, mbar);
        for (int32_t l = 0; l < L; ++l) mu0[l] = (double)Z[(int64_t)a * L + l];
        int32_t b = sel_farthest(Z, L, U, cnt, mu0);
        for (int32_t l = 0; l < L; ++l) mu1[l] = (double)Z[(int64_t)b * L + l];
        /* §3.2 Lloyd */
        for (int32_t t = 1; t <= max_iter; ++t) {
            it = t;
            int changed = 0;
            for (int64_t s = 0; s < cnt; ++s) {
                const float *z = Z + (int64_t)U[s] * L;
                uint8_t c = sel_sqdist(z, mu1, L) < sel_sqdist(z, mu0, L) ? 1 : 0;
                if (t > 1 && c != prev[s]) changed = 1;
                side[s] = c;
            }
            if (t > 1 && !changed) break;
            sel_centroid(Z, L, U, cnt, side, 0, mu0);   /* an empty side keeps its centre */
            sel_centroid(Z, L, U, cnt, side, 1, mu1);
            memcpy(prev, side, (size_t)cnt);
        }
    }
    free(mu0);
    free(mu1);
    free(mbar);
    free(prev);
    return it;
}

/* Alg. 1 lines 2 and 4 via SELECT_SPEC §4: returns 1 iff U (members U[t], KMeans sides side[t]) becomes a
 * block. two_E = 2|E| (degree sum of G); rule 0 = global 2e = two_E, 1 = local 2e = T.
 * where: scratch int32[n], all zero on entry and on return. */
int oracle_split_stops(const int64_t *row_ptr, const int32_t *col, int64_t two_E, const int32_t *U, int64_t cnt,
                       const uint8_t *side, int32_t eps, int32_t rule, int32_t *where) {
    int64_t n1 = 0, n2 = 0, mb1 = 0, mb2 = 0, cut = 0;
    for (int64_t t = 0; t < cnt; ++t) where[U[t]] = side[t] ? 2 : 1;
    for (int64_t t = 0; t < cnt; ++t) {
        int32_t i = U[t];
        int64_t d = row_ptr[i + 1] - row_ptr[i];
        if (side[t]) { n2++; mb2 += d; }
        else {
            n1++;
            mb1 += d;
            for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
                if (where[col[p]] == 2) cut++;   /* each U_1-U_2 edge is seen once, from its U_1 end */
        }
    }
    for (int64_t t = 0; t < cnt; ++t) where[U[t]] = 0;
    int64_t T = mb1 + mb2;
    __int128 two_e = rule == 1 ? (__int128)T : (__int128)two_E;
    /* m_1 > m_2  <=>  2e * c > mbar_1 * mbar_2 */
    return n1 <= eps || n2 <= eps || T == 0 || two_e * (__int128)cut > (__int128)mb1 * (__int128)mb2;
}

typedef struct {
    const int64_t *row_ptr;
    const int32_t *col;
    const float *Z;
    int32_t L, eps, max_iter, rule;   /* rule: 0 = global e (reading #28), 1 = local e (PAPER.md:167 literal) */
    int64_t two_E;       /* global degree sum 2|E| */
    int32_t *block_of;   /* discovery-order block id per node */
    int32_t nblocks;
    int32_t *where;      /* scratch: 1 = in U_1, 2 = in U_2, 0 = elsewhere */
    int64_t splits, kmeans_iters;
    int32_t depth;
} sel_state;

/* PARTITION(U, G) of Alg. 1 on the members U[0..cnt) (reordered in place: U_1 first, then U_2). */
static void sel_partition(sel_state *st, int32_t *U, int64_t cnt, int32_t depth) {
    if (depth + 1 > st->depth) st->depth = depth + 1;
    uint8_t *side = (uint8_t *)malloc((size_t)cnt + 1);
    st->kmeans_iters += oracle_kmeans2(st->Z, st->L, U, cnt, st->max_iter, side);      /* line 3 */
    /* lines 2 and 4 (m_1, m_2 and their comparison, SELECT_SPEC §4) */
    int stop = oracle_split_stops(st->row_ptr, st->col, st->two_E, U, cnt, side, st->eps, st->rule, st->where);
    int64_t n1 = 0, n2 = 0;
    for (int64_t t = 0; t < cnt; ++t) { if (side[t]) n2++; else n1++; }
    if (stop) {                                                                           /* line 5 */
        for (int64_t t = 0; t < cnt; ++t) st->block_of[U[t]] = st->nblocks;
        st->nblocks++;
        free(side);
        return;
    }
    st->splits++;
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)cnt);
    int64_t a = 0, b = n1;
    for (int64_t t = 0; t < cnt; ++t) tmp[side[t] ? b++ : a++] = U[t];
    memcpy(U, tmp, sizeof(int32_t) * (size_t)cnt);
    free(tmp);
    free(side);
    sel_partition(st, U, n1, depth + 1);                                                  /* line 7 */
    sel_partition(st, U + n1, n2, depth + 1);                                             /* line 8 */
}

/* Alg. 1 from U = V. labels[i] = canonical block label (SELECT_SPEC §5: blocks numbered by smallest member);
 * rule: 0 = e = |E| of G (SELECT_SPEC §4 default), 1 = 2e = total degree of U (PAPER.md:167 literal).
 * stats (optional, int64[4]): blocks, splits, total Lloyd iterations, tree depth.
 * Errors: 2 (L <= 0, eps < 0, max_iter < 1, rule not 0/1), 3 (|z| > 1). */
int oracle_model_select(int64_t n, const int64_t *row_ptr, const int32_t *col, const float *Z, int32_t L,
                        int32_t eps, int32_t max_iter, int32_t rule, int32_t *labels, int32_t *num_blocks,
                        int64_t *stats) {
    if (L <= 0 || eps < 0 || max_iter < 1 || n < 0 || rule < 0 || rule > 1) return 2;
    for (int64_t i = 0; i < n * (int64_t)L; ++i)
        if (!(Z[i] >= -1.0f && Z[i] <= 1.0f)) return 3;
    sel_state st;
    memset(&st, 0, sizeof st);
    st.row_ptr = row_ptr; st.col = col; st.Z = Z; st.L = L; st.eps = eps; st.max_iter = max_iter; st.rule = rule; st.two_E = row_ptr[n];
    st.block_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    st.where = (int32_t *)calloc((size_t)(n + 1), sizeof(int32_t));
    int32_t *U = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) U[i] = (int32_t)i;
    if (n > 0) sel_partition(&st, U, n, 0);
    /* canonical labels: first appearance in increasing node id */
    int32_t *canon = (int32_t *)malloc(sizeof(int32_t) * (size_t)(st.nblocks + 1));
    for (int32_t b = 0; b < st.nblocks; ++b) canon[b] = -1;
    int32_t next = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (canon[st.block_of[i]] < 0) canon[st.block_of[i]] = next++;
        labels[i] = canon[st.block_of[i]];
    }
    *num_blocks = st.nblocks;
    if (stats) { stats[0] = st.nblocks; stats[1] = st.splits; stats[2] = st.kmeans_iters; stats[3] = st.depth; }
    free(canon);
    free(U);
    free(st.where);
    free(st.block_of);
    return 0;
}

/* ---------------------------------------------------------------- Alg. 2: exact SBM sampler (NEXT-3)
 * docs/SBM_SPEC.md (Def. 5). Plain loops in the spec's order. */

/* SBM_SPEC §6 */
double oracle_ln_spec64(double u) {
    uint64_t bits;
    memcpy(&bits, &u, 8);
    int e = (int)((bits >> 52) & 0x7FF) - 1023;
    uint64_t mb = (bits & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    double m;
    memcpy(&m, &mb, 8);
    if (m > 0x1.6a09e667f3bcdp+0) { m = m * 0.5; e = e + 1; }
    double t = (m - 1.0) / (m + 1.0);
    double t2 = t * t;
    double s = 2.0 / 25.0;
    for (int k = 11; k >= 0; --k) s = fma(t2, s, 2.0 / (double)(2 * k + 1));
    double lnm = t * s;
    return fma((double)e, 0x1.62e42fefa39efp-1, fma((double)e, 0x1.abc9e3b39803fp-56, lnm));
}

/* SBM_SPEC §5 */
double oracle_sbm_uniform(uint64_t seed, uint32_t p, uint32_t k, uint32_t d) {
    uint32_t ctr[4] = {p, k, d, 0x53424D31u}, key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)}, x[4];
    oracle_philox4x32_10(ctr, key, x);
    uint64_t v = ((uint64_t)(x[0] >> 5) << 26) + (uint64_t)(x[1] >> 6) + 1u;
    return (double)v * 0x1p-53;
}

typedef struct {
    int diag;                 /* r == s */
    int64_t nr, ns;
    const int32_t *Cr, *Cs;   /* members (ascending ids) */
    const double *th;         /* theta of all nodes */
    const double *Pr, *Ps, *Q;
    double omega;
} sbm_pair;

static int64_t tri_row_start(int64_t n, int64_t a) { return a * n - a * (a + 1) / 2; }

/* SBM_SPEC §3: cell -> (a, b) */
static void sbm_cell(const sbm_pair *P, int64_t x, int64_t *a, int64_t *b) {
    if (!P->diag) { *a = x / P->ns; *b = x % P->ns; return; }
    int64_t n = P->nr, lo = 0, hi = n - 2;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (tri_row_start(n, mid) <= x) lo = mid; else hi = mid - 1;
    }
    *a = lo;
    *b = lo + 1 + (x - tri_row_start(n, lo));
}

/* SBM_SPEC §3: RangeSum(x, y), cells inclusive */
double oracle_sbm_range_sum(const sbm_pair *P, int64_t x, int64_t y) {
    int64_t a1, b1, a2, b2;
    sbm_cell(P, x, &a1, &b1);
    sbm_cell(P, y, &a2, &b2);
    double t1 = P->th[P->Cr[a1]], t2 = P->th[P->Cr[a2]];
    if (!P->diag) {
        if (a1 == a2) return P->omega * (t1 * (P->Ps[b2 + 1] - P->Ps[b1]));
        return P->omega * ((t1 * (P->Ps[P->ns] - P->Ps[b1]) + (P->Pr[a2] - P->Pr[a1 + 1]) * P->Ps[P->ns]) +
                           t2 * P->Ps[b2 + 1]);
    }
    const double *Pp = P->Pr;
    int64_t n = P->nr;
    if (a1 == a2) return P->omega * (t1 * (Pp[b2 + 1] - Pp[b1]));
    return P->omega * ((t1 * (Pp[n] - Pp[b1]) + (P->Q[a2] - P->Q[a1 + 1])) + t2 * (Pp[b2 + 1] - Pp[a2 + 1]));
}

/* Alg. 2 (SBM_SPEC §4) for all pairs. Edges (src < dst not implied: src from the row block) are appended in
 * (pair, chunk, cell) order to out_src/out_dst (capacity cap; the total count is returned in *m_out even when
 * it exceeds cap). Errors: 2 (bad arguments: K <= 0, a label outside [0,K), theta <= 0, omega < 0 or not
 * symmetric, q outside [4, 30]). */
int oracle_sbm_sample(int64_t n, int32_t K, const int32_t *c, const double *theta, const double *omega,
                      uint64_t seed, int32_t q, int32_t *out_src, int32_t *out_dst, int64_t cap, int64_t *m_out) {
    if (n < 0 || K <= 0 || q < 4 || q > 30) return 2;
    for (int64_t i = 0; i < n; ++i) if (c[i] < 0 || c[i] >= K || !(theta[i] > 0.0)) return 2;
    for (int32_t r = 0; r < K; ++r)
        for (int32_t s = 0; s < K; ++s)
            if (!(omega[r * K + s] >= 0.0) || omega[r * K + s] != omega[s * K + r]) return 2;
    /* members per block in ascending id */
    int64_t *cnt = (int64_t *)calloc((size_t)K + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[c[i] + 1]++;
    for (int32_t r = 0; r < K; ++r) cnt[r + 1] += cnt[r];
    int32_t *mem = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(K + 1));
    memcpy(fill, cnt, sizeof(int64_t) * (size_t)(K + 1));
    for (int64_t i = 0; i < n; ++i) mem[fill[c[i]]++] = (int32_t)i;
    /* SBM_SPEC §2 tables, per block */
    double *P = (double *)malloc(sizeof(double) * (size_t)(n + K + 1));
    double *Qt = (double *)malloc(sizeof(double) * (size_t)(n + K + 1));
    for (int32_t r = 0; r < K; ++r) {
        int64_t nr = cnt[r + 1] - cnt[r], o = cnt[r] + r;
        P[o] = 0.0;
        for (int64_t a = 0; a < nr; ++a) P[o + a + 1] = P[o + a] + theta[mem[cnt[r] + a]];
        Qt[o] = 0.0;
        for (int64_t a = 0; a < nr; ++a) Qt[o + a + 1] = Qt[o + a] + theta[mem[cnt[r] + a]] * (P[o + nr] - P[o + a + 1]);
    }
    int64_t m = 0;
    uint32_t pidx = 0;
    for (int32_t r = 0; r < K; ++r) {
        for (int32_t s = r; s < K; ++s, ++pidx) {
            sbm_pair pr;
            pr.diag = r == s;
            pr.nr = cnt[r + 1] - cnt[r];
            pr.ns = cnt[s + 1] - cnt[s];
            pr.Cr = mem + cnt[r];
            pr.Cs = mem + cnt[s];
            pr.th = theta;
            pr.Pr = P + cnt[r] + r;
            pr.Ps = P + cnt[s] + s;
            pr.Q = Qt + cnt[r] + r;
            pr.omega = omega[r * K + s];
            int64_t T = pr.diag ? pr.nr * (pr.nr - 1) / 2 : pr.nr * pr.ns;
            if (pr.omega == 0.0 || T <= 0) continue;
            /* SBM_SPEC §4: q_p, the largest q' in [4, q] with R_p 2^q' <= 8 T (else 4) */
            double Rp = oracle_sbm_range_sum(&pr, 0, T - 1);
            int qp = 4;
            for (int qq = q; qq >= 4; --qq)
                if (ldexp(Rp, qq) <= 8.0 * (double)T) { qp = qq; break; }
            const int64_t chunk = (int64_t)1 << qp;
            for (int64_t k = 0; k * chunk < T; ++k) {
                int64_t x0 = k * chunk, x1 = x0 + chunk < T ? x0 + chunk : T, mm = x0;
                uint32_t d = 0;
                for (;;) {
                    double u = oracle_sbm_uniform(seed, pidx, (uint32_t)k, d++);
                    double E = -oracle_ln_spec64(u);
                    if (!(oracle_sbm_range_sum(&pr, mm, x1 - 1) > E)) break;
                    int64_t lo = mm, hi = x1 - 1;
                    while (lo < hi) {
                        int64_t mid = lo + (hi - lo) / 2;
                        if (oracle_sbm_range_sum(&pr, mm, mid) > E) hi = mid; else lo = mid + 1;
                    }
                    int64_t a, b;
                    sbm_cell(&pr, lo, &a, &b);
                    if (m < cap) { out_src[m] = pr.Cr[a]; out_dst[m] = pr.diag ? pr.Cr[b] : pr.Cs[b]; }
                    m++;
                    mm = lo + 1;
                    if (mm == x1) break;
                }
            }
        }
    }
    *m_out = m;
    free(cnt); free(mem); free(fill); free(P); free(Qt);
    return 0;
}

/* Test hook: RangeSum(x, y) of one block pair given the member thetas (rows theta_r[n_r], cols theta_s[n_s];
 * diag: the upper triangle of one block, theta_s ignored). Builds the §2 tables like oracle_sbm_sample. */
double oracle_sbm_range_sum_hook(int diag, int64_t nr, const double *theta_r, int64_t ns, const double *theta_s,
                                 double omega, int64_t x, int64_t y) {
    int64_t nt = nr + (diag ? 0 : ns);
    double *th = (double *)malloc(sizeof(double) * (size_t)(nt + 1));
    int32_t *Cr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nr + 1));
    int32_t *Cs = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ns + 1));
    for (int64_t a = 0; a < nr; ++a) { th[a] = theta_r[a]; Cr[a] = (int32_t)a; }
    if (!diag) for (int64_t b = 0; b < ns; ++b) { th[nr + b] = theta_s[b]; Cs[b] = (int32_t)(nr + b); }
    double *Pr = (double *)malloc(sizeof(double) * (size_t)(nr + 1)), *Ps = (double *)malloc(sizeof(double) * (size_t)(ns + 1));
    double *Q = (double *)malloc(sizeof(double) * (size_t)(nr + 1));
    Pr[0] = 0.0;
    for (int64_t a = 0; a < nr; ++a) Pr[a + 1] = Pr[a] + th[Cr[a]];
    Q[0] = 0.0;
    for (int64_t a = 0; a < nr; ++a) Q[a + 1] = Q[a] + th[Cr[a]] * (Pr[nr] - Pr[a + 1]);
    Ps[0] = 0.0;
    if (!diag) for (int64_t b = 0; b < ns; ++b) Ps[b + 1] = Ps[b] + th[Cs[b]];
    sbm_pair P;
    P.diag = diag; P.nr = nr; P.ns = diag ? nr : ns; P.Cr = Cr; P.Cs = diag ? Cr : Cs; P.th = th;
    P.Pr = Pr; P.Ps = diag ? Pr : Ps; P.Q = Q; P.omega = omega;
    double v = oracle_sbm_range_sum(&P, x, y);
    free(th); free(Cr); free(Cs); free(Pr); free(Ps); free(Q);
    return v;
}
