/*
 * synth/dcsbm.c — seeded DC-SBM edge sampler (bench/test INPUT tooling; untimed).
 *
 * Holds none of the method's arithmetic: it only draws a degree-corrected SBM multigraph
 * (Def. 5: A_ij ~ Pois(theta_i theta_j Omega_{c_i c_j})) as a raw edge list, with
 * duplicates, both orientations and self-pairs left in, so that the CSR build of the method
 * (simple undirected graph) has real canonicalisation work to do.
 *
 * Sampling scheme: lambda_ij = theta_i theta_j [f_in d(c_i,c_j)/kappa_{c_i}
 * + (1-f_in)/2m]. Two independent Poisson pair processes:
 *   - within block r: Pois(f_in kappa_r / 2) ordered pairs, both endpoints ~ theta inside r;
 *   - global:         Pois((1-f_in) m) ordered pairs, both endpoints ~ theta over all nodes.
 * Counts are drawn by the Python caller (numpy) and passed in; this file draws the endpoints.
 * Endpoints are drawn as sorted uniforms (exponential spacings) merged against the theta prefix
 * sums (cache friendly), the second endpoint list is Fisher-Yates shuffled within its segment so
 * that the pairs are independent.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static void rng_seed(rng_t *r, uint64_t seed, uint64_t stream) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull ^ (stream + 0x632BE59BD9B4E019ull);
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t rng_next(rng_t *r) {
    uint64_t *s = r->s;
    uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return res;
}
/* uniform in (0,1] */
static inline double rng_u01(rng_t *r) { return ((rng_next(r) >> 11) + 1) * 0x1.0p-53; }

/* Draw `cnt` node indices in [lo, hi) with P(i) = w_i / W, returned in sorted order, using the
 * prefix sums cum (cum[i] = sum_{k<i} w_k over the global array). */
static void draw_sorted(rng_t *r, const double *cum, int64_t lo, int64_t hi, int64_t cnt, int32_t *out) {
    if (cnt <= 0) return;
    double base = cum[lo], W = cum[hi] - cum[lo];
    /* sorted uniforms via normalised exponential spacings */
    double total = 0.0;
    double *e = (double *)malloc(sizeof(double) * (size_t)(cnt + 1));
    for (int64_t k = 0; k <= cnt; ++k) { total += -log(rng_u01(r)); e[k] = total; }
    int64_t i = lo;
    for (int64_t k = 0; k < cnt; ++k) {
        double target = base + W * (e[k] / total);
        while (i < hi - 1 && cum[i + 1] <= target) ++i;
        out[k] = (int32_t)i;
    }
    free(e);
}

static void shuffle(rng_t *r, int32_t *a, int64_t n) {
    for (int64_t k = n - 1; k > 0; --k) {
        int64_t j = (int64_t)(rng_next(r) % (uint64_t)(k + 1));
        int32_t t = a[k]; a[k] = a[j]; a[j] = t;
    }
}

/*
 * theta_cum: prefix sums of theta in block-sorted node order, length n+1.
 * block_start: length nblocks+1 (node ranges per block, block-sorted order).
 * seg_count: number of pairs per segment; segments 0..nblocks-1 are the within-block processes,
 *            segments nblocks..nblocks+nglobal-1 are chunks of the global process.
 * seg_offset: output offset per segment (prefix sums of seg_count), length nseg+1.
 * perm: node relabelling (block-sorted id -> output id), length n.
 * src, dst: outputs, length seg_offset[nseg].
 */
int dcsbm_sample(int64_t n, const double *theta_cum, int64_t nblocks, const int64_t *block_start,
                 int64_t nglobal, const int64_t *seg_count, const int64_t *seg_offset,
                 const int32_t *perm, uint64_t seed, int32_t *src, int32_t *dst) {
    int64_t nseg = nblocks + nglobal;
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t s = 0; s < nseg; ++s) {
        rng_t r;
        rng_seed(&r, seed, (uint64_t)s);
        int64_t lo, hi;
        if (s < nblocks) { lo = block_start[s]; hi = block_start[s + 1]; }
        else { lo = 0; hi = n; }
        int64_t cnt = seg_count[s], off = seg_offset[s];
        if (cnt == 0 || hi <= lo) continue;
        draw_sorted(&r, theta_cum, lo, hi, cnt, src + off);
        draw_sorted(&r, theta_cum, lo, hi, cnt, dst + off);
        shuffle(&r, dst + off, cnt);
        for (int64_t k = 0; k < cnt; ++k) {
            int32_t a = perm[src[off + k]], b = perm[dst[off + k]];
            if (rng_next(&r) & 1) { int32_t t = a; a = b; b = t; }
            src[off + k] = a; dst[off + k] = b;
        }
    }
    return fail;
}
