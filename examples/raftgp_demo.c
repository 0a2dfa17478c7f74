/* raftgp_demo.c — the C-ABI used from plain C (no Python, no torch): build the CSR of a small graph from host
 * edge arrays, embed it with both feature operators (RaftGP-C: NCut, RaftGP-M: full modularity) and the
 * 2-layer untrained GCN, score a labelling, and print checksums. Built by __graft_entry__.build();
 * tests/test_gpu_c_api.py runs it and compares with the Python binding on the same inputs.
 *
 * usage: raftgp_demo [n] [seed]   (graph: ring i -- i+1 plus chords i -- (7 i + 3) mod n)
 *        raftgp_demo n seed rank world idfile   (row-partitioned: `world` processes, one per GPU; rank 0 writes the
 *        NCCL unique id to idfile, the others read it; each process prints the checksums of ITS rows of Z) */
#define _DEFAULT_SOURCE   /* usleep */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

#include "raftgp.h"

#define CHECK(call)                                                                                   \
    do {                                                                                              \
        raftgp_status st_ = (call);                                                                   \
        if (st_ != RAFTGP_OK) {                                                                       \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)st_, raftgp_last_error());           \
            return 1;                                                                                 \
        }                                                                                             \
    } while (0)

/* the row-partitioned step through raftgp_ctx_create_dist + raftgp_build_embed */
static int run_dist(int64_t n, uint64_t seed, int rank, int world, const char *idfile, const int32_t *src,
                    const int32_t *dst, int64_t m) {
    unsigned char id[128];
    if (rank == 0) {
        char tmp[4096];
        snprintf(tmp, sizeof tmp, "%s.tmp", idfile);
        CHECK(raftgp_nccl_unique_id(id));
        FILE *f = fopen(tmp, "wb");
        if (!f || fwrite(id, 1, 128, f) != 128) return 1;
        fclose(f);
        if (rename(tmp, idfile) != 0) return 1;
    } else {
        FILE *f = NULL;
        for (int t = 0; t < 6000 && !(f = fopen(idfile, "rb")); ++t) usleep(10000);
        if (!f || fread(id, 1, 128, f) != 128) return 1;
        fclose(f);
    }
    int ndev = 1;
    cudaGetDeviceCount(&ndev);
    raftgp_ctx ctx = NULL;
    CHECK(raftgp_ctx_create_dist(rank % ndev, NULL, rank, world, id, &ctx));
    const int64_t R = (n + world - 1) / world;
    const int64_t rb = rank * R < n ? rank * R : n, re = (rank + 1) * R < n ? (rank + 1) * R : n;
    const int32_t dims[3] = {64, 64, 32};
    const int32_t variants[2] = {RAFTGP_NCUT, RAFTGP_MOD};
    float *Zd[2] = {NULL, NULL};
    const size_t bytes = sizeof(float) * (size_t)(re - rb > 0 ? re - rb : 1) * dims[2];
    for (int v = 0; v < 2; ++v)
        if (cudaMalloc((void **)&Zd[v], bytes) != cudaSuccess) return 1;
    CHECK(raftgp_build_embed(ctx, n, m, src, dst, RAFTGP_HOST_PTRS, 2, variants, 2, dims, seed, Zd, NULL));
    CHECK(raftgp_ctx_sync(ctx));
    float *Z = (float *)malloc(bytes);
    printf("rank %d world %d rows %lld %lld\n", rank, world, (long long)rb, (long long)re);
    for (int v = 0; v < 2; ++v) {
        if (cudaMemcpy(Z, Zd[v], bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
        double sum = 0.0, sq = 0.0;
        for (int64_t i = 0; i < (re - rb) * dims[2]; ++i) {
            sum += Z[i];
            sq += (double)Z[i] * Z[i];
        }
        printf("%s sum %.9e sumsq %.9e z00 %.9e\n", v == 0 ? "ncut" : "mod", sum, sq, re > rb ? Z[0] : 0.0f);
        cudaFree(Zd[v]);
    }
    free(Z);
    CHECK(raftgp_ctx_destroy(ctx));   /* collective on a distributed context */
    return 0;
}

int main(int argc, char **argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000;
    const uint64_t seed = argc > 2 ? strtoull(argv[2], NULL, 10) : 1;
    const int64_t m = 2 * n;
    int32_t *src = (int32_t *)malloc(sizeof(int32_t) * m), *dst = (int32_t *)malloc(sizeof(int32_t) * m);
    for (int64_t i = 0; i < n; ++i) {
        src[2 * i] = (int32_t)i;
        dst[2 * i] = (int32_t)((i + 1) % n);
        src[2 * i + 1] = (int32_t)i;
        dst[2 * i + 1] = (int32_t)((7 * i + 3) % n);
    }
    if (argc > 5) {
        const int rc = run_dist(n, seed, atoi(argv[3]), atoi(argv[4]), argv[5], src, dst, m);
        free(src); free(dst);
        return rc;
    }
    raftgp_ctx ctx = NULL;
    raftgp_graph g = NULL;
    CHECK(raftgp_ctx_create(0, NULL, &ctx));
    CHECK(raftgp_build_csr(ctx, n, m, src, dst, 0, n, RAFTGP_HOST_PTRS, &g));
    int64_t gn = 0, rb = 0, re = 0, nnz = 0, two_e = 0;
    CHECK(raftgp_graph_info(g, &gn, &rb, &re, &nnz, &two_e));

    const int32_t dims[3] = {64, 64, 32};
    const int32_t variants[2] = {RAFTGP_NCUT, RAFTGP_MOD};
    float *Zd[2] = {NULL, NULL};
    for (int v = 0; v < 2; ++v)
        if (cudaMalloc((void **)&Zd[v], sizeof(float) * (size_t)n * dims[2]) != cudaSuccess) return 1;
    CHECK(raftgp_embed_multi(g, 2, variants, 2, dims, seed, NULL, Zd));
    CHECK(raftgp_ctx_sync(ctx));
    float *Z = (float *)malloc(sizeof(float) * (size_t)n * dims[2]);
    printf("n %lld nnz %lld two_e %lld\n", (long long)gn, (long long)nnz, (long long)two_e);
    for (int v = 0; v < 2; ++v) {
        if (cudaMemcpy(Z, Zd[v], sizeof(float) * (size_t)n * dims[2], cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
        double sum = 0.0, sq = 0.0, first = Z[0];
        for (int64_t i = 0; i < n * dims[2]; ++i) {
            sum += Z[i];
            sq += (double)Z[i] * Z[i];
        }
        printf("%s sum %.9e sumsq %.9e z00 %.9e\n", v == 0 ? "ncut" : "mod", sum, sq, first);
    }
    int32_t *lab = (int32_t *)malloc(sizeof(int32_t) * n);
    for (int64_t i = 0; i < n; ++i) lab[i] = (int32_t)((i * 4) / n);   /* 4 contiguous arcs of the ring */
    double q = 0.0, nc = 0.0;
    CHECK(raftgp_modularity(g, lab, 4, &q));
    CHECK(raftgp_ncut(g, lab, 4, &nc));
    printf("modularity %.12f ncut %.12f\n", q, nc);
    for (int v = 0; v < 2; ++v) cudaFree(Zd[v]);
    CHECK(raftgp_graph_destroy(g));
    CHECK(raftgp_ctx_destroy(ctx));
    free(src); free(dst); free(Z); free(lab);
    return 0;
}
