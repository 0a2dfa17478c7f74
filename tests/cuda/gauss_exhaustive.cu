// Exhaustive check of the branch-free generator steps (gauss.cuh) against the library's generic forms
// (__fdiv_rn / __fsqrt_rn / switch): every 24-bit u1 input of the radius and every 24-bit k2 of sincos2pi.
// Prints the mismatch counts; tests/test_gpu_gauss_exhaustive.py requires zeros.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2312_01560_b200/csrc/gauss.cuh"

__global__ void check(unsigned long long *bad) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;   // 0 .. 2^24 - 1
    const uint32_t xa = k << 8;
    const float r0 = raftgp::spec_radius<true>(xa), r1 = raftgp::spec_radius<false>(xa);
    const float u1 = __fmul_rn(static_cast<float>(k + 1u), 0x1p-24f);
    const float l0 = raftgp::spec_ln<true>(u1), l1 = raftgp::spec_ln<false>(u1);
    float c0, s0, c1, s1;
    raftgp::spec_sincos2pi<true>(k, c0, s0);
    raftgp::spec_sincos2pi<false>(k, c1, s1);
    if (__float_as_uint(r0) != __float_as_uint(r1)) atomicAdd(bad + 0, 1ull);
    if (__float_as_uint(l0) != __float_as_uint(l1)) atomicAdd(bad + 1, 1ull);
    if (__float_as_uint(c0) != __float_as_uint(c1) || __float_as_uint(s0) != __float_as_uint(s1)) atomicAdd(bad + 2, 1ull);
}

int main() {
    unsigned long long *bad, h[3];
    cudaMalloc(&bad, sizeof(h));
    cudaMemset(bad, 0, sizeof(h));
    check<<<(1u << 24) / 256, 256>>>(bad);
    cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    printf("radius %llu ln %llu sincos %llu %s\n", h[0], h[1], h[2], cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
