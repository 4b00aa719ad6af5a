// Bit-exactness check of pairmath.cuh's call-free IEEE fast paths (div_rn_fast, rcp_rn_fast, sqrt_rn_fast)
// against the compiler's __fdiv_rn / __fsqrt_rn over random operands in the energy kernels'
// domain: r2 in [1e-6, 1e12] (sqrt and 1/sqrt), numerators |n| in [1e-30, 1e30] of either sign
// over divisors in [1, 1e12] (the fitted Ewald rationals' denominators are >= 1).
// Built and run by tests/test_ieee_fast.py: prints "mismatches <n> of <N>".
#include <cstdio>
#include <cstdint>

#include "pairmath.cuh"

__device__ __forceinline__ uint32_t hash(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ float loguni(uint32_t h, float lo_log2, float hi_log2)
{
    const float u = (h >> 8) * (1.0f / 16777216.0f);
    return exp2f(lo_log2 + u * (hi_log2 - lo_log2));
}

__global__ void k_check(uint64_t n, uint32_t seed, unsigned long long* bad)
{
    unsigned long long nb = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t h1 = hash((uint32_t)i * 2654435761u ^ seed), h2 = hash(h1 ^ 0x9e3779b9u);
        const float r2 = loguni(h1, -19.93f, 39.86f);          // 1e-6 .. 1e12
        const float b = loguni(h2, 0.0f, 39.86f);              // 1 .. 1e12
        float a = loguni(hash(h2), -99.6f, 99.6f);             // 1e-30 .. 1e30
        if (h1 & 1u) a = -a;
        const float s1 = nbx::sqrt_rn_fast(r2), s2 = __fsqrt_rn(r2);
        const float i1 = nbx::rcp_rn_fast(s1), i2 = __fdiv_rn(1.0f, s2);
        const float d1 = nbx::div_rn_fast(a, b), d2 = __fdiv_rn(a, b);
        nb += (__float_as_uint(s1) != __float_as_uint(s2)) + (__float_as_uint(i1) != __float_as_uint(i2)) +
              (__float_as_uint(d1) != __float_as_uint(d2));
    }
    atomicAdd(bad, nb);
}

int main(int argc, char** argv)
{
    const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (1ull << 28);
    unsigned long long* d = nullptr;
    cudaMalloc(&d, sizeof(*d));
    cudaMemset(d, 0, sizeof(*d));
    k_check<<<148 * 16, 256>>>(n, 12345u, d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("cuda error %s\n", cudaGetErrorString(e));
        return 2;
    }
    printf("mismatches %llu of %llu\n", h, 3ull * n);
    return h ? 1 : 0;
}
