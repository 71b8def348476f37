// Philox4x32-10 throughput on B200: (A) __umulhi + mul, (B) 64-bit multiply (IMAD.WIDE),
// (C) B with the key schedule precomputed in kernel parameters (constant bank operands).
// Measured on B200 (round 1): A 4.72e11, B 4.73e11, C 4.94e11 Philox blocks/s for the whole
// GPU = ~75 cycles per warp-block per SM sub-partition (20 IMAD.WIDE on the FMA-heavy pipe
// at 4 cycles each).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_bench philox_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct KS { uint32_t k[20]; };

__device__ __forceinline__ uint4 phA(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ uint4 phB(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ uint4 phC(uint4 c, const KS& ks) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ ks.k[2 * r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ ks.k[2 * r + 1], (uint32_t)p0);
    }
    return c;
}

template <int V>
__global__ void bench(uint32_t k0, uint32_t k1, const __grid_constant__ KS ks, int iters, uint32_t* out) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        uint4 c = make_uint4(t, i, 3u << 24, 0u);
        uint4 r = V == 0 ? phA(c, k0, k1) : (V == 1 ? phB(c, k0, k1) : phC(c, ks));
        acc ^= r.x ^ r.y ^ r.z ^ r.w;
    }
    out[t] = acc;
}

int main() {
    const int blocks = 148 * 8, threads = 256, iters = 2048;
    uint32_t* out;
    cudaMalloc(&out, blocks * threads * 4);
    KS ks;
    uint32_t k0 = 12345, k1 = 678;
    for (int r = 0; r < 10; ++r) { ks.k[2 * r] = k0 + r * 0x9E3779B9u; ks.k[2 * r + 1] = k1 + r * 0xBB67AE85u; }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (v == 0) bench<0><<<blocks, threads>>>(k0, k1, ks, iters, out);
            if (v == 1) bench<1><<<blocks, threads>>>(k0, k1, ks, iters, out);
            if (v == 2) bench<2><<<blocks, threads>>>(k0, k1, ks, iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("variant %c: %.3f ms, %.3e Philox blocks/s\n", 'A' + v, ms, (double)blocks * threads * iters / (ms * 1e-3));
        }
    }
    return 0;
}
