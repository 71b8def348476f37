// Microbenchmark: random-gather rate vs streaming on B200 (informs the state-layout choice).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_gather4(const float4* __restrict__ x, const int* __restrict__ idx, float4* __restrict__ out, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        out[i] = __ldg(x + idx[i]);
}
__global__ void k_gather1(const float* __restrict__ x, const int* __restrict__ idx, float* __restrict__ out, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        out[i] = __ldg(x + idx[i]);
}
__global__ void k_copy4(const float4* __restrict__ x, float4* __restrict__ out, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        out[i] = __ldg(x + i);
}
__global__ void k_fill_idx(int* idx, long n, long range, unsigned seed, int local) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
        if (local) idx[i] = (int)((i & ~(long)(local - 1)) + (h % local));  // random within a window
        else idx[i] = (int)(h % range);
    }
}
int main() {
    const long n = 1L << 28;
    float4 *x, *out; int* idx;
    cudaMalloc(&x, n * 16); cudaMalloc(&out, n * 16); cudaMalloc(&idx, n * 4);
    cudaMemset(x, 0, n * 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    int grid = 148 * 16, thr = 256;
    for (int local : {0, 1 << 20, 1 << 14, 4096, 64}) {
        k_fill_idx<<<grid, thr>>>(idx, n, n, 12345u, local);
        k_gather4<<<grid, thr>>>(x, idx, out, n);
        cudaEventRecord(a); k_gather4<<<grid, thr>>>(x, idx, out, n); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("gather float4 window=%ld: %.3f ms  %.3g gathers/s  useful %.0f GB/s\n", local ? (long)local : n, ms, n / (ms * 1e-3), n * (16.0 + 4 + 16) / (ms * 1e-3) / 1e9);
        k_gather1<<<grid, thr>>>((float*)x, idx, (float*)out, n);
        cudaEventRecord(a); k_gather1<<<grid, thr>>>((float*)x, idx, (float*)out, n); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("gather float1 window=%ld: %.3f ms  %.3g gathers/s\n", local ? (long)local : n, ms, n / (ms * 1e-3));
    }
    k_copy4<<<grid, thr>>>(x, out, n);
    cudaEventRecord(a); k_copy4<<<grid, thr>>>(x, out, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy float4: %.3f ms  %.0f GB/s (r+w)\n", ms, n * 32.0 / (ms * 1e-3) / 1e9);
    return 0;
}
