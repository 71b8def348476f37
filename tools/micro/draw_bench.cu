// Micro-benchmark of the k_stages draw loop (Philox4x32-10 block + side/index logic + the
// 16-bit table store) on B200: cycles per warp-block for formulations of the side test.
//   P : Philox only (words XOR-accumulated)
//   D0: (r >> b) >= P, entry = (hi ? bhi : blo) | (r & mask)           (round-1 kernel)
//   D2: (r | mask) > T, T = P ? P 2^b - 1 : 0 (exact for P in [0, 2^(32-b)]),
//       entry = ((r & mask) | blo) + (hi ? bit 2^b : 0)
//   D3: D2 with the compare on the FMA pipe: hi = carry of (r | mask) + (2^32 - 1 - T)
//   D4: D2, two stages' Philox blocks interleaved (unroll 2)
//   D5: D0 with the shifted group bases pinned in registers (the compiler otherwise sinks
//       the shift below the select) and PRMT packing
//   D6: byte entries (side << 7 | index), PRMT packing
//   D7: 16-bit entries, side from the SIGN of (r >> b) - P (exact: both < 2^31), the sign
//       replicated over each halfword by PRMT's sign-extension, entries assembled by LOP3
//       two at a time
//   D8: byte entries with the same sign trick
//   D9: D7 with the sign extension done by inline-PTX prmt (CUDA's __byte_perm drops the
//       selector's sign-extension bit)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o draw_bench draw_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct KS {
    uint32_t k[20];
};

__device__ __forceinline__ uint4 philox(uint4 c, const KS& ks) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ ks.k[2 * r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ ks.k[2 * r + 1],
                       (uint32_t)p0);
    }
    return c;
}

constexpr int K = 6;
constexpr int P = 2048;  // tile positions per thread-quad layout (table bytes 6 x 4 KB)

template <int V>
__device__ __forceinline__ uint2 draw(const uint4 blk, uint32_t Praw, uint32_t j, uint32_t st, uint32_t b) {
    const uint32_t mask = (1u << b) - 1u, bit = 1u << st;
    const uint32_t rw[4] = {blk.x, blk.y, blk.z, blk.w};
    uint32_t en[4];
    if constexpr (V == 0) {
        const uint32_t blo = (j & ~bit) << b, bhi = (j | bit) << b;
#pragma unroll
        for (int e = 0; e < 4; ++e) en[e] = (((rw[e] >> b) >= Praw) ? bhi : blo) | (rw[e] & mask);
        return make_uint2(en[0] | (en[1] << 16), en[2] | (en[3] << 16));
    } else if constexpr (V == 5) {
        uint32_t blo = (j & ~bit) << b, bhi = (j | bit) << b;
        asm volatile("" : "+r"(blo), "+r"(bhi));
#pragma unroll
        for (int e = 0; e < 4; ++e) en[e] = (((rw[e] >> b) >= Praw) ? bhi : blo) | (rw[e] & mask);
        return make_uint2(__byte_perm(en[0], en[1], 0x5410u), __byte_perm(en[2], en[3], 0x5410u));
    } else if constexpr (V == 6) {
#pragma unroll
        for (int e = 0; e < 4; ++e) en[e] = (rw[e] & mask) | (((rw[e] >> b) >= Praw) ? 0x80u : 0u);
        const uint32_t w = __byte_perm(__byte_perm(en[0], en[1], 0x0040u), __byte_perm(en[2], en[3], 0x0040u), 0x5410u);
        return make_uint2(w, 0u);
    } else if constexpr (V == 7) {
        const uint32_t blo = (j & ~bit) << b, bitb = bit << b;
        const uint32_t blo2 = blo | (blo << 16), bitb2 = bitb | (bitb << 16), mask2 = mask | (mask << 16);
        int32_t dd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) dd[e] = (int32_t)(rw[e] >> b) - (int32_t)Praw;  // < 0: the lower side
        const uint32_t s01 = __byte_perm((uint32_t)dd[0], (uint32_t)dd[1], 0xFFBBu);  // 0xffff where lower
        const uint32_t s23 = __byte_perm((uint32_t)dd[2], (uint32_t)dd[3], 0xFFBBu);
        const uint32_t w01 = __byte_perm(rw[0], rw[1], 0x5410u), w23 = __byte_perm(rw[2], rw[3], 0x5410u);
        return make_uint2(((w01 & mask2) | blo2) | (~s01 & bitb2), ((w23 & mask2) | blo2) | (~s23 & bitb2));
    } else if constexpr (V == 9) {
        const uint32_t blo = (j & ~bit) << b, bitb = bit << b;
        const uint32_t blo2 = blo | (blo << 16), bitb2 = bitb | (bitb << 16), mask2 = mask | (mask << 16);
        uint32_t dd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) dd[e] = (uint32_t)((int32_t)(rw[e] >> b) - (int32_t)Praw);  // < 0: lower side
        uint32_t s01, s23;
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s01) : "r"(dd[0]), "r"(dd[1]));  // 0xffff where lower
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s23) : "r"(dd[2]), "r"(dd[3]));
        const uint32_t w01 = __byte_perm(rw[0], rw[1], 0x5410u), w23 = __byte_perm(rw[2], rw[3], 0x5410u);
        return make_uint2(((w01 & mask2) | blo2) | (~s01 & bitb2), ((w23 & mask2) | blo2) | (~s23 & bitb2));
    } else if constexpr (V == 8) {
        int32_t dd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) dd[e] = (int32_t)(rw[e] >> b) - (int32_t)Praw;
        const uint32_t sg = __byte_perm(__byte_perm((uint32_t)dd[0], (uint32_t)dd[1], 0x00FBu),
                                        __byte_perm((uint32_t)dd[2], (uint32_t)dd[3], 0x00FBu), 0x5410u);
        const uint32_t w = __byte_perm(__byte_perm(rw[0], rw[1], 0x0040u), __byte_perm(rw[2], rw[3], 0x0040u), 0x5410u);
        const uint32_t m4 = mask * 0x01010101u;
        return make_uint2((w & m4) | (~sg & ~m4), 0u);
    } else if constexpr (V == 2 || V == 4) {
        const uint32_t T = Praw ? (Praw << b) - 1u : 0u;
        const uint32_t blo = (j & ~bit) << b, bitb = bit << b;
#pragma unroll
        for (int e = 0; e < 4; ++e) en[e] = ((rw[e] & mask) | blo) + (((rw[e] | mask) > T) ? bitb : 0u);
        return make_uint2(__byte_perm(en[0], en[1], 0x5410u), __byte_perm(en[2], en[3], 0x5410u));
    } else {
        const uint32_t T = Praw ? (Praw << b) - 1u : 0u;
        const uint64_t C = (uint64_t)(0xffffffffu - T);
        const uint32_t blo = (j & ~bit) << b, bitb = bit << b;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t hi = (uint32_t)(((uint64_t)(rw[e] | mask) + C) >> 32);  // carry: (r | mask) > T
            en[e] = hi * bitb + ((rw[e] & mask) | blo);
        }
        return make_uint2(__byte_perm(en[0], en[1], 0x5410u), __byte_perm(en[2], en[3], 0x5410u));
    }
}

template <int V>
__global__ void __launch_bounds__(1024, 1) bench(const __grid_constant__ KS ks, int tiles, uint32_t b, uint32_t* out) {
    __shared__ __align__(16) uint16_t tab[K * P];
    __shared__ uint32_t ths[64];
    if (threadIdx.x < 64) ths[threadIdx.x] = (threadIdx.x * 0x9E3779B9u) >> (b + 1);
    __syncthreads();
    uint32_t acc = 0;
    const uint32_t q = threadIdx.x, l0 = (4 * q) % P, j = (4 * q) >> b;
    for (int t = 0; t < tiles; ++t) {
        const uint32_t c0 = (blockIdx.x * tiles + t) * 1024u + q;
        if constexpr (V == 1) {  // Philox only
#pragma unroll 1
            for (uint32_t st = 0; st < K; ++st) {
                const uint4 blk = philox(make_uint4(c0, 7u, (3u << 24) | (st + 2u), 0u), ks);
                acc ^= blk.x ^ blk.y ^ blk.z ^ blk.w;
            }
        } else if constexpr (V == 4) {
#pragma unroll 1
            for (uint32_t st = 0; st < K; st += 2) {
                const uint4 b0 = philox(make_uint4(c0, 7u, (3u << 24) | (st + 2u), 0u), ks);
                const uint4 b1 = philox(make_uint4(c0, 7u, (3u << 24) | (st + 3u), 0u), ks);
                *reinterpret_cast<uint2*>(tab + st * P + l0) = draw<V>(b0, ths[(j >> (st + 1)) & 63u], j, st, b);
                *reinterpret_cast<uint2*>(tab + (st + 1) * P + l0) = draw<V>(b1, ths[(j >> (st + 2)) & 63u], j, st + 1, b);
            }
        } else if constexpr (V == 6 || V == 8) {
#pragma unroll 1
            for (uint32_t st = 0; st < K; ++st) {
                const uint4 blk = philox(make_uint4(c0, 7u, (3u << 24) | (st + 2u), 0u), ks);
                reinterpret_cast<uint32_t*>(tab)[(st * P + l0) >> 2] = draw<V>(blk, ths[(j >> (st + 1)) & 63u], j, st, b).x;
            }
        } else {
#pragma unroll 1
            for (uint32_t st = 0; st < K; ++st) {
                const uint4 blk = philox(make_uint4(c0, 7u, (3u << 24) | (st + 2u), 0u), ks);
                *reinterpret_cast<uint2*>(tab + st * P + l0) = draw<V>(blk, ths[(j >> (st + 1)) & 63u], j, st, b);
            }
        }
        acc += tab[(t * 977u + q) % (K * P)];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// exactness of the sign trick against the plain rule, over random words and edge thresholds
__global__ void check(uint32_t b, uint32_t* bad) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t Ps[6] = {0u, 1u, (1u << (32 - b)) - 1u, 1u << (32 - b), 12345u << (20 - b), t >> b};
    for (int pi = 0; pi < 6; ++pi) {
        const uint32_t Pr = Ps[pi] > (1u << (32 - b)) ? (1u << (32 - b)) : Ps[pi];
        uint4 blk = make_uint4(t * 2654435761u, ~t * 40503u, t ^ 0xdeadbeefu, t | 0xffffff00u);
        if (t < 4) blk = make_uint4(0xffffffffu, 0u, (Pr << b) - 1u, Pr << b);
        const uint32_t j = t & 63u, st = t % 6u;
        const uint2 r0 = draw<0>(blk, Pr, j, st, b), r7 = draw<7>(blk, Pr, j, st, b);
        const uint2 r6 = draw<6>(blk, Pr, j, st, b), r8 = draw<8>(blk, Pr, j, st, b);
        const uint2 r9 = draw<9>(blk, Pr, j, st, b);
        if (r0.x != r7.x || r0.y != r7.y) atomicAdd(bad, 1u);
        if (r0.x != r9.x || r0.y != r9.y) atomicAdd(bad + 2, 1u);
        const uint32_t m4 = ((1u << b) - 1u) * 0x01010101u | 0x80808080u;
        if ((r6.x & m4) != (r8.x & m4)) atomicAdd(bad + 1, 1u);
    }
}

int main() {
    {
        uint32_t* bad;
        cudaMalloc(&bad, 12);
        cudaMemset(bad, 0, 12);
        for (uint32_t b = 1; b <= 7; ++b) check<<<256, 256>>>(b, bad);
        uint32_t hb[3];
        cudaMemcpy(hb, bad, 12, cudaMemcpyDeviceToHost);
        printf("sign-trick exactness: %u (16-bit) / %u (byte) / %u (16-bit, PTX prmt) mismatches\n", hb[0], hb[1], hb[2]);
    }
    const int blocks = 148, threads = 1024, tiles = 400;
    uint32_t* out;
    cudaMalloc(&out, blocks * threads * 4);
    KS ks;
    for (int r = 0; r < 10; ++r) {
        ks.k[2 * r] = 12345u + r * 0x9E3779B9u;
        ks.k[2 * r + 1] = 678u + r * 0xBB67AE85u;
    }
    cudaEvent_t a, e;
    cudaEventCreate(&a);
    cudaEventCreate(&e);
    const char* names[] = {"D0 shift-compare", "P  Philox only", "D2 (r|mask)>T", "D3 carry on FMA pipe",
                           "D4 D2 x2 interleaved", "D5 pinned bases+PRMT", "D6 byte entries", "D7 sign trick 16-bit",
                           "D8 sign trick bytes", "D9 sign trick 16-bit PTX"};
    for (int v = 0; v < 10; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            switch (v) {
                case 0: bench<0><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 1: bench<1><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 2: bench<2><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 3: bench<3><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 4: bench<4><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 5: bench<5><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 6: bench<6><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 7: bench<7><<<blocks, threads>>>(ks, tiles, 6, out); break;
                case 8: bench<8><<<blocks, threads>>>(ks, tiles, 6, out); break;
                default: bench<9><<<blocks, threads>>>(ks, tiles, 6, out); break;
            }
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms;
            cudaEventElapsedTime(&ms, a, e);
            const double blocks_total = (double)blocks * threads * tiles * K;
            if (rep == 2)
                printf("%-22s %.3f ms  %.3e blocks/s  (%.1f SM-cycles/warp-block at 1965 MHz per SMSP)\n", names[v], ms,
                       blocks_total / (ms * 1e-3), (ms * 1e-3) * 1.965e9 * 148 * 4 / (blocks_total / 32));
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(err));
    return 0;
}
