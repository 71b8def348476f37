// pf_multinomial.cu -- multinomial resampling over the whole population (Alg. 2,
// PAPER.md:309-319), the resampler of the plain BPF that the paper improves upon; here as
// the comparison baseline on the same weigh pass (k_pass1, kPass1Weigh).
//
//   k_mn_tile_cdf  one CTA per tile of kMnTile particles: tile max m_T, fp32 inclusive
//                  scan of e^{lw - m_T} (the tile's local CDF), tile record {m_T, total}
//   k_mn_offsets   one CTA: fp64 exclusive scan of the tile masses total_T e^{m_T - L}
//                  (L = max lw from the weigh pass) -> the tiles' offsets in the global CDF
//   k_mn_draw      thread per quad: u from the MULTI Philox block (reading R22), t = u C,
//                  bisection of the tile offsets, then of the tile's local CDF rescaled,
//                  a(i) = #{k < N-1 : C_k <= t}; gathers x_hat^i = x^{a(i)} (the one random
//                  HBM access of this algorithm)
#include "pf_launch.h"
#include "pf_kernels.cuh"

namespace pfk {

__device__ __forceinline__ float mn_float_from_order_bits(unsigned int u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void __launch_bounds__(kMnTile) k_mn_tile_cdf(const float* __restrict__ lw, float* __restrict__ cdf,
                                                        float* __restrict__ cdf32, double* __restrict__ trec,
                                                        uint64_t N) {
    __shared__ float red[32];
    const uint64_t i = (uint64_t)blockIdx.x * kMnTile + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const float v = i < N ? lw[i] : -CUDART_INF_F;
    float mx = v;
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    float m = red[lane];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();
    const bool dead = m == -CUDART_INF_F;  // no weight in the tile: its mass is 0
    float c = (i < N && !dead) ? expf(v - m) : 0.0f;
    for (int o = 1; o < 32; o <<= 1) {  // inclusive warp scan
        const float t = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= (uint32_t)o) c += t;
    }
    if (lane == 31) red[warp] = c;
    __syncthreads();
    if (warp == 0) {
        float w = red[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += t;
        }
        red[lane] = w;
    }
    __syncthreads();
    if (warp > 0) c += red[warp - 1];
    if (i < N) cdf[i] = c;
    if (lane == 31) cdf32[(uint64_t)blockIdx.x * (kMnTile / 32) + warp] = c;  // chunk ends (L2-resident)
    if (threadIdx.x == kMnTile - 1) {
        trec[2 * blockIdx.x] = dead ? -CUDART_INF : (double)m;
        trec[2 * blockIdx.x + 1] = (double)c;
    }
}

// offsets[T] = sum_{T' < T} total_T' e^{m_T' - L}, offsets[NT] = C (fixed order: thread t
// sums a contiguous run of tiles, then a block scan of the run totals)
__global__ void __launch_bounds__(1024) k_mn_offsets(const double* __restrict__ trec, double* __restrict__ off,
                                                     const unsigned int* __restrict__ lmax, uint32_t NT) {
    __shared__ double run[1024];
    const double L = (double)mn_float_from_order_bits(*lmax);
    const uint32_t per = (NT + blockDim.x - 1) / blockDim.x;
    const uint32_t t0 = threadIdx.x * per, t1 = min(NT, t0 + per);
    auto mass = [&](uint32_t T) {
        const double m = trec[2 * T];
        return m == -CUDART_INF ? 0.0 : trec[2 * T + 1] * exp(m - L);
    };
    double s = 0.0;
    for (uint32_t T = t0; T < t1; ++T) s += mass(T);
    run[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential exclusive scan of the 1024 run totals (fixed order)
        double acc = 0.0;
        for (uint32_t k = 0; k < blockDim.x; ++k) {
            const double r = run[k];
            run[k] = acc;
            acc += r;
        }
        off[NT] = acc;
    }
    __syncthreads();
    double acc = run[threadIdx.x];
    for (uint32_t T = t0; T < t1; ++T) {
        off[T] = acc;
        acc += mass(T);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_mn_draw(MultinomialArgs a) {
    const uint64_t nq = a.N >> 2;
    const double C = a.off[a.NT];
    const double L = (double)mn_float_from_order_bits(*a.lmax);
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 blk = rng_block(a.key, (uint32_t)q, a.n, kDomainMulti, 0u);
        const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
        uint64_t anc[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double t = (double)(r[e] >> 8) * 0x1p-24 * C;
            // tile: the last T with off[T] <= t (off[0] = 0)
            uint32_t lo = 0, hi = a.NT - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (__ldg(a.off + mid) <= t) lo = mid;
                else hi = mid - 1;
            }
            const double m = __ldg(a.trec + 2 * lo);
            const double tl = m == -CUDART_INF ? 0.0 : (t - __ldg(a.off + lo)) * exp(L - m);  // local CDF units
            const uint64_t base = (uint64_t)lo * kMnTile;
            const uint64_t rest = a.N - base;
            const uint32_t n_in = rest < kMnTile ? (uint32_t)rest : kMnTile;
            // count of local CDF values <= tl: first over the chunk ends (one cache line of
            // cdf32, L2-resident), then inside the chunk (one line of cdf)
            const uint32_t nch = (n_in + 31u) >> 5;
            uint32_t c0 = 0, c1 = nch;  // chunks whose end is <= tl (all of their values are)
            while (c0 < c1) {
                const uint32_t mid = (c0 + c1) >> 1;
                if ((double)__ldg(a.cdf32 + (uint64_t)lo * (kMnTile / 32) + mid) <= tl) c0 = mid + 1;
                else c1 = mid;
            }
            uint32_t k0 = c0 << 5, k1 = min(n_in, k0 + 32u);
            while (k0 < k1) {
                const uint32_t mid = (k0 + k1) >> 1;
                if ((double)__ldg(a.cdf + base + mid) <= tl) k0 = mid + 1;
                else k1 = mid;
            }
            uint64_t ai = base + k0;
            if (ai > a.N - 1) ai = a.N - 1;  // rounding at the very top (the count excludes k = N-1)
            anc[e] = ai;
            if (a.dbg_anc) a.dbg_anc[4 * q + e] = (int32_t)ai;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if constexpr (D == 1) {
                a.xhat[4 * q + e] = __ldg(a.x + anc[e]);
            } else if constexpr (D == 2) {
                reinterpret_cast<float2*>(a.xhat)[4 * q + e] = __ldg(reinterpret_cast<const float2*>(a.x) + anc[e]);
            } else {
#pragma unroll
                for (int c = 0; c < D / 4; ++c)
                    reinterpret_cast<float4*>(a.xhat)[(4 * q + e) * (D / 4) + c] =
                        __ldg(reinterpret_cast<const float4*>(a.x) + anc[e] * (D / 4) + c);
            }
        }
    }
}

void launch_multinomial(int D, cudaStream_t st, const MultinomialArgs& a, const float* lw) {
    k_mn_tile_cdf<<<a.NT, kMnTile, 0, st>>>(lw, a.cdf, a.cdf32, a.trec, a.N);
    k_mn_offsets<<<1, 1024, 0, st>>>(a.trec, a.off, a.lmax, a.NT);
    const uint32_t grid = (uint32_t)std::min<uint64_t>((a.N / 4 + 255) / 256, 148ull * 8);
    switch (D) {
        case 1: k_mn_draw<1><<<grid, 256, 0, st>>>(a); break;
        case 2: k_mn_draw<2><<<grid, 256, 0, st>>>(a); break;
        case 4: k_mn_draw<4><<<grid, 256, 0, st>>>(a); break;
        default: k_mn_draw<8><<<grid, 256, 0, st>>>(a); break;
    }
}

}  // namespace pfk
