// Instantiations of k_init, k_cascade and the debug kernels.
#include <algorithm>

#include "pf_launch.h"
#include "pf_kernels.cuh"

namespace pfk {

// The ESS kernels (declarations and EssArgs in pf_kernels.cuh) live in this unit only.
__device__ __forceinline__ float float_from_order_bits(unsigned int u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void __launch_bounds__(kEssThreads) k_ess_chunks(const __grid_constant__ EssArgs a) {
    __shared__ double r1[kEssThreads], r2[kEssThreads];
    uint32_t c = blockIdx.x, s = 0, nc;
    for (;; ++s) {  // which level, which chunk of it
        nc = (ess_level_count(a, s) + kEssChunk - 1) / kEssChunk;
        if (c < nc) break;
        c -= nc;
    }
    const double L = (double)float_from_order_bits(*a.lmax);
    const uint32_t n = ess_level_count(a, s), j0 = c * kEssChunk, j1 = min(n, j0 + kEssChunk);
    double s1 = 0.0, s2 = 0.0;
    if (L != -CUDART_INF) {
        for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
            if (s == 0 && a.lv0) {  // AIRPF2: the island weights
                const double f = exp(a.lv0[j] - L);
                s1 += f;
                s2 += f * f;
            } else if (s == 0) {
                const double* t = a.ess_part + (uint64_t)j * 3;
                if (t[0] == -CUDART_INF) continue;
                const double f = exp(t[0] - L);
                s1 += t[1] * f;
                s2 += t[2] * f * f;
            } else {
                const double f = exp(a.logV[level_offset(a.m, (int)s) + j] - L);
                s1 += f;
                s2 += f * f;
            }
        }
    }
    r1[threadIdx.x] = s1;
    r2[threadIdx.x] = s2;
    __syncthreads();
    for (uint32_t h = blockDim.x / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            r1[threadIdx.x] += r1[threadIdx.x + h];
            r2[threadIdx.x] += r2[threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.chunks[2 * blockIdx.x] = r1[0];
        a.chunks[2 * blockIdx.x + 1] = r2[0];
    }
}

__global__ void k_ess_final(const __grid_constant__ EssArgs a) {
    // warp s sums level s's chunk partials: lane-strided in a fixed order, then a fixed
    // shuffle tree (deterministic)
    const uint32_t s = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    if (s <= a.S) {
        uint32_t c0 = 0;
        for (uint32_t t = 0; t < s; ++t) c0 += (ess_level_count(a, t) + kEssChunk - 1) / kEssChunk;
        const uint32_t nc = (ess_level_count(a, s) + kEssChunk - 1) / kEssChunk;
        double s1 = 0.0, s2 = 0.0;
        for (uint32_t c = lane; c < nc; c += 32u) {
            s1 += a.chunks[2 * (c0 + c)];
            s2 += a.chunks[2 * (c0 + c) + 1];
        }
        for (int o = 16; o > 0; o >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        const double units = s == 0 ? (a.lv0 ? (double)a.m : (double)a.N) : (double)(a.m >> s);
        if (lane == 0) a.out[s] = (s2 > 0.0) ? s1 * s1 / (units * s2) : 1.0;  // no weight at all: equal
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t ss = a.S;
        for (uint32_t t = 0; t < a.S; ++t)
            if (a.out[t] >= a.theta) {
                ss = t;
                break;
            }
        a.out[a.S + 1] = (double)ss;
        a.out[a.S + 2] = a.logV[level_offset(a.m, (int)a.S)];
        *a.lmax = 0u;
    }
}


// Side draws of the four islands of quad c4 at stage s: bit e set = island 4 c4 + e takes
// its partner's block (before Alg. 7's exchange rule).
__device__ __forceinline__ uint32_t island_takes(const IslandArgs& a, uint32_t c4, uint32_t s) {
    const uint4 blk = rng_block(a.key, (a.island0 >> 2) + c4, a.n, kDomainIsland, s);  // global island quad
    const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
    const uint32_t bit = 1u << (s - 1);
    uint32_t take = 0u;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t i = 4u * c4 + (uint32_t)e;
        if (i >= a.m) break;
        const uint32_t P = a.thr[level_offset(a.m, (int)s) + (i >> s)];
        const bool left = (r[e] >> 1) < P;   // the pair's lower island is chosen
        const bool i_is_left = (i & bit) == 0u;
        if (left != i_is_left) take |= 1u << e;
    }
    return take;
}

// Thread per pair of partner quads (stages s >= 3: quads c4 and c4 ^ 2^{s-3}, the same
// lane e holding partners) or per quad (s <= 2: the partner lies in the same quad): every
// Philox block is computed once and Alg. 7's rule sees both sides' draws.
__global__ void __launch_bounds__(256) k_island_draw(const __grid_constant__ IslandArgs a) {
    const uint32_t nq = (a.m + 3u) >> 2;
    const uint32_t np = nq >= 2u ? nq >> 1 : 1u;  // work items per stage (upper bound)
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= (uint64_t)nq * a.S) return;
    const uint32_t s = (uint32_t)(t / nq) + 1u, w = (uint32_t)(t % nq);
    const uint32_t bit = 1u << (s - 1);
    if (bit < 4u) {  // partners inside the quad
        const uint32_t c4 = w;
        uint32_t take = island_takes(a, c4, s);
        if (a.modified) {
            uint32_t keep = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t eh = (uint32_t)e ^ bit;
                if (((take >> e) & 1u) && ((take >> eh) & 1u)) keep |= 1u << e;
            }
            take &= ~keep;
        }
        a.choice[(uint64_t)(s - 1) * nq + c4] = (uint8_t)take;
        return;
    }
    if (w >= np) return;
    const uint32_t qb = bit >> 2;  // quad-index bit of the partner
    const uint32_t lo4 = ((w & ~(qb - 1u)) << 1) | (w & (qb - 1u));  // insert a 0 at bit log2(qb)
    const uint32_t hi4 = lo4 | qb;
    uint32_t tl = island_takes(a, lo4, s), th = island_takes(a, hi4, s);
    if (a.modified) {  // lane e of the low quad and lane e of the high quad are partners
        const uint32_t keep = tl & th;
        tl &= ~keep;
        th &= ~keep;
    }
    a.choice[(uint64_t)(s - 1) * nq + lo4] = (uint8_t)tl;
    a.choice[(uint64_t)(s - 1) * nq + hi4] = (uint8_t)th;
}

__global__ void __launch_bounds__(256) k_island_compose(const __grid_constant__ IslandArgs a) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.m) return;
    const uint32_t nq = (a.m + 3u) >> 2;
    uint32_t c = g;
    for (uint32_t s = a.S; s >= 1u; --s) {
        const uint32_t take = (__ldg(a.choice + (uint64_t)(s - 1) * nq + (c >> 2)) >> (c & 3u)) & 1u;
        c ^= take << (s - 1);
    }
    a.A[g] = (int32_t)(a.island0 + c);
}

void launch_island(cudaStream_t st, const IslandArgs& a) {
    const uint64_t work = (uint64_t)((a.m + 3u) >> 2) * a.S;
    if (work) k_island_draw<<<(uint32_t)((work + 255) / 256), 256, 0, st>>>(a);  // S* = 0 (AIRPF2): no stage
    k_island_compose<<<(a.m + 255) / 256, 256, 0, st>>>(a);
}

// Cross island stage (sharded AIRPF, R27): thread per quad of this shard's islands.
__global__ void __launch_bounds__(256) k_island_cross(const __grid_constant__ IslandCrossArgs a) {
    const uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x;
    if (4u * c4 >= a.m) return;
    const uint32_t P = __ldg(a.thr), bit = 1u << (a.s - 1);
    const uint32_t g0 = a.island0 + 4u * c4;                      // global islands g0..g0+3
    const uint4 bo = rng_block(a.key, g0 >> 2, a.n, kDomainIsland, a.s);
    const uint4 bp = rng_block(a.key, (g0 ^ bit) >> 2, a.n, kDomainIsland, a.s);  // the partners' quad
    const uint32_t ro[4] = {bo.x, bo.y, bo.z, bo.w}, rp[4] = {bp.x, bp.y, bp.z, bp.w};
    const bool own_low = (g0 & bit) == 0u;
    uint32_t take = 0u;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const bool to = ((ro[e] >> 1) < P) != own_low;   // island g0+e takes its partner's block
        const bool tp = ((rp[e] >> 1) < P) != !own_low;  // the partner takes g0+e's block
        if (to && !(a.modified && tp)) take |= 1u << e;  // Alg. 7: a pure exchange is undone
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if ((take >> e) & 1u) a.A[4u * c4 + e] = a.Apar[4u * c4 + e];
    if (a.choice) a.choice[c4] = (uint8_t)take;
}

void launch_island_cross(cudaStream_t st, const IslandCrossArgs& a) {
    k_island_cross<<<((a.m + 3u) / 4u + 255u) / 256u, 256, 0, st>>>(a);
}

// x_hat of a sharded AIRPF step for the debug interface: local block g = owner's block.
__global__ void k_block_gather_peer(const PeerArgs p, float* out, const int32_t* A, uint64_t N, uint32_t b, uint32_t D,
                                    uint32_t shift) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < N * D; f += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = f / D, k = f % D;
        const uint32_t gb = (uint32_t)A[i >> b];
        const uint64_t src = ((uint64_t)(gb & ((1u << shift) - 1u)) << b) | (i & ((1ull << b) - 1ull));
        out[f] = p.x[gb >> shift][src * D + k];
    }
}

void launch_block_gather_peer(cudaStream_t st, const PeerArgs& p, float* out, const int32_t* A, uint64_t N, uint32_t b,
                              uint32_t D, uint32_t shift) {
    k_block_gather_peer<<<1184, 256, 0, st>>>(p, out, A, N, b, D, shift);
}

// x_hat of an AIRPF step for the debug interface: out[g M + j] = in[A[g] M + j].
__global__ void k_block_gather(const float* in, float* out, const int32_t* A, uint64_t N, uint32_t b, uint32_t D) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < N * D; f += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = f / D, k = f % D;
        const uint64_t src = ((uint64_t)A[i >> b] << b) | (i & ((1ull << b) - 1ull));
        out[f] = in[src * D + k];
    }
}

void launch_block_gather(cudaStream_t st, const float* in, float* out, const int32_t* A, uint64_t N, uint32_t b,
                         uint32_t D) {
    k_block_gather<<<1184, 256, 0, st>>>(in, out, A, N, b, D);
}

// rows x cols doubles from a pitch-sp array to a pitch-dp array (pf_run_dev's estimate rows)
__global__ void k_rows_copy(const double* __restrict__ src, uint32_t sp, double* __restrict__ dst, uint32_t dp,
                            uint32_t rows) {
    const uint32_t i = threadIdx.x, r = i / dp, c = i % dp;
    if (r < rows) dst[r * dp + c] = src[r * sp + c];
}

void launch_rows_copy(cudaStream_t st, const double* src, uint32_t sp, double* dst, uint32_t dp, uint32_t rows) {
    k_rows_copy<<<1, rows * dp, 0, st>>>(src, sp, dst, dp, rows);
}

// ---- PF_EST_RESAMPLED: N^-1 sum_i phi(x_hat^i), phi in {x, x^2} ----------
// Computed on demand from the step's output buffer (through the island map of an AIRPF
// step, whose x_hat is never materialised).  Fixed grid, fixed order: thread partials in
// fp32 over a strided range, warp and CTA sums in fp64, then one CTA sums the CTA
// partials in index order -- deterministic.
constexpr uint32_t kMomGrid = 592, kMomThreads = 256;

template <int D>
__global__ void __launch_bounds__(kMomThreads) k_moments(const float* __restrict__ x, const int32_t* __restrict__ isl,
                                                         uint32_t b, uint64_t N, double* __restrict__ part) {
    __shared__ double red[kMomThreads / 32][2 * D];
    float s1[D], s2[D];
#pragma unroll
    for (int k = 0; k < D; ++k) s1[k] = s2[k] = 0.0f;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t src = i;
        if (isl) src = ((uint64_t)__ldg(isl + (i >> b)) << b) | (i & ((1ull << b) - 1ull));
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const float v = __ldg(x + src * D + k);
            s1[k] += v;
            s2[k] = fmaf(v, v, s2[k]);
        }
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        double a = s1[k], q = s2[k];
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            q += __shfl_xor_sync(0xffffffffu, q, o);
        }
        if (lane == 0) {
            red[warp][k] = a;
            red[warp][D + k] = q;
        }
    }
    __syncthreads();
    if (threadIdx.x < 2u * D) {
        double t = 0.0;
        for (uint32_t w = 0; w < kMomThreads / 32; ++w) t += red[w][threadIdx.x];
        part[(uint64_t)blockIdx.x * 2 * D + threadIdx.x] = t;
    }
}

template <int D>
__global__ void k_moments_final(const double* __restrict__ part, uint64_t N, double* __restrict__ out) {
    if (threadIdx.x < 2u * D) {
        double t = 0.0;
        for (uint32_t c = 0; c < kMomGrid; ++c) t += part[(uint64_t)c * 2 * D + threadIdx.x];
        out[threadIdx.x] = t / (double)N;
    }
}

void launch_moments(cudaStream_t st, int D, const float* x, const int32_t* isl, uint32_t b, uint64_t N, double* part,
                    double* out) {
    switch (D) {
        case 1: k_moments<1><<<kMomGrid, kMomThreads, 0, st>>>(x, isl, b, N, part);
                k_moments_final<1><<<1, 32, 0, st>>>(part, N, out); break;
        case 2: k_moments<2><<<kMomGrid, kMomThreads, 0, st>>>(x, isl, b, N, part);
                k_moments_final<2><<<1, 32, 0, st>>>(part, N, out); break;
        case 4: k_moments<4><<<kMomGrid, kMomThreads, 0, st>>>(x, isl, b, N, part);
                k_moments_final<4><<<1, 32, 0, st>>>(part, N, out); break;
        default: k_moments<8><<<kMomGrid, kMomThreads, 0, st>>>(x, isl, b, N, part);
                 k_moments_final<8><<<1, 32, 0, st>>>(part, N, out); break;
    }
}

// ---- pull exchange (PullArgs in pf_kernels.cuh) ---------------------------------------
// Requests per owner: a shared-memory histogram per CTA, one global atomic per bin per CTA
// (G <= 64 bins).
constexpr uint32_t kPullMaxG = 64;

// Stage-S_loc source (owner rank c, local position lc) of output l: the L cross-stage
// draws composed from the last stage back (counter-based, thresholds from pf_step_top).
// Cross stages t0 .. 1 from (rank c, local position lc) at stage S_loc + t0.
__device__ __forceinline__ void compose_cross_from(const PullArgs& a, uint32_t t0, uint32_t& c, uint32_t& lc) {
    for (uint32_t t = t0; t >= 1u; --t) {  // the stage S_loc + t draw at the current position
        const uint64_t gpos = (uint64_t)c * a.Nloc + lc;
        const uint4 blk = rng_block(a.key, (uint32_t)(gpos >> 2), a.n, kDomainResample, a.S_loc + t);
        const uint32_t r = word_of(blk, (int)(gpos & 3u));
        const uint32_t P = __ldg(a.top_thr + (a.G - (a.G >> (t - 1))) + (c >> t));
        const uint32_t bit = 1u << (t - 1);
        c = ((r >> a.b) < P) ? (c & ~bit) : (c | bit);
        lc = ((lc >> a.b) << a.b) | (r & (a.M - 1u));
    }
}

__device__ __forceinline__ void compose_cross(const PullArgs& a, uint64_t l, uint32_t& c, uint32_t& lc) {
    c = a.rank;
    lc = (uint32_t)l;
    for (uint32_t t = a.L; t >= 1u; --t) {  // the stage S_loc + t draw at the current position
        const uint64_t gpos = (uint64_t)c * a.Nloc + lc;
        const uint4 blk = rng_block(a.key, (uint32_t)(gpos >> 2), a.n, kDomainResample, a.S_loc + t);
        const uint32_t r = word_of(blk, (int)(gpos & 3u));
        const uint32_t P = __ldg(a.top_thr + (a.G - (a.G >> (t - 1))) + (c >> t));
        const uint32_t bit = 1u << (t - 1);
        c = ((r >> a.b) < P) ? (c & ~bit) : (c | bit);
        lc = ((lc >> a.b) << a.b) | (r & (a.M - 1u));
    }
}

__global__ void __launch_bounds__(256) k_pull_compose(const __grid_constant__ PullArgs a) {
    __shared__ unsigned int hist[kPullMaxG];
    for (uint32_t t = threadIdx.x; t < a.G; t += blockDim.x) hist[t] = 0u;
    __syncthreads();
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < a.Nloc;
         l += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c, lc;
        compose_cross(a, l, c, lc);
        a.src_local[l] = lc;
        a.src_rank[l] = c;
        atomicAdd(hist + c, 1u);
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < a.G; t += blockDim.x)
        if (hist[t]) atomicAdd(a.counts + t, (unsigned long long)hist[t]);
}

// Slots: per 256 outputs, warp ballots per owner give each request its rank inside the
// warp, a small scan over the warps its rank inside the CTA, and one global atomic per
// owner reserves the CTA's range (outputs keep their order inside a CTA chunk).
__global__ void __launch_bounds__(256) k_pull_pack(const __grid_constant__ PullArgs a) {
    __shared__ unsigned int wcnt[8][kPullMaxG];
    __shared__ unsigned int wbase[8][kPullMaxG];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < a.Nloc; base += stride) {
        const uint64_t l = base + threadIdx.x;
        const bool valid = l < a.Nloc;
        const uint32_t c = valid ? a.src_rank[l] : 0xffffffffu;
        uint32_t myrank = 0u;
        for (uint32_t bn = 0; bn < a.G; ++bn) {
            const unsigned int m = __ballot_sync(0xffffffffu, c == bn);
            if (c == bn) myrank = __popc(m & ((1u << lane) - 1u));
            if (lane == 0) wcnt[warp][bn] = __popc(m);
        }
        __syncthreads();
        for (uint32_t bn = threadIdx.x; bn < a.G; bn += blockDim.x) {
            unsigned int tot = 0u;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) tot += wcnt[w][bn];
            unsigned int off = tot ? atomicAdd(a.fill + bn, tot) : 0u;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
                wbase[w][bn] = off;
                off += wcnt[w][bn];
            }
        }
        __syncthreads();
        if (valid) {
            const uint64_t k = a.offsets[c] + wbase[warp][c] + myrank;
            a.req[k] = a.src_local[l];
            a.outpos[l] = (uint32_t)k;  // where output l's state will arrive
        }
        __syncthreads();
    }
}

// stage tables of the cross stages for the debug interface (every local position's draw)
__global__ void k_pull_debug_tables(const __grid_constant__ PullArgs a) {
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < a.Nloc;
         l += (uint64_t)gridDim.x * blockDim.x)
        for (uint32_t t = 1; t <= a.L; ++t) {
            const uint64_t gpos = (uint64_t)a.rank * a.Nloc + l;
            const uint4 blk = rng_block(a.key, (uint32_t)(gpos >> 2), a.n, kDomainResample, a.S_loc + t);
            const uint32_t r = word_of(blk, (int)(gpos & 3u));
            const uint32_t P = __ldg(a.top_thr + (a.G - (a.G >> (t - 1))) + (a.rank >> t));
            const uint32_t bit = 1u << (t - 1);
            const uint32_t c = ((r >> a.b) < P) ? (a.rank & ~bit) : (a.rank | bit);
            const uint64_t src = (uint64_t)c * a.Nloc + ((((uint32_t)l >> a.b) << a.b) | (r & (a.M - 1u)));
            a.dbg_anc[(uint64_t)(a.S_loc + t - 1) * a.Nloc + l] = (int32_t)src;
        }
}

template <int D>
__global__ void __launch_bounds__(256) k_pull_gather(const float* __restrict__ x, const uint32_t* __restrict__ idx,
                                                     float* __restrict__ out, uint64_t n) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = idx[k];
        if constexpr (D % 4 == 0) {
#pragma unroll
            for (int c = 0; c < D / 4; ++c)
                reinterpret_cast<float4*>(out)[k * (D / 4) + c] = __ldg(reinterpret_cast<const float4*>(x) + i * (D / 4) + c);
        } else {
#pragma unroll
            for (int c = 0; c < D; ++c) out[k * D + c] = __ldg(x + i * D + c);
        }
    }
}

// output l's state from the received buffer (x[l] = in[slot[l]]: the writes stream)
template <int D>
__global__ void __launch_bounds__(256) k_pull_scatter(const float* __restrict__ in, const uint32_t* __restrict__ slot,
                                                      float* __restrict__ x, uint64_t n) {
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n; l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = slot[l];
        if constexpr (D % 4 == 0) {
#pragma unroll
            for (int c = 0; c < D / 4; ++c)
                reinterpret_cast<float4*>(x)[l * (D / 4) + c] = __ldg(reinterpret_cast<const float4*>(in) + k * (D / 4) + c);
        } else {
#pragma unroll
            for (int c = 0; c < D; ++c) x[l * D + c] = __ldg(in + k * D + c);
        }
    }
}

// Peer-memory exchange: output l composes its source and reads the state straight from
// the owner's buffer (a peer pointer over NVLink, or a local one) — the compose and the
// transfer in one pass, no request/reply round.  Four outputs per thread: their loads
// are issued together so that four remote reads are in flight per thread.
template <int D>
__global__ void __launch_bounds__(256) k_peer_gather(const __grid_constant__ PullArgs a,
                                                     const __grid_constant__ PeerArgs p) {
    // one quad of consecutive outputs per thread: the last cross stage's draws of the four
    // are the four words of ONE Philox block (the draw contract keys them by the output
    // quad), so only the earlier cross stages, at the outputs' scattered positions, draw a
    // block per output (L - 1 + 1/4 blocks per output instead of L)
    const uint64_t nq = a.Nloc >> 2;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t l0 = 4u * q;
        uint32_t c[4], lc[4];
        {
            const uint32_t t = a.L;
            const uint64_t gpos = (uint64_t)a.rank * a.Nloc + l0;
            const uint4 blk = rng_block(a.key, (uint32_t)(gpos >> 2), a.n, kDomainResample, a.S_loc + t);
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
            const uint32_t P = __ldg(a.top_thr + (a.G - (a.G >> (t - 1))) + (a.rank >> t));
            const uint32_t bit = 1u << (t - 1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                c[e] = ((r[e] >> a.b) < P) ? (a.rank & ~bit) : (a.rank | bit);
                lc[e] = (((uint32_t)(l0 + e) >> a.b) << a.b) | (r[e] & (a.M - 1u));
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) compose_cross_from(a, a.L - 1u, c[e], lc[e]);
        if constexpr (D % 4 == 0) {
            float4 v[4][D / 4];  // (the four loads of a thread in flight together)
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int k = 0; k < D / 4; ++k) v[e][k] = __ldg(reinterpret_cast<const float4*>(p.x[c[e]] + (uint64_t)lc[e] * D) + k);
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int k = 0; k < D / 4; ++k) reinterpret_cast<float4*>(p.out)[(l0 + e) * (D / 4) + k] = v[e][k];
        } else {
            float v[4][D];
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int k = 0; k < D; ++k) v[e][k] = __ldg(p.x[c[e]] + (uint64_t)lc[e] * D + k);
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int k = 0; k < D; ++k) p.out[(l0 + e) * D + k] = v[e][k];
        }
    }
    // a shard of fewer than 4 or a non-multiple of 4 outputs (not produced by the plans; kept exact)
    for (uint64_t l = 4u * nq + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < a.Nloc; l += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c, lc;
        compose_cross(a, l, c, lc);
        for (int k = 0; k < D; ++k) p.out[l * D + k] = __ldg(p.x[c] + (uint64_t)lc * D + k);
    }
}

void launch_peer_gather(cudaStream_t st, int D, const PullArgs& a, const PeerArgs& p, bool debug) {
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((a.Nloc / 4 + 255) / 256, 148ull * 8));
    switch (D) {
        case 1: k_peer_gather<1><<<grid, 256, 0, st>>>(a, p); break;
        case 2: k_peer_gather<2><<<grid, 256, 0, st>>>(a, p); break;
        case 4: k_peer_gather<4><<<grid, 256, 0, st>>>(a, p); break;
        default: k_peer_gather<8><<<grid, 256, 0, st>>>(a, p); break;
    }
    if (debug) k_pull_debug_tables<<<grid, 256, 0, st>>>(a);
}

// PF_FLAG_GUARD: count the gap bytes that differ from the fill byte
__global__ void __launch_bounds__(256) k_guard_check(const unsigned char* __restrict__ p, size_t n, unsigned char fill,
                                                     unsigned long long* bad) {
    unsigned int c = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        c += p[i] != fill;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31u) == 0u && c) atomicAdd(bad, (unsigned long long)c);
}

void launch_guard_check(cudaStream_t st, const unsigned char* p, size_t n, unsigned char fill, unsigned long long* bad) {
    k_guard_check<<<(uint32_t)((n + 255) / 256), 256, 0, st>>>(p, n, fill, bad);
}

void launch_pull_compose(cudaStream_t st, const PullArgs& a, bool debug) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((a.Nloc + 255) / 256, 148ull * 8);
    k_pull_compose<<<grid, 256, 0, st>>>(a);
    if (debug) k_pull_debug_tables<<<grid, 256, 0, st>>>(a);
}

void launch_pull_pack(cudaStream_t st, const PullArgs& a) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((a.Nloc + 255) / 256, 148ull * 8);
    k_pull_pack<<<grid, 256, 0, st>>>(a);
}

void launch_pull_move(cudaStream_t st, int D, bool gather, const float* src, const uint32_t* idx, float* dst,
                      uint64_t n) {
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 8));
    if (gather) {
        switch (D) {
            case 1: k_pull_gather<1><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            case 2: k_pull_gather<2><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            case 4: k_pull_gather<4><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            default: k_pull_gather<8><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
        }
    } else {
        switch (D) {
            case 1: k_pull_scatter<1><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            case 2: k_pull_scatter<2><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            case 4: k_pull_scatter<4><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
            default: k_pull_scatter<8><<<grid, 256, 0, st>>>(src, idx, dst, n); break;
        }
    }
}

void launch_cascade(int D, const LaunchCfg& c, const CascadeArgs& a) {
    switch (D) {
        case 1: k_cascade<1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_cascade<2><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_cascade<4><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_cascade<8><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

void launch_ess(const LaunchCfg& chunks, const EssArgs& a) {
    k_ess_chunks<<<ess_chunks_total(a), kEssThreads, 0, chunks.stream>>>(a);
    k_ess_final<<<1, 32 * (a.S + 1), 0, chunks.stream>>>(a);
}

void launch_init(int D, int kind, const LaunchCfg& c, const InitArgs& a) {
    if (kind == 2) {
        k_init<1, 2><<<c.grid, c.threads, 0, c.stream>>>(a);
        return;
    }
    switch (D) {
        case 1: k_init<1, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_init<2, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_init<4, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_init<8, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

void launch_top(int D, const LaunchCfg& c, const TopArgs& a) {
    switch (D) {
        case 1: k_top<1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_top<2><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_top<4><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_top<8><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

template <typename T>
static void cross_t(bool dbg, const LaunchCfg& c, const CrossArgs& a) {
    if (dbg) k_cross<T, true><<<c.grid, c.threads, 0, c.stream>>>(a);
    else k_cross<T, false><<<c.grid, c.threads, 0, c.stream>>>(a);
}

void launch_cross(int payload, bool dbg, const LaunchCfg& c, const CrossArgs& a) {
    switch (payload) {
        case kPayloadF1: cross_t<float>(dbg, c, a); break;
        case kPayloadF2: cross_t<float2>(dbg, c, a); break;
        case kPayloadF4: cross_t<float4>(dbg, c, a); break;
        default: cross_t<State8>(dbg, c, a); break;
    }
}

void launch_debug_compose(const LaunchCfg& c, const int32_t* anc, uint64_t N, uint32_t S, int32_t* A) {
    k_debug_compose<0><<<c.grid, c.threads, 0, c.stream>>>(anc, N, S, A);
}

}  // namespace pfk
