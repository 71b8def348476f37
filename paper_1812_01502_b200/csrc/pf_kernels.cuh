// pf_kernels.cuh -- the kernels of one BPF time step with augmented resampling.
//
//   k_init      x_0^i ~ pi_0                                   (Alg. 1 l.1-3)
//   k_pass1     per tile of T1 = 2^k1 consecutive groups (P1 = T1 M particles):
//               [gather/load xhat] -> mutate (Alg. 1 l.303) -> log g_n
//               -> stage 1 (pairs (2p, 2p+1): warp-shuffle segmented max/scan +
//               branch-free binary search) -> V levels 1..k1 and stages 2..k1 inside the
//               tile (Alg. 3 l.346-349) -> the tile's particles written once, already
//               moved to their stage-k1 positions
//   k_cascade   V levels k1+1..S (log-domain pair means, eq. V_defn_proofs),
//               the stage side thresholds, and the fixed-tree combination of the
//               estimate partials (single launch, last-CTA-finishes pattern)
//   k_compose   stages s0..s0+k-1 for a tile of 2^k groups spaced 2^{s0-1} apart
//               (exactly the groups the butterfly pairs at those stages): composes the
//               ancestor maps in shared memory and moves a payload (an int32 ancestor
//               index, or the fp32 state itself for d <= 2) once per pass
//
// Draw contract: every resampling word is word (i & 3) of Philox block
// (i >> 2, n, RESAMPLE<<24 | s, 0); stage 1 u = (r>>8) 2^-24 with a = #{k < 2M-1 :
// C_k <= u C_{2M-1}}; stage s >= 2: side L iff (r >> b) < floor(p 2^{32-b}),
// index r & (M-1).  Noise: flat coordinate c = i d + k is normal (c & 3) of block
// (c >> 2, n, MUTATE<<24, 0).
//
// Thread layout: a CTA of `threads` threads owns nq = threads * QPT quads (4 consecutive
// tile positions); thread t handles quads t + it * threads, it < QPT, so every warp
// touches 32 consecutive quads (coalesced, and pair segments of <= 32 quads live in
// one warp).
#pragma once
#include <cstdint>

#include "pf_device.cuh"

namespace pfk {

constexpr int kCascadeThreads = 1024;
constexpr uint32_t FULL = 0xffffffffu;

__host__ __device__ inline uint64_t level_offset(uint64_t m, int s) { return m - (m >> (s - 1)); }

// -------------------------------------------------------------------------------------
// Per-particle state I/O (packed AoS: particle i occupies floats [i*D, i*D+D)).
template <int D>
__device__ __forceinline__ void load_particle(const float* __restrict__ x, uint32_t i, float* v) {
    if constexpr (D == 1) {
        v[0] = __ldg(x + i);
    } else if constexpr (D == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(x) + i);
        v[0] = t.x;
        v[1] = t.y;
    } else {
#pragma unroll
        for (int c = 0; c < D / 4; ++c) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(x + (uint64_t)i * D) + c);
            v[4 * c] = t.x;
            v[4 * c + 1] = t.y;
            v[4 * c + 2] = t.z;
            v[4 * c + 3] = t.w;
        }
    }
}

// Four consecutive particles i0..i0+3 (i0 % 4 == 0): 4*D contiguous floats.
template <int D>
__device__ __forceinline__ void load_quad(const float* __restrict__ x, uint64_t i0, float* v) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(x + i0 * D) + c);
        v[4 * c] = t.x;
        v[4 * c + 1] = t.y;
        v[4 * c + 2] = t.z;
        v[4 * c + 3] = t.w;
    }
}

template <int D>
__device__ __forceinline__ void store_quad(float* __restrict__ x, uint64_t i0, const float* v) {
#pragma unroll
    for (int c = 0; c < D; ++c)
        reinterpret_cast<float4*>(x + i0 * D)[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

// -------------------------------------------------------------------------------------
struct InitArgs {
    ModelParams mp;
    Key key;
    uint64_t N;     // particles of this shard
    uint32_t pos0;  // global index of its first particle (multiple of 4)
    float* x;
};

template <int D, int KIND>
__global__ void __launch_bounds__(256) k_init(const __grid_constant__ InitArgs a) {
    const uint64_t nq = a.N >> 2;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        float z[4 * D], v[4 * D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint4 blk = rng_block(a.key, (uint32_t)(((a.pos0 >> 2) + q) * D + j), 0u, kDomainInit, 0u);
            normals4(blk, z + 4 * j);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) init_state<D, KIND>(a.mp, z + e * D, v + e * D);
        store_quad<D>(a.x, q * 4, v);
    }
}

// -------------------------------------------------------------------------------------
// Butterfly stages s >= 2 on a tile held as uint16 pointer arrays in shared memory.
//
// The tile's group j is global group gof(j) = tlo | (j << lowbits) | thi; stage
// s = s0 + st pairs j with j ^ (1 << st).  thr_s points at the tile's thresholds of
// that stage (entry j >> (st+1)).  Lo -> Ln: Ln[l] = Lo[a_s(l)] (forward composition).
struct TileGeom {
    uint32_t tlo, thi, lowbits, b, M;
    __device__ __forceinline__ uint32_t gof(uint32_t j) const { return tlo | (j << lowbits) | thi; }
    __device__ __forceinline__ uint32_t gpos(uint32_t l) const { return (gof(l >> b) << b) | (l & (M - 1)); }
};

template <bool DBG, int QPT>
__device__ __forceinline__ void tile_stage(const Key key, uint32_t n, uint32_t s, uint32_t st, const TileGeom& G,
                                           const uint32_t* __restrict__ thr_s, const uint16_t* Lo, uint16_t* Ln,
                                           uint32_t nq, int32_t* __restrict__ dbg_s, uint32_t pos0) {
    const uint32_t b = G.b, mask = G.M - 1u, bit = 1u << st;
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        uint32_t res[4];
        if (G.M >= 4u) {
            const uint32_t j = l0 >> b;
            const uint32_t g = G.gof(j);
            const uint32_t c0 = (pos0 + ((g << b) | (l0 & mask))) >> 2;
            const uint4 blk = rng_block(key, c0, n, kDomainResample, s);
            const uint32_t P = thr_s[j >> (st + 1)];
            const uint32_t bl = (j & ~bit) << b, br = (j | bit) << b;
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) res[e] = (((r[e] >> b) < P) ? bl : br) | (r[e] & mask);
        } else {  // M == 2: the quad spans groups j, j+1 (possibly two global Philox quads)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t l = l0 + e;
                const uint32_t j = l >> 1;
                const uint32_t gi = pos0 + ((G.gof(j) << 1) | (l & 1u));
                const uint4 blk = rng_block(key, gi >> 2, n, kDomainResample, s);
                const uint32_t r = word_of(blk, (int)(gi & 3u));
                const uint32_t P = thr_s[j >> (st + 1)];
                const uint32_t jj = ((r >> 1) < P) ? (j & ~bit) : (j | bit);
                res[e] = (jj << 1) | (r & 1u);
            }
        }
        const uint16_t v0 = Lo[res[0]], v1 = Lo[res[1]], v2 = Lo[res[2]], v3 = Lo[res[3]];
        *reinterpret_cast<uint2*>(Ln + l0) = make_uint2((uint32_t)v0 | ((uint32_t)v1 << 16), (uint32_t)v2 | ((uint32_t)v3 << 16));
        if constexpr (DBG) {
#pragma unroll
            for (int e = 0; e < 4; ++e) dbg_s[G.gpos(l0 + e)] = (int32_t)(pos0 + G.gpos(res[e]));
        }
    }
}

// -------------------------------------------------------------------------------------
// Shared-memory carve-up of k_pass1 (host and device agree through this function).
struct Pass1Smem {
    uint32_t xs, w, L1, tab, chunk, pm, ct, lv, th, red, wred, total;
};
__host__ __device__ inline Pass1Smem pass1_smem(int D, uint32_t P1, uint32_t M, uint32_t k1, uint32_t threads) {
    Pass1Smem s;
    uint32_t off = 0;
    auto take = [&](uint32_t bytes) {
        const uint32_t o = off;
        off += (bytes + 15u) & ~15u;
        return o;
    };
    const uint32_t T1 = P1 / M;
    s.xs = take(P1 * 4u * (uint32_t)D);
    s.w = take(P1 * 4u);
    s.L1 = take(P1 * 2u);                               // stage-1 ancestors (tile-local)
    s.tab = take(k1 >= 2 ? (k1 - 1u) * P1 * 2u : 0u);  // stage 2..k1 ancestor tables
    s.chunk = take(M > 64 ? (P1 / 128u) * 4u : 0u);     // per-warp-chunk totals (pairs > 32 quads)
    s.pm = take((T1 / 2) * 4u);
    s.ct = take((T1 / 2) * 4u);
    s.lv = take(T1 * 8u);
    s.th = take(T1 * 4u);
    s.red = take((threads / 32u) * (2u + 4u * (uint32_t)D) * 4u);
    s.wred = take((threads / 32u) * (2u + 4u * (uint32_t)D) * 33u * 4u);
    s.total = off;
    return s;
}

struct Pass1Args {
    ModelParams mp;
    Key key;
    uint32_t n;
    int do_mutate;
    const float* y_dev;  // if non-null, y is read from device memory
    float y[8];
    uint64_t N;           // particles of this shard
    uint32_t pos0;        // global index of the shard's first particle (RNG counters)
    uint32_t m, M, b, S, k1, P1, T1;
    Pass1Smem sl;         // shared-memory layout (pass1_smem)
    const float* x_in;    // xhat_{n-1} source (or x_0)
    const int32_t* A_in;  // gather map into x_in (GATHER only)
    float* x_out;         // particles moved to their stage-k1 positions
    double* logV;         // level table (m - 1)
    uint32_t* thr;        // threshold table (m - 1)
    double* part;         // per-tile estimate partials, (2 + 4D) doubles each
    float* dbg_x;
    float* dbg_lw;
    int32_t* dbg_anc;
};

// One CTA per tile of T1 = 2^k1 consecutive groups.  Barriers: B (stage-1 tables and
// per-warp partials complete), C (V levels / thresholds ready), D (stage tables ready).
template <int D, int KIND, bool GATHER, bool DBG, int QPT>
__global__ void __launch_bounds__(1024) k_pass1(const __grid_constant__ Pass1Args a) {
    constexpr int PS = 2 + 4 * D;  // partial: max, sw, s1[D], s2[D], p1[D], p2[D]
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t threads = blockDim.x;
    const Pass1Smem& SL = a.sl;
    float* xs = reinterpret_cast<float*>(smem + SL.xs);
    float* w = reinterpret_cast<float*>(smem + SL.w);
    uint16_t* L1 = reinterpret_cast<uint16_t*>(smem + SL.L1);
    uint16_t* tab = reinterpret_cast<uint16_t*>(smem + SL.tab);
    float* chunk = reinterpret_cast<float*>(smem + SL.chunk);
    float* pmax = reinterpret_cast<float*>(smem + SL.pm);
    float* ctot = reinterpret_cast<float*>(smem + SL.ct);
    double* lv = reinterpret_cast<double*>(smem + SL.lv);
    uint32_t* th = reinterpret_cast<uint32_t*>(smem + SL.th);
    float* red = reinterpret_cast<float*>(smem + SL.red);
    float* wred = reinterpret_cast<float*>(smem + SL.wred);

    const uint32_t P1 = a.P1, M = a.M, b = a.b, nq = P1 >> 2;
    const uint32_t T1 = a.T1;  // groups per tile
    const uint32_t tile = blockIdx.x;
    const uint32_t base = tile * P1;  // N < 2^31
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nwarps = threads >> 5;
    const uint32_t Z = M >> 1;  // quads per stage-1 pair (2M positions)

    float y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = a.y_dev ? (k < a.mp.dy ? __ldg(a.y_dev + k) : 0.0f) : a.y[k];

    // ---- 1. load / gather xhat_{n-1} (all slots first: independent loads in flight) ----
    float xh[QPT][4 * D];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) {  // tiny tiles only (P1 < 128)
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) xh[it][k] = 0.0f;
            continue;
        }
        const uint32_t i0 = base + 4u * q;
        if constexpr (GATHER) {
            const int4 src = __ldg(reinterpret_cast<const int4*>(a.A_in + i0));
            load_particle<D>(a.x_in, (uint32_t)src.x, xh[it]);
            load_particle<D>(a.x_in, (uint32_t)src.y, xh[it] + D);
            load_particle<D>(a.x_in, (uint32_t)src.z, xh[it] + 2 * D);
            load_particle<D>(a.x_in, (uint32_t)src.w, xh[it] + 3 * D);
        } else {
            load_quad<D>(a.x_in, i0, xh[it]);
        }
    }

    // ---- 2. mutate, weight; estimate partial accumulated online (running max) --------
    float lw[QPT][4];
    // states stay in registers for the estimate when small, else they are re-read from xs
    constexpr bool KEEPX = 4 * D * QPT <= 32;
    float xr[KEEPX ? QPT : 1][KEEPX ? 4 * D : 1];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        const bool valid = q < nq;
        const uint32_t i0 = base + 4u * q;
        float x[4 * D];
        if (a.do_mutate) {
            float z[4 * D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 blk = rng_block(a.key, ((a.pos0 + i0) >> 2) * D + j, a.n, kDomainMutate, 0u);
                normals4(blk, z + 4 * j);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) mutate<D, KIND>(a.mp, xh[it] + e * D, z + e * D, x + e * D);
        } else {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) x[k] = xh[it][k];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) lw[it][e] = valid ? log_potential<D, KIND>(a.mp, y, x + e * D) : -CUDART_INF_F;
        if constexpr (KEEPX) {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) xr[it][k] = valid ? x[k] : 0.0f;
        }
        if (!valid) continue;
#pragma unroll
        for (int c = 0; c < D; ++c)
            reinterpret_cast<float4*>(xs)[q * D + c] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        if constexpr (DBG) {
            store_quad<D>(a.dbg_x, i0, x);
            reinterpret_cast<float4*>(a.dbg_lw + i0)[0] = make_float4(lw[it][0], lw[it][1], lw[it][2], lw[it][3]);
        }
    }

    // ---- 3. stage 1: pair max, weights, segmented scan, inverse-CDF draws --------------
    const uint32_t zw = Z < 32u ? Z : 32u;
    float pm[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        float v = fmaxf(fmaxf(lw[it][0], lw[it][1]), fmaxf(lw[it][2], lw[it][3]));
        for (uint32_t o = 1; o < zw; o <<= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
        pm[it] = v;
    }
    if (Z > 32u) {  // pair spans several warp-chunks of 32 quads
#pragma unroll
        for (int it = 0; it < QPT; ++it)
            if (lane == 0 && tid + it * threads < nq) chunk[(tid + it * threads) >> 5] = pm[it];
        __syncthreads();
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t c0 = ((tid + it * threads) >> 5) & ~((Z >> 5) - 1u);
            float v = -CUDART_INF_F;
            for (uint32_t c = lane; c < (Z >> 5); c += 32u) v = fmaxf(v, chunk[c0 + c]);
            for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
            pm[it] = v;
        }
        __syncthreads();
    }
    // stage-1 weights c = exp(lw - pair max); they also weight the estimate partial,
    // rescaled to the thread's largest pair max (one exp per slot)
    float mthr = -CUDART_INF_F;
#pragma unroll
    for (int it = 0; it < QPT; ++it)
        if (tid + it * threads < nq) mthr = fmaxf(mthr, pm[it]);
    float acc[PS];
#pragma unroll
    for (int k = 0; k < PS; ++k) acc[k] = 0.0f;
    float run[QPT][4], incl[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        const bool valid = q < nq;
        const bool dead = pm[it] == -CUDART_INF_F;  // all of the pair's weights are zero
        const float f = (dead || !valid) ? 0.0f : (QPT == 1 ? 1.0f : expf(pm[it] - mthr));
        float r = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float c = dead ? 1.0f : expf(lw[it][e] - pm[it]);
            r += c;
            run[it][e] = r;
            const float wf = c * f;
            acc[1] += wf;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                float xv;
                if constexpr (KEEPX) xv = xr[it][e * D + k];
                else xv = valid ? xs[(4 * q + e) * D + k] : 0.0f;
                acc[2 + k] = fmaf(wf, xv, acc[2 + k]);
                acc[2 + D + k] = fmaf(wf * xv, xv, acc[2 + D + k]);
                acc[2 + 2 * D + k] += xv;
                acc[2 + 3 * D + k] = fmaf(xv, xv, acc[2 + 3 * D + k]);
            }
        }
        float v = r;  // inclusive scan of quad totals within the segment (<= 32 quads)
        for (uint32_t o = 1; o < zw; o <<= 1) {
            const float t = __shfl_up_sync(FULL, v, o, zw);
            if ((lane & (zw - 1u)) >= o) v += t;
        }
        incl[it] = v;
    }
    float excl[QPT], tot[QPT];
    if (Z <= 32u) {
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const float up = __shfl_up_sync(FULL, incl[it], 1, Z);
            excl[it] = (lane & (Z - 1u)) ? up : 0.0f;
            tot[it] = __shfl_sync(FULL, incl[it], lane | (Z - 1u));
        }
    } else {
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const float up = __shfl_up_sync(FULL, incl[it], 1);
            excl[it] = lane ? up : 0.0f;
            if (lane == 31 && tid + it * threads < nq) chunk[(tid + it * threads) >> 5] = incl[it];
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t cq = (tid + it * threads) >> 5;
            const uint32_t c0 = cq & ~((Z >> 5) - 1u);
            float before = 0.0f, all = 0.0f;
            for (uint32_t c = lane; c < (Z >> 5); c += 32u) {
                const float t = chunk[c0 + c];
                all += t;
                if (c0 + c < cq) before += t;
            }
            for (int o = 16; o > 0; o >>= 1) {
                before += __shfl_xor_sync(FULL, before, o);
                all += __shfl_xor_sync(FULL, all, o);
            }
            excl[it] += before;
            tot[it] = all;
        }
    }
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) continue;
        reinterpret_cast<float4*>(w)[q] =
            make_float4(excl[it] + run[it][0], excl[it] + run[it][1], excl[it] + run[it][2], excl[it] + run[it][3]);
        if (((4u * q) & (2u * M - 1u)) == 0u) {  // first quad of its pair
            const uint32_t p = (4u * q) >> (b + 1);
            pmax[p] = pm[it];
            ctot[p] = tot[it];
        }
    }
    if (Z <= 32u) __syncwarp();  // a pair's CDF was written by this warp
    else __syncthreads();
    {   // all QPT x 4 branch-free binary searches advance together (independent smem loads)
        uint32_t lo[QPT][4];
        float tq[QPT][4];
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * threads;
            const bool valid = q < nq;
            const uint4 blk = rng_block(a.key, ((a.pos0 + base) >> 2) + q, a.n, kDomainResample, 1u);
            const uint32_t pb = valid ? (((4u * q) >> (b + 1)) << (b + 1)) : 0u;
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                lo[it][e] = pb;
                tq[it][e] = valid ? u01f(r[e]) * tot[it] : -1.0f;
            }
        }
        for (uint32_t step = M; step >= 1u; step >>= 1) {
#pragma unroll
            for (int it = 0; it < QPT; ++it)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (w[lo[it][e] + step - 1u] <= tq[it][e]) lo[it][e] += step;
        }
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * threads;
            if (q >= nq) continue;
            if constexpr (DBG)
                reinterpret_cast<int4*>(a.dbg_anc + base + 4u * q)[0] =
                    make_int4((int)(a.pos0 + base + lo[it][0]), (int)(a.pos0 + base + lo[it][1]),
                              (int)(a.pos0 + base + lo[it][2]), (int)(a.pos0 + base + lo[it][3]));
            *reinterpret_cast<uint2*>(L1 + 4u * q) =
                make_uint2(lo[it][0] | (lo[it][1] << 16), lo[it][2] | (lo[it][3] << 16));
        }
    }

    // per-warp estimate partial: rescale to the warp max, then a transposed sum through
    // shared memory (row k of 33 floats per warp: conflict-free), lane k-1 sums row k
    {
        float wmax = mthr;
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(FULL, wmax, o));
        const float f = (mthr == -CUDART_INF_F) ? 0.0f : expf(mthr - wmax);
        float* W = wred + warp * (PS * 33);
#pragma unroll
        for (int k = 1; k < PS; ++k) W[k * 33 + lane] = (k < 2 + 2 * D) ? acc[k] * f : acc[k];
        __syncwarp();
        for (uint32_t k = lane + 1; k < (uint32_t)PS; k += 32u) {  // PS - 1 can exceed 32 (d = 8)
            const float* row = W + k * 33;
            float sacc = 0.0f;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) sacc += row[j];
            red[warp * PS + k] = sacc;
        }
        if (lane == 0) red[warp * PS] = wmax;
    }
    __syncthreads();  // B: pmax, ctot, red, L1 complete

    // warp 0: tile estimate partial, V levels 1..k1, thresholds (stage s uses level s-1)
    if (warp == 0) {
        {
            float tmax = -CUDART_INF_F;
            for (uint32_t wv = 0; wv < nwarps; ++wv) tmax = fmaxf(tmax, red[wv * PS]);
            for (uint32_t k = lane; k < (uint32_t)PS; k += 32u) {  // PS can exceed 32 (d = 8)
                double v;
                if (k == 0) {
                    v = (double)tmax;
                } else {
                    v = 0.0;
                    for (uint32_t wv = 0; wv < nwarps; ++wv) {
                        const float wm = red[wv * PS];
                        const float f = (k < (uint32_t)(2 + 2 * D)) ? (wm == -CUDART_INF_F ? 0.0f : expf(wm - tmax)) : 1.0f;
                        v += (double)(red[wv * PS + k] * f);
                    }
                }
                a.part[(uint64_t)tile * PS + k] = v;
            }
        }
        const float log2M = logf((float)(2u * M));
        for (uint32_t p = lane; p < T1 / 2; p += 32u) {
            const float pmv = pmax[p];
            const double v = (pmv == -CUDART_INF_F) ? -CUDART_INF : (double)pmv + (double)(logf(ctot[p]) - log2M);
            lv[p] = v;  // tile-local level s at offset T1 - (T1 >> (s-1))
            a.logV[level_offset(a.m, 1) + (uint64_t)tile * (T1 / 2) + p] = v;
        }
        __syncwarp();
        for (uint32_t s = 2; s <= a.k1; ++s) {
            const uint32_t cnt = T1 >> s;
            const uint32_t po = T1 - (T1 >> (s - 2)), co = T1 - (T1 >> (s - 1));
            for (uint32_t bk = lane; bk < cnt; bk += 32u) {
                const double vl = lv[po + 2 * bk], vr = lv[po + 2 * bk + 1];
                const double v = log_pair_mean_fast(vl, vr);
                const uint32_t P = side_threshold_fast(vl, vr, (int)b);
                lv[co + bk] = v;
                th[co + bk] = P;
                a.logV[level_offset(a.m, (int)s) + (uint64_t)tile * cnt + bk] = v;
                a.thr[level_offset(a.m, (int)s) + (uint64_t)tile * cnt + bk] = P;
            }
            __syncwarp();
        }
    }
    if (a.k1 >= 2) {
        __syncthreads();  // C: thresholds ready
        // ---- 4. stages 2..k1: every stage's draws are independent of the others (they
        // depend only on the thresholds), so all tables are filled in one phase ---------
        const uint32_t mask = M - 1u;
        for (uint32_t s = 2; s <= a.k1; ++s) {
            const uint32_t bit = 1u << (s - 1);
            const uint32_t* ths = th + (T1 - (T1 >> (s - 1)));
            uint16_t* Ts = tab + (s - 2) * P1;
#pragma unroll
            for (int it = 0; it < QPT; ++it) {
                const uint32_t q = tid + it * threads;
                if (q >= nq) continue;
                const uint32_t l0 = 4u * q;
                const uint4 blk = rng_block(a.key, ((a.pos0 + base) >> 2) + q, a.n, kDomainResample, s);
                const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
                uint32_t res[4];
                if (M >= 4u) {
                    const uint32_t j = l0 >> b;
                    const uint32_t P = ths[j >> s];
                    const uint32_t bl = (j & ~bit) << b, br = (j | bit) << b;
#pragma unroll
                    for (int e = 0; e < 4; ++e) res[e] = (((r[e] >> b) < P) ? bl : br) | (r[e] & mask);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t j = (l0 + e) >> b;
                        const uint32_t jj = ((r[e] >> b) < ths[j >> s]) ? (j & ~bit) : (j | bit);
                        res[e] = (jj << b) | (r[e] & mask);
                    }
                }
                *reinterpret_cast<uint2*>(Ts + l0) = make_uint2(res[0] | (res[1] << 16), res[2] | (res[3] << 16));
                if constexpr (DBG)
                    reinterpret_cast<int4*>(a.dbg_anc + (uint64_t)(s - 1) * a.N + base + l0)[0] =
                        make_int4((int)(a.pos0 + base + res[0]), (int)(a.pos0 + base + res[1]),
                                  (int)(a.pos0 + base + res[2]), (int)(a.pos0 + base + res[3]));
            }
        }
    }
    __syncthreads();  // D: all stage tables ready

    // ---- 5. compose backwards (l -> a_k1(l) -> ... -> a_1(.)) and write the tile,
    //         moved to its stage-k1 positions ------------------------------------------
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) continue;
        uint32_t src[4] = {4u * q, 4u * q + 1u, 4u * q + 2u, 4u * q + 3u};
        for (uint32_t s = a.k1; s >= 2u; --s) {
            const uint16_t* Ts = tab + (s - 2) * P1;
#pragma unroll
            for (int e = 0; e < 4; ++e) src[e] = Ts[src[e]];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) src[e] = L1[src[e]];
        float v[4 * D];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if constexpr (D == 1) {
                v[e] = xs[src[e]];
            } else if constexpr (D == 2) {
                const float2 t = reinterpret_cast<const float2*>(xs)[src[e]];
                v[2 * e] = t.x;
                v[2 * e + 1] = t.y;
            } else {
#pragma unroll
                for (int c = 0; c < D / 4; ++c) {
                    const float4 t = reinterpret_cast<const float4*>(xs)[src[e] * (D / 4) + c];
                    v[e * D + 4 * c] = t.x;
                    v[e * D + 4 * c + 1] = t.y;
                    v[e * D + 4 * c + 2] = t.z;
                    v[e * D + 4 * c + 3] = t.w;
                }
            }
        }
        store_quad<D>(a.x_out, (uint64_t)base + 4u * q, v);
    }
}

// -------------------------------------------------------------------------------------
struct CascadeArgs {
    double* logV;
    uint32_t* thr;
    const double* part;  // NT tile partials
    double* scratch;     // >= NT + 2 partials (tree levels)
    double* est;         // outputs: filter[2D], predict[2D] (single shard)
    double* shard_rec;   // sharded runs: {log V at level S (= S_loc), root partial[2+4D]}
    uint32_t* ticket;
    uint64_t N;
    uint32_t m, S, k1, b, NT, LPC;
};

template <int D>
__device__ __forceinline__ void combine_partial(const double* x, const double* y, double* out) {
    constexpr int PS = 2 + 4 * D;
    const double mx = x[0] > y[0] ? x[0] : y[0];
    const double fx = (x[0] == -CUDART_INF) ? 0.0 : exp(x[0] - mx);
    const double fy = (y[0] == -CUDART_INF) ? 0.0 : exp(y[0] - mx);
    double r[PS];
    r[0] = mx;
#pragma unroll
    for (int k = 1; k < 2 + 2 * D; ++k) r[k] = x[k] * fx + y[k] * fy;
#pragma unroll
    for (int k = 2 + 2 * D; k < PS; ++k) r[k] = x[k] + y[k];
#pragma unroll
    for (int k = 0; k < PS; ++k) out[k] = r[k];
}

// Perfect binary tree over cnt (power of two, <= 2 * blockDim) partials: src -> dst[0]
// (dst: a scratch area of >= cnt/2 partials).  Block-wide; deterministic.
template <int D>
__device__ void tree_combine(const double* src, uint32_t cnt, double* dst) {
    constexpr int PS = 2 + 4 * D;
    if (cnt == 1) {
        if (threadIdx.x < PS) dst[threadIdx.x] = src[threadIdx.x];
        __syncthreads();
        return;
    }
    for (uint32_t i = threadIdx.x; i < cnt / 2; i += blockDim.x)
        combine_partial<D>(src + (2 * i) * PS, src + (2 * i + 1) * PS, dst + i * PS);
    __syncthreads();
    for (uint32_t c = cnt / 2; c > 1; c >>= 1) {
        double tmp[PS];
        const uint32_t i = threadIdx.x;
        const bool act = i < c / 2;
        if (act) combine_partial<D>(dst + (2 * i) * PS, dst + (2 * i + 1) * PS, tmp);
        __syncthreads();
        if (act)
            for (int k = 0; k < PS; ++k) dst[i * PS + k] = tmp[k];
        __syncthreads();
    }
}

template <int D>
__global__ void __launch_bounds__(kCascadeThreads) k_cascade(const __grid_constant__ CascadeArgs a) {
    constexpr int PS = 2 + 4 * D;
    __shared__ double vb[2048];
    __shared__ int s_last;
    const uint32_t c = blockIdx.x;
    const uint32_t LPC = a.LPC;
    const uint32_t tid = threadIdx.x;

    // levels k1+1 .. k1+log2(LPC) over this CTA's leaves (level k1 entries)
    for (uint32_t i = tid; i < LPC; i += blockDim.x) vb[i] = a.logV[level_offset(a.m, (int)a.k1) + (uint64_t)c * LPC + i];
    __syncthreads();
    uint32_t s = a.k1 + 1;
    for (uint32_t cnt = LPC / 2; cnt >= 1 && s <= a.S; cnt >>= 1, ++s) {
        double nv = 0.0;
        const bool act = tid < cnt;
        if (act) {
            const double vl = vb[2 * tid], vr = vb[2 * tid + 1];
            nv = log_pair_mean(vl, vr);
            a.logV[level_offset(a.m, (int)s) + (uint64_t)c * cnt + tid] = nv;
            a.thr[level_offset(a.m, (int)s) + (uint64_t)c * cnt + tid] = side_threshold(vl, vr, (int)a.b);
        }
        __syncthreads();
        if (act) vb[tid] = nv;
        __syncthreads();
        if (cnt == 1) break;
    }
    // estimate partials of this CTA's leaves -> root slot (NT/2 + c)
    double* myroot = a.scratch + (uint64_t)(a.NT / 2 + c) * PS;
    tree_combine<D>(a.part + (uint64_t)c * LPC * PS, LPC, a.scratch + (uint64_t)c * (LPC / 2) * PS);
    if (tid < PS) myroot[tid] = (LPC == 1) ? a.part[(uint64_t)c * PS + tid] : a.scratch[(uint64_t)c * (LPC / 2) * PS + tid];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // last CTA: levels above the CTA subtrees
    const uint32_t R = gridDim.x;
    const uint32_t lvl0 = a.k1 + (31 - __clz(LPC));  // level of the CTA roots
    if (R > 1) {
        for (uint32_t i = tid; i < R; i += blockDim.x) vb[i] = a.logV[level_offset(a.m, (int)lvl0) + i];
        __syncthreads();
        s = lvl0 + 1;
        for (uint32_t cnt = R / 2; cnt >= 1 && s <= a.S; cnt >>= 1, ++s) {
            double nv = 0.0;
            const bool act = tid < cnt;
            if (act) {
                const double vl = vb[2 * tid], vr = vb[2 * tid + 1];
                nv = log_pair_mean(vl, vr);
                a.logV[level_offset(a.m, (int)s) + tid] = nv;
                a.thr[level_offset(a.m, (int)s) + tid] = side_threshold(vl, vr, (int)a.b);
            }
            __syncthreads();
            if (act) vb[tid] = nv;
            __syncthreads();
            if (cnt == 1) break;
        }
    }
    // final estimate partial: tree over the R CTA roots (stored contiguously)
    double* roots = a.scratch + (uint64_t)(a.NT / 2) * PS;
    double* fin = a.scratch;  // reuse (all CTAs are done with their subtrees)
    tree_combine<D>(roots, R, fin);
    if (a.shard_rec) {  // this shard's root record for the cross-shard top levels
        if (tid == 0) a.shard_rec[0] = a.logV[level_offset(a.m, (int)a.S)];
        if (tid < PS) a.shard_rec[1 + tid] = fin[tid];
        __syncthreads();
        if (tid == 0) *a.ticket = 0u;
        return;
    }
    if (tid == 0) {
        const double sw = fin[1];
        for (int k = 0; k < D; ++k) {
            a.est[k] = fin[2 + k] / sw;
            a.est[D + k] = fin[2 + D + k] / sw;
            a.est[2 * D + k] = fin[2 + 2 * D + k] / (double)a.N;
            a.est[3 * D + k] = fin[2 + 3 * D + k] / (double)a.N;
        }
        *a.ticket = 0u;
    }
}

// -------------------------------------------------------------------------------------
struct ComposeArgs {
    Key key;
    uint32_t n;
    uint64_t N;     // particles of this shard
    uint32_t pos0;  // global index of the shard's first particle
    uint32_t m, M, b, s0, k, P, lowbits;
    const void* pin;
    void* pout;
    const uint32_t* thr;
    int32_t* dbg_anc;
};

__host__ __device__ inline uint32_t compose_smem(uint32_t P, uint32_t payload_bytes, uint32_t k) {
    return P * payload_bytes + 4u * P + 4u * (1u << k);
}

// Thresholds of a tile for stages s0..s0+k-1 into shared memory: stage st has
// 2^{k-st-1} entries at offset 2^k - 2^{k-st}.  One flat index space, so every thread's
// loads are independent (a per-stage loop would serialise k global-load latencies).
__device__ __forceinline__ void load_tile_thresholds(const ComposeArgs& a, const TileGeom& G, uint32_t k,
                                                     uint32_t* ths) {
    const uint32_t E = (1u << k) - 1u;
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        const uint32_t u = (1u << k) - e;                    // in (2^{k-st-1}, 2^{k-st}]
        const uint32_t st = k - (32u - __clz(u - 1u));       // k - ceil(log2 u)
        const uint32_t off = (1u << k) - (1u << (k - st));
        const uint32_t s = a.s0 + st;
        ths[e] = __ldg(a.thr + level_offset(a.m, (int)s) + (G.thi >> s) + (e - off));
    }
}

template <typename T>
struct __align__(4 * sizeof(T) <= 16 ? 4 * sizeof(T) : 16) Vec4 {
    T v[4];
};

// T: payload (int32 ancestor index, float or float2 state).  IDENT: the input payload
// of position i is i itself (first index pass), so nothing is loaded.
template <typename T, bool IDENT, bool DBG, int QPT>
__global__ void __launch_bounds__(1024) k_compose(const __grid_constant__ ComposeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = a.P, M = a.M, b = a.b, nq = P >> 2, k = a.k;
    T* pin_s = reinterpret_cast<T*>(smem);
    uint16_t* Lo = reinterpret_cast<uint16_t*>(smem + (IDENT ? 0u : P * (uint32_t)sizeof(T)));
    uint16_t* Ln = Lo + P;
    uint32_t* ths = reinterpret_cast<uint32_t*>(Ln + P);
    const uint32_t t = blockIdx.x;
    TileGeom G;
    G.lowbits = a.lowbits;
    G.tlo = t & ((1u << a.lowbits) - 1u);
    G.thi = (t >> a.lowbits) << (a.lowbits + k);
    G.b = b;
    G.M = M;
    const T* pin = reinterpret_cast<const T*>(a.pin);
    T* pout = reinterpret_cast<T*>(a.pout);

    load_tile_thresholds(a, G, k, ths);
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        *reinterpret_cast<uint2*>(Lo + l0) = make_uint2(l0 | ((l0 + 1u) << 16), (l0 + 2u) | ((l0 + 3u) << 16));
        if constexpr (!IDENT) {
            if (M >= 4u) {
                *reinterpret_cast<Vec4<T>*>(pin_s + l0) = *reinterpret_cast<const Vec4<T>*>(pin + G.gpos(l0));
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) pin_s[l0 + e] = pin[G.gpos(l0 + e)];
            }
        }
    }
    for (uint32_t st = 0; st < k; ++st) {
        __syncthreads();
        const uint32_t s = a.s0 + st;
        tile_stage<DBG, QPT>(a.key, a.n, s, st, G, ths + ((1u << k) - (1u << (k - st))), Lo, Ln, nq,
                             DBG ? a.dbg_anc + (uint64_t)(s - 1) * a.N : nullptr, a.pos0);
        uint16_t* tmp = Lo;
        Lo = Ln;
        Ln = tmp;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        const uint2 src2 = *reinterpret_cast<const uint2*>(Lo + l0);
        const uint32_t src[4] = {src2.x & 0xffffu, src2.x >> 16, src2.y & 0xffffu, src2.y >> 16};
        Vec4<T> o;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if constexpr (IDENT) o.v[e] = (T)G.gpos(src[e]);
            else o.v[e] = pin_s[src[e]];
        }
        if (M >= 4u) {
            *reinterpret_cast<Vec4<T>*>(pout + G.gpos(l0)) = o;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) pout[G.gpos(l0 + e)] = o.v[e];
        }
    }
}

// -------------------------------------------------------------------------------------
// k_move: the state-moving form of a compose pass (default for every d).  Three phases,
// one barrier between the draws and the moves:
//   A  the tile's payload (particle states at stage s0-1) is copied global -> shared with
//      cp.async (coalesced, no registers), and stays in flight during phase B;
//   B  every stage's draws are filled into per-stage tables T_st[l] = a_s(l) (tile-local
//      positions): a draw depends only on its Philox word and the stage threshold, never
//      on another stage, so all k stages are drawn without barriers;
//   C  each output walks its ancestry back through the tables,
//      l -> a_{s0+k-1}(l) -> ... -> a_{s0}(.), and writes that payload (coalesced).
__host__ __device__ inline uint32_t move_smem(uint32_t P, uint32_t payload_bytes, uint32_t k) {
    return P * payload_bytes + 2u * k * P + 4u * (1u << k);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

template <typename T, bool DBG, int QPT>
__global__ void __launch_bounds__(1024) k_move(const __grid_constant__ ComposeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = a.P, M = a.M, b = a.b, nq = P >> 2, k = a.k;
    T* pin_s = reinterpret_cast<T*>(smem);
    uint16_t* tabs = reinterpret_cast<uint16_t*>(smem + P * (uint32_t)sizeof(T));
    uint32_t* ths = reinterpret_cast<uint32_t*>(tabs + k * P);
    const uint32_t t = blockIdx.x;
    TileGeom G;
    G.lowbits = a.lowbits;
    G.tlo = t & ((1u << a.lowbits) - 1u);
    G.thi = (t >> a.lowbits) << (a.lowbits + k);
    G.b = b;
    G.M = M;
    const T* pin = reinterpret_cast<const T*>(a.pin);
    T* pout = reinterpret_cast<T*>(a.pout);
    const uint32_t mask = M - 1u;

    // A: payload copy in flight
    if (M >= 4u) {
        constexpr uint32_t CH = (4u * sizeof(T)) / 16u;  // 16-byte chunks per quad
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = threadIdx.x + it * blockDim.x;
            if (q >= nq) break;
            const char* src = reinterpret_cast<const char*>(pin + G.gpos(4u * q));
            char* dst = reinterpret_cast<char*>(pin_s + 4u * q);
#pragma unroll
            for (uint32_t c = 0; c < CH; ++c) cp_async16(dst + 16u * c, src + 16u * c);
        }
    } else {
        for (uint32_t l = threadIdx.x; l < P; l += blockDim.x) pin_s[l] = pin[G.gpos(l)];
    }
    load_tile_thresholds(a, G, k, ths);
    __syncthreads();

    // B: all stages' draws
    for (uint32_t st = 0; st < k; ++st) {
        const uint32_t s = a.s0 + st, bit = 1u << st;
        const uint32_t* thr_s = ths + ((1u << k) - (1u << (k - st)));
        uint16_t* Ts = tabs + st * P;
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = threadIdx.x + it * blockDim.x;
            if (q >= nq) break;
            const uint32_t l0 = 4u * q;
            uint32_t res[4];
            if (M >= 4u) {
                const uint32_t j = l0 >> b;
                const uint32_t c0 = (a.pos0 + ((G.gof(j) << b) | (l0 & mask))) >> 2;
                const uint4 blk = rng_block(a.key, c0, a.n, kDomainResample, s);
                const uint32_t Pt = thr_s[j >> (st + 1)];
                const uint32_t bl = (j & ~bit) << b, br = (j | bit) << b;
                const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) res[e] = (((r[e] >> b) < Pt) ? bl : br) | (r[e] & mask);
            } else {  // M == 2: the quad spans groups j, j+1 (possibly two global Philox quads)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t l = l0 + e;
                    const uint32_t j = l >> 1;
                    const uint32_t gi = a.pos0 + ((G.gof(j) << 1) | (l & 1u));
                    const uint4 blk = rng_block(a.key, gi >> 2, a.n, kDomainResample, s);
                    const uint32_t r = word_of(blk, (int)(gi & 3u));
                    const uint32_t jj = ((r >> 1) < thr_s[j >> (st + 1)]) ? (j & ~bit) : (j | bit);
                    res[e] = (jj << 1) | (r & 1u);
                }
            }
            *reinterpret_cast<uint2*>(Ts + l0) = make_uint2(res[0] | (res[1] << 16), res[2] | (res[3] << 16));
            if constexpr (DBG) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    a.dbg_anc[(uint64_t)(s - 1) * a.N + G.gpos(l0 + e)] = (int32_t)(a.pos0 + G.gpos(res[e]));
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();

    // C: walk back and write
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        uint32_t src[4] = {l0, l0 + 1u, l0 + 2u, l0 + 3u};
        for (int st = (int)k - 1; st >= 0; --st) {
            const uint16_t* Ts = tabs + st * P;
#pragma unroll
            for (int e = 0; e < 4; ++e) src[e] = Ts[src[e]];
        }
        Vec4<T> o;
#pragma unroll
        for (int e = 0; e < 4; ++e) o.v[e] = pin_s[src[e]];
        if (M >= 4u) {
            *reinterpret_cast<Vec4<T>*>(pout + G.gpos(l0)) = o;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) pout[G.gpos(l0 + e)] = o.v[e];
        }
    }
}

// -------------------------------------------------------------------------------------
// Sharded runs (G = 2^L GPUs, shard r owns groups [r m/G, (r+1) m/G)).
//
// k_top: from the G shard records (rank order) every rank computes, identically, the V
// levels S_loc+1..S (same log-domain pair means and operand order as k_cascade, so the
// values are bitwise those of a single-GPU run), the cross-stage side thresholds, and the
// estimate (perfect binary tree over the shard partials = the upper levels of the
// single-GPU tree over tiles).  Top level t (= stage S_loc + t) has G >> t entries at
// offset G - (G >> (t-1)).
struct TopArgs {
    const double* recs;  // G x (1 + PS)
    double* top_logV;    // G - 1
    uint32_t* top_thr;   // G - 1
    double* est;
    double* scratch;     // >= 2 G partials
    uint64_t Nglobal;
    uint32_t G, L, b;
};

template <int D>
__global__ void __launch_bounds__(1024) k_top(const __grid_constant__ TopArgs a) {
    constexpr int PS = 2 + 4 * D;
    __shared__ double vb[1024];
    const uint32_t tid = threadIdx.x, G = a.G;
    for (uint32_t i = tid; i < G; i += blockDim.x) vb[i] = a.recs[(uint64_t)i * (1 + PS)];
    __syncthreads();
    for (uint32_t t = 1, cnt = G / 2; t <= a.L; ++t, cnt >>= 1) {
        double nv = 0.0;
        const bool act = tid < cnt;
        if (act) {
            const double vl = vb[2 * tid], vr = vb[2 * tid + 1];
            nv = log_pair_mean(vl, vr);
            a.top_logV[(G - (G >> (t - 1))) + tid] = nv;
            a.top_thr[(G - (G >> (t - 1))) + tid] = side_threshold(vl, vr, (int)a.b);
        }
        __syncthreads();
        if (act) vb[tid] = nv;
        __syncthreads();
    }
    // estimate: perfect binary tree over the G root partials (copied contiguous)
    for (uint32_t i = tid; i < G * PS; i += blockDim.x) {
        const uint32_t r = i / PS, c = i % PS;
        a.scratch[G * PS + i] = a.recs[(uint64_t)r * (1 + PS) + 1 + c];
    }
    __syncthreads();
    tree_combine<D>(a.scratch + G * PS, G, a.scratch);
    if (tid == 0) {
        const double* fin = a.scratch;
        const double sw = fin[1];
        for (int k = 0; k < D; ++k) {
            a.est[k] = fin[2 + k] / sw;
            a.est[D + k] = fin[2 + D + k] / sw;
            a.est[2 * D + k] = fin[2 + 2 * D + k] / (double)a.Nglobal;
            a.est[3 * D + k] = fin[2 + 3 * D + k] / (double)a.Nglobal;
        }
    }
}

// k_cross: cross-shard stage s = S_loc + t.  Shard r pairs with r ^ 2^{t-1}; a particle of
// local group gl pairs with the SAME local group of the partner.  Every output's draw
// (side, index) is counter-based, so each output reads its source state from this
// shard's or the partner's stage-(s-1) buffer (the partner's arrives whole over NVLink).
struct CrossArgs {
    Key key;
    uint32_t n, s, t, rank, b, M;
    uint64_t Nloc;
    uint32_t pos0, pos0_partner;
    const uint32_t* thr;    // the stage threshold (device): top_thr entry of block rank >> t
    const void* own_in;
    const void* partner_in;
    void* out;
    int32_t* dbg_anc;       // this shard's stage tables (global source positions)
};

template <typename T, bool DBG>
__global__ void __launch_bounds__(256) k_cross(const __grid_constant__ CrossArgs a) {
    const T* own = reinterpret_cast<const T*>(a.own_in);
    const T* par = reinterpret_cast<const T*>(a.partner_in);
    T* out = reinterpret_cast<T*>(a.out);
    const uint32_t mask = a.M - 1u;
    const bool own_is_low = ((a.rank >> (a.t - 1)) & 1u) == 0u;
    const uint32_t P = __ldg(a.thr);
    const uint64_t nq = a.Nloc >> 2;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l0 = (uint32_t)(4u * q);
        const uint4 blk = rng_block(a.key, (a.pos0 + l0) >> 2, a.n, kDomainResample, a.s);
        const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
        Vec4<T> o;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t l = l0 + e;
            const bool low = (r[e] >> a.b) < P;
            const bool from_own = (low == own_is_low);
            const uint32_t src = ((l >> a.b) << a.b) | (r[e] & mask);
            o.v[e] = from_own ? own[src] : par[src];
            if constexpr (DBG)
                a.dbg_anc[(uint64_t)(a.s - 1) * a.Nloc + l] = (int32_t)((from_own ? a.pos0 : a.pos0_partner) + src);
        }
        if (a.M >= 4u) {
            *reinterpret_cast<Vec4<T>*>(out + l0) = o;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) out[l0 + e] = o.v[e];
        }
    }
}

// -------------------------------------------------------------------------------------
// Debug helpers (not on the timed path).
template <int UNUSED>
__global__ void k_debug_compose(const int32_t* __restrict__ anc, uint64_t N, uint32_t S, int32_t* __restrict__ A) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t j = i;
        for (int s = (int)S; s >= 1; --s) j = (uint64_t)anc[(uint64_t)(s - 1) * N + j];
        A[i] = (int32_t)j;
    }
}

template <int D>
__global__ void k_gather(const float* __restrict__ x, const int32_t* __restrict__ A, uint64_t N, float* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = A ? (uint64_t)A[i] : i;
        for (int k = 0; k < D; ++k) out[i * D + k] = x[j * D + k];
    }
}

}  // namespace pfk
