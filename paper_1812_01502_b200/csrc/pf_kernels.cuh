// pf_kernels.cuh -- the kernels of one BPF time step with augmented resampling.
//
//   k_init      x_0^i ~ pi_0                                   (Alg. 1 l.1-3)
//   k_pass1     (pf_pass1.cuh) per tile of T1 = 2^k1 consecutive groups: load -> mutate ->
//               log g_n -> stage 1 -> V levels and stages 2..k1 -> the tile written once,
//               moved to its stage-k1 positions
//   k_cascade   V levels k1+1..S (log-domain pair means, eq. V_defn_proofs),
//               the stage side thresholds, and the fixed-tree combination of the
//               estimate partials (single launch, last-CTA-finishes pattern)
//   k_stages    (pf_stages.cuh) stages s0..s0+k-1 for a tile of 2^k groups spaced
//               2^{s0-1} apart (exactly the groups the butterfly pairs at those stages),
//               moving the particle states once per pass
//   k_top / k_cross   the cross-shard stages of a sharded run (pairwise rounds); the pull
//               exchange kernels k_pull_* live in pf_inst_misc.cu
//   next rows   k_ess_* (fully adapted scheme), k_island_* (AIRPF), MultinomialArgs
//               (Alg. 2, pf_multinomial.cu); k_pass1's weigh / resample / AIRPF modes
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
#include "pf_args.h"

namespace pfk {

constexpr uint32_t FULL = 0xffffffffu;


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
    if (gridDim.x > 1) {  // last CTA to finish does the top (one CTA: no ticket, no fence)
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
    } else {
        __syncthreads();
    }

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
        if (tid == 0 && gridDim.x > 1) *a.ticket = 0u;
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
        if (gridDim.x > 1) *a.ticket = 0u;
    }
}

// -------------------------------------------------------------------------------------
// Fully adapted scheme (R17): the ESS of the stage weights V_0 = w, V_1, ..., V_S
// and the number of stages to run, S* = min{s : E_s >= theta}.
//   k_ess_chunks  one CTA per chunk of kEssChunk entries of one level: level 0 = the tile
//                 partials {max, sum w, sum w^2} of k_pass1 (kPass1Weigh), level s >= 1 =
//                 the m / 2^s values of the V table; sums of e^{v - L}, e^{2(v - L)} with L
//                 the global max of lw (V_s <= max w, so no term overflows); fixed order
//   k_ess_final   one thread per level sums its chunks in order -> E_s; thread 0 -> S*,
//                 log V_S; resets the running max for the next step
// -------------------------------------------------------------------------------------
// AIRPF island stages (Alg. 6 / Alg. 7; R20, R21).
//   k_island_draw     thread per (stage s, quad of islands): the four islands' side draws
//                     (Philox block (quad, n, ISLAND<<24 | s)), side L iff (r >> 1) <
//                     thr_s[pair]; Alg. 7 undoes a pure exchange (needs the partner quad's
//                     block when the partner lies in another quad); writes one nibble per
//                     quad: bit e = island 4 quad + e takes its partner's block
//   k_island_compose  thread per island: walks stages S..1 through the nibbles -> A_isl
// -------------------------------------------------------------------------------------
// Multinomial resampling, Alg. 2 (kernels in pf_multinomial.cu).
// -------------------------------------------------------------------------------------
// -------------------------------------------------------------------------------------
// Sharded runs (G = 2^L GPUs, shard r owns groups [r m/G, (r+1) m/G)).
//
// k_top: from the G shard records (rank order) every rank computes, identically, the V
// levels S_loc+1..S (same log-domain pair means and operand order as k_cascade, so the
// values are bitwise those of a single-GPU run), the cross-stage side thresholds, and the
// estimate (perfect binary tree over the shard partials = the upper levels of the
// single-GPU tree over tiles).  Top level t (= stage S_loc + t) has G >> t entries at
// offset G - (G >> (t-1)).
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
// Pull exchange of the cross stages (alternative to L rounds of k_cross):
// every output of this shard composes its L cross-stage draws locally (they are
// counter-based, and every rank holds the top thresholds after k_top), giving the
// (rank, local position) of its stage-S_loc source; the requests are grouped by owner
// rank, exchanged in one all-to-all, served by a gather on the owner, and the states come
// back in a second all-to-all.  Same draws and the same x_hat as the pairwise rounds.
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

}  // namespace pfk
