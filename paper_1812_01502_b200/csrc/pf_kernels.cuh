// pf_kernels.cuh -- the kernels of one BPF time step with augmented resampling.
//
//   k_init      x_0^i ~ pi_0                                   (Alg. 1 l.1-3)
//   k_pass1     per tile of T1 = 2^k1 consecutive groups (P1 = T1 M particles):
//               [gather/load xhat] -> mutate (Alg. 1 l.303) -> log g_n
//               -> stage 1 (pairs (2p, 2p+1): smem scan + branch-free search)
//               -> V levels 1..k1 and stages 2..k1 inside the tile (Alg. 3 l.346-349)
//               -> write the tile's particles moved to their stage-k1 positions
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
#pragma once
#include <cstdint>

#include "pf_device.cuh"

namespace pfk {

constexpr int kPass1Threads = 512;
constexpr int kComposeThreads = 1024;
constexpr int kCascadeThreads = 1024;
constexpr int kMaxQuadsPerThread = 16;

__host__ __device__ inline uint64_t level_offset(uint64_t m, int s) { return m - (m >> (s - 1)); }

// -------------------------------------------------------------------------------------
// Per-particle state I/O (packed AoS: particle i occupies floats [i*D, i*D+D)).
template <int D>
__device__ __forceinline__ void load_particle(const float* __restrict__ x, uint64_t i, float* v) {
    if constexpr (D == 1) {
        v[0] = __ldg(x + i);
    } else if constexpr (D == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(x) + i);
        v[0] = t.x;
        v[1] = t.y;
    } else {
#pragma unroll
        for (int c = 0; c < D / 4; ++c) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(x + i * D) + c);
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
    uint64_t N;
    float* x;
};

template <int D, int KIND>
__global__ void __launch_bounds__(256) k_init(const __grid_constant__ InitArgs a) {
    const uint64_t nq = a.N >> 2;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        float z[4 * D], v[4 * D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint4 blk = rng_block(a.key, (uint32_t)(q * D + j), 0u, kDomainInit, 0u);
            normals4(blk, z + 4 * j);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) init_state<D, KIND>(a.mp, z + e * D, v + e * D);
        store_quad<D>(a.x, q * 4, v);
    }
}

// -------------------------------------------------------------------------------------
struct Pass1Args {
    ModelParams mp;
    Key key;
    uint32_t n;
    int do_mutate;
    const float* y_dev;  // if non-null, y is read from device memory
    float y[8];
    uint64_t N;
    uint32_t m, M, b, S, k1, P1;
    const float* x_in;    // xhat_{n-1} source (or x_0)
    const int32_t* A_in;  // gather map into x_in (nullptr: identity)
    float* x_out;         // particles moved to their stage-k1 positions
    double* logV;         // level table (m - 1)
    uint32_t* thr;        // threshold table (m - 1)
    double* part;         // per-tile estimate partials, (2 + 4D) doubles each
    float* dbg_x;
    float* dbg_lw;
    int32_t* dbg_anc;
};

// Shared-memory carve-up of k_pass1 (host and device agree through this function).
struct Pass1Smem {
    uint32_t xs, w, L0, L1, Q, pm, ct, lv, th, red, total;
};
__host__ __device__ inline Pass1Smem pass1_smem(int D, uint32_t P1, uint32_t M, uint32_t k1) {
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
    s.L0 = take(k1 >= 2 ? P1 * 2u : 0u);
    s.L1 = take(k1 >= 2 ? P1 * 2u : 0u);
    s.Q = take(P1);  // P1/4 floats
    s.pm = take((T1 / 2) * 4u);
    s.ct = take((T1 / 2) * 4u);
    s.lv = take(T1 * 8u);
    s.th = take(T1 * 4u);
    s.red = take(32u * (2u + 4u * 8u) * 8u);
    s.total = off;
    return s;
}

// Segmented inclusive scan (op = max or +) of Q[0..nq) in segments of Z quads
// (Hillis-Steele in shared memory; Z a power of two).
template <bool MAX>
__device__ __forceinline__ void seg_scan(float* Q, uint32_t nq, uint32_t Z) {
    for (uint32_t off = 1; off < Z; off <<= 1) {
        float tmp[kMaxQuadsPerThread];
        int t = 0;
        for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x, ++t)
            tmp[t] = ((q & (Z - 1)) >= off) ? Q[q - off] : (MAX ? -CUDART_INF_F : 0.0f);
        __syncthreads();
        t = 0;
        for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x, ++t)
            Q[q] = MAX ? fmaxf(Q[q], tmp[t]) : Q[q] + tmp[t];
        __syncthreads();
    }
}

template <int D>
struct Partial {
    double v[2 + 4 * D];  // tmax, sw, s1[D], s2[D], p1[D], p2[D]
};

template <int D, int KIND, bool GATHER>
__global__ void __launch_bounds__(kPass1Threads) k_pass1(const __grid_constant__ Pass1Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Pass1Smem L = pass1_smem(D, a.P1, a.M, a.k1);
    float* xs = reinterpret_cast<float*>(smem + L.xs);
    float* w = reinterpret_cast<float*>(smem + L.w);
    uint16_t* La = reinterpret_cast<uint16_t*>(smem + L.L0);
    uint16_t* Lb = reinterpret_cast<uint16_t*>(smem + L.L1);
    float* Q = reinterpret_cast<float*>(smem + L.Q);
    float* pmax = reinterpret_cast<float*>(smem + L.pm);
    float* ctot = reinterpret_cast<float*>(smem + L.ct);
    double* lv = reinterpret_cast<double*>(smem + L.lv);
    uint32_t* th = reinterpret_cast<uint32_t*>(smem + L.th);
    double* red = reinterpret_cast<double*>(smem + L.red);

    const uint32_t P1 = a.P1, M = a.M, b = a.b, nq = P1 >> 2;
    const uint32_t T1 = P1 >> b;  // groups per tile
    const uint32_t tile = blockIdx.x;
    const uint64_t base = (uint64_t)tile * P1;
    const uint64_t N = a.N;
    const uint32_t tid = threadIdx.x;

    float y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = a.y_dev ? (k < a.mp.dy ? __ldg(a.y_dev + k) : 0.0f) : a.y[k];

    // ---- 1. load / gather xhat, mutate, weight --------------------------------------
    float tmax_thread = -CUDART_INF_F;
    for (uint32_t q = tid; q < nq; q += blockDim.x) {
        const uint64_t i0 = base + 4ull * q;
        float xh[4 * D], x[4 * D];
        if (GATHER) {
            const int4 src = __ldg(reinterpret_cast<const int4*>(a.A_in + i0));
            load_particle<D>(a.x_in, (uint64_t)src.x, xh);
            load_particle<D>(a.x_in, (uint64_t)src.y, xh + D);
            load_particle<D>(a.x_in, (uint64_t)src.z, xh + 2 * D);
            load_particle<D>(a.x_in, (uint64_t)src.w, xh + 3 * D);
        } else {
            load_quad<D>(a.x_in, i0, xh);
        }
        if (a.do_mutate) {
            float z[4 * D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 blk = rng_block(a.key, (uint32_t)((i0 >> 2) * D + j), a.n, kDomainMutate, 0u);
                normals4(blk, z + 4 * j);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) mutate<D, KIND>(a.mp, xh + e * D, z + e * D, x + e * D);
        } else {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) x[k] = xh[k];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float lw = log_potential<D, KIND>(a.mp, y, x + e * D);
            w[4 * q + e] = lw;
            tmax_thread = fmaxf(tmax_thread, lw);
        }
#pragma unroll
        for (int k = 0; k < 4 * D; ++k) xs[4 * q * D + k] = x[k];
        if (a.dbg_x) {
            store_quad<D>(a.dbg_x, i0, x);
            reinterpret_cast<float4*>(a.dbg_lw + i0)[0] =
                make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
    }
    // tile max (for the estimate partials)
    for (int o = 16; o > 0; o >>= 1) tmax_thread = fmaxf(tmax_thread, __shfl_xor_sync(0xffffffffu, tmax_thread, o));
    float* redf = reinterpret_cast<float*>(red);
    if ((tid & 31) == 0) redf[tid >> 5] = tmax_thread;
    __syncthreads();
    float tmax = -CUDART_INF_F;
    for (uint32_t wv = 0; wv < (blockDim.x + 31) / 32; ++wv) tmax = fmaxf(tmax, redf[wv]);

    // ---- 2. stage 1: pair max, weights, segmented scan --------------------------------
    const uint32_t Z = M >> 1;  // quads per pair (2M positions)
    for (uint32_t q = tid; q < nq; q += blockDim.x)
        Q[q] = fmaxf(fmaxf(w[4 * q], w[4 * q + 1]), fmaxf(w[4 * q + 2], w[4 * q + 3]));
    __syncthreads();
    seg_scan<true>(Q, nq, Z);
    for (uint32_t p = tid; p < T1 / 2; p += blockDim.x) pmax[p] = Q[(p + 1) * Z - 1];
    __syncthreads();

    float acc[2 + 4 * D];
#pragma unroll
    for (int k = 0; k < 2 + 4 * D; ++k) acc[k] = 0.0f;
    for (uint32_t q = tid; q < nq; q += blockDim.x) {
        const uint32_t p = (4 * q) >> (b + 1);
        const float pm = pmax[p];
        const float f = (tmax == -CUDART_INF_F) ? 1.0f : expf(pm - tmax);
        float run = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float c = (pm == -CUDART_INF_F) ? 1.0f : expf(w[4 * q + e] - pm);
            const float wf = c * f;
            acc[1] += wf;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float xv = xs[(4 * q + e) * D + k];
                acc[2 + k] = fmaf(wf, xv, acc[2 + k]);
                acc[2 + D + k] = fmaf(wf * xv, xv, acc[2 + D + k]);
                acc[2 + 2 * D + k] += xv;
                acc[2 + 3 * D + k] = fmaf(xv, xv, acc[2 + 3 * D + k]);
            }
            run += c;
            w[4 * q + e] = run;
        }
        Q[q] = run;
    }
    __syncthreads();
    seg_scan<false>(Q, nq, Z);
    for (uint32_t q = tid; q < nq; q += blockDim.x) {
        if (q & (Z - 1)) {
            const float off = Q[q - 1];
#pragma unroll
            for (int e = 0; e < 4; ++e) w[4 * q + e] += off;
        }
    }
    for (uint32_t p = tid; p < T1 / 2; p += blockDim.x) ctot[p] = Q[(p + 1) * Z - 1];

    // estimate partials of the tile: fp64 block reduction (deterministic order)
    {
        double accd[2 + 4 * D];
#pragma unroll
        for (int k = 1; k < 2 + 4 * D; ++k) {
            double v = (double)acc[k];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            accd[k] = v;
        }
        __syncthreads();  // redf reads above are done
        const uint32_t nw = (blockDim.x + 31) / 32;
        if ((tid & 31) == 0)
            for (int k = 1; k < 2 + 4 * D; ++k) red[(tid >> 5) * (2 + 4 * D) + k] = accd[k];
        __syncthreads();
        if (tid < (uint32_t)(2 + 4 * D)) {
            double v;
            if (tid == 0) {
                v = (double)tmax;
            } else {
                v = 0.0;
                for (uint32_t wv = 0; wv < nw; ++wv) v += red[wv * (2 + 4 * D) + tid];
            }
            a.part[(uint64_t)tile * (2 + 4 * D) + tid] = v;
        }
    }

    // logV level 1 per pair, then levels 2..k1 and thresholds (stage s uses level s-1)
    const double log2M = log((double)(2u * M));
    for (uint32_t p = tid; p < T1 / 2; p += blockDim.x) {
        const float pm = pmax[p];
        const double v = (pm == -CUDART_INF_F) ? -CUDART_INF : (double)pm + log((double)ctot[p]) - log2M;
        lv[p] = v;  // tile-local level offset: T1 - (T1 >> (s-1)); level 1 at 0
        a.logV[level_offset(a.m, 1) + (uint64_t)tile * (T1 / 2) + p] = v;
    }
    __syncthreads();
    for (uint32_t s = 2; s <= a.k1; ++s) {
        const uint32_t cnt = T1 >> s;
        const uint32_t po = T1 - (T1 >> (s - 2)), co = T1 - (T1 >> (s - 1));
        for (uint32_t bk = tid; bk < cnt; bk += blockDim.x) {
            const double vl = lv[po + 2 * bk], vr = lv[po + 2 * bk + 1];
            const double v = log_pair_mean(vl, vr);
            const uint32_t P = side_threshold(vl, vr, (int)b);
            lv[co + bk] = v;
            th[co + bk] = P;
            a.logV[level_offset(a.m, (int)s) + (uint64_t)tile * cnt + bk] = v;
            a.thr[level_offset(a.m, (int)s) + (uint64_t)tile * cnt + bk] = P;
        }
        __syncthreads();
    }

    // ---- 3. stage-1 draws: inverse CDF over the pair's 2M weights ----------------------
    for (uint32_t q = tid; q < nq; q += blockDim.x) {
        const uint64_t i0 = base + 4ull * q;
        const uint4 blk = rng_block(a.key, (uint32_t)(i0 >> 2), a.n, kDomainResample, 1u);
        const uint32_t p = (4 * q) >> (b + 1);
        const uint32_t pb = p << (b + 1);
        const float tot = ctot[p];
        uint32_t res[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float t = u01f(word_of(blk, e)) * tot;
            uint32_t lo = 0;
            for (uint32_t step = M; step >= 1; step >>= 1)
                if (w[pb + lo + step - 1] <= t) lo += step;
            res[e] = pb + lo;
        }
        if (a.dbg_anc) {
            reinterpret_cast<int4*>(a.dbg_anc + i0)[0] =
                make_int4((int)(base + res[0]), (int)(base + res[1]), (int)(base + res[2]), (int)(base + res[3]));
        }
        if (a.k1 == 1) {
            float v[4 * D];
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int k = 0; k < D; ++k) v[e * D + k] = xs[res[e] * D + k];
            store_quad<D>(a.x_out, i0, v);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) La[4 * q + e] = (uint16_t)res[e];
        }
    }
    if (a.k1 == 1) return;

    // ---- 4. stages 2..k1 inside the tile (uniform-within-group side draws) ------------
    uint16_t* Lo = La;
    uint16_t* Ln = Lb;
    for (uint32_t s = 2; s <= a.k1; ++s) {
        __syncthreads();
        const uint32_t bit = 1u << (s - 1);
        const uint32_t co = T1 - (T1 >> (s - 1));
        for (uint32_t q = tid; q < nq; q += blockDim.x) {
            const uint64_t i0 = base + 4ull * q;
            const uint4 blk = rng_block(a.key, (uint32_t)(i0 >> 2), a.n, kDomainResample, s);
            int res[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t l = 4 * q + e;
                const uint32_t j = l >> b;
                const uint32_t r = word_of(blk, e);
                const uint32_t P = th[co + (j >> s)];
                const uint32_t jj = ((r >> b) < P) ? (j & ~bit) : (j | bit);
                const uint32_t al = (jj << b) | (r & (M - 1));
                Ln[l] = Lo[al];
                res[e] = (int)(base + al);
            }
            if (a.dbg_anc)
                reinterpret_cast<int4*>(a.dbg_anc + (uint64_t)(s - 1) * N + i0)[0] =
                    make_int4(res[0], res[1], res[2], res[3]);
        }
        uint16_t* t = Lo;
        Lo = Ln;
        Ln = t;
    }
    __syncthreads();
    for (uint32_t q = tid; q < nq; q += blockDim.x) {
        float v[4 * D];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t src = Lo[4 * q + e];
#pragma unroll
            for (int k = 0; k < D; ++k) v[e * D + k] = xs[src * D + k];
        }
        store_quad<D>(a.x_out, base + 4ull * q, v);
    }
}

// -------------------------------------------------------------------------------------
struct CascadeArgs {
    double* logV;
    uint32_t* thr;
    const double* part;  // NT tile partials
    double* scratch;     // >= NT/2 partials (tree levels)
    double* est;         // outputs: filter[2D], predict[2D]
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

// Perfect binary tree over cnt (power of two) partials: src -> dst[0] (dst may alias a
// scratch area of >= cnt/2 partials).  Block-wide; deterministic.
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
        // each pair combined by one thread; write after a barrier (in-place levels)
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
    // estimate partials of this CTA's leaves -> scratch slot (NT/2 + c)
    double* myroot = a.scratch + (uint64_t)(a.NT / 2 + c) * PS;
    tree_combine<D>(a.part + (uint64_t)c * LPC * PS, LPC, a.scratch + (uint64_t)c * (LPC / 2) * PS);
    if (tid < PS) myroot[tid] = a.scratch[(uint64_t)c * (LPC / 2) * PS + tid];
    if (LPC == 1 && tid < PS) myroot[tid] = a.part[(uint64_t)c * PS + tid];
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
    uint64_t N;
    uint32_t m, M, b, s0, k, P, lowbits;
    const void* pin;
    void* pout;
    const uint32_t* thr;
    int32_t* dbg_anc;
};

__host__ __device__ inline uint32_t compose_smem(uint32_t P, uint32_t payload_bytes) {
    return P * payload_bytes + 4u * P;
}

// T: payload (int32 ancestor index, float or float2 state).  IDENT: the input payload
// of position i is i itself (first index pass), so nothing is loaded.
template <typename T, bool IDENT>
__global__ void __launch_bounds__(kComposeThreads) k_compose(const __grid_constant__ ComposeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = a.P, M = a.M, b = a.b, nq = P >> 2;
    T* pin_s = reinterpret_cast<T*>(smem);
    uint16_t* Lo = reinterpret_cast<uint16_t*>(smem + (IDENT ? 0u : P * (uint32_t)sizeof(T)));
    uint16_t* Ln = Lo + P;
    const uint32_t t = blockIdx.x;
    const uint32_t lowmask = (1u << a.lowbits) - 1u;
    const uint32_t thi = (t >> a.lowbits) << (a.lowbits + a.k);
    const uint32_t tlo = t & lowmask;
    auto gof = [&](uint32_t j) -> uint32_t { return tlo | (j << a.lowbits) | thi; };
    const T* pin = reinterpret_cast<const T*>(a.pin);
    T* pout = reinterpret_cast<T*>(a.pout);

    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t l = 4 * q + e;
            Lo[l] = (uint16_t)l;
            if constexpr (!IDENT) {
                const uint64_t gi = ((uint64_t)gof(l >> b) << b) | (l & (M - 1));
                pin_s[l] = pin[gi];
            }
        }
    }
    for (uint32_t st = 0; st < a.k; ++st) {
        __syncthreads();
        const uint32_t s = a.s0 + st;
        const uint32_t bitj = 1u << st;
        const uint64_t toff = level_offset(a.m, (int)s);
        for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
            uint32_t cached = 0xffffffffu;
            uint4 blk = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t l = 4 * q + e;
                const uint32_t j = l >> b;
                const uint32_t g = gof(j);
                const uint64_t gi = ((uint64_t)g << b) | (l & (M - 1));
                const uint32_t c0 = (uint32_t)(gi >> 2);
                if (c0 != cached) {
                    blk = rng_block(a.key, c0, a.n, kDomainResample, s);
                    cached = c0;
                }
                const uint32_t r = word_of(blk, (int)(gi & 3));
                const uint32_t Pth = __ldg(a.thr + toff + (g >> s));
                const uint32_t jj = ((r >> b) < Pth) ? (j & ~bitj) : (j | bitj);
                const uint32_t al = (jj << b) | (r & (M - 1));
                Ln[l] = Lo[al];
                if (a.dbg_anc)
                    a.dbg_anc[(uint64_t)(s - 1) * a.N + gi] = (int32_t)((gof(jj) << b) | (r & (M - 1)));
            }
        }
        uint16_t* tmp = Lo;
        Lo = Ln;
        Ln = tmp;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t l = 4 * q + e;
            const uint64_t gi = ((uint64_t)gof(l >> b) << b) | (l & (M - 1));
            const uint32_t src = Lo[l];
            if constexpr (IDENT) {
                pout[gi] = (T)(((uint64_t)gof(src >> b) << b) | (src & (M - 1)));
            } else {
                pout[gi] = pin_s[src];
            }
        }
    }
}

// -------------------------------------------------------------------------------------
// Debug helpers (not on the timed path).
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
