// pf_pass1c.cuh -- k_pass1c: the fused pass 1 (k_pass1, kPass1Fused, pf_pass1.cuh) with the
// group size M = 2^B, the tile depth K1 and the quads per thread fixed at compile time, for
// the plans the benchmark configurations run (C4: d = 4, B = 6, K1 = 4, QPT = 2).
//
// Same arithmetic in the same order as k_pass1 (Alg. 1 l.302-303 mutation, PAPER.md:291
// weighting, Alg. 3 stage 1 over the pair pools, V levels eq. V_defn_proofs and the
// stages 2..K1, composition by Lemma facts_about_Vs (a)), so the outputs are bitwise
// k_pass1's (tests/test_gpu_stage_spec.py); what changes is the instruction count:
//   * every loop bound, shift and mask is an immediate (no tail guards: the tile is full);
//   * the stage-1 search walks BYTE offsets of the quad-end array (one LDS, one compare,
//     one predicated add per step, immediates for the probe offsets);
//   * the stage tables (stage 1 and stages 2..K1) hold the source's byte offset (tile
//     position x 2), so a walk step is a single LDS.U16, and the stage 2..K1 entries are
//     built two per word with the sign trick of k_stages_ws (pf_stages.cuh).
// Restrictions (the launcher falls back to k_pass1 otherwise): 16-bit tables (TB = 2), a
// stage-1 pool of at most 32 quads (B <= 6), no debug tables, no adaptive modes; the AIRPF
// mode has an instance of its own (MODE = kPass1Airpf).
#pragma once
#include <cstdint>

#include "pf_args.h"
#include "pf_pass1.cuh"
#include "pf_stages.cuh"

namespace pfk {

// The linear-Gaussian model with LQ diagonal and the diagonal observation fast path
// (mp.diag_lq, mp.diag_obs: C1, C2, C4) as compile-time branches; same operations and order
// as mutate / log_potential (pf_device.cuh).
template <int D>
__device__ __forceinline__ void mutate_lg_diag(const ModelParams& mp, const float* xh, const float* z, float* x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float v = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) v = fmaf(mp.A[k * D + j], xh[j], v);
        x[k] = fmaf(mp.LQ[k * D + k], z[k], v);
    }
}
template <int D>
__device__ __forceinline__ float log_potential_lg_diag(const ModelParams& mp, const float* y, const float* x) {
    float v = 0.0f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float r = y[k] - x[k];
        v = fmaf(mp.rdiag[k] * r, r, v);
    }
    return (v == v && v != INFINITY && v != -INFINITY) ? v : -INFINITY;
}

// DIAG: the LG model takes the diagonal paths (the launcher checks mp.diag_lq && mp.diag_obs).
// MODE: kPass1Fused (the step's pass 1) or kPass1Airpf (AIRPF, k_pass1's AIRPF mode: island
// blocks read through the previous island map, carried island weights (AIRPF2), the
// within-island resample with pools of one island, island levels 1..K1 with 31-bit
// thresholds (R20), no stage tables: the tile is written in natural order).
template <int D, int KIND, int B, int K1, int QPT, int MINB, bool DIAG, int MODE = kPass1Fused>
__global__ void __launch_bounds__(((1 << (B + K1)) / 4) / QPT, MINB) k_pass1c(const __grid_constant__ Pass1Args a) {
    constexpr bool AIR = MODE == kPass1Airpf, WEIGH = MODE == kPass1Weigh, RES = MODE == kPass1Resample;
    constexpr uint32_t M = 1u << B, P1 = M << K1, T1 = 1u << K1, nq = P1 / 4u;
    constexpr uint32_t NTHR = nq / QPT, NWARP = NTHR / 32u;
    constexpr uint32_t Z = AIR ? (M >> 2) : (M >> 1);  // quads per stage-1 pool (2M positions; AIRPF: one island)
    constexpr uint32_t pool_sh = AIR ? B : B + 1u;
    constexpr int PS = 2 + 4 * D;
    static_assert(B >= 2 && B <= 6 && K1 >= 1 && K1 <= 6 && NTHR % 32u == 0u && 2u * P1 <= 65536u, "k_pass1c plan");
    extern __shared__ __align__(16) unsigned char smem[];
    const Pass1Smem& SL = a.sl;
    float* xs = reinterpret_cast<float*>(smem + SL.xs);
    float* w = reinterpret_cast<float*>(smem + SL.w);
    float* qe = reinterpret_cast<float*>(smem + SL.qe);
    unsigned char* L1 = smem + SL.L1;
    unsigned char* tab = smem + SL.tab;
    double* lv1 = reinterpret_cast<double*>(smem + SL.lv1);
    float* red = reinterpret_cast<float*>(smem + SL.red);
    float* essw = reinterpret_cast<float*>(smem + SL.ess);
    // stages drawn: K1 (the tile depth) except in the resample half of an early-stopped
    // adaptive step, which draws stages 1..min(K1, S*) of the same tile
    const uint32_t kd = RES ? a.k1 : (uint32_t)K1;

    const uint32_t tile = blockIdx.x;
    const uint32_t base = tile * P1;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t c0t = (a.pos0 + base) >> 2;

    // ---- 1. load xhat_{n-1} ------------------------------------------------------------
    float xh[QPT][4 * D];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * NTHR;
        uint32_t src_q = base + 4u * q;  // AIRPF: the quad's position inside the island block it reads
        const float* xsrc = a.x_in;
        if constexpr (AIR)
            if (a.isl_src) {
                const uint32_t gblk = (uint32_t)a.isl_src[src_q >> B];
                if (a.xpeer[0]) {  // sharded (R27): the block's owner, over NVLink when remote
                    xsrc = a.xpeer[gblk >> a.peer_shift];
                    src_q = ((gblk & ((1u << a.peer_shift) - 1u)) << B) | (src_q & (M - 1u));
                } else {
                    src_q = (gblk << B) | (src_q & (M - 1u));
                }
            }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(xsrc + (uint64_t)src_q * D) + c);
            xh[it][4 * c] = t.x;
            xh[it][4 * c + 1] = t.y;
            xh[it][4 * c + 2] = t.z;
            xh[it][4 * c + 3] = t.w;
        }
    }
    float y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = a.y_dev ? (k < a.mp.dy ? __ldg(a.y_dev + k) : 0.0f) : a.y[k];

    // ---- 2. mutate, weight (k_pass1 section 2) ------------------------------------------
    float lw[QPT][4];
    float xr[QPT][4 * D];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * NTHR;
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
            for (int e = 0; e < 4; ++e) {
                if constexpr (KIND == 1 && DIAG) mutate_lg_diag<D>(a.mp, xh[it] + e * D, z + e * D, x + e * D);
                else mutate<D, KIND>(a.mp, xh[it] + e * D, z + e * D, x + e * D);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) x[k] = xh[it][k];
        }
        if constexpr (RES) {  // the weigh half's log-weights, read back
            const float4 t = __ldg(reinterpret_cast<const float4*>(a.lw_in + i0));
            lw[it][0] = t.x;
            lw[it][1] = t.y;
            lw[it][2] = t.z;
            lw[it][3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if constexpr (KIND == 1 && DIAG) lw[it][e] = log_potential_lg_diag<D>(a.mp, y, x + e * D);
                else lw[it][e] = log_potential<D, KIND>(a.mp, y, x + e * D);
            }
        }
        if constexpr (AIR || WEIGH) {  // carried weight (R18; AIRPF2: R26; k_pass1 section 2)
            if (a.carry_mode != 0) {
                float cw[4];
                if (a.carry_mode == 1) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(a.carry_lw + i0));
                    cw[0] = (float)((double)t.x - a.carry_c);
                    cw[1] = (float)((double)t.y - a.carry_c);
                    cw[2] = (float)((double)t.z - a.carry_c);
                    cw[3] = (float)((double)t.w - a.carry_c);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        cw[e] = (float)(__ldg(a.carry_lv + (((((uint64_t)a.pos0 + i0 + e) >> B) >> a.carry_shift) &
                                                            a.carry_mask)) - a.carry_c);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) lw[it][e] += cw[e];
            }
        }
        if constexpr (WEIGH) {  // x_n and lw in natural order for the resample half
            reinterpret_cast<float4*>(a.lw_out + i0)[0] = make_float4(lw[it][0], lw[it][1], lw[it][2], lw[it][3]);
#pragma unroll
            for (int c = 0; c < D; ++c)
                reinterpret_cast<float4*>(a.x_out + (uint64_t)i0 * D)[c] =
                    make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        }
#pragma unroll
        for (int k = 0; k < 4 * D; ++k) xr[it][k] = x[k];
        if constexpr (!WEIGH) {
#pragma unroll
            for (int c = 0; c < D; ++c)
                reinterpret_cast<float4*>(xs)[q * D + c] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        }
    }

    // ---- 3. stage 1 (k_pass1 section 3, Z <= 32: one pool per warp segment) -------------
    float pm[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        float v = fmaxf(fmaxf(lw[it][0], lw[it][1]), fmaxf(lw[it][2], lw[it][3]));
#pragma unroll
        for (uint32_t o = 1; o < Z; o <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
        pm[it] = v;
    }
    float mthr = -CUDART_INF_F;
#pragma unroll
    for (int it = 0; it < QPT; ++it) mthr = fmaxf(mthr, pm[it]);
    float acc[PS], accsq = 0.0f;
#pragma unroll
    for (int k = 0; k < PS; ++k) acc[k] = 0.0f;
    float run[QPT][4], incl[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const bool dead = pm[it] == -CUDART_INF_F;
        const float f = dead ? 0.0f : (QPT == 1 ? 1.0f : exp_ftz(pm[it] - mthr));
        float r = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float c = dead ? 1.0f : exp_ftz(lw[it][e] - pm[it]);  // MUFU ex2: see DESIGN.md §5
            r += c;
            run[it][e] = r;
            const float wf = c * f;
            acc[1] += wf;
            if constexpr (WEIGH) accsq = fmaf(wf, wf, accsq);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float xv = xr[it][e * D + k];
                acc[2 + k] = fmaf(wf, xv, acc[2 + k]);
                acc[2 + D + k] = fmaf(wf * xv, xv, acc[2 + D + k]);
                acc[2 + 2 * D + k] += xv;
                acc[2 + 3 * D + k] = fmaf(xv, xv, acc[2 + 3 * D + k]);
            }
        }
        float v = r;
#pragma unroll
        for (uint32_t o = 1; o < Z; o <<= 1) {
            const float t = __shfl_up_sync(kFull, v, o, Z);
            if ((lane & (Z - 1u)) >= o) v += t;
        }
        incl[it] = v;
    }
    float excl[QPT], tot[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const float up = __shfl_up_sync(kFull, incl[it], 1, Z);
        excl[it] = (lane & (Z - 1u)) ? up : 0.0f;
        tot[it] = __shfl_sync(kFull, incl[it], lane | (Z - 1u));
    }
    const float log2M = logf((float)(4u * Z));
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * NTHR;
        if constexpr (!WEIGH) {
            reinterpret_cast<float4*>(w)[q] =
                make_float4(excl[it] + run[it][0], excl[it] + run[it][1], excl[it] + run[it][2], excl[it] + run[it][3]);
            qe[q] = excl[it] + run[it][3];
        }
        if (((4u * q) & ((1u << pool_sh) - 1u)) == 0u) {
            const double lm = pm[it] == -CUDART_INF_F ? -CUDART_INF : (double)pm[it] + (double)(logf(tot[it]) - log2M);
            lv1[(4u * q) >> pool_sh] = lm;
            if constexpr (AIR) a.logW[((uint64_t)base >> B) + ((4u * q) >> B)] = lm;
        }
    }
    __syncwarp();
    if constexpr (!WEIGH) {
        uint32_t jb[QPT][4];  // byte offset of the quad-end probe base (4 x quad index)
        float tq[QPT][4];
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * NTHR;
            const uint4 blk = AIR ? rng_block(a.key, c0t + q, a.n, kDomainWithin, 0u)
                                  : rng_block(a.key, c0t + q, a.n, kDomainResample, 1u);
            const uint32_t pq = ((4u * q) >> pool_sh) << (pool_sh - 2u);  // the pool's first quad
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
            const float totc = w[4u * pq + 4u * Z - 1u];  // the pool total as stored (reading R3)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                jb[it][e] = 4u * pq;
                tq[it][e] = u01f(r[e]) * totc;
            }
        }
        const unsigned char* qeb = reinterpret_cast<const unsigned char*>(qe);
#pragma unroll
        for (uint32_t step = Z >> 1; step >= 1u; step >>= 1) {
#pragma unroll
            for (int it = 0; it < QPT; ++it)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (*reinterpret_cast<const float*>(qeb + jb[it][e] + 4u * (step - 1u)) <= tq[it][e]) jb[it][e] += 4u * step;
        }
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * NTHR;
            uint32_t lo2[4];  // 2 x tile position of the drawn pool entry
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const unsigned char*>(w) + 4u * jb[it][e]);
                const float t = tq[it][e];
                lo2[e] = 2u * jb[it][e] + 2u * ((uint32_t)(v.x <= t) + (uint32_t)(v.y <= t) + (uint32_t)(v.z <= t));
            }
            *reinterpret_cast<uint2*>(L1 + 8u * q) = make_uint2(lo2[0] | (lo2[1] << 16), lo2[2] | (lo2[3] << 16));
        }
    }

    // per-warp estimate partial (k_pass1 section 3, end)
    {
        float wmax = mthr;
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(kFull, wmax, o));
        const float f = (mthr == -CUDART_INF_F) ? 0.0f : expf(mthr - wmax);
        float sw = acc[1] * f;
        for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(kFull, sw, o);
        float v[4 * D];
#pragma unroll
        for (int k = 0; k < 4 * D; ++k) v[k] = (k < 2 * D) ? acc[2 + k] * f : acc[2 + k];
        const float tot4 = warp_sum_transpose<4 * D>(v, lane);
        constexpr int LV = (4 * D == 4) ? 2 : ((4 * D == 8) ? 3 : ((4 * D == 16) ? 4 : 5));
        if ((lane & ((32u >> LV) - 1u)) == 0u) red[warp * PS + 2 + (lane >> (5 - LV))] = tot4;
        if (lane == 0) {
            red[warp * PS] = wmax;
            red[warp * PS + 1] = sw;
        }
        if constexpr (WEIGH) {
            float sq = accsq * f * f;
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (lane == 0) essw[warp] = sq;
        }
    }
    __syncthreads();  // L1, lv1, red complete

    // ---- 4. V levels 2..K1 and thresholds (k_pass1 section 4), by warp 0 alone (k_pass1
    // has every warp build them redundantly), the thresholds handed to the other warps in
    // shared memory: 4.30 -> 4.12 ms per C4 launch.  AIRPF: level 1 = pair means of the
    // island log-means, every level with 31-bit thresholds (R20), nothing handed over.
    uint32_t* thr_s = reinterpret_cast<uint32_t*>(smem + SL.thr);
    if (warp == 0) {
        constexpr uint32_t npair = T1 >> 1;
        constexpr int tb_bits = AIR ? 1 : B;
        double v;
        if constexpr (AIR) {
            double nv = -CUDART_INF;
            uint32_t Pt = 0u;
            if (lane < npair) pair_level_fast(lv1[2u * lane], lv1[2u * lane + 1u], 1, &nv, &Pt);
            v = nv;
            if (lane < npair) a.thr[level_offset(a.m, 1) + (uint64_t)tile * npair + lane] = Pt;
        } else {
            v = lane < npair ? lv1[lane] : -CUDART_INF;
        }
        if (lane < npair) a.logV[level_offset(a.m, 1) + (uint64_t)tile * npair + lane] = v;
#pragma unroll
        for (int s = 2; s <= K1; ++s) {
            if ((uint32_t)s > kd) break;
            const uint32_t stp = 1u << (s - 2);
            const double vr = __shfl_down_sync(kFull, v, stp);
            const bool act = (lane & (2u * stp - 1u)) == 0u && lane < npair;
            uint32_t Pt;
            double nv;
            pair_level_fast(v, vr, tb_bits, &nv, &Pt);
            if (act) {
                v = nv;
                const uint64_t at = level_offset(a.m, s) + (uint64_t)tile * (T1 >> s) + (lane >> (s - 1));
                a.logV[at] = nv;
                a.thr[at] = Pt;
                if constexpr (!AIR) thr_s[(s - 2) * (T1 / 4u) + (lane >> (s - 1))] = Pt;
            }
        }
    }
    if constexpr (!AIR && !WEIGH) __syncthreads();  // thresholds ready

    // ---- 5. stages 2..K1: entries = source byte offsets, two per word ----------------------
    if constexpr (!AIR && !WEIGH) {
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * NTHR;
        const uint32_t l0 = 4u * q;
        const uint32_t j0 = l0 >> B;
        const uint32_t jb2 = (j0 << (B + 1)) * 0x10001u;
#pragma unroll
        for (int s = 2; s <= K1; ++s) {
            if ((uint32_t)s > kd) break;
            const uint32_t P0 = thr_s[(s - 2) * (T1 / 4u) + (j0 >> s)];
            const uint32_t bitb2 = ((1u << (s - 1)) << (B + 1)) * 0x10001u;
            const uint4 blk = rng_block(a.key, c0t + q, a.n, kDomainResample, (uint32_t)s);
            *reinterpret_cast<uint2*>(tab + (uint32_t)(s - 2) * 2u * P1 + 2u * l0) =
                wsc_pair_entries<B>(blk, P0, jb2 & ~bitb2, bitb2);
        }
    }
    __syncthreads();  // all stage tables ready
    }  // !AIR

    // ---- 6. compose backwards (byte offsets) and write the tile at its stage-K1 positions
    if constexpr (!WEIGH) {
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * NTHR;
        uint32_t t2[4] = {8u * q, 8u * q + 2u, 8u * q + 4u, 8u * q + 6u};
        if constexpr (!AIR) {  // AIRPF: the within-island draw only
#pragma unroll
            for (int s = K1; s >= 2; --s) {
                if ((uint32_t)s > kd) continue;
#pragma unroll
                for (int e = 0; e < 4; ++e) t2[e] = *reinterpret_cast<const uint16_t*>(tab + (uint32_t)(s - 2) * 2u * P1 + t2[e]);
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) t2[e] = *reinterpret_cast<const uint16_t*>(L1 + t2[e]);
        float v[4 * D];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(xs) + t2[e] * (2u * D);
            if constexpr (D == 1) {
                v[e] = *reinterpret_cast<const float*>(src);
            } else if constexpr (D == 2) {
                const float2 t = *reinterpret_cast<const float2*>(src);
                v[2 * e] = t.x;
                v[2 * e + 1] = t.y;
            } else {
#pragma unroll
                for (int c = 0; c < D / 4; ++c) {
                    const float4 t = reinterpret_cast<const float4*>(src)[c];
                    v[e * D + 4 * c] = t.x;
                    v[e * D + 4 * c + 1] = t.y;
                    v[e * D + 4 * c + 2] = t.z;
                    v[e * D + 4 * c + 3] = t.w;
                }
            }
        }
        uint32_t dst = base + 4u * q;
        if (!AIR && a.out_rot) dst = (rotr_group(dst >> B, a.out_rot, a.S) << B) | (dst & (M - 1u));
#pragma unroll
        for (int c = 0; c < D; ++c)
            reinterpret_cast<float4*>(a.x_out + (uint64_t)dst * D)[c] =
                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    }  // !WEIGH

    // ---- 7. warp 0: the tile's estimate partial (k_pass1 section 7) -----------------------
    if (warp == 0) {
        float tmax = -CUDART_INF_F;
#pragma unroll
        for (uint32_t wv = 0; wv < NWARP; ++wv) tmax = fmaxf(tmax, red[wv * PS]);
        for (uint32_t k = lane; k < (uint32_t)PS; k += 32u) {
            double v;
            if (k == 0) {
                v = (double)tmax;
            } else {
                v = 0.0;
#pragma unroll
                for (uint32_t wv = 0; wv < NWARP; ++wv) {
                    const float wm = red[wv * PS];
                    const float f = (k < (uint32_t)(2 + 2 * D)) ? (wm == -CUDART_INF_F ? 0.0f : expf(wm - tmax)) : 1.0f;
                    v += (double)(red[wv * PS + k] * f);
                }
            }
            a.part[(uint64_t)tile * PS + k] = v;
        }
        if constexpr (AIR) {  // AIRPF2: the running max of lw shifts the island ESS sums
            if (lane == 0 && a.ess_lmax) atomicMax(a.ess_lmax, float_order_bits(tmax));
        }
        if constexpr (WEIGH) {  // ESS partial {max, sum w, sum w^2} (R17)
            if (lane == 0) {
                double sw = 0.0, sq = 0.0;
#pragma unroll
                for (uint32_t wv = 0; wv < NWARP; ++wv) {
                    const float wm = red[wv * PS];
                    const double f = (wm == -CUDART_INF_F) ? 0.0 : exp((double)wm - (double)tmax);
                    sw += (double)red[wv * PS + 1] * f;
                    sq += (double)essw[wv] * f * f;
                }
                a.ess_part[(uint64_t)tile * 3] = (double)tmax;
                a.ess_part[(uint64_t)tile * 3 + 1] = sw;
                a.ess_part[(uint64_t)tile * 3 + 2] = sq;
                atomicMax(a.ess_lmax, float_order_bits(tmax));
            }
        }
    }
}

}  // namespace pfk
