// pf_pass1.cuh -- k_pass1: one CTA per tile of T1 = 2^k1 consecutive groups (P1 = T1 M
// particles, T1 <= 64):
//
//   load xhat_{n-1} (coalesced) -> mutate (Alg. 1 l.303) -> log g_n
//    -> stage 1 over the pairs (2p, 2p+1) (Alg. 3 l.346-349): pair max,
//   weights c = exp(lw - max), warp-shuffle segmented inclusive scan, branch-free binary
//   searches of the inverse CDF -> V level 1 per pair; then every warp redundantly builds
//   the tile's V levels 2..k1 and side thresholds in its lanes (log-domain pair means,
//   eq. V_defn_proofs) -> draws of stages 2..k1 into per-stage tables ->
//   each output walks its ancestry back through the tables and writes its state, already
//   moved to its stage-k1 position (composition licensed by Lemma facts_about_Vs (a),
//   PAPER.md:645).
//
// Barriers: B (stage-1 tables, pair V_1 and per-warp estimate partials in shared memory),
// D (all stage tables complete); pairs wider than one warp (M > 64) add two for the
// cross-warp max and scan.
//
// Table entries (TB = 1, M <= 128): stage 1 stores the pool index a in [0, 2M) (the source
// is pair base + a); stage s >= 2 stores side << 7 | index.  TB = 2: the 16-bit tile
// position of the source.
#pragma once
#include <cstdint>
#include <cstring>

#include "pf_args.h"

namespace pfk {

// Sum of NV = 2^v values over the 32 lanes of a warp by recursive halving: after the
// call, lane l holds the total of value (l >> (5 - v)) in v[0].
template <int NV>
__device__ __forceinline__ float warp_sum_transpose(float* v, uint32_t lane) {
    constexpr int LV = NV == 1 ? 0 : (NV == 2 ? 1 : (NV == 4 ? 2 : (NV == 8 ? 3 : (NV == 16 ? 4 : 5))));
    static_assert((1 << LV) == NV && LV <= 5, "NV must be a power of two <= 32");
#pragma unroll
    for (int t = 0; t < LV; ++t) {
        const uint32_t o = 16u >> t;
        const int half = NV >> (t + 1);
        const bool upper = (lane & o) != 0u;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = upper ? v[i] : v[half + i];
            const float keep = upper ? v[half + i] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, o);
        }
    }
#pragma unroll
    for (int t = LV; t < 5; ++t) v[0] += __shfl_xor_sync(kFull, v[0], 16u >> t);
    return v[0];
}

// Shared-memory slot of float4 s of the state tile: a thread writes its quad's D float4s
// (one per store instruction), so without a swizzle the 8 threads of a store phase hit
// only 2 (D = 4) or 1 (D = 8) of the 8 16-byte bank groups.  XOR-ing the low log2(D) bits
// with bits 3.. of the index spreads them over all 8; it stays inside the quad.  Measured
// (profiles/r1_ab_xs_swizzle.txt): AIRPF mode -3.8% and d = 8 -11% per k_pass1 launch,
// the fused d = 4 pass +0.3% (its extra XORs cost more than the conflicts), so it is on
// for d = 8 and the AIRPF mode only.
template <int D, bool ON>
__device__ __forceinline__ uint32_t xs_swz(uint32_t s) {
    if constexpr (ON) return s ^ ((s >> 3) & (uint32_t)(D - 1));
    else return s;
}

// experiment knobs (tools/build_variant.sh): the register budget of the fused mode and the
// largest state block kept in registers for the estimate
#ifndef PF_P1_MINB
#define PF_P1_MINB 1
#endif
#ifndef PF_KEEPX_MAX
#define PF_KEEPX_MAX 32
#endif
// cost probes (experiment builds with -DPF_PROBES only; a.probe from PF_PASS1_PROBE): bit 0
// drops the mutation noise (no Philox, no Box-Muller), bit 1 the stage-1 searches, bit 2
// the stage 2..k1 Philox blocks (identity draws), bit 3 the walk (tile written in place)
#ifdef PF_PROBES
#define PF_PROBE(bit) ((a.probe >> (bit)) & 1u)
#else
#define PF_PROBE(bit) false
#endif

// Launch bounds of the fused d = 4 pass: 128 threads, 6 CTAs per SM (80 registers, no new
// spill): 5.55 -> 5.27 ms per C4 launch against (512, 1) = 96 registers and 5 CTAs per SM;
// 7 CTAs (72 registers) measured 5.42 (profiles/r2_pass1_launch_bounds.txt).  make_plan
// keeps d = 4 at <= 128 threads per CTA below 8 quads per thread; the QPT = 8 instance
// (tiles of M >= 4096 only) keeps the general 512-thread bound.
#ifndef PF_P1_D4_MAXT
#define PF_P1_D4_MAXT 128
#define PF_P1_D4_MINB 6
#endif
constexpr bool pass1_d4_fused(int D, int MODE, int QPT) { return D == 4 && MODE == kPass1Fused && QPT < 8; }
constexpr int pass1_maxt(int D, int MODE, int QPT) { return pass1_d4_fused(D, MODE, QPT) ? PF_P1_D4_MAXT : 512; }
constexpr int pass1_minb(int D, int MODE, int QPT) {
    return (MODE == kPass1Airpf && D >= 4) ? 2 : (pass1_d4_fused(D, MODE, QPT) ? PF_P1_D4_MINB : PF_P1_MINB);
}

template <int D, int KIND, bool DBG, int QPT, int TB, int MODE = kPass1Fused>
__global__ void __launch_bounds__(pass1_maxt(D, MODE, QPT), pass1_minb(D, MODE, QPT)) k_pass1(const __grid_constant__ Pass1Args a) {
    constexpr int PS = 2 + 4 * D;  // partial: max, sw, s1[D], s2[D], p1[D], p2[D]
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t threads = blockDim.x;
    const Pass1Smem& SL = a.sl;
    float* xs = reinterpret_cast<float*>(smem + SL.xs);
    float* w = reinterpret_cast<float*>(smem + SL.w);
    float* qe = reinterpret_cast<float*>(smem + SL.qe);
    float* ey = reinterpret_cast<float*>(smem + SL.ey);
    unsigned char* L1 = smem + SL.L1;
    unsigned char* tab = smem + SL.tab;
    float* chunk = reinterpret_cast<float*>(smem + SL.chunk);
    double* lv1 = reinterpret_cast<double*>(smem + SL.lv1);
    float* red = reinterpret_cast<float*>(smem + SL.red);
    float* essw = reinterpret_cast<float*>(smem + SL.ess);

    const uint32_t P1 = a.P1, M = a.M, b = a.b, nq = P1 >> 2, k1 = a.k1;
    const uint32_t T1 = a.T1;  // groups per tile (<= 64)
    const uint32_t tile = blockIdx.x;
    const uint32_t base = tile * P1;  // N < 2^31
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nwarps = threads >> 5;
    constexpr bool AIR = MODE == kPass1Airpf;
    constexpr bool SWZ = AIR || D == 8;  // swizzled state tile (xs_swz)
    const uint32_t Z = AIR ? (M >> 2) : (M >> 1);  // quads per stage-1 pool (2M positions; AIRPF: one island of M)
    const uint32_t pool_sh = AIR ? b : b + 1u;      // log2 of the pool size
    const uint32_t c0t = (a.pos0 + base) >> 2;  // Philox counter of the tile's first quad

    // ---- 1. load xhat_{n-1} (all slots first: independent loads in flight) -------------
    float xh[QPT][4 * D];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) {  // tiny tiles only (P1 < 128)
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) xh[it][k] = 0.0f;
            continue;
        }
        uint32_t src_q = base + 4u * q;  // AIRPF: the quad's position inside the island block it reads
        const float* xsrc = a.x_in;
        if constexpr (AIR)
            if (a.isl_src) {
                const uint32_t gblk = (uint32_t)a.isl_src[src_q >> b];
                if (a.xpeer[0]) {  // sharded (R27): the block's owner, over NVLink when remote
                    xsrc = a.xpeer[gblk >> a.peer_shift];
                    src_q = ((gblk & ((1u << a.peer_shift) - 1u)) << b) | (src_q & (M - 1u));
                } else {
                    src_q = (gblk << b) | (src_q & (M - 1u));
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

    float y[8];  // after the state loads: its latency overlaps theirs
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = a.y_dev ? (k < a.mp.dy ? __ldg(a.y_dev + k) : 0.0f) : a.y[k];

    // ---- 2. mutate, weight ---------------------------------------------------------------
    float lw[QPT][4];
    constexpr bool KEEPX = 4 * D * QPT <= PF_KEEPX_MAX;  // states stay in registers for the estimate
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
                if (PF_PROBE(0)) {
#pragma unroll
                    for (int w = 0; w < 4; ++w) z[4 * j + w] = 0.0f;
                    continue;
                }
                const uint4 blk = rng_block(a.key, ((a.pos0 + i0) >> 2) * D + j, a.n, kDomainMutate, 0u);
                normals4(blk, z + 4 * j);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) mutate<D, KIND>(a.mp, xh[it] + e * D, z + e * D, x + e * D);
        } else {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) x[k] = xh[it][k];
        }
        if constexpr (MODE == kPass1Resample) {
            const float4 t = valid ? __ldg(reinterpret_cast<const float4*>(a.lw_in + i0))
                                   : make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
            lw[it][0] = t.x;
            lw[it][1] = t.y;
            lw[it][2] = t.z;
            lw[it][3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) lw[it][e] = valid ? log_potential<D, KIND>(a.mp, y, x + e * D) : -CUDART_INF_F;
        }
        if constexpr (MODE == kPass1Weigh || MODE == kPass1Airpf) {  // carried weight (R18; AIRPF2: R26)
            if (valid && a.carry_mode != 0) {
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
                        cw[e] = (float)(__ldg(a.carry_lv + (((((uint64_t)a.pos0 + i0 + e) >> b) >> a.carry_shift) &
                                                            a.carry_mask)) - a.carry_c);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) lw[it][e] += cw[e];
            }
            if (MODE == kPass1Weigh && valid) {
                reinterpret_cast<float4*>(a.lw_out + i0)[0] = make_float4(lw[it][0], lw[it][1], lw[it][2], lw[it][3]);
#pragma unroll
                for (int c = 0; c < D; ++c)
                    reinterpret_cast<float4*>(a.x_out + (uint64_t)i0 * D)[c] =
                        make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
            }
        }
        if constexpr (KEEPX) {
#pragma unroll
            for (int k = 0; k < 4 * D; ++k) xr[it][k] = valid ? x[k] : 0.0f;
        }
        if (!valid) continue;
        if constexpr (!(MODE == kPass1Weigh && KEEPX)) {  // the weigh pass has no walk: the tile is read
#pragma unroll                                              // back only by a non-KEEPX estimate
            for (int c = 0; c < D; ++c)
                reinterpret_cast<float4*>(xs)[xs_swz<D, SWZ>(q * D + c)] =
                    make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        }
        if constexpr (DBG) {
#pragma unroll
            for (int c = 0; c < D; ++c)
                reinterpret_cast<float4*>(a.dbg_x + (uint64_t)i0 * D)[c] =
                    make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
            reinterpret_cast<float4*>(a.dbg_lw + i0)[0] = make_float4(lw[it][0], lw[it][1], lw[it][2], lw[it][3]);
        }
    }

    // ---- 3. stage 1: pair max, weights, segmented scan, inverse-CDF draws --------------
    const uint32_t zw = Z < 32u ? Z : 32u;
    float pm[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        float v = fmaxf(fmaxf(lw[it][0], lw[it][1]), fmaxf(lw[it][2], lw[it][3]));
        for (uint32_t o = 1; o < zw; o <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
        pm[it] = v;
    }
    if (Z > 32u) {  // a pair spans several warp-chunks of 32 quads
#pragma unroll
        for (int it = 0; it < QPT; ++it)
            if (lane == 0 && tid + it * threads < nq) chunk[(tid + it * threads) >> 5] = pm[it];
        __syncthreads();
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t c0 = ((tid + it * threads) >> 5) & ~((Z >> 5) - 1u);
            float v = -CUDART_INF_F;
            for (uint32_t c = lane; c < (Z >> 5); c += 32u) v = fmaxf(v, chunk[c0 + c]);
            for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
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
    float acc[PS], accsq = 0.0f;
#pragma unroll
    for (int k = 0; k < PS; ++k) acc[k] = 0.0f;
    float run[QPT][4], incl[QPT];
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        const bool valid = q < nq;
        const bool dead = pm[it] == -CUDART_INF_F;  // all of the pair's weights are zero
        const float f = (dead || !valid) ? 0.0f : (QPT == 1 ? 1.0f : exp_ftz(pm[it] - mthr));
        float r = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float c = dead ? 1.0f : exp_ftz(lw[it][e] - pm[it]);  // MUFU ex2: see DESIGN.md §5
            r += c;
            run[it][e] = r;
            const float wf = c * f;
            acc[1] += wf;
            if constexpr (MODE == kPass1Weigh) accsq = fmaf(wf, wf, accsq);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                float xv;
                if constexpr (KEEPX) xv = xr[it][e * D + k];
                else {
                    const uint32_t fi = (4u * q + e) * D + k;
                    xv = valid ? xs[(xs_swz<D, SWZ>(fi >> 2) << 2) | (fi & 3u)] : 0.0f;
                }
                acc[2 + k] = fmaf(wf, xv, acc[2 + k]);
                acc[2 + D + k] = fmaf(wf * xv, xv, acc[2 + D + k]);
                acc[2 + 2 * D + k] += xv;
                acc[2 + 3 * D + k] = fmaf(xv, xv, acc[2 + 3 * D + k]);
            }
        }
        float v = r;  // inclusive scan of quad totals within the segment (<= 32 quads)
        for (uint32_t o = 1; o < zw; o <<= 1) {
            const float t = __shfl_up_sync(kFull, v, o, zw);
            if ((lane & (zw - 1u)) >= o) v += t;
        }
        incl[it] = v;
    }
    float excl[QPT], tot[QPT];
    if (Z <= 32u) {
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const float up = __shfl_up_sync(kFull, incl[it], 1, Z);
            excl[it] = (lane & (Z - 1u)) ? up : 0.0f;
            tot[it] = __shfl_sync(kFull, incl[it], lane | (Z - 1u));
        }
    } else {
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const float up = __shfl_up_sync(kFull, incl[it], 1);
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
                before += __shfl_xor_sync(kFull, before, o);
                all += __shfl_xor_sync(kFull, all, o);
            }
            excl[it] += before;
            tot[it] = all;
        }
    }
    const float log2M = logf((float)(4u * Z));  // log of the pool size
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) continue;
        reinterpret_cast<float4*>(w)[q] =
            make_float4(excl[it] + run[it][0], excl[it] + run[it][1], excl[it] + run[it][2], excl[it] + run[it][3]);
        qe[q] = excl[it] + run[it][3];
        if (Z > 32u && MODE != kPass1Weigh) {
            // pools of > 32 quads: the quad ends again in BFS (Eytzinger) order of the search
            // tree -- the probe of level L, node m (quad m 2 step + step - 1, step = Z >> (L+1))
            // at pool offset 2^L - 1 + m -- so one level's probes are consecutive words (the
            // flat order put every probe of a level with step >= 32 in one bank)
            const uint32_t j = q & (Z - 1u);
            if (j + 1u < Z) {
                const uint32_t v = j + 1u, ls = __ffs(v) - 1u, lz = __ffs(Z) - 1u;
                ey[(q - j) + (1u << (lz - 1u - ls)) - 1u + (v >> (ls + 1u))] = excl[it] + run[it][3];
            }
        }
        if (((4u * q) & ((1u << pool_sh) - 1u)) == 0u) {  // first quad of its pool: log mean of the pool
            const double lm = pm[it] == -CUDART_INF_F ? -CUDART_INF : (double)pm[it] + (double)(logf(tot[it]) - log2M);
            lv1[(4u * q) >> pool_sh] = lm;
            if constexpr (AIR) a.logW[((uint64_t)base >> b) + ((4u * q) >> b)] = lm;
        }
    }
    if (Z <= 32u) __syncwarp();  // a pair's CDF was written by this warp
    else __syncthreads();
    if constexpr (MODE != kPass1Weigh) {  // all QPT x 4 branch-free binary searches advance together
        uint32_t lo[QPT][4];
        float tq[QPT][4];
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * threads;
            const bool valid = q < nq;
            const uint4 blk = AIR ? rng_block(a.key, c0t + q, a.n, kDomainWithin, 0u)
                                  : rng_block(a.key, c0t + q, a.n, kDomainResample, 1u);
            const uint32_t pb = valid ? (((4u * q) >> pool_sh) << pool_sh) : 0u;
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
            // the search target scales the pool total AS STORED in the CDF (same summation
            // order as the entries it is compared with), so t <= C_{2M-1} and a zero-weight
            // last entry can never be selected (reading R3)
            const float totc = valid ? w[pb + 4u * Z - 1u] : 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                lo[it][e] = pb;
                tq[it][e] = valid ? u01f(r[e]) * totc : -1.0f;
            }
        }
        // two levels: the quad among the pool's Z quad ends (qe, consecutive words: <= 32
        // of them hit distinct banks), then the entry inside the quad from one 16-byte load
        // a = 4 j + #{e < 3 : C_{4j+e} <= t} with j = #{quads j' < Z-1 : C_{4j'+3} <= t}
        // -- the same count as the flat binary search, in 5 conflict-free steps plus one
        // vector load instead of 7 scalar steps (2M = 128)
        uint32_t jq[QPT][4];
#pragma unroll
        for (int it = 0; it < QPT; ++it)
#pragma unroll
            for (int e = 0; e < 4; ++e) jq[it][e] = lo[it][e] >> 2;  // the pool's first quad
        if (Z <= 32u) {
            for (uint32_t step = Z >> 1; step >= 1u && !PF_PROBE(1); step >>= 1) {
#pragma unroll
                for (int it = 0; it < QPT; ++it)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (qe[jq[it][e] + step - 1u] <= tq[it][e]) jq[it][e] += step;
            }
        } else {  // the same probes, read from the BFS-ordered copy (level L, node jr >> (lz - L))
            const uint32_t lz = __ffs(Z) - 1u;
            uint32_t jr[QPT][4];
#pragma unroll
            for (int it = 0; it < QPT; ++it)
#pragma unroll
                for (int e = 0; e < 4; ++e) jr[it][e] = 0u;
            for (uint32_t L = 0; L < lz && !PF_PROBE(1); ++L) {
                const uint32_t step = Z >> (L + 1u), sh = lz - L, lvl = (1u << L) - 1u;
#pragma unroll
                for (int it = 0; it < QPT; ++it)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (ey[jq[it][e] + lvl + (jr[it][e] >> sh)] <= tq[it][e]) jr[it][e] += step;
            }
#pragma unroll
            for (int it = 0; it < QPT; ++it)
#pragma unroll
                for (int e = 0; e < 4; ++e) jq[it][e] += jr[it][e];
        }
#pragma unroll
        for (int it = 0; it < QPT; ++it)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float4 v = reinterpret_cast<const float4*>(w)[jq[it][e]];
                const float t = tq[it][e];
                lo[it][e] = 4u * jq[it][e] + (uint32_t)(v.x <= t) + (uint32_t)(v.y <= t) + (uint32_t)(v.z <= t);
            }
#pragma unroll
        for (int it = 0; it < QPT; ++it) {
            const uint32_t q = tid + it * threads;
            if (q >= nq) continue;
            if constexpr (DBG)
                reinterpret_cast<int4*>(a.dbg_anc + base + 4u * q)[0] =
                    make_int4((int)(a.pos0 + base + lo[it][0]), (int)(a.pos0 + base + lo[it][1]),
                              (int)(a.pos0 + base + lo[it][2]), (int)(a.pos0 + base + lo[it][3]));
            if constexpr (TB == 1) {
                const uint32_t pm2 = 4u * Z - 1u;  // pool index a = lo - pool base
                *reinterpret_cast<uint32_t*>(L1 + 4u * q) = (lo[it][0] & pm2) | ((lo[it][1] & pm2) << 8) |
                                                             ((lo[it][2] & pm2) << 16) | ((lo[it][3] & pm2) << 24);
            } else {
                *reinterpret_cast<uint2*>(L1 + 8u * q) =
                    make_uint2(lo[it][0] | (lo[it][1] << 16), lo[it][2] | (lo[it][3] << 16));
            }
        }
    }

    // per-warp estimate partial: rescale to the warp max, then a transposed warp sum
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
        if constexpr (MODE == kPass1Weigh) {
            float sq = accsq * f * f;
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (lane == 0) essw[warp] = sq;
        }
    }
    __syncthreads();  // B: L1, lv1, red complete

    // ---- 4. V levels 2..k1 and thresholds, redundantly in every warp (lane i holds
    //         block i << (s-2) of level s-1 before step s) -----------------------------
    uint32_t thr[7];
    {
        const uint32_t npair = T1 >> 1;
        const int tb_bits = AIR ? 1 : (int)b;  // threshold resolution 2^-(32-tb_bits) (R1; AIRPF R20)
        double v;
        if constexpr (AIR) {  // level 1 = pair means of the island log-means; stage-1 island thresholds
            double nv = -CUDART_INF;
            uint32_t Pt = 0u;
            if (lane < npair) pair_level_fast(lv1[2u * lane], lv1[2u * lane + 1u], 1, &nv, &Pt);
            v = nv;
            if (warp == 0 && lane < npair) a.thr[level_offset(a.m, 1) + (uint64_t)tile * npair + lane] = Pt;
        } else {
            v = lane < npair ? lv1[lane] : -CUDART_INF;
        }
        if (warp == 0 && lane < npair) a.logV[level_offset(a.m, 1) + (uint64_t)tile * npair + lane] = v;
#pragma unroll
        for (int s = 2; s <= 6; ++s) {
            thr[s] = 0u;
            if ((uint32_t)s > k1) continue;
            const uint32_t stp = 1u << (s - 2);
            const double vr = __shfl_down_sync(kFull, v, stp);
            const bool act = (lane & (2u * stp - 1u)) == 0u && lane < npair;
            uint32_t Pt;
            double nv;
            pair_level_fast(v, vr, tb_bits, &nv, &Pt);
            thr[s] = Pt;
            if (act) {
                v = nv;
                if (warp == 0) {
                    const uint64_t at = level_offset(a.m, s) + (uint64_t)tile * (T1 >> s) + (lane >> (s - 1));
                    a.logV[at] = nv;
                    a.thr[at] = Pt;
                }
            }
        }
    }

    if constexpr (MODE != kPass1Weigh) {  // sections 5-6: the draws and the walk
    // ---- 5. stages 2..k1: every draw depends only on its word and the threshold ---------
    const uint32_t mask = M - 1u;
    if constexpr (!AIR) {
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        const bool valid = q < nq;
        const uint32_t l0 = valid ? 4u * q : 0u;
        const uint32_t j0 = l0 >> b, j1 = (l0 + 2u) >> b;  // quad groups (differ only when M == 2)
#pragma unroll
        for (int s = 2; s <= 6; ++s) {
            if ((uint32_t)s > k1) continue;
            const uint32_t P0 = __shfl_sync(kFull, thr[s], (j0 >> s) << (s - 1));
            const uint32_t Pq1 = __shfl_sync(kFull, thr[s], (j1 >> s) << (s - 1));
            if (!valid) continue;
            const uint32_t bit = 1u << (s - 1);
            const uint4 blk = PF_PROBE(2) ? make_uint4(q, q + 1u, q + 2u, q + 3u)
                                          : rng_block(a.key, c0t + q, a.n, kDomainResample, (uint32_t)s);
            const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
            uint32_t en[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t je = e < 2 ? j0 : j1;
                const bool hi = (r[e] >> b) >= (e < 2 ? P0 : Pq1);
                if constexpr (TB == 1) en[e] = (r[e] & mask) | (hi ? 0x80u : 0u);
                else en[e] = ((hi ? (je | bit) : (je & ~bit)) << b) | (r[e] & mask);
                if constexpr (DBG) {
                    const uint32_t src = ((hi ? (je | bit) : (je & ~bit)) << b) | (r[e] & mask);
                    a.dbg_anc[(uint64_t)(s - 1) * a.N + base + l0 + e] = (int32_t)(a.pos0 + base + src);
                }
            }
            unsigned char* Ts = tab + (uint32_t)(s - 2) * P1 * TB;
            if constexpr (TB == 1)
                *reinterpret_cast<uint32_t*>(Ts + l0) = en[0] | (en[1] << 8) | (en[2] << 16) | (en[3] << 24);
            else
                *reinterpret_cast<uint2*>(Ts + 2u * l0) = make_uint2(en[0] | (en[1] << 16), en[2] | (en[3] << 16));
        }
    }
    __syncthreads();  // D: all stage tables ready
    }  // !AIR

    // ---- 6. compose backwards and write the tile at its stage-k1 positions ------------
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = tid + it * threads;
        if (q >= nq) continue;
        uint32_t tp[4] = {4u * q, 4u * q + 1u, 4u * q + 2u, 4u * q + 3u};
        // (keeping stage k1's own entries in registers instead of the table measured 3%
        // slower: the extra live registers of the fused d = 4 kernel, profiles/r2_bench_C4_z.json)
        for (uint32_t s = AIR ? 1u : k1; s >= 2u && !PF_PROBE(3); --s) {  // AIRPF: the within-island draw only
            const unsigned char* Ts = tab + (s - 2u) * P1 * TB;
            if constexpr (TB == 1) {
                const uint32_t sh = s - 1u + b;
                const uint32_t keep = ~(mask | (1u << sh));
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t en = Ts[tp[e]];
                    tp[e] = (tp[e] & keep) | (en & 0x7fu) | ((en >> 7) << sh);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) tp[e] = reinterpret_cast<const uint16_t*>(Ts)[tp[e]];
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if constexpr (TB == 1) tp[e] = (tp[e] & ~(4u * Z - 1u)) | L1[tp[e]];
            else tp[e] = reinterpret_cast<const uint16_t*>(L1)[tp[e]];
        }
        float v[4 * D];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if constexpr (D == 1) {
                v[e] = xs[tp[e]];
            } else if constexpr (D == 2) {
                const float2 t = reinterpret_cast<const float2*>(xs)[(xs_swz<D, SWZ>(tp[e] >> 1) << 1) | (tp[e] & 1u)];
                v[2 * e] = t.x;
                v[2 * e + 1] = t.y;
            } else {
#pragma unroll
                for (int c = 0; c < D / 4; ++c) {
                    const float4 t = reinterpret_cast<const float4*>(xs)[xs_swz<D, SWZ>(tp[e] * (D / 4) + c)];
                    v[e * D + 4 * c] = t.x;
                    v[e * D + 4 * c + 1] = t.y;
                    v[e * D + 4 * c + 2] = t.z;
                    v[e * D + 4 * c + 3] = t.w;
                }
            }
        }
        uint32_t dst = base + 4u * q;
        if (a.out_rot) dst = (rotr_group(dst >> b, a.out_rot, a.S) << b) | (dst & (M - 1u));
#pragma unroll
        for (int c = 0; c < D; ++c)
            reinterpret_cast<float4*>(a.x_out + (uint64_t)dst * D)[c] =
                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    }

    // ---- 7. warp 0: the tile's estimate partial (off the critical path) ----------------
    if (warp == 0) {
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
        if constexpr (MODE == kPass1Weigh) {  // ESS partial {max, sum w, sum w^2} (R17)
            if (lane == 0) {
                double sw = 0.0, sq = 0.0;
                for (uint32_t wv = 0; wv < nwarps; ++wv) {
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
        if constexpr (MODE == kPass1Airpf) {  // AIRPF2: the running max of lw shifts the island ESS sums
            if (lane == 0 && a.ess_lmax) atomicMax(a.ess_lmax, float_order_bits(tmax));
        }
    }
}

}  // namespace pfk
