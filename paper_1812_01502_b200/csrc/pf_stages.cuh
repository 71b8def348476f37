// pf_stages.cuh -- k_stages: butterfly stages s0 .. s0+k-1 (s0 >= 2) over one tile held in
// shared memory, moving the particle states once per pass.
//
// Tile: the 2^k groups that the butterfly pairs at stages s0..s0+k-1, i.e. global groups
//   g(j) = tlo | (j << (s0-1)) | thi,   j in [0, 2^k)   (tile-local group index j)
// so stage s0+st pairs j with j ^ 2^st (eq. `A matrices`; pairing by
// Lemma `facts about A`).  Tile position tp = (j << b) | i, i < M = 2^b.
//
//   A  the tile's states (stage s0-1) are copied global -> shared with TMA bulk copies
//      (one per group of M contiguous particles);
//   B  every stage's draws: a draw depends only on its Philox word and the stage's side
//      threshold (reading R1; for s >= 2, V_{s-1} is constant over each group,
//      SURVEY.md App. A.2), never on another stage, so all k stages are drawn without
//      barriers into per-stage tables T_st[tp]: 1 byte (side << 7 | index) when M <= 128,
//      else the 16-bit tile position of the source;
//   C  each output walks its ancestry back, tp -> a_{s0+k-1}(tp) -> ... -> a_{s0}(.)
//      (the composition of Alg. 3's stages, licensed by Lemma facts_about_Vs (a),
//      PAPER.md:645), reads that state from shared memory and writes it coalesced.
// The kernel is persistent and software-pipelined (see k_stages below).
//
// Measured and rejected: spreading a larger tile over a thread-block cluster and reading
// the sources through DSMEM (random 16-byte remote reads ran ~4x slower than a whole
// extra HBM pass; profiles/r1_ncu_k_stages_v1_cluster_experiment.txt).
#pragma once
#include <cstdint>

#include "pf_args.h"

namespace pfk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async_bytes(void* smem_dst, const void* gsrc, int bytes) {
    const uint32_t d = smem_u32(smem_dst);
    if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
    else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc));
}

// mbarrier + TMA bulk copy (global -> shared, completion counted in bytes on the barrier)
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// The same wait with a suspend-time hint: a waiting warp sleeps until the phase completes
// (or the hint elapses) instead of spinning -- in k_stages_ws the spinning waiters took
// ~30% of the issued instructions from the working warps (ncu source page)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns = 1000000u) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct StageTile {
    uint32_t tlo, thi;
};

__device__ __forceinline__ StageTile stage_tile_geom(const StageArgs& a, uint32_t t) {
    StageTile g;
    g.tlo = t & ((1u << a.lowbits) - 1u);
    g.thi = (t >> a.lowbits) << (a.lowbits + a.k);
    return g;
}

// Copies of tile t's states (stage s0-1): one TMA bulk copy per group (M contiguous
// particles) completing on `bar`, or per-thread cp.async when a group is < 16 bytes.
template <typename T>
__device__ __forceinline__ void stage_states_load(const StageArgs& a, const StageTile& g, T* xs, uint64_t* bar) {
    const uint32_t b = a.b, lowbits = a.lowbits, G = 1u << a.k;
    constexpr uint32_t SB = (uint32_t)sizeof(T);
    const uint32_t gbytes = a.M * SB;
    const char* gin = reinterpret_cast<const char*>(a.pin);
    char* sdst = reinterpret_cast<char*>(xs);
    if (gbytes >= 16u) {
        if (threadIdx.x < 32u) {
            if (threadIdx.x == 0) mbar_expect_tx(bar, G * gbytes);
            __syncwarp();
            for (uint32_t j = threadIdx.x; j < G; j += 32u) {
                const uint64_t gg = g.tlo | (j << lowbits) | g.thi;
                bulk_g2s(sdst + (size_t)j * gbytes, gin + (gg << b) * SB, gbytes, bar);
            }
        }
    } else {  // d = 1, M = 2: 8-byte groups
        for (uint32_t j = threadIdx.x; j < G; j += blockDim.x) {
            const uint64_t gg = g.tlo | (j << lowbits) | g.thi;
            cp_async_bytes(sdst + (size_t)j * gbytes, gin + (gg << b) * SB, (int)gbytes);
        }
    }
}

// Tile t's thresholds: stage st has 2^{k-st-1} entries at offset 2^k - 2^{k-st}.
__device__ __forceinline__ void stage_thresholds_load(const StageArgs& a, const StageTile& g, uint32_t* ths) {
    const uint32_t k = a.k, E = (1u << k) - 1u;
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        const uint32_t u = (1u << k) - e;
        const uint32_t st = k - (32u - __clz(u - 1u));
        const uint32_t off = (1u << k) - (1u << (k - st));
        const uint32_t s = a.s0 + st;
        cp_async_bytes(ths + e, a.thr + level_offset(a.m, (int)s) + (g.thi >> s) + (e - off), 4);
    }
}

// B: all k stages' draws of the thread's quads of one tile into the tables.
template <int TB, bool DBG, int QPT>
__device__ __forceinline__ void stage_draws(const StageArgs& a, const StageTile& g, const uint32_t* ths,
                                            unsigned char* tabs) {
    const uint32_t M = a.M, b = a.b, k = a.k, kd = a.kd, P = a.P, mask = M - 1u, nq = P >> 2, lowbits = a.lowbits;
    const uint32_t tlo = g.tlo, thi = g.thi;
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        if (M >= 4u) {  // the quad lies in one group: one Philox block per stage
            const uint32_t j = l0 >> b;
            const uint32_t gp0 = ((tlo | (j << lowbits) | thi) << b) | (l0 & mask);
            const uint32_t c0 = (a.pos0 + gp0) >> 2;
            uint32_t toff = 0;  // offset of stage st's thresholds
            for (uint32_t st = 0; st < kd; ++st) {
                const uint32_t s = a.s0 + st, bit = 1u << st;
                const uint4 blk = rng_block(a.key, c0, a.n, kDomainResample, s);
                const uint32_t Pt = ths[toff + (j >> (st + 1))];
                toff += (1u << k) >> (st + 1);
                const uint32_t rw[4] = {blk.x, blk.y, blk.z, blk.w};
                const uint32_t blo = (j & ~bit) << b, bhi = (j | bit) << b;
                uint32_t en[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool hi = (rw[e] >> b) >= Pt;
                    if constexpr (TB == 1) en[e] = (rw[e] & mask) | (hi ? 0x80u : 0u);
                    else en[e] = (hi ? bhi : blo) | (rw[e] & mask);
                }
                if constexpr (TB == 1)
                    *reinterpret_cast<uint32_t*>(tabs + st * P + l0) = en[0] | (en[1] << 8) | (en[2] << 16) | (en[3] << 24);
                else
                    *reinterpret_cast<uint2*>(tabs + 2u * (st * P + l0)) = make_uint2(en[0] | (en[1] << 16), en[2] | (en[3] << 16));
                if constexpr (DBG) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool hi = (rw[e] >> b) >= Pt;
                        const uint32_t jj = hi ? (j | bit) : (j & ~bit);
                        const uint32_t gsrc = ((tlo | (jj << lowbits) | thi) << b) | (rw[e] & mask);
                        a.dbg_anc[(uint64_t)(s - 1) * a.N + gp0 + e] = (int32_t)(a.pos0 + gsrc);
                    }
                }
            }
        } else {  // M == 2: the quad spans tile groups j0, j0+1 (two Philox blocks per stage)
            const uint32_t j0 = l0 >> 1;
            uint32_t gpa[2], c0[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                gpa[h] = (tlo | ((j0 + h) << lowbits) | thi) << 1;
                c0[h] = (a.pos0 + gpa[h]) >> 2;
            }
            uint32_t toff = 0;
            for (uint32_t st = 0; st < kd; ++st) {
                const uint32_t s = a.s0 + st, bit = 1u << st;
                uint32_t en[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t j = j0 + h;
                    const uint4 blk = rng_block(a.key, c0[h], a.n, kDomainResample, s);
                    const bool upper = ((a.pos0 + gpa[h]) & 2u) != 0u;
                    const uint32_t w0 = upper ? blk.z : blk.x, w1 = upper ? blk.w : blk.y;
                    const uint32_t Pt = ths[toff + (j >> (st + 1))];
                    const uint32_t w[2] = {w0, w1};
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const bool hi = (w[e] >> 1) >= Pt;
                        if constexpr (TB == 1) en[2 * h + e] = (w[e] & 1u) | (hi ? 0x80u : 0u);
                        else en[2 * h + e] = ((hi ? (j | bit) : (j & ~bit)) << 1) | (w[e] & 1u);
                        if constexpr (DBG) {
                            const uint32_t jj = hi ? (j | bit) : (j & ~bit);
                            const uint32_t gsrc = ((tlo | (jj << lowbits) | thi) << 1) | (w[e] & 1u);
                            a.dbg_anc[(uint64_t)(s - 1) * a.N + gpa[h] + e] = (int32_t)(a.pos0 + gsrc);
                        }
                    }
                }
                toff += (1u << k) >> (st + 1);
                if constexpr (TB == 1)
                    *reinterpret_cast<uint32_t*>(tabs + st * P + l0) = en[0] | (en[1] << 8) | (en[2] << 16) | (en[3] << 24);
                else
                    *reinterpret_cast<uint2*>(tabs + 2u * (st * P + l0)) = make_uint2(en[0] | (en[1] << 16), en[2] | (en[3] << 16));
            }
        }
    }
}

// C: each of the thread's outputs walks back through the tables, reads its source state
// and writes it coalesced.
template <typename T, int TB, int QPT>
__device__ __forceinline__ void stage_walk(const StageArgs& a, const StageTile& g, const T* xs,
                                           const unsigned char* tabs) {
    const uint32_t M = a.M, b = a.b, kd = a.kd, P = a.P, mask = M - 1u, nq = P >> 2, lowbits = a.lowbits;
    T* pout = reinterpret_cast<T*>(a.pout);
#pragma unroll
    for (int it = 0; it < QPT; ++it) {
        const uint32_t q = threadIdx.x + it * blockDim.x;
        if (q >= nq) break;
        const uint32_t l0 = 4u * q;
        uint32_t tp[4] = {l0, l0 + 1u, l0 + 2u, l0 + 3u};
        for (int st = (int)kd - 1; st >= 0; --st) {
            if constexpr (TB == 1) {
                const unsigned char* Ts = tabs + (uint32_t)st * P;
                const uint32_t sh = (uint32_t)st + b;
                const uint32_t keep = ~(mask | (1u << sh));
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t en = Ts[tp[e]];
                    tp[e] = (tp[e] & keep) | (en & 0x7fu) | ((en >> 7) << sh);
                }
            } else {
                const uint16_t* Ts = reinterpret_cast<const uint16_t*>(tabs) + (uint32_t)st * P;
#pragma unroll
                for (int e = 0; e < 4; ++e) tp[e] = Ts[tp[e]];
            }
        }
        Vec4<T> v;
#pragma unroll
        for (int e = 0; e < 4; ++e) v.v[e] = xs[tp[e]];
        const uint32_t j = l0 >> b;
        uint32_t gp0 = ((g.tlo | (j << lowbits) | g.thi) << b) | (l0 & mask);
        if (M >= 4u) {
            if (a.out_rot) gp0 = (rotr_group(gp0 >> b, a.out_rot, a.out_S) << b) | (gp0 & mask);
            *reinterpret_cast<Vec4<T>*>(pout + gp0) = v;
        } else {
            const uint32_t gp1 = (g.tlo | ((j + 1u) << lowbits) | g.thi) << 1;
            pout[gp0] = v.v[0];
            pout[gp0 + 1] = v.v[1];
            pout[gp1] = v.v[2];
            pout[gp1 + 1] = v.v[3];
        }
    }
}

// Persistent and software-pipelined: CTA c owns tiles t_i = c + i gridDim.x.  Iteration i
// walks and writes tile t_{i-1} (tables and states of slot (i-1) & 1) while drawing tile
// t_i into the other table set; the states of t_i are copied (TMA bulk) during iteration
// i and consumed in iteration i+1; the thresholds of t_{i+1} arrive during iteration i.
// Even warps walk first and odd warps draw first, so the Philox-heavy draws and the
// shared-memory-heavy walk overlap on every SM sub-partition.  One barrier per tile.
template <typename T, int TB, bool DBG, int QPT>
__global__ void __launch_bounds__(1024, 1) k_stages(const __grid_constant__ StageArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k = a.k, P = a.P;
    const uint32_t ntiles = (uint32_t)(a.N / P);
    const uint32_t stb = (P * (uint32_t)sizeof(T) + 15u) & ~15u;
    const uint32_t ttb = (k * P * TB + 15u) & ~15u;
    const uint32_t nb = a.pipe ? 2u : 1u;
    unsigned char* tab0 = smem + nb * stb;
    uint32_t* th0 = reinterpret_cast<uint32_t*>(tab0 + nb * ttb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(th0 + (nb << k));
    auto xbuf = [&](uint32_t sl) { return reinterpret_cast<T*>(smem + sl * stb); };
    auto tbuf = [&](uint32_t sl) { return tab0 + sl * ttb; };
    auto thbuf = [&](uint32_t sl) { return th0 + (sl << k); };
    const bool bulk = a.M * (uint32_t)sizeof(T) >= 16u;

    const uint32_t t0 = blockIdx.x;
    if (t0 >= ntiles) return;
    const uint32_t nt = (ntiles - t0 + gridDim.x - 1u) / gridDim.x;  // tiles of this CTA
    if (threadIdx.x == 0) {
        mbar_init(bars, 1u);
        mbar_init(bars + 1, 1u);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (!a.pipe) {  // one buffer: load, draw, walk, tile after tile
        for (uint32_t i = 0; i < nt; ++i) {
            const StageTile g = stage_tile_geom(a, t0 + i * gridDim.x);
            stage_states_load<T>(a, g, xbuf(0u), bars);
            stage_thresholds_load(a, g, thbuf(0u));
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
            __syncthreads();
            stage_draws<TB, DBG, QPT>(a, g, thbuf(0u), tbuf(0u));
            if (bulk) mbar_wait(bars, i & 1u);
            __syncthreads();
            stage_walk<T, TB, QPT>(a, g, xbuf(0u), tbuf(0u));
            __syncthreads();
        }
        return;
    }
    stage_thresholds_load(a, stage_tile_geom(a, t0), thbuf(0u));
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
    __syncthreads();

    const bool walk_first = ((threadIdx.x >> 5) & 1u) == 0u;
    for (uint32_t i = 0; i <= nt; ++i) {
        const uint32_t sl = i & 1u;
        const StageTile gi = stage_tile_geom(a, t0 + i * gridDim.x);
        const StageTile gp = stage_tile_geom(a, t0 + (i - 1u) * gridDim.x);
        if (i < nt) stage_states_load<T>(a, gi, xbuf(sl), bars + sl);      // consumed in iteration i+1
        if (i + 1 < nt) stage_thresholds_load(a, stage_tile_geom(a, t0 + (i + 1) * gridDim.x), thbuf(sl ^ 1u));
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (i >= 1u && bulk) mbar_wait(bars + (sl ^ 1u), ((i - 1u) >> 1) & 1u);
        if (walk_first) {
            if (i >= 1u) stage_walk<T, TB, QPT>(a, gp, xbuf(sl ^ 1u), tbuf(sl ^ 1u));
            if (i < nt) stage_draws<TB, DBG, QPT>(a, gi, thbuf(sl), tbuf(sl));
        } else {
            if (i < nt) stage_draws<TB, DBG, QPT>(a, gi, thbuf(sl), tbuf(sl));
            if (i >= 1u) stage_walk<T, TB, QPT>(a, gp, xbuf(sl ^ 1u), tbuf(sl ^ 1u));
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// k_stages_ws: the same pass, warp-specialised so that the Philox-bound draws and the
// shared-memory-bound walk run concurrently on every SM sub-partition instead of in
// alternating phases separated by a CTA barrier.
//   warps [0, nw/2)   walkers: wait for tile t's tables and states, walk and store the
//                     outputs, release the slot; walker warp 0 then issues the TMA bulk
//                     copies of tile t+2 into the slot it just released
//   warps [nw/2, nw)  drawers: wait for the slot's release, copy tile t's thresholds
//                     (drawer-only named barrier), draw the k stages into the slot's tables
// Two slots of {states, tables, thresholds}; mbarriers per slot: st_full (TMA bytes),
// tab_full (every drawer thread arrives), slot_free (every walker thread arrives); the
// parity of tile t's phase is (t >> 1) & 1.  Same tables, same outputs as k_stages.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// One stage's draws of quad l0 (tile position; M >= 4: the quad lies in one group j):
// the table entry of each of its 4 outputs
template <int TB>
__device__ __forceinline__ void ws_entries(const StageArgs& a, const uint4 blk, uint32_t Pt, uint32_t j, uint32_t st,
                                           unsigned char* tabs, uint32_t l0) {
    const uint32_t b = a.b, mask = a.M - 1u, bit = 1u << st;
    const uint32_t rw[4] = {blk.x, blk.y, blk.z, blk.w};
    if constexpr (TB == 1) {
        uint32_t en[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) en[e] = (rw[e] & mask) | (((rw[e] >> b) >= Pt) ? 0x80u : 0u);
        *reinterpret_cast<uint32_t*>(tabs + st * a.P + l0) =
            __byte_perm(__byte_perm(en[0], en[1], 0x0040u), __byte_perm(en[2], en[3], 0x0040u), 0x5410u);
    } else {
        // side from the SIGN of (r >> b) - P: both are < 2^31 (b >= 1), so the difference is
        // negative exactly when the lower side is drawn, for every P in [0, 2^{32-b}];
        // prmt's sign-extending selector spreads it over each 16-bit entry of a pair and
        // three LOP3s assemble two entries: (r & mask) | lower-base | (upper ? bit 2^b : 0)
        // -- 4% fewer cycles per block than select-and-shift (profiles/r2_micro_draw_variants.txt)
        const uint32_t blo = (j & ~bit) << b, bitb = bit << b;
        const uint32_t blo2 = blo | (blo << 16), bitb2 = bitb | (bitb << 16), mask2 = mask | (mask << 16);
        uint32_t dd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) dd[e] = (uint32_t)((int32_t)(rw[e] >> b) - (int32_t)Pt);
        uint32_t s01, s23;  // 0xffff per entry where the lower side is drawn
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s01) : "r"(dd[0]), "r"(dd[1]));
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s23) : "r"(dd[2]), "r"(dd[3]));
        const uint32_t w01 = __byte_perm(rw[0], rw[1], 0x5410u), w23 = __byte_perm(rw[2], rw[3], 0x5410u);
        *reinterpret_cast<uint2*>(tabs + 2u * (st * a.P + l0)) =
            make_uint2(((w01 & mask2) | blo2) | (~s01 & bitb2), ((w23 & mask2) | blo2) | (~s23 & bitb2));
    }
}

// The drawers' share of a tile: quads rt, rt + nthr, ...; two quads per iteration, their
// Philox blocks of a stage computed side by side (two independent chains in flight).
// (Measured against a flat (stage, quad) order balanced to one block per thread: that
// was 6% slower, profiles/r2_k_stages_ws_variants.txt.)
template <int TB, bool DBG>
__device__ __forceinline__ void ws_draws(const StageArgs& a, const StageTile& g, const uint32_t* ths,
                                         unsigned char* tabs, uint32_t rt, uint32_t nthr) {
    const uint32_t b = a.b, k = a.k, kd = a.kd, nq = a.P >> 2, lowbits = a.lowbits, mask = a.M - 1u;
    const uint32_t tlo = g.tlo, thi = g.thi;
    for (uint32_t q0 = rt; q0 < nq; q0 += 2u * nthr) {
        const uint32_t q1 = q0 + nthr;
        const bool two = q1 < nq;
        const uint32_t l0 = 4u * q0, l1 = 4u * (two ? q1 : q0);
        const uint32_t j0 = l0 >> b, j1 = l1 >> b;
        const uint32_t gp0 = ((tlo | (j0 << lowbits) | thi) << b) | (l0 & mask);
        const uint32_t gp1 = ((tlo | (j1 << lowbits) | thi) << b) | (l1 & mask);
        const uint32_t c0 = (a.pos0 + gp0) >> 2, c1 = (a.pos0 + gp1) >> 2;
        uint32_t toff = 0;
        for (uint32_t st = 0; st + 1u < kd; ++st) {  // the last stage: in the walk (ws_walk)
            const uint32_t s = a.s0 + st;
            const uint4 b0 = rng_block(a.key, c0, a.n, kDomainResample, s);
            const uint4 b1 = rng_block(a.key, c1, a.n, kDomainResample, s);
            const uint32_t P0 = ths[toff + (j0 >> (st + 1))], P1 = ths[toff + (j1 >> (st + 1))];
            toff += (1u << k) >> (st + 1);
            ws_entries<TB>(a, b0, P0, j0, st, tabs, l0);
            if (two) ws_entries<TB>(a, b1, P1, j1, st, tabs, l1);
            if constexpr (DBG) {
                const uint32_t bit = 1u << st;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && !two) break;
                    const uint4 bb = h ? b1 : b0;
                    const uint32_t jj0 = h ? j1 : j0, PP = h ? P1 : P0, gp = h ? gp1 : gp0;
                    const uint32_t rw[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool hi = (rw[e] >> b) >= PP;
                        const uint32_t jj = hi ? (jj0 | bit) : (jj0 & ~bit);
                        const uint32_t gsrc = ((tlo | (jj << lowbits) | thi) << b) | (rw[e] & mask);
                        a.dbg_anc[(uint64_t)(s - 1) * a.N + gp + e] = (int32_t)(a.pos0 + gsrc);
                    }
                }
            }
        }
    }
}

// The walkers' share: quads tid, tid + nthr, ...  The pass's LAST stage is drawn here from
// the output quad's own Philox block (its 4 words are exactly these 4 outputs' draws, and
// the walk starts at the output), so the drawers skip it and no table holds it: 1/k of the
// draw work moves to the walkers, which wait on the drawers otherwise (ncu, round 2).
template <typename T, int TB, bool DBG>
__device__ __forceinline__ void ws_walk(const StageArgs& a, const StageTile& g, const T* xs, const unsigned char* tabs,
                                        const uint32_t* ths, uint32_t tid, uint32_t nthr) {
    const uint32_t M = a.M, b = a.b, k = a.k, P = a.P, mask = M - 1u, nq = P >> 2, lowbits = a.lowbits;
    const uint32_t stl = a.kd - 1u, sl = a.s0 + stl, bitl = 1u << stl;
    // the last drawn stage's thresholds (one when kd = k: the tile's two halves pair)
    const uint32_t* thl = ths + ((1u << k) - (1u << (k - stl)));
    T* pout = reinterpret_cast<T*>(a.pout);
    for (uint32_t q = tid; q < nq; q += nthr) {
        const uint32_t l0 = 4u * q;
        const uint32_t j = l0 >> b;
        const uint32_t Pl = thl[j >> (stl + 1u)];
        const uint32_t gp = ((g.tlo | (j << lowbits) | g.thi) << b) | (l0 & mask);
        const uint4 blk = rng_block(a.key, (a.pos0 + gp) >> 2, a.n, kDomainResample, sl);
        const uint32_t rw[4] = {blk.x, blk.y, blk.z, blk.w};
        uint32_t tp[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t jj = ((rw[e] >> b) >= Pl) ? (j | bitl) : (j & ~bitl);
            tp[e] = (jj << b) | (rw[e] & mask);
            if constexpr (DBG)
                a.dbg_anc[(uint64_t)(sl - 1) * a.N + gp + e] =
                    (int32_t)(a.pos0 + (((g.tlo | (jj << lowbits) | g.thi) << b) | (rw[e] & mask)));
        }
        for (int st = (int)stl - 1; st >= 0; --st) {
            if constexpr (TB == 1) {
                const unsigned char* Ts = tabs + (uint32_t)st * P;
                const uint32_t sh = (uint32_t)st + b;
                const uint32_t keep = ~(mask | (1u << sh));
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t en = Ts[tp[e]];
                    tp[e] = (tp[e] & keep) | (en & 0x7fu) | ((en >> 7) << sh);
                }
            } else {
                const uint16_t* Ts = reinterpret_cast<const uint16_t*>(tabs) + (uint32_t)st * P;
#pragma unroll
                for (int e = 0; e < 4; ++e) tp[e] = Ts[tp[e]];
            }
        }
        Vec4<T> v;
#pragma unroll
        for (int e = 0; e < 4; ++e) v.v[e] = xs[tp[e]];
        uint32_t gp0 = gp;
        if (a.out_rot) gp0 = (rotr_group(gp0 >> b, a.out_rot, a.out_S) << b) | (gp0 & mask);
        *reinterpret_cast<Vec4<T>*>(pout + gp0) = v;
    }
}

// a.ws_walkers threads walk (a multiple of 32), the rest draw; QPT is unused (runtime
// loops over the quads); needs M >= 4 and the bulk-copy path (M * sizeof(T) >= 16)
template <typename T, int TB, bool DBG, int QPT>
__global__ void __launch_bounds__(1024, 1) k_stages_ws(const __grid_constant__ StageArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k = a.k, P = a.P;
    const uint32_t ntiles = (uint32_t)(a.N / P);
    const uint32_t stb = (P * (uint32_t)sizeof(T) + 15u) & ~15u;
    const uint32_t ttb = (k * P * TB + 15u) & ~15u;
    unsigned char* tab0 = smem + 2u * stb;
    uint32_t* th0 = reinterpret_cast<uint32_t*>(tab0 + 2u * ttb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(th0 + (2u << k));
    uint64_t* st_full = bars;        // [2]
    uint64_t* tab_full = bars + 2;   // [2]
    uint64_t* slot_free = bars + 4;  // [2]
    auto xbuf = [&](uint32_t sl) { return reinterpret_cast<T*>(smem + sl * stb); };
    auto tbuf = [&](uint32_t sl) { return tab0 + sl * ttb; };
    auto thbuf = [&](uint32_t sl) { return th0 + (sl << k); };

    const uint32_t t0 = blockIdx.x;
    if (t0 >= ntiles) return;
    const uint32_t nt = (ntiles - t0 + gridDim.x - 1u) / gridDim.x;
    const uint32_t nwalk = a.ws_walkers, ndraw = blockDim.x - nwalk;
    const bool walker = threadIdx.x < nwalk;
    const uint32_t rt = walker ? threadIdx.x : threadIdx.x - nwalk;  // thread index within the role
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(st_full + i, 1u);
            mbar_init(tab_full + i, ndraw);
            mbar_init(slot_free + i, nwalk);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (walker) {
        // the first two tiles' states
        for (uint32_t i = 0; i < 2u && i < nt; ++i)
            stage_states_load<T>(a, stage_tile_geom(a, t0 + i * gridDim.x), xbuf(i), st_full + i);
        for (uint32_t i = 0; i < nt; ++i) {
            const uint32_t sl = i & 1u, par = (i >> 1) & 1u;
            mbar_wait_sleep(st_full + sl, par);
            mbar_wait_sleep(tab_full + sl, par);
            ws_walk<T, TB, DBG>(a, stage_tile_geom(a, t0 + i * gridDim.x), xbuf(sl), tbuf(sl), thbuf(sl), rt, nwalk);
            mbar_arrive(slot_free + sl);
            if (i + 2u < nt && threadIdx.x < 32u) {  // refill the slot once every walker has left it
                mbar_wait_sleep(slot_free + sl, par);
                stage_states_load<T>(a, stage_tile_geom(a, t0 + (i + 2u) * gridDim.x), xbuf(sl), st_full + sl);
            }
        }
    } else {
        // drawers; tile i+1's thresholds (<= 2^k - 1 entries, one per drawer thread) are
        // loaded while tile i is drawn and stored into the other threshold slot afterwards
        const uint32_t E = (1u << k) - 1u;
        auto thr_of = [&](uint32_t tile_i) -> uint32_t {
            const StageTile g = stage_tile_geom(a, t0 + tile_i * gridDim.x);
            const uint32_t e = rt, u = (1u << k) - e;
            const uint32_t st = k - (32u - __clz(u - 1u));
            const uint32_t off = (1u << k) - (1u << (k - st));
            const uint32_t s = a.s0 + st;
            return __ldg(a.thr + level_offset(a.m, (int)s) + (g.thi >> s) + (e - off));
        };
        uint32_t nxt = rt < E ? thr_of(0) : 0u;
        for (uint32_t i = 0; i < nt; ++i) {
            const uint32_t sl = i & 1u, par = (i >> 1) & 1u;
            if (i >= 2u) mbar_wait_sleep(slot_free + sl, par ^ 1u);  // tile i-2 walked: the slot is free
            if (rt < E) thbuf(sl)[rt] = nxt;                         // (the walkers read its threshold too)
            named_bar_sync(1u, ndraw);                               // tile i's thresholds stored
            nxt = (rt < E && i + 1u < nt) ? thr_of(i + 1u) : 0u;     // in flight during the draws
            ws_draws<TB, DBG>(a, stage_tile_geom(a, t0 + i * gridDim.x), thbuf(sl), tbuf(sl), rt, ndraw);
            mbar_arrive(tab_full + sl);
        }
    }
}

// ---------------------------------------------------------------------------------------
// k_stages_wsc: k_stages_ws with the pass depth K and b = log2 M fixed at compile time
// (16-bit tables, no debug tables), for the plans the benchmark configurations run (C4:
// K = 6, b = 6).  Same draws, same outputs, bit for bit (tests/test_gpu_stage_spec.py);
// what changes is the instruction count per particle:
//   * the stage loop unrolls, so every stage's bit, table offset and threshold offset is
//     an immediate and the Philox counter's (n, stage) words fold where uniform;
//   * table entries hold the source's BYTE offset in the previous stage's table (tile
//     position x 2): a walk step is one LDS.U16 at [entry + stage offset], no address
//     arithmetic (the drawers pay one shift per pair of entries for it);
//   * the drawers compose two entries with three LOP3-class operations after the sign
//     trick of ws_entries.
// Entries of one stage for one quad: e = ((r & mask) << 1) | (side ? hi : lo) << (b + 1),
// two per 32-bit word (outputs 4q, 4q+1 | 4q+2, 4q+3).
template <int B>
__device__ __forceinline__ uint2 wsc_pair_entries(const uint4 blk, uint32_t Pt, uint32_t blo2, uint32_t bitb2) {
    constexpr uint32_t mask2s = (((1u << B) - 1u) << 1) * 0x10001u;
    const int32_t ip = (int32_t)Pt;
    const uint32_t d0 = (uint32_t)((int32_t)(blk.x >> B) - ip), d1 = (uint32_t)((int32_t)(blk.y >> B) - ip);
    const uint32_t d2 = (uint32_t)((int32_t)(blk.z >> B) - ip), d3 = (uint32_t)((int32_t)(blk.w >> B) - ip);
    uint32_t s01, s23;  // 0xffff per entry where the lower side is drawn
    asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s01) : "r"(d0), "r"(d1));
    asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(s23) : "r"(d2), "r"(d3));
    const uint32_t w01 = __byte_perm(blk.x, blk.y, 0x5410u) << 1, w23 = __byte_perm(blk.z, blk.w, 0x5410u) << 1;
    return make_uint2(((w01 & mask2s) | blo2) | (~s01 & bitb2), ((w23 & mask2s) | blo2) | (~s23 & bitb2));
}

// The drawers' stages ST..K-2 of two quads (q0, q1), NS stages at a time: 2 NS Philox chains
// in lockstep (philox10_lockstep: the drawers are bound by the latency of the multiply
// chain, not by its pipe; one stage at a time, 2 chains, measured 2.056 ms per C4 pass,
// two stages 1.972, three stages (-DPF_WSC_CHUNK=3) 1.975; profiles/r2_wsc_lockstep_s4.txt).
// The last stage of the pass is drawn in the walk (wsc_walk).
#ifndef PF_WSC_CHUNK
#define PF_WSC_CHUNK 2
#endif
struct WscQuadPair {
    uint32_t l0, l1, j0, j1, c0, c1, jb0, jb1;
    bool two;
};
template <int K, int B, int ST>
__device__ __forceinline__ void wsc_draw_from(const StageArgs& a, const WscQuadPair& w, const uint32_t* ths, uint16_t* tabs) {
    constexpr uint32_t P = (1u << B) << K;
    constexpr int rem = K - 1 - ST;
    if constexpr (rem > 0) {
        constexpr int NS = (PF_WSC_CHUNK == 3 && (rem == 3 || rem >= 5)) ? 3 : (rem >= 2 ? 2 : 1);
        uint4 c[2 * NS];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
            c[2 * h] = rng_counter(w.c0, a.n, kDomainResample, a.s0 + (uint32_t)(ST + h));
            c[2 * h + 1] = rng_counter(w.c1, a.n, kDomainResample, a.s0 + (uint32_t)(ST + h));
        }
        philox10_lockstep<2 * NS>(c, a.key);
#pragma unroll
        for (int h = 0; h < NS; ++h) {
            constexpr uint32_t one = 1u;
            const int sh = ST + h;
            const uint32_t bitb2 = ((one << sh) << (B + 1)) * 0x10001u;
            const uint32_t toff = (one << K) - (one << (K - sh));
            const uint32_t P0 = ths[toff + (w.j0 >> (sh + 1))], P1 = ths[toff + (w.j1 >> (sh + 1))];
            *reinterpret_cast<uint2*>(tabs + sh * P + w.l0) = wsc_pair_entries<B>(c[2 * h], P0, w.jb0 & ~bitb2, bitb2);
            if (w.two) *reinterpret_cast<uint2*>(tabs + sh * P + w.l1) = wsc_pair_entries<B>(c[2 * h + 1], P1, w.jb1 & ~bitb2, bitb2);
        }
        wsc_draw_from<K, B, ST + NS>(a, w, ths, tabs);
    }
}

template <int K, int B>
__device__ __forceinline__ void wsc_draws(const StageArgs& a, const StageTile& g, const uint32_t* ths, uint16_t* tabs,
                                          uint32_t rt, uint32_t nthr) {
    constexpr uint32_t M = 1u << B, P = M << K, nq = P >> 2, mask = M - 1u;
    const uint32_t lowbits = a.lowbits;
    for (uint32_t q0 = rt; q0 < nq; q0 += 2u * nthr) {
        const uint32_t q1 = q0 + nthr;
        WscQuadPair w;
        w.two = q1 < nq;
        w.l0 = 4u * q0;
        w.l1 = 4u * (w.two ? q1 : q0);
        w.j0 = w.l0 >> B;
        w.j1 = w.l1 >> B;
        w.c0 = (a.pos0 + (((g.tlo | (w.j0 << lowbits) | g.thi) << B) | (w.l0 & mask))) >> 2;
        w.c1 = (a.pos0 + (((g.tlo | (w.j1 << lowbits) | g.thi) << B) | (w.l1 & mask))) >> 2;
        w.jb0 = (w.j0 << (B + 1)) * 0x10001u;
        w.jb1 = (w.j1 << (B + 1)) * 0x10001u;
        wsc_draw_from<K, B, 0>(a, w, ths, tabs);
    }
}

template <typename T, int K, int B>
__device__ __forceinline__ void wsc_walk(const StageArgs& a, const StageTile& g, const T* xs, const uint16_t* tabs,
                                         const uint32_t* ths, uint32_t tid, uint32_t nthr) {
    constexpr uint32_t M = 1u << B, P = M << K, nq = P >> 2, mask = M - 1u;
    constexpr uint32_t bitlb = (1u << (K - 1)) << (B + 1);  // the last stage's bit, as a byte offset
    const uint32_t lowbits = a.lowbits, sl = a.s0 + (uint32_t)K - 1u;
    const uint32_t Pl = ths[(1u << K) - 2u];  // the last stage pairs the tile's two halves: one threshold
    const unsigned char* tb = reinterpret_cast<const unsigned char*>(tabs);
    T* pout = reinterpret_cast<T*>(a.pout);
    for (uint32_t q = tid; q < nq; q += nthr) {
        const uint32_t l0 = 4u * q;
        const uint32_t j = l0 >> B;
        const uint32_t gp = ((g.tlo | (j << lowbits) | g.thi) << B) | (l0 & mask);
        const uint4 blk = rng_block(a.key, (a.pos0 + gp) >> 2, a.n, kDomainResample, sl);
        const uint32_t rw[4] = {blk.x, blk.y, blk.z, blk.w};
        const uint32_t jlo = (j << (B + 1)) & ~bitlb;
        uint32_t t2[4];  // byte offsets (tile position x 2)
#pragma unroll
        for (int e = 0; e < 4; ++e) t2[e] = ((rw[e] & mask) << 1) | jlo | (((rw[e] >> B) >= Pl) ? bitlb : 0u);
#pragma unroll
        for (int st = K - 2; st >= 0; --st)
#pragma unroll
            for (int e = 0; e < 4; ++e) t2[e] = *reinterpret_cast<const uint16_t*>(tb + st * (2u * P) + t2[e]);
        Vec4<T> v;
#pragma unroll
        for (int e = 0; e < 4; ++e) v.v[e] = *reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(xs) + t2[e] * (sizeof(T) / 2));
        uint32_t gp0 = gp;
        if (a.out_rot) gp0 = (rotr_group(gp0 >> B, a.out_rot, a.out_S) << B) | (gp0 & mask);
        *reinterpret_cast<Vec4<T>*>(pout + gp0) = v;
    }
}

template <typename T, int K, int B>
__global__ void __launch_bounds__(1024, 1) k_stages_wsc(const __grid_constant__ StageArgs a) {
    static_assert(B >= 2 && ((1u << B) * sizeof(T)) >= 16u && ((1u << (B + K)) * 2u) <= 65536u, "wsc: M >= 4, bulk groups, 16-bit byte offsets");
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr uint32_t P = (1u << B) << K;
    constexpr uint32_t stb = (P * (uint32_t)sizeof(T) + 15u) & ~15u;
    constexpr uint32_t ttb = (K * P * 2u + 15u) & ~15u;  // the layout of stages_smem(P, ., K, 2, 2)
    const uint32_t ntiles = (uint32_t)(a.N / P);
    unsigned char* tab0 = smem + 2u * stb;
    uint32_t* th0 = reinterpret_cast<uint32_t*>(tab0 + 2u * ttb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(th0 + (2u << K));
    uint64_t* st_full = bars;        // [2]
    uint64_t* tab_full = bars + 2;   // [2]
    uint64_t* slot_free = bars + 4;  // [2]
    auto xbuf = [&](uint32_t sl) { return reinterpret_cast<T*>(smem + sl * stb); };
    auto tbuf = [&](uint32_t sl) { return reinterpret_cast<uint16_t*>(tab0 + sl * ttb); };
    auto thbuf = [&](uint32_t sl) { return th0 + (sl << K); };

    const uint32_t t0 = blockIdx.x;
    if (t0 >= ntiles) return;
    const uint32_t nt = (ntiles - t0 + gridDim.x - 1u) / gridDim.x;
    const uint32_t nwalk = a.ws_walkers, ndraw = blockDim.x - nwalk;
    const bool walker = threadIdx.x < nwalk;
    const uint32_t rt = walker ? threadIdx.x : threadIdx.x - nwalk;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(st_full + i, 1u);
            mbar_init(tab_full + i, ndraw);
            mbar_init(slot_free + i, nwalk);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (walker) {
        for (uint32_t i = 0; i < 2u && i < nt; ++i)
            stage_states_load<T>(a, stage_tile_geom(a, t0 + i * gridDim.x), xbuf(i), st_full + i);
        for (uint32_t i = 0; i < nt; ++i) {
            const uint32_t sl = i & 1u, par = (i >> 1) & 1u;
            mbar_wait_sleep(st_full + sl, par);
            mbar_wait_sleep(tab_full + sl, par);
            wsc_walk<T, K, B>(a, stage_tile_geom(a, t0 + i * gridDim.x), xbuf(sl), tbuf(sl), thbuf(sl), rt, nwalk);
            mbar_arrive(slot_free + sl);
            if (i + 2u < nt && threadIdx.x < 32u) {
                mbar_wait_sleep(slot_free + sl, par);
                stage_states_load<T>(a, stage_tile_geom(a, t0 + (i + 2u) * gridDim.x), xbuf(sl), st_full + sl);
            }
        }
    } else {
        constexpr uint32_t E = (1u << K) - 1u;
        auto thr_of = [&](uint32_t tile_i) -> uint32_t {
            const StageTile g = stage_tile_geom(a, t0 + tile_i * gridDim.x);
            const uint32_t e = rt, u = (1u << K) - e;
            const uint32_t st = K - (32u - __clz(u - 1u));
            const uint32_t off = (1u << K) - (1u << (K - st));
            const uint32_t s = a.s0 + st;
            return __ldg(a.thr + level_offset(a.m, (int)s) + (g.thi >> s) + (e - off));
        };
        uint32_t nxt = rt < E ? thr_of(0) : 0u;
        for (uint32_t i = 0; i < nt; ++i) {
            const uint32_t sl = i & 1u, par = (i >> 1) & 1u;
            if (i >= 2u) mbar_wait_sleep(slot_free + sl, par ^ 1u);
            if (rt < E) thbuf(sl)[rt] = nxt;
            named_bar_sync(1u, ndraw);
            nxt = (rt < E && i + 1u < nt) ? thr_of(i + 1u) : 0u;
            wsc_draws<K, B>(a, stage_tile_geom(a, t0 + i * gridDim.x), thbuf(sl), tbuf(sl), rt, ndraw);
            mbar_arrive(tab_full + sl);
        }
    }
}

}  // namespace pfk
