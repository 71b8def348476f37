// pf_device.cuh -- device building blocks of the BPF step (sm_100a).
//
// * Philox4x32-10 counter-based generator (Salmon et al., SC'11), written for the
//   GPU from its published definition; the draw contract keys every
//   32-bit word by (seed, n, domain, stage, particle quad).
// * Box-Muller normals in fp32 (accurate logf / sqrtf / sincospif, no fast-math).
// * Model evaluation: mutation f (Alg. 1 l.303) and log-potential
//   log g_n, templated on the state dimension D.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace pfk {

constexpr uint32_t kDomainInit = 1u;
constexpr uint32_t kDomainMutate = 2u;
constexpr uint32_t kDomainResample = 3u;
constexpr uint32_t kDomainWithin = 4u;  // AIRPF within-island draws (R19)
constexpr uint32_t kDomainIsland = 5u;  // AIRPF island side draws (R20)
constexpr uint32_t kDomainMulti = 6u;   // Alg. 2 multinomial draws (R22)

// Stage rotation (R23): group g of the current layout lands in group
// rotr_S(g, k) of the next one.
__host__ __device__ inline uint32_t rotr_group(uint32_t g, uint32_t k, uint32_t S) {
    if (k == 0u || S == 0u) return g;
    const uint32_t mask = S >= 32u ? 0xffffffffu : ((1u << S) - 1u);
    return ((g >> k) | (g << (S - k))) & mask;
}

// Offset of V level s (s >= 1) in the (m - 1)-entry level tables: level s has m / 2^s
// entries (blocks of 2^s groups).
__host__ __device__ inline uint64_t level_offset(uint64_t m, int s) { return m - (m >> (s - 1)); }

// Philox key schedule: round r uses (k[2r], k[2r+1]) = (k0 + r W0, k1 + r W1).  Computed
// once on the host and passed inside the kernel parameters, so every round's key XOR reads
// a constant-bank operand (no per-thread key registers or adds).
struct Key {
    uint32_t k[20];
};

__host__ __device__ inline Key make_key(uint64_t seed) {
    Key key;
    const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        key.k[2 * r] = k0 + (uint32_t)r * 0x9E3779B9u;
        key.k[2 * r + 1] = k1 + (uint32_t)r * 0xBB67AE85u;
    }
    return key;
}

// Philox4x32-10: per round (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
// c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key += (W0, W1) between rounds.
__device__ __forceinline__ uint4 philox10(uint4 c, const Key& key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ key.k[2 * r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ key.k[2 * r + 1],
                       (uint32_t)p0);
    }
    return c;
}

// NB independent blocks advanced round by round in lockstep: the same values as NB calls of
// philox10, but the NB multiply chains are interleaved in program order, so a warp has
// 2 NB independent IMAD.WIDE in flight per round instead of 2 (the drawers of k_stages_wsc
// and the pass-1 noise are bound by the latency of that chain, not by its pipe).
template <int NB>
__device__ __forceinline__ void philox10_lockstep(uint4 (&c)[NB], const Key& key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t p0[NB], p1[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            p0[i] = (uint64_t)0xD2511F53u * c[i].x;
            p1[i] = (uint64_t)0xCD9E8D57u * c[i].z;
        }
#pragma unroll
        for (int i = 0; i < NB; ++i)
            c[i] = make_uint4((uint32_t)(p1[i] >> 32) ^ c[i].y ^ key.k[2 * r], (uint32_t)p1[i],
                              (uint32_t)(p0[i] >> 32) ^ c[i].w ^ key.k[2 * r + 1], (uint32_t)p0[i]);
    }
}
__device__ __forceinline__ uint4 rng_counter(uint32_t c0, uint32_t n, uint32_t domain, uint32_t sub) {
    return make_uint4(c0, n, (domain << 24) | sub, 0u);
}

// Block (c0, n, domain<<24 | sub, 0) of the draw contract.
__device__ __forceinline__ uint4 rng_block(const Key& key, uint32_t c0, uint32_t n, uint32_t domain, uint32_t sub) {
    return philox10(make_uint4(c0, n, (domain << 24) | sub, 0u), key);
}

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// MUFU approximations without the denormal fix-ups of __log2f / rsqrtf / __expf (the
// .ftz PTX forms): for normal inputs and outputs the same MUFU results, three instructions
// fewer each.  Every input below is normal by construction (u1 >= 2^-24, r2 >= 1e-30); the
// stage-1 weights e^x (x = lw - max <= 0) flush to 0 below e^-87 instead of going denormal.
__device__ __forceinline__ float lg2_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float exp_ftz(float x) {  // e^x = 2^(x log2 e), as __expf
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.4426950408889634f));
    return r;
}

// u in [0,1) from the 24 high bits (exact in fp32).
__device__ __forceinline__ float u01f(uint32_t r) { return (float)(r >> 8) * 0x1p-24f; }

// -2 ln u1 for u1 = n 2^-24, n = (a >> 8) + 1 in [1, 2^24].  With n = 2^e m, m in
// [0.75, 1.5): ln u1 = (e - 24) ln 2 + log1p(f), f = m - 1 exact, and
// log1p(f) = 2 atanh(t) = 2t (1 + t^2/3 + t^4/5 + t^6/7 + t^8/9), t = f / (2 + f),
// |t| <= 0.2 (truncation < 4e-9).  Relative accuracy ~1e-7 everywhere, including
// u1 -> 1 where R = sqrt(-2 ln u1) -> 0 is most sensitive (no cancellation).
__device__ __forceinline__ float neg2_log_u1(uint32_t a) {
    const float nf = (float)((a >> 8) + 1u);  // exact
    const int bits = __float_as_int(nf);
    int e = (bits >> 23) - 127;
    float m = __int_as_float((bits & 0x007fffff) | 0x3f800000);  // [1, 2)
    const bool hi = m >= 1.5f;
    m = hi ? 0.5f * m : m;
    e = hi ? e + 1 : e;
    const float f = m - 1.0f;
    const float t = __fdividef(f, 2.0f + f);
    const float t2 = t * t;
    const float poly = fmaf(t2, fmaf(t2, fmaf(t2, fmaf(t2, 1.0f / 9.0f, 1.0f / 7.0f), 1.0f / 5.0f), 1.0f / 3.0f), 1.0f);
    const float l1p = 2.0f * t * poly;
    const float k = (float)(24 - e);
    return 2.0f * fmaf(k, 0.693145751953125f, fmaf(k, 1.428606765330187e-06f, -l1p));  // ln2 = hi + lo
}

// Box-Muller: (a, b) -> (R cos 2 pi u2, R sin 2 pi u2), R = sqrt(-2 ln u1), with
// u1 = ((a>>8)+1) 2^-24 in (0,1] and u2 = (b>>8) 2^-24 in [0,1).
// The square root uses MUFU.RSQ and the angle the MUFU sin/cos on [-pi, pi):
// cos(2 pi u2) = -cos(th), sin(2 pi u2) = -sin(th) with th = 2 pi u2 - pi.
// Absolute error <= ~3e-6.  -2 ln u1 takes the MUFU lg2 unless u1 is within
// 2^-10 of 1 (kFastLogLimit).
// Fast branch of -2 ln u1: MUFU lg2 has absolute error <= 2^-22.6 on [0.5, 1) and relative
// error <= 2^-22 below, so for u1 < 1 - 2^-10 the radius R = sqrt(-2 ln u1) is within
// ~2.5e-6 of exact (worst case at the limit, R ~ 0.045); above the limit (probability
// 2^-10 per pair) the precise neg2_log_u1 runs.
constexpr uint32_t kFastLogLimit = (1u << 24) - (1u << 14);  // u1 = n 2^-24 < 1 - 2^-10

template <int FAST>  // 1: u1 < 1 - 2^-10 is known (the MUFU branch), 0: decide here
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
    const uint32_t na = (a >> 8) + 1u;
    float r2;
    if (FAST || na < kFastLogLimit) r2 = -1.3862943611198906f * lg2_ftz((float)na * 0x1p-24f);  // -2 ln 2 lg2(u1)
    else r2 = neg2_log_u1(a);
    const float rad = r2 * rsqrt_ftz(fmaxf(r2, 1e-30f));
    const float th = fmaf((float)(b >> 8), 6.28318530717958647692f * 0x1p-24f, -3.14159265358979323846f);
    float s, c;
    __sincosf(th, &s, &c);
    return make_float2(-rad * c, -rad * s);
}

// Four normals of one block: coordinates 4j..4j+3.  One branch decides the radius path of
// both pairs (each pair's value is the one box_muller<0> gives it).
__device__ __forceinline__ void normals4(const uint4& v, float* z) {
    float2 p, q;
    if (max(v.x, v.z) < ((kFastLogLimit - 1u) << 8)) {  // both u1 below the limit: (a >> 8) + 1 < limit
        p = box_muller<1>(v.x, v.y);
        q = box_muller<1>(v.z, v.w);
    } else {
        p = box_muller<0>(v.x, v.y);
        q = box_muller<0>(v.z, v.w);
    }
    z[0] = p.x;
    z[1] = p.y;
    z[2] = q.x;
    z[3] = q.y;
}

// Model constants, copied once at pf_init and passed by value to the kernels.
struct ModelParams {
    int kind;  // 1 LG, 2 SV
    int d, dy;
    int diag_obs;  // H == I (dy == d) and Rinv diagonal: fast weighting path
    int diag_lq;   // LQ diagonal: fast noise path
    float A[64], LQ[64], H[64], Rinv[64], m0[8], L0[64];
    float rdiag[8];  // -0.5 * Rinv_kk (fast path)
    float phi, sigma, beta, sv_m0, sv_s0;
    float sv_c;  // 1 / (2 beta^2)
};

// x = A xhat + LQ z  (LG)  |  x = phi xhat + sigma z  (SV)      [PAPER.md:302-303]
template <int D, int KIND>
__device__ __forceinline__ void mutate(const ModelParams& mp, const float* xh, const float* z, float* x) {
    if (KIND == 2) {
        x[0] = fmaf(mp.phi, xh[0], mp.sigma * z[0]);
    } else {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            float v = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) v = fmaf(mp.A[k * D + j], xh[j], v);
            if (mp.diag_lq) {
                v = fmaf(mp.LQ[k * D + k], z[k], v);
            } else {
#pragma unroll
                for (int j = 0; j <= k; ++j) v = fmaf(mp.LQ[k * D + j], z[j], v);
            }
            x[k] = v;
        }
    }
}

// x_0 = m0 + L0 z (LG) | sv_m0 + sv_s0 z (SV)                    [PAPER.md:296-298]
template <int D, int KIND>
__device__ __forceinline__ void init_state(const ModelParams& mp, const float* z, float* x) {
    if (KIND == 2) {
        x[0] = fmaf(mp.sv_s0, z[0], mp.sv_m0);
    } else {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            float v = mp.m0[k];
#pragma unroll
            for (int j = 0; j <= k; ++j) v = fmaf(mp.L0[k * D + j], z[j], v);
            x[k] = v;
        }
    }
}

// log g_n(x), constants dropped (reading R9):
//   LG: -1/2 (y - Hx)^T Rinv (y - Hx);  SV: -x/2 - y^2 e^{-x} / (2 beta^2).
// Non-finite -> -inf.
template <int D, int KIND>
__device__ __forceinline__ float log_potential(const ModelParams& mp, const float* y, const float* x) {
    float v;
    if (KIND == 2) {
        v = fmaf(-0.5f, x[0], -(y[0] * y[0] * mp.sv_c) * expf(-x[0]));
    } else if (mp.diag_obs) {
        v = 0.0f;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const float r = y[k] - x[k];
            v = fmaf(mp.rdiag[k] * r, r, v);
        }
    } else {
        // static trip counts with dy guards: y and r stay in registers (a dynamic index
        // would put them, and the kernel's y, in local memory); same summation order
        float r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float hx = 0.0f;
            if (k < mp.dy) {
#pragma unroll
                for (int j = 0; j < D; ++j) hx = fmaf(mp.H[k * D + j], x[j], hx);
            }
            r[k] = y[k] - hx;
        }
        float q = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k < mp.dy) {
                float t = 0.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < mp.dy) t = fmaf(mp.Rinv[k * mp.dy + j], r[j], t);
                q = fmaf(r[k], t, q);
            }
        }
        v = -0.5f * q;
    }
    return (v == v && v != INFINITY && v != -INFINITY) ? v : -INFINITY;
}

// log((e^a + e^b)/2): the pair average V_s = A_s V_{s-1} in the log domain (fp64).
__device__ __forceinline__ double log_pair_mean(double a, double b) {
    const double c = a > b ? a : b;
    if (c == -CUDART_INF) return -CUDART_INF;
    return c + log((exp(a - c) + exp(b - c)) * 0.5);
}

// Stage-s (s >= 2) side threshold floor(p 2^{32-b}), p = V_L / (V_L + V_R).
__device__ __forceinline__ uint32_t side_threshold(double vl, double vr, int b) {
    double p;
    if (vl == -CUDART_INF && vr == -CUDART_INF) p = 0.5;
    else p = 1.0 / (1.0 + exp(vr - vl));
    return (uint32_t)floor(p * ldexp(1.0, 32 - b));
}

// The same two quantities for the in-tile levels of k_pass1: the large common offset stays
// fp64, the O(1) part uses the MUFU exp2/log2/rcp (|error| ~3e-7 in log V and in p, inside
// the 1e-6 decision window of the parity contract).  One exp serves both outputs.
__device__ __forceinline__ void pair_level_fast(double vl, double vr, int b, double* v, uint32_t* P) {
    const double mx = vl > vr ? vl : vr, mn = vl > vr ? vr : vl;
    if (mx == -CUDART_INF) {  // both halves dead: V = 0, p = 1/2
        *v = -CUDART_INF;
        *P = 1u << (31 - b);
        return;
    }
    const float t = exp2f((float)(mn - mx) * 1.4426950408889634f);  // e^{mn - mx} in [0, 1]
    const float op = 1.0f + t;
    *v = mx + (double)(__log2f(op) * 0.6931471805599453f - 0.6931471805599453f);
    const float q = __frcp_rn(op);
    const float p = vl >= vr ? q : t * q;
    *P = (uint32_t)(p * __int_as_float((127 + 32 - b) << 23));  // floor(p 2^(32-b)), p 2^(32-b) >= 0
}

// Four consecutive payload elements moved as one vector.
template <typename T>
struct __align__(4 * sizeof(T) <= 16 ? 4 * sizeof(T) : 16) Vec4 {
    T v[4];
};

}  // namespace pfk
