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

struct Key {
    uint32_t k0, k1;
};

// Philox4x32-10: per round (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
// c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key += (W0, W1) between rounds.
__device__ __forceinline__ uint4 philox10(uint4 c, Key key) {
    uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Block (c0, n, domain<<24 | sub, 0) of the draw contract.
__device__ __forceinline__ uint4 rng_block(Key key, uint32_t c0, uint32_t n, uint32_t domain, uint32_t sub) {
    return philox10(make_uint4(c0, n, (domain << 24) | sub, 0u), key);
}

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// u in [0,1) from the 24 high bits (exact in fp32).
__device__ __forceinline__ float u01f(uint32_t r) { return (float)(r >> 8) * 0x1p-24f; }

// Box-Muller: (a, b) -> two normals (cos, sin) with u1 = ((a>>8)+1) 2^-24 in (0,1].
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
    const float u1 = (float)((a >> 8) + 1u) * 0x1p-24f;
    const float u2 = (float)(b >> 8) * 0x1p-24f;
    const float rad = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    return make_float2(rad * c, rad * s);
}

// Four normals of one block: coordinates 4j..4j+3.
__device__ __forceinline__ void normals4(const uint4& v, float* z) {
    const float2 p = box_muller(v.x, v.y);
    const float2 q = box_muller(v.z, v.w);
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
#pragma unroll
            for (int j = 0; j <= k; ++j) v = fmaf(mp.LQ[k * D + j], z[j], v);
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
        float r[8];
        for (int k = 0; k < mp.dy; ++k) {
            float hx = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) hx = fmaf(mp.H[k * D + j], x[j], hx);
            r[k] = y[k] - hx;
        }
        float q = 0.0f;
        for (int k = 0; k < mp.dy; ++k) {
            float t = 0.0f;
            for (int j = 0; j < mp.dy; ++j) t = fmaf(mp.Rinv[k * mp.dy + j], r[j], t);
            q = fmaf(r[k], t, q);
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

}  // namespace pfk
