/*
 * pf_oracle.c -- plain, slow, fp64 CPU oracle for ONE bootstrap-particle-filter
 * time step with augmented resampling (arXiv 1812.01502, Heine, Whiteley, Cemgil).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1812_01502_b200/
 * csrc); it re-implements the Philox4x32-10 generator independently from its
 * published definition (Salmon et al., SC'11) and the draw contract of
 * DESIGN.md §3.
 *
 * Every function cites the passage of PAPER.md it follows.  Everything is fp64
 * except the input particle states and model constants, which the method's
 * configurations fix as fp32 values (BASELINE.json configs: "fp32 particles");
 * they are widened to fp64 on entry.
 *
 * Pins (what checks this file against something other than itself) are listed in
 * DESIGN.md §6; every function here has at least one.
 *
 * Step, in the paper's order (Alg. 1 with Alg. 3 as RESAMPLE):
 *   1. mutation   zeta_{n}^i ~ f(zhat_{n-1}^i, .)         (Alg. 1 l.302-303; skipped at n=0)
 *   2. weighting  V_0^i = g_n(xi_0^i)  (log domain)        (Alg. 3 l.343-344)
 *   3. for s = 1..S:  V_s = A_s V_{s-1};  xi_s^i ~ (V_s^i)^-1 sum_j A_s^ij V_{s-1}^j delta_{xi_{s-1}^j}
 *                                                          (Alg. 3 l.346-349; eq. A matrices 357-360)
 *   4. composition A(i) = a_1(a_2(...a_S(i))), xhat^i = x^{A(i)}  (xi_s^i = xi_{s-1}^{a_s(i)})
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-2)

/* RNG domains (draw contract). */
#define ORC_DOMAIN_INIT 1u
#define ORC_DOMAIN_MUTATE 2u
#define ORC_DOMAIN_RESAMPLE 3u
#define ORC_DOMAIN_WITHIN 4u /* AIRPF within-island draws (reading R19) */
#define ORC_DOMAIN_ISLAND 5u /* AIRPF island side draws (reading R20) */
#define ORC_DOMAIN_MULTI 6u  /* Alg. 2 multinomial draws (reading R22) */

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers:
 * as easy as 1, 2, 3"): 10 rounds of
 *   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 *   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0),
 * with the key bumped by the Weyl constants (W0, W1) before every round but the
 * first.  Pinned against cuRAND's curand_Philox4x32_10 (tests/test_philox.py). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += W0;
            k1 += W1;
        }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One 32-bit word of the draw contract: block counter (c0, n, domain<<24 | sub, 0),
 * key (seed lo, seed hi), word w in 0..3. */
static uint32_t rng_word(uint64_t seed, uint32_t c0, uint32_t n, uint32_t domain,
                         uint32_t sub, int w)
{
    uint32_t ctr[4] = {c0, n, (domain << 24) | sub, 0u};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[w];
}

/* u in [0,1): 24 high bits, exact in fp32 and fp64. */
static double u01(uint32_t r) { return (double)(r >> 8) * 0x1p-24; }
/* u in (0,1]: used for the Box-Muller radius so log(u) is finite. */
static double u01_open0(uint32_t r) { return ((double)(r >> 8) + 1.0) * 0x1p-24; }

/* Standard normal for flat coordinate c of the (domain, n) noise field.
 * Block c/4 gives words (w0,w1,w2,w3); Box-Muller on (w0,w1) gives coordinates
 * 4j, 4j+1 (cos, sin) and on (w2,w3) coordinates 4j+2, 4j+3. */
double orc_normal(uint64_t seed, uint32_t domain, uint32_t n, uint64_t c)
{
    uint32_t ctr[4] = {(uint32_t)(c >> 2), n, domain << 24, 0u};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    int w = (int)(c & 3u);
    int pair = w >> 1;
    double radius = sqrt(-2.0 * log(u01_open0(out[2 * pair])));
    double theta = 2.0 * M_PI * u01(out[2 * pair + 1]);
    return (w & 1) ? radius * sin(theta) : radius * cos(theta);
}

/* ------------------------------------------------------------------------- */
/* The HMM of eq. HMM for the two model families of
 * BASELINE.json: linear-Gaussian (LG) and stochastic volatility (SV). */
typedef struct {
    int kind; /* 1 = LG, 2 = SV */
    int d, dy;
    float A[64], LQ[64], H[64], Rinv[64], m0[8], L0[64]; /* row-major */
    float sv_phi, sv_sigma, sv_beta, sv_m0, sv_s0;
} orc_model;

/* Alg. 1 l.296-298: zeta_0^i iid pi_0.  LG: m0 + L0 z; SV: m0 + s0 z. */
/* x_0 of particle i (global index: the INIT counter). */
static void init_one(const orc_model* mdl, uint64_t seed, uint64_t i, double* x)
{
    int d = mdl->d;
    double z[8];
    for (int k = 0; k < d; ++k)
        z[k] = orc_normal(seed, ORC_DOMAIN_INIT, 0u, i * (uint64_t)d + (uint64_t)k);
    for (int k = 0; k < d; ++k) {
        double v;
        if (mdl->kind == 2) {
            v = (double)mdl->sv_m0 + (double)mdl->sv_s0 * z[k];
        } else {
            v = (double)mdl->m0[k];
            for (int j = 0; j < d; ++j) v += (double)mdl->L0[k * d + j] * z[j];
        }
        x[k] = v;
    }
}

void orc_init(const orc_model* mdl, uint64_t N, uint64_t seed, double* x0)
{
    for (uint64_t i = 0; i < N; ++i) init_one(mdl, seed, i, x0 + i * (uint64_t)mdl->d);
}

/* orc_init evaluated on k given particle indices rows[] (full-size sampled parity). */
void orc_init_rows(const orc_model* mdl, uint64_t seed, uint64_t k, const int64_t* rows, double* x0)
{
    for (uint64_t r = 0; r < k; ++r) init_one(mdl, seed, (uint64_t)rows[r], x0 + r * (uint64_t)mdl->d);
}

/* Alg. 1 l.302-303: zeta_n^i ~ f(zhat_{n-1}^i, .).
 * LG: x = A xhat + LQ z;  SV: x = phi xhat + sigma z.  z from the MUTATE field at n.
 * mutate_one: particle i (global index, the noise counter) from its xhat row. */
static void mutate_one(const orc_model* mdl, uint64_t seed, uint32_t n, uint64_t i, const double* xh, double* x)
{
    int d = mdl->d;
    double z[8];
    for (int k = 0; k < d; ++k)
        z[k] = orc_normal(seed, ORC_DOMAIN_MUTATE, n, i * (uint64_t)d + (uint64_t)k);
    for (int k = 0; k < d; ++k) {
        double v;
        if (mdl->kind == 2) {
            v = (double)mdl->sv_phi * xh[0] + (double)mdl->sv_sigma * z[0];
        } else {
            v = 0.0;
            for (int j = 0; j < d; ++j) v += (double)mdl->A[k * d + j] * xh[j];
            for (int j = 0; j < d; ++j) v += (double)mdl->LQ[k * d + j] * z[j];
        }
        x[k] = v;
    }
}

void orc_mutate(const orc_model* mdl, uint64_t N, uint64_t seed, uint32_t n,
                const double* xhat, double* x)
{
    int d = mdl->d;
    for (uint64_t i = 0; i < N; ++i) mutate_one(mdl, seed, n, i, xhat + i * d, x + i * d);
}

/* g_n(x) = g(x, y_n), in the log domain with normalising constants
 * dropped (reading R9).
 * LG: log g = -1/2 (y - Hx)^T Rinv (y - Hx).
 * SV: y | x ~ N(0, beta^2 e^x)  =>  log g = -x/2 - y^2 e^{-x} / (2 beta^2).
 * A non-finite result (non-finite x) is -inf. */
static double logweight_one(const orc_model* mdl, const float* y, const double* x)
{
    int d = mdl->d, dy = mdl->dy;
    double v;
    if (mdl->kind == 2) {
        double xv = x[0];
        double yv = (double)y[0];
        double beta = (double)mdl->sv_beta;
        v = -0.5 * xv - yv * yv * exp(-xv) / (2.0 * beta * beta);
    } else {
        double r[8];
        for (int k = 0; k < dy; ++k) {
            double hx = 0.0;
            for (int j = 0; j < d; ++j) hx += (double)mdl->H[k * d + j] * x[j];
            r[k] = (double)y[k] - hx;
        }
        double q = 0.0;
        for (int k = 0; k < dy; ++k)
            for (int j = 0; j < dy; ++j) q += r[k] * (double)mdl->Rinv[k * dy + j] * r[j];
        v = -0.5 * q;
    }
    return isfinite(v) ? v : -INFINITY;
}

void orc_logweight(const orc_model* mdl, uint64_t N, const float* y, const double* x,
                   double* lw)
{
    int d = mdl->d;
    for (uint64_t i = 0; i < N; ++i) lw[i] = logweight_one(mdl, y, x + i * d);
}

/* ------------------------------------------------------------------------- */
/* Augmented resampling, Alg. 3 with A_s of eq. A matrices
 * (PAPER.md:357-360).  Groups are 0-based; group g holds particles g*M..g*M+M-1.
 *
 * By Lemma `facts about A`, at stage s group g interacts with
 * exactly one other group, h = g XOR 2^{s-1}; block (g,h) of A_s is (1/2M) 1.
 * By eq. V_defn_proofs, V_s^i = (1/2M) sum over the pair's 2M
 * particles of V_{s-1}^j, so V_s is constant over blocks of 2^s groups; we store
 * it per block:  logV[off(s) + b], b = g >> s, off(s) = m - m/2^{s-1}.
 *
 * Draw law: P(xi_s^i = xi_{s-1}^j) = A_s^ij V_{s-1}^j / V_s^i.
 *   s = 1: the 2M pool (lower group first) with weights g(xi_0^j): inverse CDF,
 *          u = U(RESAMPLE, n, s=1, i); a_1(i) = base + #{k < 2M-1 : C_k <= u C_{2M-1}}
 *          (readings R1-R4).
 *   s >= 2: V_{s-1} is constant over each of the two groups, so the law is
 *          "side L w.p. p = V_L/(V_L+V_R), then uniform index": with M = 2^b and
 *          r = RESAMPLE word, side = L iff (r >> b) < floor(p 2^{32-b}),
 *          index = r & (M-1) (reading R1).
 * RESAMPLE word for (s, i): word i%4 of block (i/4, n, RESAMPLE<<24 | s).
 *
 * Outputs (any may be NULL):
 *   a[(s-1)*N + i]     = a_s(i), the stage-(s-1) position of the stage-s particle i;
 *   delta[(s-1)*N + i] = distance of draw (s,i) to its nearest decision boundary in
 *                        uniform units (stage 1: min_k |u - C_k/C_{2M-1}|;
 *                        s >= 2: |p - ((r>>b)+1)/2^{32-b}|);
 *   logV[m-1]          = all levels s = 1..S (see off(s));
 *   A[N]               = composed ancestor A(i) = a_1(a_2(...a_S(i))).
 */
static int ilog2_exact(uint64_t v)
{
    if (v == 0 || (v & (v - 1)) != 0) return -1;
    int k = 0;
    while ((1ull << k) < v) ++k;
    return k;
}

static uint64_t level_offset(uint64_t m, int s) { return m - (m >> (s - 1)); }

/* log((e^a + e^b)/2): the pair average of eq. V_defn_proofs in the log domain. */
static double log_pair_mean(double a, double b)
{
    double c = a > b ? a : b;
    if (c == -INFINITY) return -INFINITY;
    return c + log((exp(a - c) + exp(b - c)) / 2.0);
}

/* Stage-1 draw for output i of the pool starting at `base` (2M entries, CDF C). */
static void stage1_draw(uint64_t M, uint64_t seed, uint32_t n, uint64_t base, const double* C,
                        uint64_t i, int64_t* a_out, double* delta_out)
{
    uint64_t twoM = 2 * M;
    double u = u01(rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_RESAMPLE, 1u, (int)(i & 3u)));
    double total = C[twoM - 1];
    double t = u * total;
    uint64_t k = 0;
    for (uint64_t kk = 0; kk + 1 < twoM; ++kk)
        if (C[kk] <= t) ++k;
    *a_out = (int64_t)(base + k);
    if (delta_out) {
        double dmin = INFINITY;
        for (uint64_t kk = 0; kk + 1 < twoM; ++kk) {
            double dd = fabs(u - C[kk] / total);
            if (dd < dmin) dmin = dd;
        }
        *delta_out = dmin;
    }
}

/* Stage-s (s >= 2) draw for output i, given the level-(s-1) table. */
static void stage_s_draw(uint64_t M, int b, int s, uint64_t seed, uint32_t n, const double* lv_prev,
                         uint64_t i, int64_t* a_out, double* delta_out)
{
    uint64_t g = i / M;
    uint64_t h = g ^ (1ull << (s - 1));
    uint64_t gl = g < h ? g : h, gr = g < h ? h : g;
    double vl = lv_prev[gl >> (s - 1)], vr = lv_prev[gr >> (s - 1)];
    /* p = V_L / (V_L + V_R) */
    double p = 1.0 / (1.0 + exp(vr - vl));
    if (vl == -INFINITY && vr == -INFINITY) p = 0.5; /* both zero: undefined; never happens for g > 0 */
    double scale = ldexp(1.0, 32 - b);
    uint64_t P = (uint64_t)floor(p * scale);
    uint32_t r = rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_RESAMPLE, (uint32_t)s, (int)(i & 3u));
    uint64_t hi = (uint64_t)(r >> b);
    uint64_t idx = (uint64_t)r & (M - 1);
    uint64_t chosen = (hi < P) ? gl : gr;
    *a_out = (int64_t)(chosen * M + idx);
    if (delta_out) *delta_out = fabs(p - (double)(hi + 1) / scale);
}

/* Stage-1 CDF of the pair starting at base: C_k = sum_{j<=k} exp(lw_j - mx),
 * sequential.  Returns mx. */
static double pair_cdf(const double* lw, uint64_t base, uint64_t twoM, double* C)
{
    double mx = -INFINITY;
    for (uint64_t j = 0; j < twoM; ++j)
        if (lw[base + j] > mx) mx = lw[base + j];
    double acc = 0.0;
    for (uint64_t j = 0; j < twoM; ++j) {
        acc += (mx == -INFINITY) ? 1.0 : exp(lw[base + j] - mx);
        C[j] = acc;
    }
    return mx;
}

/* Alg. 3 with only the first S_exec stages executed (0 <= S_exec <= S): the V levels are
 * computed for every s = 1..S (they depend on the weights only, eq. V_defn_proofs), the
 * draws and the composition for s <= S_exec.  S_exec = S is Alg. 3; S_exec < S is the
 * early stop of the fully adapted scheme.  Stage tables of stages
 * > S_exec are left untouched. */
static int augmented_resample_upto(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw,
                                   int S_exec, int32_t* a, float* delta, double* logV, int64_t* A);

int orc_augmented_resample(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw,
                           int32_t* a, float* delta, double* logV, int64_t* A)
{
    uint64_t m = (M == 0) ? 0 : N / M;
    int S = ilog2_exact(m);
    if (S < 1) return ORC_EINVAL;
    return augmented_resample_upto(N, M, seed, n, lw, S, a, delta, logV, A);
}

int orc_augmented_resample_partial(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw,
                                   int S_exec, int32_t* a, float* delta, double* logV, int64_t* A)
{
    return augmented_resample_upto(N, M, seed, n, lw, S_exec, a, delta, logV, A);
}

static int augmented_resample_upto(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw,
                                   int S_exec, int32_t* a, float* delta, double* logV, int64_t* A)
{
    if (M == 0 || N % M != 0) return ORC_EINVAL;
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    int b = ilog2_exact(M);
    if (S < 1 || b < 0 || S_exec < 0 || S_exec > S) return ORC_EINVAL;
    uint64_t twoM = 2 * M;
    double* lv = (double*)malloc(sizeof(double) * (m - 1));
    double* C = (double*)malloc(sizeof(double) * twoM);
    int32_t* as = (int32_t*)malloc(sizeof(int32_t) * N * (uint64_t)S);
    if (!lv || !C || !as) {
        free(lv); free(C); free(as);
        return ORC_ENOMEM;
    }

    /* Stage s = 1 (Alg. 3 l.346-349 with A_1: pairs (2p, 2p+1)). */
    for (uint64_t p = 0; p < m / 2; ++p) {
        uint64_t base = 2 * p * M;
        double mx = pair_cdf(lw, base, twoM, C);
        /* V_1 = (1/2M) sum_pool g  (eq. V_defn_proofs) */
        lv[level_offset(m, 1) + p] = (mx == -INFINITY) ? -INFINITY : mx + log(C[twoM - 1]) - log((double)twoM);
        for (uint64_t j = 0; j < twoM && S_exec >= 1; ++j) {
            uint64_t i = base + j;
            int64_t ai;
            double dl;
            stage1_draw(M, seed, n, base, C, i, &ai, &dl);
            as[i] = (int32_t)ai;
            if (delta) delta[i] = (float)dl;
        }
    }
    /* Stages s = 2..S (Alg. 3 l.346-349). */
    for (int s = 2; s <= S; ++s) {
        const double* prev = lv + level_offset(m, s - 1);
        double* cur = lv + level_offset(m, s);
        /* V_s = A_s V_{s-1}: block b of level s is the pair mean of blocks 2b, 2b+1. */
        for (uint64_t bk = 0; bk < (m >> s); ++bk) cur[bk] = log_pair_mean(prev[2 * bk], prev[2 * bk + 1]);
        for (uint64_t i = 0; i < N && s <= S_exec; ++i) {
            int64_t ai;
            double dl;
            stage_s_draw(M, b, s, seed, n, prev, i, &ai, &dl);
            as[(uint64_t)(s - 1) * N + i] = (int32_t)ai;
            if (delta) delta[(uint64_t)(s - 1) * N + i] = (float)dl;
        }
    }
    /* Composition: xi_{S_exec}^i = xi_0^{a_1(a_2(...a_{S_exec}(i)))}. */
    if (A) {
        for (uint64_t i = 0; i < N; ++i) {
            uint64_t j = i;
            for (int s = S_exec; s >= 1; --s) j = (uint64_t)as[(uint64_t)(s - 1) * N + j];
            A[i] = (int64_t)j;
        }
    }
    if (a) memcpy(a, as, sizeof(int32_t) * N * (uint64_t)S_exec);
    if (logV) memcpy(logV, lv, sizeof(double) * (m - 1));
    free(lv); free(C); free(as);
    return ORC_OK;
}

/* V table of Alg. 3 (levels 1..S, layout of orc_augmented_resample) from the weights. */
static int v_table(uint64_t N, uint64_t M, const double* lw, double* lv)
{
    uint64_t m = N / M, twoM = 2 * M;
    int S = ilog2_exact(m);
    double* C = (double*)malloc(sizeof(double) * twoM);
    if (!C) return ORC_ENOMEM;
    for (uint64_t p = 0; p < m / 2; ++p) {
        double mx = pair_cdf(lw, 2 * p * M, twoM, C);
        lv[level_offset(m, 1) + p] = (mx == -INFINITY) ? -INFINITY : mx + log(C[twoM - 1]) - log((double)twoM);
    }
    for (int s = 2; s <= S; ++s) {
        const double* prev = lv + level_offset(m, s - 1);
        double* cur = lv + level_offset(m, s);
        for (uint64_t bk = 0; bk < (m >> s); ++bk) cur[bk] = log_pair_mean(prev[2 * bk], prev[2 * bk + 1]);
    }
    free(C);
    return ORC_OK;
}

/* The draws of stages S_exec..1 along the ancestral path of each sampled output (the same
 * draws as orc_augmented_resample).  path/anc/pdelta: k*S + (s-1); stages above S_exec
 * are not drawn (pdelta = +inf, path = anc = -1). */
static int sampled_draws(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw, const double* lv,
                         uint64_t nsamp, const int64_t* outputs, int S_exec, int64_t* path, int64_t* anc,
                         float* pdelta, int64_t* A_out)
{
    uint64_t m = N / M, twoM = 2 * M;
    int S = ilog2_exact(m), b = ilog2_exact(M);
    double* C = (double*)malloc(sizeof(double) * twoM);
    if (!C) return ORC_ENOMEM;
    for (uint64_t k = 0; k < nsamp; ++k) {
        uint64_t j = (uint64_t)outputs[k];
        for (int s = S; s > S_exec; --s) {
            if (path) path[k * S + (uint64_t)(s - 1)] = -1;
            if (anc) anc[k * S + (uint64_t)(s - 1)] = -1;
            if (pdelta) pdelta[k * S + (uint64_t)(s - 1)] = INFINITY;
        }
        for (int s = S_exec; s >= 1; --s) {
            int64_t aj;
            double dl;
            if (s >= 2) {
                stage_s_draw(M, b, s, seed, n, lv + level_offset(m, s - 1), j, &aj, &dl);
            } else {
                uint64_t base = (j / twoM) * twoM;
                pair_cdf(lw, base, twoM, C);
                stage1_draw(M, seed, n, base, C, j, &aj, &dl);
            }
            if (path) path[k * S + (uint64_t)(s - 1)] = (int64_t)j;
            if (anc) anc[k * S + (uint64_t)(s - 1)] = aj;
            if (pdelta) pdelta[k * S + (uint64_t)(s - 1)] = (float)dl;
            j = (uint64_t)aj;
        }
        if (A_out) A_out[k] = (int64_t)j;
    }
    free(C);
    return ORC_OK;
}

/* Same draws, evaluated only along the ancestral paths of `nsamp` sampled outputs
 * (for full-size configurations where S x N tables do not fit).  The V tables are
 * computed in full, exactly as above.  For each sample k and stage s:
 *   path[k*S + (s-1)]  = the stage-s position on the path (path[k*S+S-1] = output),
 *   anc[k*S + (s-1)]   = a_s(path position),  pdelta likewise;  A_out[k] = A(output). */
int orc_augmented_resample_sampled(uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                                   const double* lw, uint64_t nsamp, const int64_t* outputs,
                                   int64_t* path, int64_t* anc, float* pdelta, double* logV,
                                   int64_t* A_out)
{
    if (M == 0 || N % M != 0) return ORC_EINVAL;
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    int b = ilog2_exact(M);
    if (S < 1 || b < 0) return ORC_EINVAL;
    double* lv = (double*)malloc(sizeof(double) * (m - 1));
    if (!lv) return ORC_ENOMEM;
    int rc = v_table(N, M, lw, lv);
    if (rc == ORC_OK) rc = sampled_draws(N, M, seed, n, lw, lv, nsamp, outputs, S, path, anc, pdelta, A_out);
    if (rc == ORC_OK && logV) memcpy(logV, lv, sizeof(double) * (m - 1));
    free(lv);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Estimates of one step (reading R8):
 *   filter   pi_hat_n(phi) = sum_i g_n(x^i) phi(x^i) / sum_i g_n(x^i)
 *   predict  pi_n^N(phi)   = N^-1 sum_i phi(x^i)
 *   resampled N^-1 sum_i phi(xhat^i)
 * for phi = x_k (out[0..d)) and phi = x_k^2 (out[d..2d)), sequential fp64 sums. */
void orc_estimates(int d, uint64_t N, const double* lw, const double* x, const int64_t* A,
                   double* filt, double* pred, double* resamp)
{
    double L = -INFINITY;
    for (uint64_t i = 0; i < N; ++i)
        if (lw[i] > L) L = lw[i];
    double sw = 0.0;
    double s1[8] = {0}, s2[8] = {0}, p1[8] = {0}, p2[8] = {0}, r1[8] = {0}, r2[8] = {0};
    for (uint64_t i = 0; i < N; ++i) {
        double w = exp(lw[i] - L);
        sw += w;
        for (int k = 0; k < d; ++k) {
            double v = x[i * d + k];
            s1[k] += w * v;
            s2[k] += w * v * v;
            p1[k] += v;
            p2[k] += v * v;
            if (A) {
                double vr = x[(uint64_t)A[i] * d + k];
                r1[k] += vr;
                r2[k] += vr * vr;
            }
        }
    }
    for (int k = 0; k < d; ++k) {
        if (filt) { filt[k] = s1[k] / sw; filt[d + k] = s2[k] / sw; }
        if (pred) { pred[k] = p1[k] / (double)N; pred[d + k] = p2[k] / (double)N; }
        if (resamp && A) { resamp[k] = r1[k] / (double)N; resamp[d + k] = r2[k] / (double)N; }
    }
}

/* ------------------------------------------------------------------------- */
/* A whole step of Alg. 1 deploying Alg. 3, from a given xhat_{n-1} (or x_0 when
 * n == 0, when no mutation happens: DESIGN.md reading R7).  Outputs x (N*d), lw,
 * per-stage tables, estimates, and xhat_n (N*d).  Returns an ORC_* code. */
int orc_step(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
             const float* y, const float* xin, double* x, double* lw, int32_t* a, float* delta,
             double* logV, int64_t* A, double* xhat_out, double* filt, double* pred, double* resamp)
{
    int d = mdl->d;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    int64_t* Aloc = (int64_t*)malloc(sizeof(int64_t) * N);
    if (!xprev || !Aloc) {
        free(xprev); free(Aloc);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    orc_logweight(mdl, N, y, x, lw);
    int rc = orc_augmented_resample(N, M, seed, n, lw, a, delta, logV, Aloc);
    if (rc == ORC_OK) {
        if (A) memcpy(A, Aloc, sizeof(int64_t) * N);
        if (xhat_out)
            for (uint64_t i = 0; i < N; ++i)
                for (int k = 0; k < d; ++k) xhat_out[i * d + k] = x[(uint64_t)Aloc[i] * d + k];
        orc_estimates(d, N, lw, x, Aloc, filt, pred, resamp);
    }
    free(xprev); free(Aloc);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Fully adapted augmented resampling (AIRPF2 of PAPER.md:1279).
 *
 * ESS of a weight vector w over n equally sized units:
 *     E = (n^-1 sum w)^2 / (n^-1 sum w^2)  in [1/n, 1],
 * evaluated "after every stage of augmented resampling" on the stage
 * weights V_s: s = 0 on the particle weights V_0 = w (N units); s >= 1 on the level-s
 * values of the V table, which are constant over blocks of 2^s groups, so the N-particle
 * ESS equals the ESS of the m / 2^s block values.  Log domain, shifted by the max;
 * sequential fp64 sums.  ess[0..S]. */
static double ess_of(const double* lv, uint64_t n)
{
    double L = -INFINITY;
    for (uint64_t i = 0; i < n; ++i)
        if (lv[i] > L) L = lv[i];
    if (L == -INFINITY) return 1.0; /* all weights zero: no information, treat as equal */
    double s1 = 0.0, s2 = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double w = exp(lv[i] - L);
        s1 += w;
        s2 += w * w;
    }
    return s1 * s1 / ((double)n * s2);
}

void orc_ess_levels(uint64_t N, uint64_t M, const double* lw, const double* logV, double* ess)
{
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    ess[0] = ess_of(lw, N);
    for (int s = 1; s <= S; ++s) ess[s] = ess_of(logV + level_offset(m, s), m >> s);
}

/* Controller: stage s + 1 runs iff ESS after stage s is below theta (PAPER.md:574,
 * "executes the resampling step only if E_n is below some predetermined threshold";
 * strict rule, reading R17).  Returns S* = min{s in 0..S : ess[s] >= theta};
 * ess[S] = 1 (V_S is constant, Lemma facts_about_Vs (c)) so S* <= S for theta <= 1. */
int orc_stages_to_run(int S, const double* ess, double theta)
{
    for (int s = 0; s < S; ++s)
        if (ess[s] >= theta) return s;
    return S;
}

/* One step of the fully adapted filter from (xin, lwc_in): xin = the state after the
 * previous step (resampled or not), lwc_in[i] = its carried log-weight (0 after a step
 * that ran all S stages).  lw = lwc_in + log g_n(x); stages 1..S* run (S* from the ESS
 * levels of lw); the particles then carry the stage-S* weights V_{S*} (Prop. 1 holds for
 * the partial product A_{S*}...A_1: sum_i V_{S*}^i P(xi_{S*}^i = xi_0^j) = g_j), stored as
 *   lwc_out[i] = log V_{S*}(block of i) - log V_S   (S* >= 1; block = group >> S*),
 *   lwc_out[i] = lw[i] - log V_S                    (S* = 0),
 * i.e. shifted by the global constant log V_S = log N^-1 sum w, which changes no
 * normalised quantity (reading R18).  Outputs as orc_step plus ess[S+1], *sstar. */
int orc_step_adaptive_rot(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                          const float* y, const float* xin, const double* lwc_in, double theta, int rotate,
                          double* x, double* lw, int32_t* a, float* delta, double* logV, int64_t* A,
                          double* xhat_out, double* lwc_out, double* filt, double* pred, double* ess,
                          int* sstar);

/* Stage rotation: the next step starts at the stage after the last one
 * executed.  Realised as a relabelling of the groups (reading R23): the particle arrays
 * are kept in the current layout, where the stage at position t pairs bit t-1 of the
 * layout group index g' = rotr_S(g, rho) (g the natural group, rho the rotation offset);
 * after a step that ran S* >= 1 stages, rho += S* and the outputs move to the next
 * layout, group g' -> rotr_S(g', S*).  All draws are keyed by layout positions.  rotate =
 * 0 leaves the layout fixed (every step starts at stage 1). */
static uint64_t rotr_bits(uint64_t g, int k, int S)
{
    k %= S;
    if (k == 0) return g;
    uint64_t mask = (S >= 64) ? ~0ull : ((1ull << S) - 1);
    return ((g >> k) | (g << (S - k))) & mask;
}

int orc_step_adaptive(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                      const float* y, const float* xin, const double* lwc_in, double theta,
                      double* x, double* lw, int32_t* a, float* delta, double* logV, int64_t* A,
                      double* xhat_out, double* lwc_out, double* filt, double* pred, double* ess,
                      int* sstar)
{
    return orc_step_adaptive_rot(mdl, N, M, seed, n, y, xin, lwc_in, theta, 0, x, lw, a, delta, logV, A, xhat_out,
                                 lwc_out, filt, pred, ess, sstar);
}

int orc_step_adaptive_rot(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                          const float* y, const float* xin, const double* lwc_in, double theta, int rotate,
                          double* x, double* lw, int32_t* a, float* delta, double* logV, int64_t* A,
                          double* xhat_out, double* lwc_out, double* filt, double* pred, double* ess,
                          int* sstar)
{
    int d = mdl->d;
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    if (S < 1) return ORC_EINVAL;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    int64_t* Aloc = (int64_t*)malloc(sizeof(int64_t) * N);
    double* lvl = (double*)malloc(sizeof(double) * (m - 1));
    if (!xprev || !Aloc || !lvl) {
        free(xprev); free(Aloc); free(lvl);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    orc_logweight(mdl, N, y, x, lw);
    for (uint64_t i = 0; i < N; ++i) lw[i] += lwc_in[i];
    /* levels first (S_exec = 0), then the controller, then the stages */
    int rc = augmented_resample_upto(N, M, seed, n, lw, 0, NULL, NULL, lvl, NULL);
    if (rc == ORC_OK) {
        orc_ess_levels(N, M, lw, lvl, ess);
        int ss = orc_stages_to_run(S, ess, theta);
        *sstar = ss;
        rc = augmented_resample_upto(N, M, seed, n, lw, ss, a, delta, logV, Aloc);
        if (rc == ORC_OK) {
            double lvS = lvl[level_offset(m, S)];
            if (A) memcpy(A, Aloc, sizeof(int64_t) * N);
            if (xhat_out)
                for (uint64_t i = 0; i < N; ++i)
                    for (int k = 0; k < d; ++k) xhat_out[i * d + k] = x[(uint64_t)Aloc[i] * d + k];
            for (uint64_t i = 0; i < N; ++i)
                lwc_out[i] = (ss == 0) ? lw[i] - lvS : lvl[level_offset(m, ss) + ((i / M) >> ss)] - lvS;
            orc_estimates(d, N, lw, x, Aloc, filt, pred, NULL);
            if (rotate && ss >= 1 && (ss % S) != 0) {  /* move to the next layout (R23) */
                double* tx = (double*)malloc(sizeof(double) * N * (uint64_t)d);
                double* tc = (double*)malloc(sizeof(double) * N);
                if (!tx || !tc) {
                    free(tx); free(tc);
                    rc = ORC_ENOMEM;
                } else {
                    for (uint64_t i = 0; i < N; ++i) {
                        uint64_t g = i / M, j = i % M;
                        uint64_t dst = rotr_bits(g, ss, S) * M + j;
                        for (int k = 0; k < d; ++k) tx[dst * d + k] = xhat_out[i * d + k];
                        tc[dst] = lwc_out[i];
                    }
                    memcpy(xhat_out, tx, sizeof(double) * N * (uint64_t)d);
                    memcpy(lwc_out, tc, sizeof(double) * N);
                    free(tx); free(tc);
                }
            }
        }
    }
    free(xprev); free(Aloc); free(lvl);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* AIRPF: the augmented island resampling particle filter (Alg. 4)
 * with the within-island resample (Alg. 5) and the augmented
 * island resampling (Alg. 6) or its modified form (Alg. 7,
 * PAPER.md:1137-1160).  Draw contract: DESIGN.md readings R19-R21. */

/* Alg. 5: every output i of island k (particles kM..kM+M-1) draws its source from the
 * island's M particles with probability g_j / sum_island g (the rows of A = I_m (x)
 * 1_{1/M} restricted to the island); W_out = the island mean of g (eq. out weight,
 * PAPER.md:918-922), returned as logW[k].  Inverse CDF with the island's particles in
 * ascending order, u = (r >> 8) 2^-24 from word (i & 3) of block (i >> 2, n,
 * WITHIN << 24), a_w(i) = kM + #{c < M-1 : C_c <= u C_{M-1}}; delta as for stage 1. */
int orc_within_island(uint64_t N, uint64_t M, uint64_t seed, uint32_t n, const double* lw,
                      int64_t* a_w, float* delta, double* logW)
{
    if (M == 0 || N % M != 0) return ORC_EINVAL;
    uint64_t m = N / M;
    double* C = (double*)malloc(sizeof(double) * M);
    if (!C) return ORC_ENOMEM;
    for (uint64_t k = 0; k < m; ++k) {
        uint64_t base = k * M;
        double mx = -INFINITY;
        for (uint64_t j = 0; j < M; ++j)
            if (lw[base + j] > mx) mx = lw[base + j];
        double acc = 0.0;
        for (uint64_t j = 0; j < M; ++j) {
            acc += (mx == -INFINITY) ? 1.0 : exp(lw[base + j] - mx);
            C[j] = acc;
        }
        logW[k] = (mx == -INFINITY) ? -INFINITY : mx + log(C[M - 1]) - log((double)M);
        for (uint64_t j = 0; j < M; ++j) {
            uint64_t i = base + j;
            double u = u01(rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_WITHIN, 0u, (int)(i & 3u)));
            double t = u * C[M - 1];
            uint64_t c = 0;
            for (uint64_t kk = 0; kk + 1 < M; ++kk)
                if (C[kk] <= t) ++c;
            a_w[i] = (int64_t)(base + c);
            if (delta) {
                double dmin = INFINITY;
                for (uint64_t kk = 0; kk + 1 < M; ++kk) {
                    double dd = fabs(u - C[kk] / C[M - 1]);
                    if (dd < dmin) dmin = dd;
                }
                delta[i] = (float)dmin;
            }
        }
    }
    free(C);
    return ORC_OK;
}

/* Alg. 6 (modified = 0) / Alg. 7 (modified = 1) on the island log-weights logW (m):
 *   V_bar_0 = W, V_bar_s = A_bar_s V_bar_{s-1} (pair means; stored in logVbar with the
 *   level layout of orc_augmented_resample, levels 1..S);
 *   at stage s island i draws its whole block from island j in {i, i ^ 2^{s-1}} with
 *   probability V_bar_{s-1}^j / (V_bar_{s-1}^L + V_bar_{s-1}^R) (line 'sampling aug
 *   island'): word (i & 3) of block (i >> 2, n, ISLAND << 24 | s), side L iff
 *   (r >> 1) < floor(p 2^31), p = V_L / (V_L + V_R) (reading R20);
 *   Alg. 7: a pure exchange of a pair (L took R's block and R took L's) is undone
 *   (lines 'loop'/'exchange'; reading R21).
 * src[(s-1) m + i] = the island whose stage-(s-1) block island i holds after stage s;
 * delta as for stage s >= 2; Aisl[i] = src_1(src_2(...src_S(i))). */
static int island_resample_upto(uint64_t m, uint64_t seed, uint32_t n, const double* logW, int modified,
                                int S_exec, int32_t* src, float* delta, double* logVbar, int64_t* Aisl);

int orc_island_resample(uint64_t m, uint64_t seed, uint32_t n, const double* logW, int modified,
                        int32_t* src, float* delta, double* logVbar, int64_t* Aisl)
{
    return island_resample_upto(m, seed, n, logW, modified, ilog2_exact(m), src, delta, logVbar, Aisl);
}

/* Alg. 6/7 with only the island stages 1..S_exec executed (the fully adapted AIRPF,
 * AIRPF2 of PAPER.md:1279; reading R26): every V_bar level is computed, the
 * draws and the composition for s <= S_exec; src rows of later stages are untouched. */
int orc_island_resample_partial(uint64_t m, uint64_t seed, uint32_t n, const double* logW, int modified,
                                int S_exec, int32_t* src, float* delta, double* logVbar, int64_t* Aisl)
{
    return island_resample_upto(m, seed, n, logW, modified, S_exec, src, delta, logVbar, Aisl);
}

static int island_resample_upto(uint64_t m, uint64_t seed, uint32_t n, const double* logW, int modified,
                                int S_exec, int32_t* src, float* delta, double* logVbar, int64_t* Aisl)
{
    int S = ilog2_exact(m);
    if (S < 1 || S_exec < 0 || S_exec > S) return ORC_EINVAL;
    double* lv = (double*)malloc(sizeof(double) * (m - 1));
    int32_t* sr = (int32_t*)malloc(sizeof(int32_t) * m * (uint64_t)S);
    if (!lv || !sr) {
        free(lv); free(sr);
        return ORC_ENOMEM;
    }
    const double scale = ldexp(1.0, 31);
    for (int s = 1; s <= S; ++s) {
        const double* prev = (s == 1) ? logW : lv + level_offset(m, s - 1);
        double* cur = lv + level_offset(m, s);
        for (uint64_t bk = 0; bk < (m >> s); ++bk) cur[bk] = log_pair_mean(prev[2 * bk], prev[2 * bk + 1]);
        if (s > S_exec) continue;
        uint64_t bit = 1ull << (s - 1);
        for (uint64_t i = 0; i < m; ++i) {
            uint64_t h = i ^ bit;
            uint64_t L = i < h ? i : h, R = i < h ? h : i;
            double vl = prev[L >> (s - 1)], vr = prev[R >> (s - 1)];
            double p = (vl == -INFINITY && vr == -INFINITY) ? 0.5 : 1.0 / (1.0 + exp(vr - vl));
            uint64_t P = (uint64_t)floor(p * scale);
            uint32_t r = rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_ISLAND, (uint32_t)s, (int)(i & 3u));
            uint64_t hi = (uint64_t)(r >> 1);
            sr[(uint64_t)(s - 1) * m + i] = (int32_t)((hi < P) ? L : R);
            if (delta) delta[(uint64_t)(s - 1) * m + i] = (float)fabs(p - (double)(hi + 1) / scale);
        }
        if (modified) {
            for (uint64_t L = 0; L < m; ++L) {
                if (L & bit) continue;
                uint64_t R = L | bit;
                int32_t* sl = &sr[(uint64_t)(s - 1) * m + L];
                int32_t* sR = &sr[(uint64_t)(s - 1) * m + R];
                if (*sl == (int32_t)R && *sR == (int32_t)L) {
                    *sl = (int32_t)L;
                    *sR = (int32_t)R;
                }
            }
        }
    }
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t c = i;
        for (int s = S_exec; s >= 1; --s) c = (uint64_t)sr[(uint64_t)(s - 1) * m + c];
        Aisl[i] = (int64_t)c;
    }
    if (src) memcpy(src, sr, sizeof(int32_t) * m * (uint64_t)S_exec);
    if (logVbar) memcpy(logVbar, lv, sizeof(double) * (m - 1));
    free(lv); free(sr);
    return ORC_OK;
}

/* One AIRPF step (Alg. 4 rotated like Alg. 1, reading R7): mutate xin (n >= 1), weight,
 * estimates (before resampling, as orc_step), within-island resample (Alg. 5), augmented
 * island resample (Alg. 6/7) of the island blocks; xhat[i M + j] = x[a_w(Aisl(i) M + j)]. */
int orc_step_airpf(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                   const float* y, const float* xin, int modified, double* x, double* lw, int64_t* a_w,
                   float* wdelta, double* logW, int32_t* src, float* idelta, double* logVbar, int64_t* Aisl,
                   double* xhat_out, double* filt, double* pred)
{
    int d = mdl->d;
    uint64_t m = N / M;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    if (!xprev) return ORC_ENOMEM;
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    free(xprev);
    orc_logweight(mdl, N, y, x, lw);
    orc_estimates(d, N, lw, x, NULL, filt, pred, NULL);
    int rc = orc_within_island(N, M, seed, n, lw, a_w, wdelta, logW);
    if (rc != ORC_OK) return rc;
    rc = orc_island_resample(m, seed, n, logW, modified, src, idelta, logVbar, Aisl);
    if (rc != ORC_OK) return rc;
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < M; ++j) {
            uint64_t a = (uint64_t)a_w[(uint64_t)Aisl[i] * M + j];
            for (int k = 0; k < d; ++k) xhat_out[(i * M + j) * d + k] = x[a * d + k];
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Alg. 2, multinomial resampling: every output i draws its source from
 * all N particles with probability g_j / sum g.  Inverse CDF over the whole population in
 * ascending order (reading R22): C_k = sum_{j<=k} e^{lw_j - L} (sequential, L = max lw),
 * u = (r >> 8) 2^-24 from word (i & 3) of block (i >> 2, n, MULTI << 24),
 * a(i) = #{k < N-1 : C_k <= u C_{N-1}}, found by bisection of the non-decreasing C (the
 * count, pinned against the literal count in tests); delta = distance of u to the nearest
 * C_k / C_{N-1}. */
int orc_multinomial(uint64_t N, uint64_t seed, uint32_t n, const double* lw, int64_t* a, float* delta)
{
    if (N == 0) return ORC_EINVAL;
    double* C = (double*)malloc(sizeof(double) * N);
    if (!C) return ORC_ENOMEM;
    double L = -INFINITY;
    for (uint64_t j = 0; j < N; ++j)
        if (lw[j] > L) L = lw[j];
    double acc = 0.0;
    for (uint64_t j = 0; j < N; ++j) {
        acc += (L == -INFINITY) ? 1.0 : exp(lw[j] - L);
        C[j] = acc;
    }
    const double total = C[N - 1];
    for (uint64_t i = 0; i < N; ++i) {
        double u = u01(rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_MULTI, 0u, (int)(i & 3u)));
        double t = u * total;
        /* smallest k in [0, N-1] with C_k > t, restricted to k < N-1: the count of C_k <= t */
        uint64_t lo = 0, hi = N - 1; /* answer in [0, N-1] */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (C[mid] <= t) lo = mid + 1;
            else hi = mid;
        }
        a[i] = (int64_t)lo;
        if (delta) {
            double d1 = (lo < N - 1) ? fabs(u - C[lo] / total) : INFINITY;
            double d0 = (lo > 0) ? fabs(u - C[lo - 1] / total) : INFINITY;
            delta[i] = (float)(d0 < d1 ? d0 : d1);
        }
    }
    free(C);
    return ORC_OK;
}

/* One step of Alg. 1 with Alg. 2 (rotated as orc_step). */
int orc_step_multinomial(const orc_model* mdl, uint64_t N, uint64_t seed, uint32_t n, const float* y,
                         const float* xin, double* x, double* lw, int64_t* a, float* delta, double* xhat_out,
                         double* filt, double* pred)
{
    int d = mdl->d;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    if (!xprev) return ORC_ENOMEM;
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    free(xprev);
    orc_logweight(mdl, N, y, x, lw);
    orc_estimates(d, N, lw, x, NULL, filt, pred, NULL);
    int rc = orc_multinomial(N, seed, n, lw, a, delta);
    if (rc != ORC_OK) return rc;
    for (uint64_t i = 0; i < N; ++i)
        for (int k = 0; k < d; ++k) xhat_out[i * d + k] = x[(uint64_t)a[i] * d + k];
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Full-size checks on sampled outputs (C4: N = 2^28).  lw_pass: x_n (mutated from xin
 * when n >= 1) and lw for all N particles (lw kept, x not), with the estimates accumulated
 * in the same pass: Sum g phi / Sum g with the weights shifted by the running maximum of
 * lw (rescaled whenever it grows) -- the same quantity as orc_estimates' shift by the final
 * maximum, in one pass.  filt / pred: 2d each (phi = x, then x^2). */
static void lw_pass(const orc_model* mdl, uint64_t N, uint64_t seed, uint32_t n, const float* y, const float* xin,
                    double* lw, double* filt, double* pred)
{
    int d = mdl->d;
    double L = -INFINITY, sw = 0.0;
    double s1[8] = {0}, s2[8] = {0}, p1[8] = {0}, p2[8] = {0};
    for (uint64_t i = 0; i < N; ++i) {
        double xh[8], x[8];
        for (int k = 0; k < d; ++k) xh[k] = (double)xin[i * d + k];
        if (n == 0) memcpy(x, xh, sizeof(double) * d);
        else mutate_one(mdl, seed, n, i, xh, x);
        lw[i] = logweight_one(mdl, y, x);
        if (lw[i] > L) {  /* new running maximum: rescale what was accumulated */
            double f = (L == -INFINITY) ? 0.0 : exp(L - lw[i]);
            sw *= f;
            for (int k = 0; k < d; ++k) { s1[k] *= f; s2[k] *= f; }
            L = lw[i];
        }
        double w = (lw[i] == -INFINITY) ? 0.0 : exp(lw[i] - L);
        sw += w;
        for (int k = 0; k < d; ++k) {
            s1[k] += w * x[k];
            s2[k] += w * x[k] * x[k];
            p1[k] += x[k];
            p2[k] += x[k] * x[k];
        }
    }
    for (int k = 0; k < d; ++k) {
        filt[k] = s1[k] / sw; filt[d + k] = s2[k] / sw;
        pred[k] = p1[k] / (double)N; pred[d + k] = p2[k] / (double)N;
    }
}

/* x_n of particle j (recomputed from its xin row). */
static void x_of(const orc_model* mdl, uint64_t seed, uint32_t n, const float* xin, uint64_t j, double* x)
{
    int d = mdl->d;
    double xh[8];
    for (int c = 0; c < d; ++c) xh[c] = (double)xin[j * d + c];
    if (n == 0) memcpy(x, xh, sizeof(double) * d);
    else mutate_one(mdl, seed, n, j, xh, x);
}

/* One step (plain, or fully adapted with theta > 0) at full size, on sampled outputs:
 * the whole V table (logV, m - 1), the estimates, with theta > 0 the ESS levels (ess,
 * S + 1) and S* (*sstar; the stop rule of orc_stages_to_run), and for each sampled output
 * its composed ancestor A (stages S*..1), the boundary distances on its path (pdelta,
 * nsamp x S, +inf above S*) and its resampled state (xhat_out, nsamp x d). */
int orc_step_sampled(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                     const float* y, const float* xin, double theta, uint64_t nsamp, const int64_t* outputs,
                     double* logV, double* ess, int* sstar, int64_t* A_out, float* pdelta, double* xhat_out,
                     double* filt, double* pred)
{
    if (M == 0 || N % M != 0 || ilog2_exact(N / M) < 1) return ORC_EINVAL;
    int S = ilog2_exact(N / M);
    double* lw = (double*)malloc(sizeof(double) * N);
    if (!lw) return ORC_ENOMEM;
    lw_pass(mdl, N, seed, n, y, xin, lw, filt, pred);
    int rc = v_table(N, M, lw, logV);
    int se = S;
    if (rc == ORC_OK && theta > 0.0) {
        orc_ess_levels(N, M, lw, logV, ess);
        se = orc_stages_to_run(S, ess, theta);
    }
    if (sstar) *sstar = se;
    if (rc == ORC_OK) rc = sampled_draws(N, M, seed, n, lw, logV, nsamp, outputs, se, NULL, NULL, pdelta, A_out);
    if (rc == ORC_OK)
        for (uint64_t k = 0; k < nsamp; ++k) x_of(mdl, seed, n, xin, (uint64_t)A_out[k], xhat_out + k * mdl->d);
    free(lw);
    return rc;
}

/* One AIRPF step (orc_step_airpf) at full size, on sampled outputs: the island
 * log-means (logW, m), the island map (Aisl, m), the estimates, and for each sampled
 * output i = b M + j its resampled state x[a_w(Aisl(b) M + j)] (xhat_out) with the
 * smallest boundary distance on its path (sdelta): the within-island draw it takes and,
 * at every island stage, the draws of both islands of the pair (Alg. 7 couples them). */
int orc_step_airpf_sampled(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                           const float* y, const float* xin, int modified, uint64_t nsamp, const int64_t* outputs,
                           double* logW, int64_t* Aisl, float* sdelta, double* xhat_out, double* filt, double* pred)
{
    if (M == 0 || N % M != 0 || ilog2_exact(N / M) < 1) return ORC_EINVAL;
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    double* lw = (double*)malloc(sizeof(double) * N);
    int64_t* a_w = (int64_t*)malloc(sizeof(int64_t) * N);
    float* wdelta = (float*)malloc(sizeof(float) * N);
    int32_t* src = (int32_t*)malloc(sizeof(int32_t) * m * (uint64_t)S);
    float* idelta = (float*)malloc(sizeof(float) * m * (uint64_t)S);
    int rc = (lw && a_w && wdelta && src && idelta) ? ORC_OK : ORC_ENOMEM;
    if (rc == ORC_OK) {
        lw_pass(mdl, N, seed, n, y, xin, lw, filt, pred);
        rc = orc_within_island(N, M, seed, n, lw, a_w, wdelta, logW);
    }
    if (rc == ORC_OK) rc = orc_island_resample(m, seed, n, logW, modified, src, idelta, NULL, Aisl);
    if (rc == ORC_OK)
        for (uint64_t k = 0; k < nsamp; ++k) {
            uint64_t i = (uint64_t)outputs[k], c = i / M, j = i % M;
            float dmin = INFINITY;
            for (int s = S; s >= 1; --s) {
                uint64_t h = c ^ (1ull << (s - 1));
                float a = idelta[(uint64_t)(s - 1) * m + c], b = idelta[(uint64_t)(s - 1) * m + h];
                if (a < dmin) dmin = a;
                if (b < dmin) dmin = b;
                c = (uint64_t)src[(uint64_t)(s - 1) * m + c];
            }
            uint64_t q = c * M + j;  /* c = Aisl(i / M) */
            if (wdelta[q] < dmin) dmin = wdelta[q];
            sdelta[k] = dmin;
            x_of(mdl, seed, n, xin, (uint64_t)a_w[q], xhat_out + k * mdl->d);
        }
    free(lw); free(a_w); free(wdelta); free(src); free(idelta);
    return rc;
}

/* Multinomial step (orc_step_multinomial, Alg. 2) at full size on sampled outputs: the
 * estimates, and per sampled output i its ancestor a(i) (the literal CDF search of
 * orc_multinomial on the fp64 CDF of all N weights), the distance of its uniform to the
 * nearest boundary C_k / C_{N-1} (sdelta) and the states of the particles a(i) + k,
 * k = -2..2 (xnb, nsamp x 5 x d; NaN outside [0, N)), and the index window [klo, khi] of
 * the draws for the uniforms u - eps and u + eps (every ancestor a draw within eps of u in
 * uniform units could select). */
static uint64_t cdf_search(const double* C, uint64_t N, double t)
{
    uint64_t lo = 0, hi = N - 1;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (C[mid] <= t) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

int orc_step_multinomial_sampled(const orc_model* mdl, uint64_t N, uint64_t seed, uint32_t n, const float* y,
                                 const float* xin, uint64_t nsamp, const int64_t* outputs, double eps,
                                 int64_t* a_out, int64_t* klo, int64_t* khi, float* sdelta, double* xnb,
                                 double* filt, double* pred)
{
    int d = mdl->d;
    if (N == 0) return ORC_EINVAL;
    double* lw = (double*)malloc(sizeof(double) * N);
    double* C = (double*)malloc(sizeof(double) * N);
    if (!lw || !C) {
        free(lw); free(C);
        return ORC_ENOMEM;
    }
    lw_pass(mdl, N, seed, n, y, xin, lw, filt, pred);
    double L = -INFINITY;
    for (uint64_t j = 0; j < N; ++j)
        if (lw[j] > L) L = lw[j];
    double acc = 0.0;
    for (uint64_t j = 0; j < N; ++j) {
        acc += (L == -INFINITY) ? 1.0 : exp(lw[j] - L);
        C[j] = acc;
    }
    const double total = C[N - 1];
    for (uint64_t k = 0; k < nsamp; ++k) {
        uint64_t i = (uint64_t)outputs[k];
        double u = u01(rng_word(seed, (uint32_t)(i >> 2), n, ORC_DOMAIN_MULTI, 0u, (int)(i & 3u)));
        uint64_t lo = cdf_search(C, N, u * total);
        a_out[k] = (int64_t)lo;
        klo[k] = (int64_t)cdf_search(C, N, (u - eps) * total);
        khi[k] = (int64_t)cdf_search(C, N, (u + eps) * total);
        double d1 = (lo < N - 1) ? fabs(u - C[lo] / total) : INFINITY;
        double d0 = (lo > 0) ? fabs(u - C[lo - 1] / total) : INFINITY;
        sdelta[k] = (float)(d0 < d1 ? d0 : d1);
        for (int o = -2; o <= 2; ++o) {
            double* dst = xnb + (k * 5 + (uint64_t)(o + 2)) * d;
            int64_t j = (int64_t)lo + o;
            if (j < 0 || (uint64_t)j >= N) {
                for (int c = 0; c < d; ++c) dst[c] = NAN;
            } else {
                x_of(mdl, seed, n, xin, (uint64_t)j, dst);
            }
        }
    }
    free(lw); free(C);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Relabelled exchange across G shards ("keeps resampled particles on
 * the GPU holding their ancestor, ships only the per-GPU count imbalance"; the disabled
 * surplus sketch of PAPER.md:826-850: "the PEs with more resampled particles send the
 * surplus particles to the paired PE with fewer than M resampled particles";
 * DESIGN.md reading R24).
 *
 * The N particles form G = 2^L equal shards, shard r = positions [r N/G, (r+1) N/G).
 * Stage s = S - L + t (t = 1..L) pairs every group of shard r with the same local group
 * of shard r' = r ^ 2^{t-1}.  At such a stage every output first takes its Alg. 3 draw
 * (stage_s_draw).  With A_r the outputs of r whose draw lies in r' and A_r' the outputs
 * of r' whose draw lies in r, both in increasing position, the k-th outputs of the two
 * lists exchange their draws for k < min(|A_r|, |A_r'|): each then reads a particle of
 * its own shard, and only the |A_r| - |A_r'| unmatched outputs of the longer list read
 * across the pair.  The exchange permutes outputs inside a block on which V_s is
 * constant (Lemma facts_about_Vs), so the V-weighted sample after the stage -- and with
 * it the unbiasedness of Prop. 1, eq. aug_res_lack_of_bias -- is that
 * of Alg. 3 (pinned in rationals by enumeration, tests/test_oracle_relabel.py).
 *
 * orc_relabel_stage applies the exchange to one cross stage's table `as` (N entries:
 * output position -> source position at stage s-1) in place; excess[r] = the number of
 * outputs of shard r that still read across the pair (unmatched). */
int orc_relabel_stage(uint64_t N, uint64_t G, int t, int32_t* as, uint64_t* excess)
{
    int L = ilog2_exact(G);
    if (L < 1 || t < 1 || t > L || N % G != 0) return ORC_EINVAL;
    uint64_t nl = N / G;
    uint64_t half = 1ull << (t - 1);
    uint64_t* lr = (uint64_t*)malloc(sizeof(uint64_t) * nl);
    uint64_t* lp = (uint64_t*)malloc(sizeof(uint64_t) * nl);
    if (!lr || !lp) {
        free(lr); free(lp);
        return ORC_ENOMEM;
    }
    for (uint64_t r = 0; r < G; ++r) {
        if (r & half) continue; /* visit each pair once, from its lower shard */
        uint64_t rp = r | half;
        uint64_t nr = 0, np = 0;
        for (uint64_t i = r * nl; i < (r + 1) * nl; ++i)
            if ((uint64_t)as[i] / nl == rp) lr[nr++] = i;
        for (uint64_t i = rp * nl; i < (rp + 1) * nl; ++i)
            if ((uint64_t)as[i] / nl == r) lp[np++] = i;
        uint64_t k0 = nr < np ? nr : np;
        for (uint64_t k = 0; k < k0; ++k) {
            int32_t tmp = as[lr[k]];
            as[lr[k]] = as[lp[k]];
            as[lp[k]] = tmp;
        }
        if (excess) {
            excess[r] = nr - k0;
            excess[rp] = np - k0;
        }
    }
    free(lr); free(lp);
    return ORC_OK;
}

/* Alg. 3 on log-weights lw with the last L = log2 G stages relabelled (orc_relabel_stage):
 * tables a (S x N, relabelled), delta (the Alg. 3 draws' boundary distances), logV, the
 * composed ancestors A, and excess (L x G). */
int orc_augmented_resample_relabel(uint64_t N, uint64_t M, uint64_t G, uint64_t seed, uint32_t n, const double* lw,
                                   int32_t* a, float* delta, double* logV, int64_t* A, uint64_t* excess)
{
    uint64_t m = (M == 0) ? 0 : N / M;
    int S = ilog2_exact(m), L = ilog2_exact(G);
    if (S < 1 || L < 1 || (m / G) < 2 || m % G != 0) return ORC_EINVAL;
    int32_t* as = (int32_t*)malloc(sizeof(int32_t) * N * (uint64_t)S);
    if (!as) return ORC_ENOMEM;
    int rc = augmented_resample_upto(N, M, seed, n, lw, S, as, delta, logV, NULL);
    for (int t = 1; t <= L && rc == ORC_OK; ++t)
        rc = orc_relabel_stage(N, G, t, as + (uint64_t)(S - L + t - 1) * N, excess ? excess + (uint64_t)(t - 1) * G : NULL);
    if (rc == ORC_OK) {
        if (A)
            for (uint64_t i = 0; i < N; ++i) {
                uint64_t j = i;
                for (int s = S; s >= 1; --s) j = (uint64_t)as[(uint64_t)(s - 1) * N + j];
                A[i] = (int64_t)j;
            }
        if (a) memcpy(a, as, sizeof(int32_t) * N * (uint64_t)S);
    }
    free(as);
    return rc;
}

/* One step of Alg. 1 deploying Alg. 3 with the relabelled exchange on G shards (same
 * outputs as orc_step, plus excess). */
int orc_step_relabel(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t G, uint64_t seed, uint32_t n,
                     const float* y, const float* xin, double* x, double* lw, int32_t* a, float* delta,
                     double* logV, int64_t* A, double* xhat_out, double* filt, double* pred, double* resamp,
                     uint64_t* excess)
{
    int d = mdl->d;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    int64_t* Aloc = (int64_t*)malloc(sizeof(int64_t) * N);
    if (!xprev || !Aloc) {
        free(xprev); free(Aloc);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    orc_logweight(mdl, N, y, x, lw);
    int rc = orc_augmented_resample_relabel(N, M, G, seed, n, lw, a, delta, logV, Aloc, excess);
    if (rc == ORC_OK) {
        if (A) memcpy(A, Aloc, sizeof(int64_t) * N);
        if (xhat_out)
            for (uint64_t i = 0; i < N; ++i)
                for (int k = 0; k < d; ++k) xhat_out[i * d + k] = x[(uint64_t)Aloc[i] * d + k];
        orc_estimates(d, N, lw, x, Aloc, filt, pred, resamp);
    }
    free(xprev); free(Aloc);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* AIRPF with the fully adapted scheme, AIRPF2 ("AIRPF with the fully adapted
 * resampling scheme"; the scheme of PAPER.md:570-576; reading R26).  One step:
 *   mutate (n >= 1), weight: lw = log g_n + lwc_in (the weight carried from the previous
 *   step, constant over each island), estimates (before resampling, with the carried
 *   weights), within-island resample (Alg. 5, always), island log-means logW = log W_check;
 *   the ESS of the island weights E_0 = ESS(W_check) over the m islands (every particle of
 *   island k carries W_check_k after Alg. 5, so it is the particle-level ESS) and of every
 *   level E_s = ESS(V_bar_s) over the m / 2^s blocks (orc_ess_levels with M = 1);
 *   S* = min{s : E_s >= theta} (orc_stages_to_run, reading R17); the island stages
 *   1..S* (Alg. 6/7); the islands carry V_bar_{S*} of their block (S* = 0: their own
 *   W_check), normalised by V_bar_S (lwc_out per particle, reading R18). */
int orc_step_airpf_adaptive(const orc_model* mdl, uint64_t N, uint64_t M, uint64_t seed, uint32_t n,
                            const float* y, const float* xin, const double* lwc_in, double theta, int modified,
                            double* x, double* lw, int64_t* a_w, float* wdelta, double* logW, int32_t* src,
                            float* idelta, double* logVbar, int64_t* Aisl, double* xhat_out, double* lwc_out,
                            double* filt, double* pred, double* ess, int* sstar)
{
    int d = mdl->d;
    uint64_t m = N / M;
    int S = ilog2_exact(m);
    if (S < 1) return ORC_EINVAL;
    double* xprev = (double*)malloc(sizeof(double) * N * (uint64_t)d);
    double* lvb = (double*)malloc(sizeof(double) * (m - 1));
    int64_t* Ai = (int64_t*)malloc(sizeof(int64_t) * m);
    if (!xprev || !lvb || !Ai) {
        free(xprev); free(lvb); free(Ai);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < N * (uint64_t)d; ++i) xprev[i] = (double)xin[i];
    if (n == 0) memcpy(x, xprev, sizeof(double) * N * (uint64_t)d);
    else orc_mutate(mdl, N, seed, n, xprev, x);
    orc_logweight(mdl, N, y, x, lw);
    for (uint64_t i = 0; i < N; ++i) lw[i] += lwc_in[i];
    orc_estimates(d, N, lw, x, NULL, filt, pred, NULL);
    int rc = orc_within_island(N, M, seed, n, lw, a_w, wdelta, logW);
    if (rc == ORC_OK) rc = island_resample_upto(m, seed, n, logW, modified, 0, NULL, NULL, lvb, Ai);
    if (rc == ORC_OK) {
        orc_ess_levels(m, 1, logW, lvb, ess);
        int ss = orc_stages_to_run(S, ess, theta);
        *sstar = ss;
        rc = island_resample_upto(m, seed, n, logW, modified, ss, src, idelta, logVbar, Ai);
        if (rc == ORC_OK) {
            double lvS = lvb[level_offset(m, S)];
            for (uint64_t i = 0; i < m; ++i) {
                Aisl[i] = Ai[i];
                double c = (ss == 0) ? logW[i] - lvS : lvb[level_offset(m, ss) + (i >> ss)] - lvS;
                for (uint64_t j = 0; j < M; ++j) {
                    uint64_t a = (uint64_t)a_w[(uint64_t)Ai[i] * M + j];
                    for (int k = 0; k < d; ++k) xhat_out[(i * M + j) * d + k] = x[a * d + k];
                    lwc_out[i * M + j] = c;
                }
            }
        }
    }
    free(xprev); free(lvb); free(Ai);
    return rc;
}
