// pf_api.cu -- C-ABI (include/pf.h) and host orchestration of one BPF step.
//
// Launch sequence of pf_step:
//   k_pass1 (NT tiles) -> k_cascade (ceil(NT/2048) CTAs) -> k_compose x (#passes)
// Index mode (d >= 4): the passes compose int32 ancestor maps; the next step's k_pass1
// gathers x[A(i)] (one random 4d-byte read per particle).  State mode (d <= 2): the
// passes move the fp32 states themselves (a state is no bigger than an index).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pf.h"
#include "pf_kernels.cuh"

using namespace pfk;

namespace {

constexpr uint32_t kPass1SmemBudget = 112u * 1024u;
constexpr uint32_t kComposeSmemBudget = 200u * 1024u;
constexpr uint32_t kLPC = 2048u;

struct ComposePass {
    uint32_t s0, k, P;
    bool ident;
};

struct Plan {
    int D;
    bool index_mode;
    uint32_t P1, k1, NT, LPC, cascade_grid, pass1_threads;
    uint32_t pass1_smem;
    std::vector<ComposePass> passes;
};

int ilog2_exact(uint64_t v) {
    if (v == 0 || (v & (v - 1)) != 0) return -1;
    int k = 0;
    while ((1ull << k) < v) ++k;
    return k;
}

size_t align256(size_t v) { return (v + 255u) & ~size_t(255u); }

bool make_plan(int d, uint64_t N, uint32_t M, Plan* pl, std::string* err) {
    const uint64_t m = N / M;
    const int S = ilog2_exact(m);
    const int b = ilog2_exact(M);
    Plan p;
    p.D = d;
    p.index_mode = d >= 4;
    // pass-1 tile: the largest 2^k1 groups with k1 <= S whose shared memory fits
    uint32_t P1 = (uint32_t)std::min<uint64_t>(N, 65536u);
    for (;;) {
        const uint32_t k1 = (uint32_t)ilog2_exact(P1 / M);
        if (pass1_smem(d, P1, M, k1).total <= kPass1SmemBudget || P1 <= 2 * M) break;
        P1 >>= 1;
    }
    if (P1 < 2 * M) P1 = 2 * M;
    p.P1 = P1;
    p.k1 = (uint32_t)ilog2_exact(P1 / M);
    if ((int)p.k1 > S) {
        *err = "internal: k1 > S";
        return false;
    }
    p.pass1_smem = pass1_smem(d, P1, M, p.k1).total;
    if (p.pass1_smem > 227u * 1024u) {
        *err = "pass-1 tile does not fit in shared memory (M too large for d)";
        return false;
    }
    p.NT = (uint32_t)(N / P1);
    p.LPC = std::min<uint32_t>(p.NT, kLPC);
    p.cascade_grid = p.NT / p.LPC;
    if (p.cascade_grid > kLPC) {
        *err = "too many pass-1 tiles for the cascade tree";
        return false;
    }
    const uint32_t nq = P1 / 4;
    p.pass1_threads = std::max<uint32_t>(32u, std::min<uint32_t>(kPass1Threads, nq));
    if ((nq + p.pass1_threads - 1) / p.pass1_threads > (uint32_t)kMaxQuadsPerThread) {
        *err = "internal: too many quads per thread";
        return false;
    }
    // compose passes for stages k1+1..S
    uint32_t s = p.k1 + 1;
    bool first = true;
    while ((int)s <= S) {
        const bool ident = p.index_mode && first;
        const uint32_t payload = ident ? 0u : (p.index_mode ? 4u : (uint32_t)(4 * d));
        uint32_t P = 65536u;
        while (P > 2 * M && (compose_smem(P, payload) > kComposeSmemBudget || P > N)) P >>= 1;
        if (P < 2 * M) P = 2 * M;
        if (compose_smem(P, payload) > 227u * 1024u) {
            *err = "compose tile does not fit in shared memory";
            return false;
        }
        uint32_t k = (uint32_t)ilog2_exact(P / M);
        if (k > (uint32_t)S - s + 1) k = (uint32_t)S - s + 1;
        P = M << k;
        p.passes.push_back({s, k, P, ident});
        s += k;
        first = false;
    }
    (void)b;
    *pl = p;
    return true;
}

struct Layout {
    size_t X0, X1, A0, A1, logV, thr, part, scratch, est, ticket, y;
    size_t dbg_x, dbg_lw, dbg_anc, dbg_A, dbg_xhat;
    size_t total;
};

Layout make_layout(const Plan& p, uint64_t N, uint32_t M, uint32_t flags) {
    Layout L;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align256(off + bytes);
        return o;
    };
    const uint64_t m = N / M;
    const int S = ilog2_exact(m);
    const int PS = 2 + 4 * p.D;
    const size_t xb = (size_t)N * p.D * 4;
    L.X0 = take(xb);
    L.X1 = take(xb);
    L.A0 = take(p.index_mode ? N * 4 : 0);
    L.A1 = take(p.index_mode ? N * 4 : 0);
    L.logV = take(m * 8);
    L.thr = take(m * 4);
    L.part = take((size_t)p.NT * PS * 8);
    L.scratch = take((size_t)(p.NT + 2) * PS * 8);
    L.est = take(4 * 8 * 8);
    L.ticket = take(16);
    L.y = take(64);
    const bool dbg = flags & PF_FLAG_DEBUG;
    L.dbg_x = take(dbg ? xb : 0);
    L.dbg_lw = take(dbg ? N * 4 : 0);
    L.dbg_anc = take(dbg ? (size_t)N * S * 4 : 0);
    L.dbg_A = take(dbg ? N * 4 : 0);
    L.dbg_xhat = take(xb);
    L.total = off;
    return L;
}

}  // namespace

struct pf_handle {
    ModelParams mp;
    uint64_t N;
    uint32_t M, b, m, S;
    uint64_t seed;
    uint32_t flags;
    Plan plan;
    Layout lay;
    unsigned char* ws;
    cudaStream_t stream;
    // state
    uint32_t n;          // index of the next step
    int cur;             // X buffer that holds the gather source / xhat for the next step
    int amap;            // A buffer holding the next step's gather map (index mode)
    bool a_identity;     // next step reads X[cur] without a map
    bool have_step;
    int last_launches;
    std::string err;
    float* X(int i) { return reinterpret_cast<float*>(ws + (i ? lay.X1 : lay.X0)); }
    int32_t* A(int i) { return reinterpret_cast<int32_t*>(ws + (i ? lay.A1 : lay.A0)); }
    template <typename T>
    T* at(size_t off) { return reinterpret_cast<T*>(ws + off); }
};

static std::string g_init_error;

static int fail(pf_handle* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    else g_init_error = msg;
    return code;
}

static int check_cuda(pf_handle* h, const char* where) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
    return PF_OK;
}

static bool validate_model(const pf_model* mdl, std::string* err) {
    if (!mdl) {
        *err = "model is NULL";
        return false;
    }
    if (mdl->kind == PF_SV) {
        if (mdl->d != 1 || mdl->dy != 1) {
            *err = "PF_SV requires d = dy = 1";
            return false;
        }
        if (!(mdl->sv_beta > 0.0f) || !std::isfinite(mdl->sv_phi) || !std::isfinite(mdl->sv_sigma)) {
            *err = "PF_SV parameters invalid";
            return false;
        }
        return true;
    }
    if (mdl->kind != PF_LG) {
        *err = "unknown model kind";
        return false;
    }
    if (mdl->d != 1 && mdl->d != 2 && mdl->d != 4 && mdl->d != 8) {
        *err = "d must be 1, 2, 4 or 8";
        return false;
    }
    if (mdl->dy < 1 || mdl->dy > 8) {
        *err = "dy must be in 1..8";
        return false;
    }
    if (!mdl->A || !mdl->LQ || !mdl->H || !mdl->Rinv || !mdl->m0 || !mdl->L0) {
        *err = "PF_LG model matrices must be non-NULL";
        return false;
    }
    const int d = mdl->d;
    for (int k = 0; k < d; ++k)
        for (int j = k + 1; j < d; ++j)
            if (mdl->LQ[k * d + j] != 0.0f || mdl->L0[k * d + j] != 0.0f) {
                *err = "LQ and L0 must be lower triangular";
                return false;
            }
    return true;
}

static ModelParams to_params(const pf_model* mdl) {
    ModelParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.kind = mdl->kind;
    mp.d = mdl->d;
    mp.dy = mdl->dy;
    if (mdl->kind == PF_SV) {
        mp.phi = mdl->sv_phi;
        mp.sigma = mdl->sv_sigma;
        mp.beta = mdl->sv_beta;
        mp.sv_m0 = mdl->sv_m0;
        mp.sv_s0 = mdl->sv_s0;
        mp.sv_c = 1.0f / (2.0f * mdl->sv_beta * mdl->sv_beta);
        return mp;
    }
    const int d = mdl->d, dy = mdl->dy;
    std::memcpy(mp.A, mdl->A, sizeof(float) * d * d);
    std::memcpy(mp.LQ, mdl->LQ, sizeof(float) * d * d);
    std::memcpy(mp.H, mdl->H, sizeof(float) * dy * d);
    std::memcpy(mp.Rinv, mdl->Rinv, sizeof(float) * dy * dy);
    std::memcpy(mp.m0, mdl->m0, sizeof(float) * d);
    std::memcpy(mp.L0, mdl->L0, sizeof(float) * d * d);
    bool diag = (dy == d);
    for (int k = 0; k < dy && diag; ++k)
        for (int j = 0; j < d; ++j)
            if (mp.H[k * d + j] != (k == j ? 1.0f : 0.0f)) diag = false;
    for (int k = 0; k < dy && diag; ++k)
        for (int j = 0; j < dy; ++j)
            if (k != j && mp.Rinv[k * dy + j] != 0.0f) diag = false;
    mp.diag_obs = diag ? 1 : 0;
    for (int k = 0; k < dy; ++k) mp.rdiag[k] = -0.5f * mp.Rinv[k * dy + k];
    return mp;
}

static bool validate_topology(uint64_t N, uint32_t M, std::string* err) {
    if (M < 2 || M > 8192 || ilog2_exact(M) < 0) {
        *err = "M must be a power of two in [2, 8192]";
        return false;
    }
    if (N == 0 || N % M != 0) {
        *err = "N must be a positive multiple of M";
        return false;
    }
    const uint64_t m = N / M;
    if (ilog2_exact(m) < 1) {
        *err = "m = N/M must be a power of two >= 2 (S >= 1)";
        return false;
    }
    if (N >= (1ull << 31)) {
        *err = "N must be < 2^31";
        return false;
    }
    return true;
}

// ---------------------------------------------------------------------------------------
// kernel dispatch
template <int D, int KIND>
static void launch_init(pf_handle* h) {
    InitArgs a;
    a.mp = h->mp;
    a.key = {(uint32_t)(h->seed & 0xffffffffu), (uint32_t)(h->seed >> 32)};
    a.N = h->N;
    a.x = h->X(0);
    const uint64_t nq = h->N / 4;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((nq + 255) / 256, 148ull * 16);
    k_init<D, KIND><<<grid, 256, 0, h->stream>>>(a);
}

template <int D, int KIND>
static void launch_pass1(pf_handle* h, const Pass1Args& a, bool gather) {
    const Plan& p = h->plan;
    if (gather) {
        auto k = k_pass1<D, KIND, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, p.pass1_smem);
        k<<<p.NT, p.pass1_threads, p.pass1_smem, h->stream>>>(a);
    } else {
        auto k = k_pass1<D, KIND, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, p.pass1_smem);
        k<<<p.NT, p.pass1_threads, p.pass1_smem, h->stream>>>(a);
    }
}

template <int D>
static void launch_cascade(pf_handle* h) {
    const Plan& p = h->plan;
    CascadeArgs c;
    c.logV = h->at<double>(h->lay.logV);
    c.thr = h->at<uint32_t>(h->lay.thr);
    c.part = h->at<double>(h->lay.part);
    c.scratch = h->at<double>(h->lay.scratch);
    c.est = h->at<double>(h->lay.est);
    c.ticket = h->at<uint32_t>(h->lay.ticket);
    c.N = h->N;
    c.m = h->m;
    c.S = h->S;
    c.k1 = p.k1;
    c.b = h->b;
    c.NT = p.NT;
    c.LPC = p.LPC;
    k_cascade<D><<<p.cascade_grid, kCascadeThreads, 0, h->stream>>>(c);
}

template <typename T, bool IDENT>
static void launch_compose(pf_handle* h, const ComposeArgs& a, uint32_t P) {
    const uint32_t smem = compose_smem(P, IDENT ? 0u : (uint32_t)sizeof(T));
    auto k = k_compose<T, IDENT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const uint32_t grid = (uint32_t)(h->N / P);
    const uint32_t threads = std::min<uint32_t>(kComposeThreads, std::max<uint32_t>(32u, P / 4));
    k<<<grid, threads, smem, h->stream>>>(a);
}

template <int D, int KIND>
static int run_step(pf_handle* h, const float* y_host, const float* y_dev) {
    const Plan& p = h->plan;
    const bool dbg = h->flags & PF_FLAG_DEBUG;
    Pass1Args a;
    a.mp = h->mp;
    a.key = {(uint32_t)(h->seed & 0xffffffffu), (uint32_t)(h->seed >> 32)};
    a.n = h->n;
    a.do_mutate = h->n > 0 ? 1 : 0;
    a.y_dev = y_dev;
    for (int k = 0; k < 8; ++k) a.y[k] = (y_host && k < h->mp.dy) ? y_host[k] : 0.0f;
    a.N = h->N;
    a.m = h->m;
    a.M = h->M;
    a.b = h->b;
    a.S = h->S;
    a.k1 = p.k1;
    a.P1 = p.P1;
    const int src = h->cur, dst = h->cur ^ 1;
    a.x_in = h->X(src);
    const bool gather = p.index_mode && !h->a_identity;
    a.A_in = gather ? h->A(h->amap) : nullptr;
    a.x_out = h->X(dst);
    a.logV = h->at<double>(h->lay.logV);
    a.thr = h->at<uint32_t>(h->lay.thr);
    a.part = h->at<double>(h->lay.part);
    a.dbg_x = dbg ? h->at<float>(h->lay.dbg_x) : nullptr;
    a.dbg_lw = dbg ? h->at<float>(h->lay.dbg_lw) : nullptr;
    a.dbg_anc = dbg ? h->at<int32_t>(h->lay.dbg_anc) : nullptr;
    launch_pass1<D, KIND>(h, a, gather);
    int launches = 1;
    launch_cascade<D>(h);
    ++launches;

    // compose passes
    ComposeArgs c;
    c.key = a.key;
    c.n = h->n;
    c.N = h->N;
    c.m = h->m;
    c.M = h->M;
    c.b = h->b;
    c.thr = a.thr;
    c.dbg_anc = a.dbg_anc;
    int amap_out = h->amap;
    int xs = dst;  // state mode: current payload buffer
    for (size_t i = 0; i < p.passes.size(); ++i) {
        const ComposePass& cp = p.passes[i];
        c.s0 = cp.s0;
        c.k = cp.k;
        c.P = cp.P;
        c.lowbits = cp.s0 - 1;
        if (p.index_mode) {
            if (cp.ident) {
                amap_out = 0;
                c.pin = nullptr;
                c.pout = h->A(0);
                launch_compose<int32_t, true>(h, c, cp.P);
            } else {
                c.pin = h->A(amap_out);
                c.pout = h->A(amap_out ^ 1);
                amap_out ^= 1;
                launch_compose<int32_t, false>(h, c, cp.P);
            }
        } else {
            c.pin = h->X(xs);
            c.pout = h->X(xs ^ 1);
            xs ^= 1;
            if (D == 1) launch_compose<float, false>(h, c, cp.P);
            else launch_compose<float2, false>(h, c, cp.P);
        }
        ++launches;
    }
    if (p.index_mode) {
        h->cur = dst;
        h->amap = amap_out;
        h->a_identity = p.passes.empty();
    } else {
        h->cur = xs;
        h->a_identity = true;
    }
    h->n += 1;
    h->have_step = true;
    h->last_launches = launches;
    return check_cuda(h, "pf_step");
}

template <int D>
static int dispatch_kind(pf_handle* h, const float* yh, const float* yd) {
    if (h->mp.kind == PF_SV) return run_step<D, 2>(h, yh, yd);
    return run_step<D, 1>(h, yh, yd);
}

static int dispatch_step(pf_handle* h, const float* yh, const float* yd) {
    switch (h->plan.D) {
        case 1: return dispatch_kind<1>(h, yh, yd);
        case 2: return dispatch_kind<2>(h, yh, yd);
        case 4: return dispatch_kind<4>(h, yh, yd);
        case 8: return dispatch_kind<8>(h, yh, yd);
    }
    return fail(h, PF_EINVAL, "bad d");
}

// ---------------------------------------------------------------------------------------
extern "C" {

size_t pf_workspace_bytes(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags) {
    std::string err;
    if (!validate_model(model, &err) || !validate_topology(N, M, &err)) return 0;
    Plan p;
    if (!make_plan(model->d, N, M, &p, &err)) return 0;
    return make_layout(p, N, M, flags).total;
}

int pf_init(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags, void* dev_ws,
            size_t ws_bytes, void* cuda_stream, pf_handle** out) {
    if (!out) return fail(nullptr, PF_EINVAL, "out is NULL");
    *out = nullptr;
    std::string err;
    if (!validate_model(model, &err)) return fail(nullptr, PF_EINVAL, err);
    if (!validate_topology(N, M, &err)) return fail(nullptr, PF_EINVAL, err);
    Plan p;
    if (!make_plan(model->d, N, M, &p, &err)) return fail(nullptr, PF_EINVAL, err);
    Layout L = make_layout(p, N, M, flags);
    if (!dev_ws || ws_bytes < L.total) return fail(nullptr, PF_EWORKSPACE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(dev_ws) & 255u) return fail(nullptr, PF_EWORKSPACE, "workspace not 256-byte aligned");
    pf_handle* h = new pf_handle();
    h->mp = to_params(model);
    h->N = N;
    h->M = M;
    h->b = (uint32_t)ilog2_exact(M);
    h->m = (uint32_t)(N / M);
    h->S = (uint32_t)ilog2_exact(h->m);
    h->seed = seed;
    h->flags = flags;
    h->plan = p;
    h->lay = L;
    h->ws = static_cast<unsigned char*>(dev_ws);
    h->stream = static_cast<cudaStream_t>(cuda_stream);
    h->n = 0;
    h->cur = 0;
    h->amap = 0;
    h->a_identity = true;
    h->have_step = false;
    h->last_launches = 0;
    cudaMemsetAsync(h->at<uint32_t>(L.ticket), 0, 16, h->stream);
    switch (p.D * 4 + h->mp.kind) {
        case 1 * 4 + 1: launch_init<1, 1>(h); break;
        case 1 * 4 + 2: launch_init<1, 2>(h); break;
        case 2 * 4 + 1: launch_init<2, 1>(h); break;
        case 4 * 4 + 1: launch_init<4, 1>(h); break;
        case 8 * 4 + 1: launch_init<8, 1>(h); break;
        default: delete h; return fail(nullptr, PF_EINVAL, "unsupported (d, kind)");
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        delete h;
        return fail(nullptr, PF_ECUDA, std::string("pf_init: ") + cudaGetErrorString(e));
    }
    *out = h;
    return PF_OK;
}

int pf_step(pf_handle* h, const float* y_host) {
    if (!h || !y_host) return fail(h, PF_EINVAL, "NULL argument");
    for (int k = 0; k < h->mp.dy; ++k)
        if (!std::isfinite(y_host[k])) return fail(h, PF_EOBS, "non-finite observation");
    return dispatch_step(h, y_host, nullptr);
}

int pf_step_dev(pf_handle* h, const float* y_dev) {
    if (!h || !y_dev) return fail(h, PF_EINVAL, "NULL argument");
    return dispatch_step(h, nullptr, y_dev);
}

int pf_estimate(pf_handle* h, int phi, int kind, double* out) {
    if (!h || !out) return fail(h, PF_EINVAL, "NULL argument");
    if (!h->have_step) return fail(h, PF_ESTATE, "no completed step");
    if ((phi != PF_PHI_X && phi != PF_PHI_X2) || (kind != PF_EST_FILTER && kind != PF_EST_PREDICT))
        return fail(h, PF_EINVAL, "bad phi / kind");
    const int D = h->plan.D;
    const size_t off = (size_t)((kind == PF_EST_FILTER ? 0 : 2) + (phi == PF_PHI_X ? 0 : 1)) * D;
    cudaError_t e = cudaMemcpyAsync(out, h->at<double>(h->lay.est) + off, sizeof(double) * D,
                                    cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_estimate: ") + cudaGetErrorString(e));
    return PF_OK;
}

void pf_destroy(pf_handle* h) { delete h; }

const char* pf_last_error(const pf_handle* h) { return h ? h->err.c_str() : g_init_error.c_str(); }

int pf_last_step_launches(const pf_handle* h) { return h ? h->last_launches : 0; }

int pf_debug_ptr(pf_handle* h, int what, int stage, void** dev_out) {
    if (!h || !dev_out) return fail(h, PF_EINVAL, "NULL argument");
    if (!h->have_step) return fail(h, PF_ESTATE, "no completed step");
    const bool dbg = h->flags & PF_FLAG_DEBUG;
    const int D = h->plan.D;
    switch (what) {
        case PF_DBG_X:
        case PF_DBG_LOGW:
        case PF_DBG_ANC_STAGE:
        case PF_DBG_ANC_FINAL:
            if (!dbg) return fail(h, PF_ESTATE, "handle not created with PF_FLAG_DEBUG");
            break;
        default:
            break;
    }
    switch (what) {
        case PF_DBG_X: *dev_out = h->at<float>(h->lay.dbg_x); return PF_OK;
        case PF_DBG_LOGW: *dev_out = h->at<float>(h->lay.dbg_lw); return PF_OK;
        case PF_DBG_ANC_STAGE:
            if (stage < 1 || stage > (int)h->S) return fail(h, PF_EINVAL, "stage out of range");
            *dev_out = h->at<int32_t>(h->lay.dbg_anc) + (size_t)(stage - 1) * h->N;
            return PF_OK;
        case PF_DBG_ANC_FINAL: {
            int32_t* A = h->at<int32_t>(h->lay.dbg_A);
            k_debug_compose<<<1024, 256, 0, h->stream>>>(h->at<int32_t>(h->lay.dbg_anc), h->N, h->S, A);
            *dev_out = A;
            return check_cuda(h, "pf_debug_ptr");
        }
        case PF_DBG_XHAT: {
            float* out = h->at<float>(h->lay.dbg_xhat);
            const float* x = h->X(h->cur);
            const int32_t* A = (h->plan.index_mode && !h->a_identity) ? h->A(h->amap) : nullptr;
            switch (D) {
                case 1: k_gather<1><<<1024, 256, 0, h->stream>>>(x, A, h->N, out); break;
                case 2: k_gather<2><<<1024, 256, 0, h->stream>>>(x, A, h->N, out); break;
                case 4: k_gather<4><<<1024, 256, 0, h->stream>>>(x, A, h->N, out); break;
                case 8: k_gather<8><<<1024, 256, 0, h->stream>>>(x, A, h->N, out); break;
            }
            *dev_out = out;
            return check_cuda(h, "pf_debug_ptr");
        }
        case PF_DBG_LOGV: *dev_out = h->at<double>(h->lay.logV); return PF_OK;
        case PF_DBG_THRESH: *dev_out = h->at<uint32_t>(h->lay.thr); return PF_OK;
    }
    return fail(h, PF_EINVAL, "unknown debug table");
}

int pf_debug_get(pf_handle* h, int what, int stage, void* host_out, size_t bytes) {
    void* p = nullptr;
    const int rc = pf_debug_ptr(h, what, stage, &p);
    if (rc != PF_OK) return rc;
    const int D = h->plan.D;
    size_t need = 0;
    switch (what) {
        case PF_DBG_X:
        case PF_DBG_XHAT: need = (size_t)h->N * D * 4; break;
        case PF_DBG_LOGW:
        case PF_DBG_ANC_STAGE:
        case PF_DBG_ANC_FINAL: need = (size_t)h->N * 4; break;
        case PF_DBG_LOGV: need = (size_t)(h->m - 1) * 8; break;
        case PF_DBG_THRESH: need = (size_t)(h->m - 1) * 4; break;
    }
    if (!host_out || bytes < need) return fail(h, PF_EINVAL, "host buffer too small");
    cudaError_t e = cudaMemcpyAsync(host_out, p, need, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_debug_get: ") + cudaGetErrorString(e));
    return PF_OK;
}

int pf_debug_set_state(pf_handle* h, const float* host_xhat, uint32_t n) {
    if (!h || !host_xhat) return fail(h, PF_EINVAL, "NULL argument");
    cudaError_t e = cudaMemcpyAsync(h->X(h->cur), host_xhat, (size_t)h->N * h->plan.D * 4, cudaMemcpyHostToDevice,
                                    h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_debug_set_state: ") + cudaGetErrorString(e));
    h->a_identity = true;
    h->n = n;
    return PF_OK;
}

}  // extern "C"
