// pf_api.cu -- C-ABI (include/pf.h) and host orchestration of one BPF step.
//
// Launch sequence of pf_step:
//   k_pass1 (NT tiles) -> k_cascade (one wave of CTAs) -> k_stages x (#passes)
// Every pass moves the particle states through shared-memory tiles (coalesced reads and
// writes; no random HBM access anywhere on the step).  The next rows reuse the same
// kernels: run_step_adaptive (weigh -> cascade -> ESS -> resample up to S*),
// run_step_airpf (AIRPF pass -> cascade -> island stages), run_step_multinomial (weigh ->
// cascade -> global CDF search and gather); the sharded step is pf_step_local /
// pf_step_top followed by the pull exchange (pf_cross_pull_*) or pf_cross_stage rounds.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pf.h"
#include "pf_launch.h"

using namespace pfk;

namespace {

// k_pass1 tile: shared-memory budget and threads per CTA.  Smaller tiles with two quads per
// thread win for d = 4 (C4: 7.17 -> 5.62 ms per launch, one more stage moves into the
// k_stages passes at no extra pass; profiles/r1_stage_pass_experiments.md); the other
// dimensions keep the larger tile (C2, C3 measured slower with it).
constexpr uint32_t kPass1SmemBudgetDefault = 64u * 1024u;
constexpr uint32_t kPass1ThreadsDefault = 256u;
constexpr uint32_t kPass1SmemBudgetD4 = 40000u;
constexpr uint32_t kPass1ThreadsD4 = 128u;
constexpr uint32_t kStageSmemDefault = 232448u;  // one persistent CTA per SM
constexpr uint32_t kStageThreadsDefault = 1024u;
constexpr uint32_t kSmemPerSM = 233472u;          // 228 KiB (1 KiB of it reserved per CTA)

// Tuning knobs (environment, read at pf_init; for experiments only).
uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = getenv(name);
    return (v && *v) ? (uint32_t)strtoul(v, nullptr, 10) : dflt;
}
constexpr uint32_t kLPC = 2048u;    // max cascade CTAs (and max leaves per CTA)
constexpr uint32_t kLPCMin = 64u;   // min leaves per cascade CTA

struct StagePass {
    uint32_t s0, k, P, threads, qpt, smem, tb, grid, pipe;
    uint32_t kd = 0;  // stages drawn (0: k)
};

struct Plan {
    int D;
    uint32_t tb;  // k_pass1 table entry bytes (1: side|index, M <= 128; 2: tile position)
    uint32_t P1, k1, NT, LPC, cascade_grid, pass1_threads, pass1_qpt;
    uint32_t pass1_smem;
    std::vector<StagePass> passes;
};

int ilog2_exact(uint64_t v) {
    if (v == 0 || (v & (v - 1)) != 0) return -1;
    int k = 0;
    while ((1ull << k) < v) ++k;
    return k;
}

size_t align256(size_t v) { return (v + 255u) & ~size_t(255u); }

uint32_t pick_threads(uint32_t nq, uint32_t maxthr, uint32_t* qpt) {
    if (nq < 32u) {
        *qpt = 1;
        return 32u;
    }
    uint32_t t = std::min(nq, std::max(maxthr, std::min(nq / 8u, 1024u)));  // at most 8 quads per thread
    *qpt = nq / t;
    return t;
}

// N is this shard's particle count; Nglobal the whole problem's.  The pass-1 tile is
// bounded by Nglobal / kMaxShards so that, for any world size up to kMaxShards, the
// single-GPU tiles coincide with the sharded ones (bitwise G-invariance).
constexpr uint64_t kMaxShards = 8;
bool make_plan(int d, uint64_t N, uint32_t M, Plan* pl, std::string* err, uint64_t Nglobal = 0, uint32_t nsm = 148) {
    if (Nglobal == 0) Nglobal = N;
    const uint64_t m = N / M;
    const int S = ilog2_exact(m);
    Plan p;
    p.D = d;
    const uint32_t budget1 = env_u32("PF_PASS1_SMEM", d == 4 ? kPass1SmemBudgetD4 : kPass1SmemBudgetDefault);
    uint32_t threads1 = env_u32("PF_PASS1_THREADS", d == 4 ? kPass1ThreadsD4 : kPass1ThreadsDefault);
    if (d == 4) threads1 = std::min(threads1, kPass1ThreadsD4);  // the d = 4 fused kernel's launch bounds
    const uint32_t maxqpt1 = env_u32("PF_PASS1_MAXQPT", 8u);
    // pass-1 tile: the largest 2^k1 <= 64 groups (k1 <= S) whose shared memory fits the budget
    uint32_t P1 = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(N, (uint64_t)kPass1MaxGroups * M),
                                               std::max<uint64_t>(2ull * M, Nglobal / kMaxShards));
    // the kernels' launch bounds: 512 threads, except the fused d = 4 pass below 8 quads per
    // thread (128); a d = 4 tile too large for 128 x 8 quads (M >= 4096) takes more threads
    // at 8 quads each, which that kernel's QPT = 8 instantiation allows
    const uint32_t maxthr1 = 512u;
    auto threads_for = [&](uint32_t P, uint32_t* q) {
        uint32_t t = std::min(pick_threads(P / 4, threads1, q), d == 4 ? kPass1ThreadsD4 : maxthr1);
        *q = std::max(1u, (P / 4) / t);
        while (*q > maxqpt1 && t < maxthr1) {  // k_pass1 is instantiated for up to 8 quads per thread
            t *= 2;
            *q /= 2;
        }
        return t;
    };
    // table entries: 16-bit tile positions when they fit (cheapest walk), else 1 byte
    auto fits1 = [&](uint32_t P, uint32_t tb) {
        uint32_t q;
        const uint32_t thr = threads_for(P, &q);
        if (tb == 1u && M > 128u) return false;
        return thr <= maxthr1 && q <= maxqpt1 && pass1_smem(d, P, M, (uint32_t)ilog2_exact(P / M), thr, tb).total <= budget1;
    };
    p.tb = M <= 128u ? 1u : 2u;
    for (;;) {
        if (fits1(P1, 2u)) {
            p.tb = 2u;
            break;
        }
        if (fits1(P1, 1u)) {
            p.tb = 1u;
            break;
        }
        if (P1 <= 2 * M) break;
        P1 >>= 1;
    }
    if (P1 < 2 * M) P1 = 2 * M;
    p.P1 = P1;
    p.k1 = (uint32_t)ilog2_exact(P1 / M);
    if ((int)p.k1 > S) {
        *err = "internal: k1 > S";
        return false;
    }
    p.pass1_threads = threads_for(P1, &p.pass1_qpt);
    if (p.pass1_threads > maxthr1 || p.pass1_qpt > maxqpt1) {
        *err = "pass-1 tile needs more threads than its kernel's launch bounds";
        return false;
    }
    p.pass1_smem = pass1_smem(d, P1, M, p.k1, p.pass1_threads, p.tb).total;
    if (p.pass1_smem > 227u * 1024u) {
        *err = "pass-1 tile does not fit in shared memory (M too large for d)";
        return false;
    }
    p.NT = (uint32_t)(N / P1);
    // leaves per cascade CTA: as few as keep the CTA subtrees in one wave on the SMs (one
    // CTA walking the whole tree dominated small configurations; more than a wave of CTAs
    // or a wide top tree for the last CTA slows large ones), within [kLPCMin, kLPC]
    {
        uint32_t lpc = kLPCMin;
        while (lpc < kLPC && (uint64_t)lpc * nsm < p.NT) lpc <<= 1;
        p.LPC = std::min<uint32_t>(p.NT, lpc);
    }
    p.cascade_grid = p.NT / p.LPC;
    if (p.cascade_grid > kLPC) {
        *err = "too many pass-1 tiles for the cascade tree";
        return false;
    }
    // stages k1+1..S in persistent k_stages passes: the largest tile in the shared-memory
    // budget (default: one double-buffered CTA per SM), fewest passes, stages spread evenly
    uint32_t s = p.k1 + 1;
    const uint32_t sb = (uint32_t)(4 * d);
    const uint32_t budget = std::min(env_u32("PF_STAGE_SMEM", kStageSmemDefault), 232448u);
    const uint32_t rem = (uint32_t)S - p.k1;
    const uint32_t tbmin = M <= 128u ? 1u : 2u;
    auto kmax = [&](uint32_t pipe) {
        uint32_t K = 0;
        for (uint32_t k = 1; k <= rem; ++k) {
            const uint64_t P = (uint64_t)M << k;
            if (P > N || P > 65536u || P / 4u > 8u * 1024u) break;
            if (stages_smem((uint32_t)P, sb, k, tbmin, pipe) > budget) break;
            K = k;
        }
        return K;
    };
    // software-pipelined unless only the single-buffered tile fits (or it is forced)
    uint32_t pipe = env_u32("PF_STAGE_PIPE", 1u) ? 1u : 0u;
    uint32_t K = kmax(pipe);
    if (K == 0 && pipe) {
        pipe = 0u;
        K = kmax(0u);
    }
    if (rem > 0 && K == 0) {
        *err = "stage tile does not fit in shared memory";
        return false;
    }
    const uint32_t npass = rem ? (rem + K - 1) / K : 0;
    for (uint32_t i = 0; i < npass; ++i) {
        const uint32_t left = rem - (s - p.k1 - 1);
        const uint32_t k = (left + (npass - i) - 1) / (npass - i);
        StagePass sp;
        sp.s0 = s;
        sp.k = k;
        sp.P = M << k;
        sp.pipe = pipe;
        sp.tb = (env_u32("PF_STAGE_TB", 2u) == 2u && stages_smem(sp.P, sb, k, 2u, pipe) <= budget) ? 2u : tbmin;
        sp.threads = pick_threads(sp.P / 4, env_u32("PF_STAGE_THREADS", kStageThreadsDefault), &sp.qpt);
        // warp-specialised pass (k_stages_ws): half the CTA walks, half draws, each on QPT
        // quads per thread; needs whole-quad groups (M >= 4), bulk-copied groups and a CTA
        // of 2 x P/4/QPT <= 1024 threads; deep passes over tiny groups (k > 7 with M < 16,
        // d = 1) run faster on the plain pipelined kernel (profiles/r2_ws_kmax.txt)
        if (pipe && env_u32("PF_STAGE_WS", 1u) && M >= 4u && (uint64_t)M * sb >= 16u && sp.P / 4u >= 64u &&
            k <= env_u32("PF_STAGE_WS_KMAX", M >= 16u ? 16u : 7u) &&
            stages_smem(sp.P, sb, k, sp.tb, 2u) <= budget &&
            (1u << k) <= std::min<uint32_t>(1024u, sp.P / 4u * 2u) / 2u) {  // one threshold per drawer
            sp.pipe = 2u;
            sp.qpt = 1u;  // unused: runtime loops
            sp.threads = std::min<uint32_t>(1024u, sp.P / 4u * 2u);
        }
        sp.smem = stages_smem(sp.P, sb, k, sp.tb, sp.pipe);
        const uint32_t per_sm = std::max(1u, std::min(kSmemPerSM / (sp.smem + 1024u), 2048u / sp.threads));
        sp.grid = (uint32_t)std::min<uint64_t>(N / sp.P, (uint64_t)nsm * per_sm);
        p.passes.push_back(sp);
        s += k;
    }
    if (env_u32("PF_PLAN_VERBOSE", 0u)) {
        fprintf(stderr, "[pf plan] N=%llu M=%u d=%d tb=%u pass1: P1=%u k1=%u threads=%u qpt=%u smem=%u tiles=%u\n",
                (unsigned long long)N, M, p.D, p.tb, p.P1, p.k1, p.pass1_threads, p.pass1_qpt, p.pass1_smem, p.NT);
        for (const StagePass& sp : p.passes)
            fprintf(stderr, "[pf plan]   pass s0=%u k=%u P=%u tb=%u pipe=%u threads=%u qpt=%u smem=%u grid=%u\n", sp.s0,
                    sp.k, sp.P, sp.tb, sp.pipe, sp.threads, sp.qpt, sp.smem, sp.grid);
    }
    *pl = p;
    return true;
}

struct Layout {
    size_t X0, X1, logV, thr, part, scratch, est, ticket, y;
    size_t lw0, lw1, carry_lv, ess_part, ess_chunks, ess_out, ess_lmax;  // PF_FLAG_ADAPTIVE
    size_t isl_A, isl_choice, isl_logW;                                  // PF_FLAG_AIRPF
    size_t mn_cdf, mn_cdf32, mn_trec, mn_off;                            // PF_FLAG_MULTINOMIAL
    size_t shard_rec, recs, top_logV, top_thr, top_scratch;
    size_t pull_src, pull_rank, pull_counts, pull_fill, pull_off, pull_req, pull_outpos, pull_serve;  // world > 1
    size_t dbg_x, dbg_lw, dbg_anc, dbg_A;
    size_t mom_part, mom_out;          // PF_EST_RESAMPLED (k_moments)
    size_t rl_cnt, rl_off, rl_own, rl_par, rl_kidx, rl_send;  // relabelled exchange (world > 1)
    size_t guard_count;                // PF_FLAG_GUARD
    std::vector<size_t> gaps;          // PF_FLAG_GUARD: offsets of the PF_GUARD_BYTES gaps
    size_t total;
};

Layout make_layout(const Plan& p, uint64_t N, uint32_t M, uint32_t flags, uint32_t world, int Sglobal) {
    Layout L;
    size_t off = 0;
    const bool guard = flags & PF_FLAG_GUARD;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align256(off + bytes);
        if (guard) {  // a gap behind every region (PF_GUARD_BYTES is a multiple of 256)
            L.gaps.push_back(off);
            off += PF_GUARD_BYTES;
        }
        return o;
    };
    const uint64_t m = N / M;
    const int S = ilog2_exact(m);
    const int PS = 2 + 4 * p.D;
    const size_t xb = (size_t)N * p.D * 4;
    L.X0 = take(xb);
    L.X1 = take(xb);
    L.logV = take(m * 8);
    L.thr = take(m * 4);
    L.part = take((size_t)p.NT * PS * 8);
    L.scratch = take((size_t)(p.NT + 2) * PS * 8);
    L.est = take(4 * 8 * 8);
    L.ticket = take(16);
    L.y = take(64);
    L.shard_rec = take((size_t)(1 + PS) * 8);
    L.recs = take((size_t)world * (1 + PS) * 8);
    L.top_logV = take((size_t)world * 8);
    L.top_thr = take((size_t)world * 4);
    L.top_scratch = take((size_t)2 * world * PS * 8);
    const bool sh = world > 1;
    L.pull_src = take(sh ? N * 4 : 0);
    L.pull_rank = take(sh ? N * 4 : 0);
    L.pull_counts = take(sh ? (size_t)world * 8 : 0);
    L.pull_fill = take(sh ? (size_t)world * 4 : 0);
    L.pull_off = take(sh ? (size_t)world * 8 : 0);
    L.pull_req = take(sh ? N * 4 : 0);
    L.pull_outpos = take(sh ? N * 4 : 0);
    L.pull_serve = take(sh ? xb * world : 0);  // worst case: every rank reads only this shard
    const bool ad = flags & PF_FLAG_ADAPTIVE;
    const bool air_flag = flags & PF_FLAG_AIRPF;
    const bool mn = flags & PF_FLAG_MULTINOMIAL;
    L.lw0 = take((ad || mn) ? N * 4 : 0);
    L.lw1 = take(ad ? N * 4 : 0);
    L.carry_lv = take(ad ? (air_flag ? m : m / 2) * 8 : 0);
    L.ess_part = take((ad || mn) ? (size_t)p.NT * 3 * 8 : 0);
    L.ess_chunks = take(ad ? (size_t)(p.NT / kEssChunk + 3 * m / kEssChunk + 64) * 2 * 8 : 0);
    L.ess_out = take(ad ? (size_t)(S + 3) * 8 : 0);
    L.ess_lmax = take((ad || mn) ? 16 : 0);
    const size_t nt_mn = (N + kMnTile - 1) / kMnTile;
    L.mn_cdf = take(mn ? N * 4 : 0);
    L.mn_cdf32 = take(mn ? nt_mn * (kMnTile / 32) * 4 : 0);
    L.mn_trec = take(mn ? nt_mn * 16 : 0);
    L.mn_off = take(mn ? (nt_mn + 1) * 8 : 0);
    const bool air = flags & PF_FLAG_AIRPF;
    L.isl_A = take(air ? m * 4 : 0);
    L.isl_choice = take(air ? (size_t)Sglobal * ((m + 3) / 4) : 0);  // sharded: the cross stages too
    L.isl_logW = take(air ? m * 8 : 0);
    const bool dbg = flags & PF_FLAG_DEBUG;
    L.dbg_x = take(dbg ? xb : 0);
    L.dbg_lw = take(dbg ? N * 4 : 0);
    L.dbg_anc = take(dbg ? (size_t)N * Sglobal * 4 : 0);
    (void)S;
    L.dbg_A = take(dbg ? N * 4 : 0);
    {
        const size_t nch = (N + kRlChunk - 1) / kRlChunk;
        L.rl_cnt = take(sh ? 2 * nch * 4 : 0);
        L.rl_off = take(sh ? (2 * nch + 2) * 4 : 0);
        L.rl_own = take(sh ? N * 4 : 0);
        L.rl_par = take(sh ? N * 4 : 0);
        L.rl_kidx = take(sh ? N * 4 : 0);
        L.rl_send = take(sh ? xb : 0);
    }
    L.mom_part = take((size_t)kMomPartDoubles * 8);
    L.mom_out = take(16 * 8);
    L.guard_count = take(guard ? 16 : 0);
    L.total = off;
    return L;
}

}  // namespace

struct pf_handle {
    ModelParams mp;
    uint64_t N;                    // particles of this shard (= Nglobal when world == 1)
    uint32_t M, b, m, S;           // m, S: groups and local stages of this shard
    uint64_t Nglobal;
    uint32_t Sglobal, rank, world, L, pos0;
    uint32_t step_n;               // time index of the step in progress / last completed
    bool top_done;
    uint64_t seed;
    uint32_t flags;
    Plan plan;
    Layout lay;
    unsigned char* ws;
    cudaStream_t stream;
    // state
    uint32_t n;          // index of the next step
    int cur;             // X buffer that holds the gather source / xhat for the next step
    bool have_step;
    int last_launches;
    // fully adapted scheme (pf_set_adaptive)
    double theta = 0.0;
    int sstar_last = -1;
    int lwi = 0;             // lw buffer the next weigh pass writes
    int carry_mode = 0;      // 0 none, 1 particle (lw of the other buffer), 2 block (carry_lv)
    uint32_t carry_shift = 0;
    double carry_c = 0.0;
    // AIRPF (pf_set_airpf)
    int airpf = 0;           // 0 off, 1 Alg. 7 (modified), 2 Alg. 6 (plain)
    bool isl_valid = false;  // X(cur) is a within-resampled sample read through the island map
    // multinomial resampling, Alg. 2 (pf_set_multinomial)
    bool multinomial = false;
    bool rotate = false;     // stage rotation with the fully adapted scheme (pf_set_rotation)
    uint32_t carry_mask = 0xffffffffu;
    uint32_t rho = 0;        // current rotation offset (bookkeeping for pf_last_stages users)
    bool anc_ready = false;  // dbg_A holds the ancestors of the last (multinomial) step
    // peer-memory exchange (pf_peer_open / pf_peer_set / pf_cross_peer)
    std::vector<unsigned char*> peer_ws;    // every rank's workspace, mapped here
    std::vector<void*> peer_ipc;            // IPC mappings to close (allocation bases)
    bool half_step = false;  // pf_step_local_begin ran, pf_step_local_end pending
    // relabelled exchange in progress (pf_relabel_begin -> pf_relabel_end)
    int rl_t = 0;
    uint64_t rl_own = 0, rl_kmin = 0;
    // kernel timing
    bool timing;
    struct Rec {
        cudaEvent_t a, b;
        int kind;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::string err;
    cudaEvent_t ev() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    void mark(int kind, bool begin) {
        if (!timing) return;
        if (begin) {
            Rec r;
            r.a = ev();
            r.b = nullptr;
            r.kind = kind;
            cudaEventRecord(r.a, stream);
            recs.push_back(r);
        } else {
            recs.back().b = ev();
            cudaEventRecord(recs.back().b, stream);
        }
    }
    // CUDA graph of T captured steps (pf_graph_capture -> pf_graph_launch)
    cudaGraphExec_t gexec = nullptr;
    ~pf_handle() {
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
        for (void* p : peer_ipc) cudaIpcCloseMemHandle(p);
        if (gexec) cudaGraphExecDestroy(gexec);
    }
    float* X(int i) { return reinterpret_cast<float*>(ws + (i ? lay.X1 : lay.X0)); }
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
    bool dlq = true;
    for (int k = 0; k < d; ++k)
        for (int j = 0; j < d; ++j)
            if (k != j && mp.LQ[k * d + j] != 0.0f) dlq = false;
    mp.diag_lq = dlq ? 1 : 0;
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
// kernel dispatch (instantiations live in pf_inst_*.cu)
static void launch_pass1(pf_handle* h, const Pass1Args& a, int mode = kPass1Fused) {
    const Plan& p = h->plan;
    const LaunchCfg c{p.NT, p.pass1_threads, a.sl.total, h->stream};
    const bool dbg = h->flags & PF_FLAG_DEBUG;
    const int q = (int)p.pass1_qpt;
    const int k = h->mp.kind, tb = (int)p.tb;
    if (mode == kPass1Fused) {
        switch (p.D) {
            case 1: launch_pass1_d1(k, tb, dbg, q, mode, c, a); break;
            case 2: launch_pass1_d2(k, tb, dbg, q, mode, c, a); break;
            case 4: launch_pass1_d4(k, tb, dbg, q, mode, c, a); break;
            default: launch_pass1_d8(k, tb, dbg, q, mode, c, a); break;
        }
    } else {
        switch (p.D) {
            case 1: launch_pass1_ad_d1(k, tb, dbg, q, mode, c, a); break;
            case 2: launch_pass1_ad_d2(k, tb, dbg, q, mode, c, a); break;
            case 4: launch_pass1_ad_d4(k, tb, dbg, q, mode, c, a); break;
            default: launch_pass1_ad_d8(k, tb, dbg, q, mode, c, a); break;
        }
    }
}

static void launch_cascade_k(pf_handle* h) {
    const Plan& p = h->plan;
    CascadeArgs c{};
    c.logV = h->at<double>(h->lay.logV);
    c.thr = h->at<uint32_t>(h->lay.thr);
    c.part = h->at<double>(h->lay.part);
    c.scratch = h->at<double>(h->lay.scratch);
    c.est = h->at<double>(h->lay.est);
    c.shard_rec = h->world > 1 ? h->at<double>(h->lay.shard_rec) : nullptr;
    c.ticket = h->at<uint32_t>(h->lay.ticket);
    c.N = h->N;
    c.m = h->m;
    c.S = h->S;
    c.k1 = p.k1;
    c.b = h->airpf ? 1u : h->b;  // AIRPF: 31-bit island thresholds (R20)
    c.NT = p.NT;
    c.LPC = p.LPC;
    // threads: half the widest tree level the kernel builds (its leaves per CTA, or the CTA
    // roots of the last CTA), at least 64 (per-thread copies of a partial)
    uint32_t wide = std::max(p.LPC, p.cascade_grid), thr = 64;  // >= the partial size 2 + 4 d
    while (thr < 1024u && 2u * thr < wide) thr *= 2;
    launch_cascade(p.D, LaunchCfg{p.cascade_grid, thr, 0u, h->stream}, c);
}

static void launch_stages_k(pf_handle* h, const StagePass& cp, const void* pin, void* pout, uint32_t out_rot = 0u) {
    StageArgs a{};
    a.key = make_key(h->seed);
    a.n = h->n;
    a.N = h->N;
    a.pos0 = h->pos0;
    a.m = h->m;
    a.M = h->M;
    a.b = h->b;
    a.s0 = cp.s0;
    a.k = cp.k;
    a.kd = cp.kd ? cp.kd : cp.k;
    a.P = cp.P;
    a.lowbits = cp.s0 - 1;
    a.pipe = cp.pipe;
    // k_stages_ws: walkers = the given fraction (in 32ths) of the CTA, whole warps
    a.ws_walkers = std::max<uint32_t>(32u, (cp.threads * env_u32("PF_STAGE_WS_WALK32", 16u) / 32u) & ~31u);
    a.spec = env_u32("PF_STAGE_SPEC", 1u);
    a.out_rot = out_rot;
    a.out_S = h->S;
    a.pin = pin;
    a.pout = pout;
    a.thr = h->at<uint32_t>(h->lay.thr);
    a.dbg_anc = (h->flags & PF_FLAG_DEBUG) ? h->at<int32_t>(h->lay.dbg_anc) : nullptr;
    const LaunchCfg c{cp.grid, cp.threads, cp.smem, h->stream};
    launch_stages(h->plan.D, (int)cp.tb, (h->flags & PF_FLAG_DEBUG) != 0, (int)cp.qpt, c, a);
}

// A k_stages pass over stages s0..s0+k-1 (k <= the plan's pass), sized like make_plan.
static StagePass stage_pass_for(const pf_handle* h, const StagePass& sp, uint32_t k) {
    // the plan's pass (tile depth sp.k, geometry, launch size) drawing only its first k stages
    StagePass q = sp;
    q.kd = k;
    (void)h;
    return q;
}

static void fill_pass1(pf_handle* h, Pass1Args& a, const float* y_host, const float* y_dev) {
    const Plan& p = h->plan;
    const bool dbg = h->flags & PF_FLAG_DEBUG;
    a.mp = h->mp;
    a.key = make_key(h->seed);
    a.n = h->n;
    a.do_mutate = h->n > 0 ? 1 : 0;
    a.y_dev = y_dev;
    for (int k = 0; k < 8; ++k) a.y[k] = (y_host && k < h->mp.dy) ? y_host[k] : 0.0f;
    a.N = h->N;
    a.pos0 = h->pos0;
    a.m = h->m;
    a.M = h->M;
    a.b = h->b;
    a.S = h->S;
    a.k1 = p.k1;
    a.P1 = p.P1;
    a.T1 = p.P1 / h->M;
    a.probe = env_u32("PF_PASS1_PROBE", 0u);
    a.spec = env_u32("PF_PASS1_SPEC", 1u);
    a.sl = pass1_smem(p.D, p.P1, h->M, p.k1, p.pass1_threads, p.tb);
    a.logV = h->at<double>(h->lay.logV);
    a.thr = h->at<uint32_t>(h->lay.thr);
    a.part = h->at<double>(h->lay.part);
    a.dbg_x = dbg ? h->at<float>(h->lay.dbg_x) : nullptr;
    a.dbg_lw = dbg ? h->at<float>(h->lay.dbg_lw) : nullptr;
    a.dbg_anc = dbg ? h->at<int32_t>(h->lay.dbg_anc) : nullptr;
    a.lw_out = nullptr;
    a.lw_in = nullptr;
    a.carry_mode = 0;
    a.carry_lw = nullptr;
    a.carry_lv = nullptr;
    a.carry_shift = 0;
    a.carry_c = 0.0;
    a.ess_part = nullptr;
    a.ess_lmax = nullptr;
    a.isl_src = nullptr;
    a.logW = nullptr;
    a.carry_mask = 0xffffffffu;
    a.out_rot = 0u;
}

// One step of the fully adapted scheme (include/pf.h pf_set_adaptive; R17/R18):
//   k_pass1 (weigh) -> k_cascade -> k_ess -> [host reads S*] -> k_pass1 (resample,
//   stages 1..min(k1, S*)) -> k_stages passes up to stage S* -> carried weights.
static int run_step_adaptive(pf_handle* h, const float* y_host, const float* y_dev) {
    const Plan& p = h->plan;
    const int src = h->cur, mid = h->cur ^ 1;
    float* lw = h->at<float>(h->lwi ? h->lay.lw1 : h->lay.lw0);
    Pass1Args a{};
    fill_pass1(h, a, y_host, y_dev);
    a.x_in = h->X(src);
    a.x_out = h->X(mid);  // x_n in natural order
    a.lw_out = lw;
    a.carry_mode = h->carry_mode;
    a.carry_lw = h->at<float>(h->lwi ? h->lay.lw0 : h->lay.lw1);
    a.carry_lv = h->at<double>(h->lay.carry_lv);
    a.carry_shift = h->carry_shift;
    a.carry_mask = h->carry_mask;
    a.carry_c = h->carry_c;
    a.ess_part = h->at<double>(h->lay.ess_part);
    a.ess_lmax = h->at<unsigned int>(h->lay.ess_lmax);
    h->mark(PF_KERNEL_PASS1, true);
    launch_pass1(h, a, kPass1Weigh);
    h->mark(PF_KERNEL_PASS1, false);
    int launches = 1;
    h->mark(PF_KERNEL_CASCADE, true);
    launch_cascade_k(h);
    EssArgs e{};
    e.lv0 = nullptr;  // level 0 = the particle weights (tile partials)
    e.ess_part = h->at<double>(h->lay.ess_part);
    e.logV = h->at<double>(h->lay.logV);
    e.lmax = h->at<unsigned int>(h->lay.ess_lmax);
    e.chunks = h->at<double>(h->lay.ess_chunks);
    e.out = h->at<double>(h->lay.ess_out);
    e.N = h->N;
    e.NT = p.NT;
    e.m = h->m;
    e.S = h->S;
    e.theta = h->theta;
    launch_ess(LaunchCfg{0u, 0u, 0u, h->stream}, e);
    h->mark(PF_KERNEL_CASCADE, false);
    launches += 3;
    double tail[2];
    cudaError_t ce = cudaMemcpyAsync(tail, e.out + h->S + 1, sizeof(tail), cudaMemcpyDeviceToHost, h->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
    if (ce != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_step (adaptive): ") + cudaGetErrorString(ce));
    const uint32_t ss = (uint32_t)tail[0];
    const double lvS = tail[1];

    int xs = mid;  // buffer holding the current states
    // stage rotation (R23): the last kernel of the step writes the next layout
    const uint32_t rot = (h->rotate && ss >= 1u && ss < h->S) ? ss : 0u;
    if (ss >= 1u) {
        Pass1Args r{};
        fill_pass1(h, r, y_host, y_dev);
        r.do_mutate = 0;
        r.x_in = h->X(mid);
        r.x_out = h->X(mid ^ 1);
        r.lw_in = lw;
        r.k1 = std::min(p.k1, ss);
        r.out_rot = (ss <= p.k1) ? rot : 0u;
        h->mark(PF_KERNEL_PASS1, true);
        launch_pass1(h, r, kPass1Resample);
        h->mark(PF_KERNEL_PASS1, false);
        ++launches;
        xs = mid ^ 1;
        for (const StagePass& sp : p.passes) {
            if (sp.s0 > ss) break;
            const uint32_t kk = std::min(sp.k, ss - sp.s0 + 1u);
            const StagePass q = stage_pass_for(h, sp, kk);
            const bool last = sp.s0 + kk - 1u == ss;
            h->mark(PF_KERNEL_STAGES, true);
            launch_stages_k(h, q, h->X(xs), h->X(xs ^ 1), last ? rot : 0u);
            h->mark(PF_KERNEL_STAGES, false);
            xs ^= 1;
            ++launches;
        }
    }
    if (rot) h->rho = (h->rho + rot) % h->S;
    // weights carried into the next step (R18)
    if (ss == 0u) {
        h->carry_mode = 1;  // lw of this step, in buffer lwi (the next weigh pass writes the other)
        h->lwi ^= 1;
    } else if (ss < h->S) {
        h->carry_mode = 2;
        // block of level S* containing group g: g >> S* in this layout; after the rotation
        // by S* bits the same block is the low S - S* bits of the new group index
        h->carry_shift = rot ? 0u : ss;
        h->carry_mask = rot ? ((1u << (h->S - ss)) - 1u) : 0xffffffffu;
        cudaMemcpyAsync(h->at<double>(h->lay.carry_lv), h->at<double>(h->lay.logV) + level_offset(h->m, (int)ss),
                        (size_t)(h->m >> ss) * 8, cudaMemcpyDeviceToDevice, h->stream);
    } else {
        h->carry_mode = 0;
    }
    h->carry_c = lvS;
    h->sstar_last = (int)ss;
    h->cur = xs;
    h->step_n = h->n;
    h->n += 1;
    h->have_step = true;
    h->top_done = true;
    h->last_launches = launches;
    return check_cuda(h, "pf_step");
}

// One AIRPF step (Alg. 4 rotated like Alg. 1; R19-R21):
//   k_pass1 (AIRPF mode: read the island blocks named by the previous island map, mutate,
//   weight, within-island resample, island levels 1..k1) -> k_cascade (levels k1+1..S,
//   island thresholds) -> k_island_draw -> k_island_compose (the new island map).
// x_hat is never materialised: the next step reads block A_isl[g] for island g.
static int run_step_airpf(pf_handle* h, const float* y_host, const float* y_dev) {
    Pass1Args a{};
    fill_pass1(h, a, y_host, y_dev);
    a.x_in = h->X(h->cur);
    a.x_out = h->X(h->cur ^ 1);
    a.isl_src = h->isl_valid ? h->at<int32_t>(h->lay.isl_A) : nullptr;
    a.logW = h->at<double>(h->lay.isl_logW);
    if (h->world > 1 && h->isl_valid) {  // sharded (R27): the blocks live on their owners
        if (h->peer_ws.size() != h->world) return fail(h, PF_ESTATE, "sharded AIRPF needs the peer mapping (pf_peer_open/set)");
        const size_t xoff = h->cur ? h->lay.X1 : h->lay.X0;  // same layout on every rank
        for (uint32_t r = 0; r < h->world; ++r) a.xpeer[r] = reinterpret_cast<const float*>(h->peer_ws[r] + xoff);
        a.peer_shift = h->S;  // m / world = 2^S_loc islands per rank
    }
    // d >= 4: no stage tables in AIRPF mode; the smaller footprint (with <= 64 registers,
    // launch bounds of kPass1Airpf) fits 8 CTAs per SM (C4: 4.79 -> 4.42 ms per pass; the
    // same change measured slower for d = 1)
    if (h->plan.D >= 4) a.sl = pass1_smem(h->plan.D, h->plan.P1, h->M, 1u, h->plan.pass1_threads, h->plan.tb);
    const bool adaptive = h->theta > 0.0;  // AIRPF2 (reading R26)
    if (adaptive) {
        a.carry_mode = h->carry_mode;  // 0 or 2 (block carry: the island's V_bar_{S*} or W_check)
        a.carry_lv = h->at<double>(h->lay.carry_lv);
        a.carry_shift = h->carry_shift;
        a.carry_mask = h->carry_mask;
        a.carry_c = h->carry_c;
        a.ess_lmax = h->at<unsigned int>(h->lay.ess_lmax);
    }
    h->mark(PF_KERNEL_PASS1, true);
    launch_pass1(h, a, kPass1Airpf);
    h->mark(PF_KERNEL_PASS1, false);
    h->mark(PF_KERNEL_CASCADE, true);
    launch_cascade_k(h);
    uint32_t ss = h->S;
    double lvS = 0.0;
    int launches = 4;
    if (adaptive) {  // island ESS levels, S*: the island stages that run
        EssArgs e{};
        e.lv0 = h->at<double>(h->lay.isl_logW);
        e.ess_part = nullptr;
        e.logV = h->at<double>(h->lay.logV);
        e.lmax = h->at<unsigned int>(h->lay.ess_lmax);
        e.chunks = h->at<double>(h->lay.ess_chunks);
        e.out = h->at<double>(h->lay.ess_out);
        e.N = h->N;
        e.NT = h->plan.NT;
        e.m = h->m;
        e.S = h->S;
        e.theta = h->theta;
        launch_ess(LaunchCfg{0u, 0u, 0u, h->stream}, e);
        launches += 2;
        double tail[2];
        cudaError_t ce = cudaMemcpyAsync(tail, e.out + h->S + 1, sizeof(tail), cudaMemcpyDeviceToHost, h->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
        if (ce != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_step (AIRPF2): ") + cudaGetErrorString(ce));
        ss = (uint32_t)tail[0];
        lvS = tail[1];
    }
    IslandArgs ia{};
    ia.key = make_key(h->seed);
    ia.n = h->n;
    ia.m = h->m;
    ia.S = ss;  // island stages 1..S* (all S unless AIRPF2 stops early; sharded: the local ones)
    ia.island0 = h->pos0 >> h->b;
    ia.modified = h->airpf == 1;
    ia.thr = h->at<uint32_t>(h->lay.thr);
    ia.choice = h->at<uint8_t>(h->lay.isl_choice);
    ia.A = h->at<int32_t>(h->lay.isl_A);
    launch_island(h->stream, ia);
    h->mark(PF_KERNEL_CASCADE, false);
    if (adaptive) {  // the weights the islands carry into the next step (R18 / R26)
        if (ss == 0u) {
            h->carry_mode = 2;
            h->carry_shift = 0u;
            cudaMemcpyAsync(h->at<double>(h->lay.carry_lv), h->at<double>(h->lay.isl_logW), (size_t)h->m * 8,
                            cudaMemcpyDeviceToDevice, h->stream);
        } else if (ss < h->S) {
            h->carry_mode = 2;
            h->carry_shift = ss;
            cudaMemcpyAsync(h->at<double>(h->lay.carry_lv), h->at<double>(h->lay.logV) + level_offset(h->m, (int)ss),
                            (size_t)(h->m >> ss) * 8, cudaMemcpyDeviceToDevice, h->stream);
        } else {
            h->carry_mode = 0;
        }
        h->carry_mask = 0xffffffffu;
        h->carry_c = lvS;
    }
    h->cur ^= 1;
    h->isl_valid = true;
    h->sstar_last = (int)ss;
    h->step_n = h->n;
    h->n += 1;
    h->have_step = h->world == 1;  // sharded: pf_step_top and the cross island stages follow
    h->top_done = h->world == 1;
    h->last_launches = launches;
    return check_cuda(h, "pf_step (AIRPF)");
}

// One step of the plain BPF (Alg. 1 with Alg. 2): k_pass1 (weigh) -> k_cascade (the
// estimates) -> k_mn_tile_cdf -> k_mn_offsets -> k_mn_draw (search + gather).
static int run_step_multinomial(pf_handle* h, const float* y_host, const float* y_dev) {
    const int src = h->cur, mid = h->cur ^ 1;
    float* lw = h->at<float>(h->lay.lw0);
    Pass1Args a{};
    fill_pass1(h, a, y_host, y_dev);
    a.x_in = h->X(src);
    a.x_out = h->X(mid);
    a.lw_out = lw;
    a.ess_part = h->at<double>(h->lay.ess_part);
    a.ess_lmax = h->at<unsigned int>(h->lay.ess_lmax);
    h->mark(PF_KERNEL_PASS1, true);
    launch_pass1(h, a, kPass1Weigh);
    h->mark(PF_KERNEL_PASS1, false);
    h->mark(PF_KERNEL_CASCADE, true);
    launch_cascade_k(h);
    h->mark(PF_KERNEL_CASCADE, false);
    MultinomialArgs mn{};
    mn.key = make_key(h->seed);
    mn.n = h->n;
    mn.N = h->N;
    mn.NT = (uint32_t)((h->N + kMnTile - 1) / kMnTile);
    mn.cdf = h->at<float>(h->lay.mn_cdf);
    mn.cdf32 = h->at<float>(h->lay.mn_cdf32);
    mn.trec = h->at<double>(h->lay.mn_trec);
    mn.off = h->at<double>(h->lay.mn_off);
    mn.lmax = h->at<unsigned int>(h->lay.ess_lmax);
    mn.x = h->X(mid);
    mn.xhat = h->X(src);
    mn.dbg_anc = (h->flags & PF_FLAG_DEBUG) ? h->at<int32_t>(h->lay.dbg_A) : nullptr;
    h->mark(PF_KERNEL_STAGES, true);
    launch_multinomial(h->plan.D, h->stream, mn, lw);
    h->mark(PF_KERNEL_STAGES, false);
    cudaMemsetAsync(h->at<unsigned int>(h->lay.ess_lmax), 0, 4, h->stream);  // running max for the next step
    h->anc_ready = mn.dbg_anc != nullptr;
    h->sstar_last = (int)h->S;
    h->step_n = h->n;
    h->n += 1;
    h->have_step = true;
    h->top_done = true;
    h->last_launches = 5;
    return check_cuda(h, "pf_step (multinomial)");
}

// The plain step in two halves (phase bit 1: k_pass1 + k_cascade, after which the shard
// record and every V level of a sharded handle are final -- Lemma facts_about_Vs (a),
// so the records' all-gather can overlap bit 2: the k_stages passes).
static int run_step_plain(pf_handle* h, const float* y_host, const float* y_dev, int phase) {
    const Plan& p = h->plan;
    if (phase & 1) {
        Pass1Args a{};
        fill_pass1(h, a, y_host, y_dev);
        const int src = h->cur, dst = h->cur ^ 1;
        a.x_in = h->X(src);
        a.x_out = h->X(dst);
        h->mark(PF_KERNEL_PASS1, true);
        launch_pass1(h, a);
        h->mark(PF_KERNEL_PASS1, false);
        h->mark(PF_KERNEL_CASCADE, true);
        launch_cascade_k(h);
        h->mark(PF_KERNEL_CASCADE, false);
        h->cur = dst;
        h->half_step = (phase & 2) == 0;
        h->last_launches = 2;
        if (h->world > 1) {  // this step's top levels are pending (pf_step_top)
            h->top_done = false;
            h->have_step = false;
        }
    }
    if (phase & 2) {
        // stages k1+1..S: state-moving tile passes
        int xs = h->cur;
        for (const StagePass& sp : p.passes) {
            h->mark(PF_KERNEL_STAGES, true);
            launch_stages_k(h, sp, h->X(xs), h->X(xs ^ 1));
            h->mark(PF_KERNEL_STAGES, false);
            xs ^= 1;
        }
        h->cur = xs;
        h->half_step = false;
        h->last_launches = (phase & 1 ? 2 : h->last_launches) + (int)p.passes.size();
        h->sstar_last = (int)h->S;
        h->step_n = h->n;
        h->n += 1;
        if (h->world == 1) {
            h->have_step = true;
            h->top_done = true;
        }
    }
    return check_cuda(h, "pf_step");
}

static int run_step(pf_handle* h, const float* y_host, const float* y_dev) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(h->stream, &cs);
    if (h->gexec && cs == cudaStreamCaptureStatusNone)
        return fail(h, PF_ESTATE, "a captured graph is pending: pf_graph_launch first");
    if (h->airpf) return run_step_airpf(h, y_host, y_dev);  // AIRPF, or AIRPF2 with theta > 0
    if (h->theta > 0.0) return run_step_adaptive(h, y_host, y_dev);
    if (h->multinomial) return run_step_multinomial(h, y_host, y_dev);
    return run_step_plain(h, y_host, y_dev, 3);
}

static int dispatch_step(pf_handle* h, const float* yh, const float* yd) { return run_step(h, yh, yd); }

// ---------------------------------------------------------------------------------------
extern "C" {

static bool shard_geometry(uint64_t N, uint32_t M, int rank, int world, uint64_t* Nloc, std::string* err) {
    if (world < 1 || ilog2_exact((uint64_t)world) < 0 || rank < 0 || rank >= world) {
        *err = "world must be a power of two >= 1 and 0 <= rank < world";
        return false;
    }
    const uint64_t m = N / M;
    if (m % (uint64_t)world != 0 || m / (uint64_t)world < 2) {
        *err = "each shard needs >= 2 groups (m / world >= 2)";
        return false;
    }
    *Nloc = N / (uint64_t)world;
    return true;
}

static size_t workspace_bytes(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags, int world,
                              std::string* err) {
    uint64_t Nloc = 0;
    if (!validate_model(model, err) || !validate_topology(N, M, err) || !shard_geometry(N, M, 0, world, &Nloc, err))
        return 0;
    Plan p;
    if (!make_plan(model->d, Nloc, M, &p, err, N)) return 0;
    return make_layout(p, Nloc, M, flags, (uint32_t)world, ilog2_exact(N / M)).total;
}

static int init_core(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags, int rank,
                     int world, void* dev_ws, size_t ws_bytes, void* cuda_stream, pf_handle** out) {
    if (!out) return fail(nullptr, PF_EINVAL, "out is NULL");
    *out = nullptr;
    std::string err;
    uint64_t Nloc = 0;
    if (!validate_model(model, &err)) return fail(nullptr, PF_EINVAL, err);
    if (!validate_topology(N, M, &err)) return fail(nullptr, PF_EINVAL, err);
    if (!shard_geometry(N, M, rank, world, &Nloc, &err)) return fail(nullptr, PF_EINVAL, err);
    if ((flags & PF_FLAG_ADAPTIVE) && world != 1) return fail(nullptr, PF_EINVAL, "PF_FLAG_ADAPTIVE needs world = 1");
    if ((flags & PF_FLAG_MULTINOMIAL) && world != 1) return fail(nullptr, PF_EINVAL, "PF_FLAG_MULTINOMIAL needs world = 1");
    if ((flags & PF_FLAG_AIRPF) && (M < 4u || (world > 1 && ((N / M / (uint64_t)world) % 4u != 0 ||
                                                           (flags & PF_FLAG_ADAPTIVE)))))
        return fail(nullptr, PF_EINVAL, "PF_FLAG_AIRPF needs M >= 4; sharded: m / world a multiple of 4, no adaptive");
    Plan p;
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        nsm <= 0) {
        cudaGetLastError();
        nsm = 148;
    }
    if (!make_plan(model->d, Nloc, M, &p, &err, N, (uint32_t)nsm)) return fail(nullptr, PF_EINVAL, err);
    const int Sglobal = ilog2_exact(N / M);
    Layout L = make_layout(p, Nloc, M, flags, (uint32_t)world, Sglobal);
    if (!dev_ws || ws_bytes < L.total) return fail(nullptr, PF_EWORKSPACE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(dev_ws) & 255u) return fail(nullptr, PF_EWORKSPACE, "workspace not 256-byte aligned");
    pf_handle* h = new pf_handle();
    h->mp = to_params(model);
    h->N = Nloc;
    h->M = M;
    h->b = (uint32_t)ilog2_exact(M);
    h->m = (uint32_t)(Nloc / M);
    h->S = (uint32_t)ilog2_exact(h->m);
    h->Nglobal = N;
    h->Sglobal = (uint32_t)Sglobal;
    h->rank = (uint32_t)rank;
    h->world = (uint32_t)world;
    h->L = (uint32_t)ilog2_exact((uint64_t)world);
    h->pos0 = (uint32_t)(Nloc * (uint64_t)rank);
    h->step_n = 0;
    h->top_done = false;
    h->seed = seed;
    h->flags = flags;
    h->plan = p;
    h->lay = L;
    h->ws = static_cast<unsigned char*>(dev_ws);
    h->stream = static_cast<cudaStream_t>(cuda_stream);
    h->n = 0;
    h->cur = 0;
    h->have_step = false;
    h->last_launches = 0;
    h->timing = false;
    cudaMemsetAsync(h->at<uint32_t>(L.ticket), 0, 16, h->stream);
    if (flags & (PF_FLAG_ADAPTIVE | PF_FLAG_MULTINOMIAL))
        cudaMemsetAsync(h->at<uint32_t>(L.ess_lmax), 0, 16, h->stream);  // running max, reset after each use
    {
        InitArgs ia{};
        ia.mp = h->mp;
        ia.key = make_key(seed);
        ia.N = h->N;
        ia.pos0 = h->pos0;
        ia.x = h->X(0);
        const uint32_t grid = (uint32_t)std::min<uint64_t>((h->N / 4 + 255) / 256, 148ull * 16);
        launch_init(p.D, h->mp.kind, LaunchCfg{grid, 256u, 0u, h->stream}, ia);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        delete h;
        return fail(nullptr, PF_ECUDA, std::string("pf_init: ") + cudaGetErrorString(e));
    }
    *out = h;
    return PF_OK;
}

size_t pf_workspace_bytes(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags) {
    std::string err;
    return workspace_bytes(model, N, M, flags, 1, &err);
}

size_t pf_workspace_bytes_sharded(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags, int world) {
    std::string err;
    return workspace_bytes(model, N, M, flags, world, &err);
}

int pf_init(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags, void* dev_ws,
            size_t ws_bytes, void* cuda_stream, pf_handle** out) {
    return init_core(model, N, M, seed, flags, 0, 1, dev_ws, ws_bytes, cuda_stream, out);
}

int pf_init_sharded(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags, int rank, int world,
                    void* dev_ws, size_t ws_bytes, void* cuda_stream, pf_handle** out) {
    return init_core(model, N, M, seed, flags, rank, world, dev_ws, ws_bytes, cuda_stream, out);
}

int pf_step_local(pf_handle* h, const float* y_host, const float* y_dev) {
    if (!h || (!y_host && !y_dev)) return fail(h, PF_EINVAL, "NULL argument");
    if (y_host)
        for (int k = 0; k < h->mp.dy; ++k)
            if (!std::isfinite(y_host[k])) return fail(h, PF_EOBS, "non-finite observation");
    return dispatch_step(h, y_host, y_dev);
}

int pf_step_local_begin(pf_handle* h, const float* y_host, const float* y_dev) {
    if (!h || (!y_host && !y_dev)) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (h->half_step) return fail(h, PF_ESTATE, "pf_step_local_end is pending");
    if (y_host)
        for (int k = 0; k < h->mp.dy; ++k)
            if (!std::isfinite(y_host[k])) return fail(h, PF_EOBS, "non-finite observation");
    return run_step_plain(h, y_host, y_dev, 1);
}

int pf_step_local_end(pf_handle* h) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (!h->half_step) return fail(h, PF_ESTATE, "pf_step_local_begin must run first");
    return run_step_plain(h, nullptr, nullptr, 2);
}

int pf_shard_record(pf_handle* h, const double** dev_rec) {
    if (!h || !dev_rec) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    *dev_rec = h->at<double>(h->lay.shard_rec);
    return PF_OK;
}

int pf_step_top(pf_handle* h, const double* dev_all_recs) {
    if (!h || !dev_all_recs) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    TopArgs t{};
    t.recs = dev_all_recs;
    t.top_logV = h->at<double>(h->lay.top_logV);
    t.top_thr = h->at<uint32_t>(h->lay.top_thr);
    t.est = h->at<double>(h->lay.est);
    t.scratch = h->at<double>(h->lay.top_scratch);
    t.Nglobal = h->Nglobal;
    t.G = h->world;
    t.L = h->L;
    t.b = h->airpf ? 1u : h->b;  // AIRPF: 31-bit island thresholds (R20)
    h->mark(PF_KERNEL_TOP, true);
    launch_top(h->plan.D, LaunchCfg{1u, 1024u, 0u, h->stream}, t);
    h->mark(PF_KERNEL_TOP, false);
    h->top_done = true;
    h->have_step = true;
    return check_cuda(h, "pf_step_top");
}

int pf_cross_buffer(pf_handle* h, const void** dev_states, size_t* bytes) {
    if (!h || !dev_states || !bytes) return fail(h, PF_EINVAL, "NULL argument");
    *dev_states = h->X(h->cur);
    *bytes = (size_t)h->N * (size_t)h->plan.D * 4u;
    return PF_OK;
}

int pf_cross_stage(pf_handle* h, int t, const void* dev_partner_states) {
    // Stream-ordered: k_cross reads the stage threshold that k_top wrote on this stream.
    if (!h || !dev_partner_states) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2 || t < 1 || (uint32_t)t > h->L) return fail(h, PF_EINVAL, "cross stage out of range");
    if (!h->top_done) return fail(h, PF_ESTATE, "pf_step_top must run first");
    const uint32_t* top_thr = h->at<uint32_t>(h->lay.top_thr);
    const uint32_t G = h->world;
    CrossArgs c{};
    c.key = make_key(h->seed);
    c.n = h->step_n;
    c.s = h->S + (uint32_t)t;
    c.t = (uint32_t)t;
    c.rank = h->rank;
    c.b = h->b;
    c.M = h->M;
    c.Nloc = h->N;
    c.pos0 = h->pos0;
    c.pos0_partner = (uint32_t)(h->N * (uint64_t)(h->rank ^ (1u << (t - 1))));
    c.thr = top_thr + (G - (G >> (t - 1))) + (h->rank >> t);
    c.own_in = h->X(h->cur);
    c.partner_in = dev_partner_states;
    c.out = h->X(h->cur ^ 1);
    c.dbg_anc = (h->flags & PF_FLAG_DEBUG) ? h->at<int32_t>(h->lay.dbg_anc) : nullptr;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((h->N / 4 + 255) / 256, (uint64_t)148 * 8);
    const int D = h->plan.D;
    h->mark(PF_KERNEL_CROSS, true);
    launch_cross(D == 1 ? kPayloadF1 : (D == 2 ? kPayloadF2 : (D == 4 ? kPayloadF4 : kPayloadF8)),
                 (h->flags & PF_FLAG_DEBUG) != 0, LaunchCfg{grid, 256u, 0u, h->stream}, c);
    h->mark(PF_KERNEL_CROSS, false);
    h->cur ^= 1;
    return check_cuda(h, "pf_cross_stage");
}

// ---- pull exchange of the cross stages (include/pf.h) --------------------
static PullArgs pull_args(pf_handle* h) {
    PullArgs a{};
    a.key = make_key(h->seed);
    a.n = h->step_n;
    a.S_loc = h->S;
    a.L = h->L;
    a.rank = h->rank;
    a.b = h->b;
    a.M = h->M;
    a.Nloc = h->N;
    a.top_thr = h->at<uint32_t>(h->lay.top_thr);
    a.G = h->world;
    a.src_local = h->at<uint32_t>(h->lay.pull_src);
    a.src_rank = h->at<uint32_t>(h->lay.pull_rank);
    a.counts = h->at<unsigned long long>(h->lay.pull_counts);
    a.fill = h->at<uint32_t>(h->lay.pull_fill);
    a.offsets = h->at<unsigned long long>(h->lay.pull_off);
    a.req = h->at<uint32_t>(h->lay.pull_req);
    a.outpos = h->at<uint32_t>(h->lay.pull_outpos);
    a.dbg_anc = (h->flags & PF_FLAG_DEBUG) ? h->at<int32_t>(h->lay.dbg_anc) : nullptr;
    return a;
}

int pf_cross_pull_plan(pf_handle* h, uint64_t* host_counts) {
    if (!h || !host_counts) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (h->world > 64) return fail(h, PF_EINVAL, "the pull exchange supports up to 64 ranks");
    if (!h->top_done) return fail(h, PF_ESTATE, "pf_step_top must run first");
    const PullArgs a = pull_args(h);
    cudaMemsetAsync(a.counts, 0, (size_t)h->world * 8, h->stream);
    cudaMemsetAsync(a.fill, 0, (size_t)h->world * 4, h->stream);
    h->mark(PF_KERNEL_CROSS, true);
    launch_pull_compose(h->stream, a, (h->flags & PF_FLAG_DEBUG) != 0);
    h->mark(PF_KERNEL_CROSS, false);
    cudaError_t e = cudaMemcpyAsync(host_counts, a.counts, (size_t)h->world * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_cross_pull_plan: ") + cudaGetErrorString(e));
    return check_cuda(h, "pf_cross_pull_plan");
}

int pf_cross_pull_pack(pf_handle* h, const uint64_t* host_offsets, const uint32_t** dev_requests) {
    if (!h || !host_offsets || !dev_requests) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    const PullArgs a = pull_args(h);
    const cudaError_t e = cudaMemcpyAsync(const_cast<unsigned long long*>(a.offsets), host_offsets,
                                          (size_t)h->world * 8, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_cross_pull_pack: ") + cudaGetErrorString(e));
    h->mark(PF_KERNEL_CROSS, true);
    launch_pull_pack(h->stream, a);
    h->mark(PF_KERNEL_CROSS, false);
    *dev_requests = a.req;
    return check_cuda(h, "pf_cross_pull_pack");
}

int pf_cross_pull_serve(pf_handle* h, const uint32_t* dev_requests_in, uint64_t n, const void** dev_states) {
    if (!h || (n && !dev_requests_in) || !dev_states) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (n > h->N * (uint64_t)h->world) return fail(h, PF_EINVAL, "too many requests");
    float* out = h->at<float>(h->lay.pull_serve);
    h->mark(PF_KERNEL_CROSS, true);
    if (n) launch_pull_move(h->stream, h->plan.D, true, h->X(h->cur), dev_requests_in, out, n);
    h->mark(PF_KERNEL_CROSS, false);
    *dev_states = out;
    return check_cuda(h, "pf_cross_pull_serve");
}

int pf_cross_pull_finish(pf_handle* h, const void* dev_states_in) {
    if (!h || !dev_states_in) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    h->mark(PF_KERNEL_CROSS, true);
    launch_pull_move(h->stream, h->plan.D, false, static_cast<const float*>(dev_states_in),
                     h->at<uint32_t>(h->lay.pull_outpos), h->X(h->cur ^ 1), h->N);
    h->mark(PF_KERNEL_CROSS, false);
    h->cur ^= 1;
    return check_cuda(h, "pf_cross_pull_finish");
}

// ---- peer-memory exchange of the cross stages (include/pf.h) ------------
static_assert(sizeof(cudaIpcMemHandle_t) == PF_IPC_HANDLE_BYTES, "IPC handle size");
typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

int pf_peer_export(pf_handle* h, void* ipc_handle, uint64_t* offset) {
    if (!h || !ipc_handle || !offset) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess)
        return fail(h, PF_ECUDA, "pf_peer_export: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (reinterpret_cast<MemGetAddressRangeFn>(fn)(&base, &size, reinterpret_cast<unsigned long long>(h->ws)) != 0)
        return fail(h, PF_ECUDA, "pf_peer_export: the workspace is not a device allocation");
    cudaIpcMemHandle_t hd;
    e = cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_peer_export: ") + cudaGetErrorString(e));
    std::memcpy(ipc_handle, &hd, sizeof(hd));
    *offset = reinterpret_cast<unsigned long long>(h->ws) - base;
    return PF_OK;
}

int pf_peer_open(pf_handle* h, const void* ipc_handles, const uint64_t* offsets) {
    if (!h || !ipc_handles || !offsets) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (h->world > kPeerMaxG) return fail(h, PF_EINVAL, "the peer exchange supports up to 64 ranks");
    for (void* p : h->peer_ipc) cudaIpcCloseMemHandle(p);
    h->peer_ipc.clear();
    h->peer_ws.assign(h->world, nullptr);
    for (uint32_t r = 0; r < h->world; ++r) {
        if (r == h->rank) {
            h->peer_ws[r] = h->ws;
            continue;
        }
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, static_cast<const unsigned char*>(ipc_handles) + (size_t)r * PF_IPC_HANDLE_BYTES, sizeof(hd));
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            h->peer_ws.clear();
            return fail(h, PF_ECUDA, std::string("pf_peer_open: rank ") + std::to_string(r) + ": " + cudaGetErrorString(e));
        }
        h->peer_ipc.push_back(p);
        h->peer_ws[r] = static_cast<unsigned char*>(p) + offsets[r];
    }
    return PF_OK;
}

int pf_peer_set(pf_handle* h, const uint64_t* dev_workspaces) {
    if (!h || !dev_workspaces) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (h->world > kPeerMaxG) return fail(h, PF_EINVAL, "the peer exchange supports up to 64 ranks");
    if (reinterpret_cast<unsigned char*>(dev_workspaces[h->rank]) != h->ws)
        return fail(h, PF_EINVAL, "dev_workspaces[rank] must be this handle's workspace");
    for (uint32_t r = 0; r < h->world; ++r)
        if (!dev_workspaces[r] || (dev_workspaces[r] & 255u)) return fail(h, PF_EINVAL, "NULL or misaligned workspace");
    for (void* p : h->peer_ipc) cudaIpcCloseMemHandle(p);
    h->peer_ipc.clear();
    h->peer_ws.assign(h->world, nullptr);
    for (uint32_t r = 0; r < h->world; ++r) h->peer_ws[r] = reinterpret_cast<unsigned char*>(dev_workspaces[r]);
    return PF_OK;
}

int pf_cross_peer(pf_handle* h) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (!h->top_done) return fail(h, PF_ESTATE, "pf_step_top must run first");
    if (h->peer_ws.size() != h->world) return fail(h, PF_ESTATE, "no peer mapping: pf_peer_open or pf_peer_set first");
    const PullArgs a = pull_args(h);
    PeerArgs p{};
    const size_t xoff = h->cur ? h->lay.X1 : h->lay.X0;  // same layout on every rank
    for (uint32_t r = 0; r < kPeerMaxG; ++r)
        p.x[r] = r < h->world ? reinterpret_cast<const float*>(h->peer_ws[r] + xoff) : nullptr;
    p.out = h->X(h->cur ^ 1);
    h->mark(PF_KERNEL_CROSS, true);
    launch_peer_gather(h->stream, h->plan.D, a, p, (h->flags & PF_FLAG_DEBUG) != 0);
    h->mark(PF_KERNEL_CROSS, false);
    h->cur ^= 1;
    return check_cuda(h, "pf_cross_peer");
}

// ---- relabelled exchange of the cross stages (include/pf.h; reading R24) ----
static RelabelArgs relabel_args(pf_handle* h, int t) {
    RelabelArgs a{};
    a.key = make_key(h->seed);
    a.n = h->step_n;
    a.s = h->S + (uint32_t)t;
    a.b = h->b;
    a.M = h->M;
    a.Nloc = h->N;
    a.rank = h->rank;
    a.partner = h->rank ^ (1u << (t - 1));
    a.own_is_low = ((h->rank >> (t - 1)) & 1u) == 0u ? 1u : 0u;
    a.thr = h->at<uint32_t>(h->lay.top_thr) + (h->world - (h->world >> (t - 1))) + (h->rank >> t);
    a.nchunks = (uint32_t)((h->N + kRlChunk - 1) / kRlChunk);
    a.cnt = h->at<uint32_t>(h->lay.rl_cnt);
    a.off = h->at<uint32_t>(h->lay.rl_off);
    a.own = h->at<uint32_t>(h->lay.rl_own);
    a.par = h->at<uint32_t>(h->lay.rl_par);
    a.kidx = h->at<uint32_t>(h->lay.rl_kidx);
    a.x = h->X(h->cur);
    a.out = h->X(h->cur ^ 1);
    a.send = h->at<float>(h->lay.rl_send);
    a.recv = nullptr;
    a.kmin = 0;
    a.nsend = 0;
    a.dbg_anc = (h->flags & PF_FLAG_DEBUG) ? h->at<int32_t>(h->lay.dbg_anc) + (size_t)(a.s - 1) * h->N : nullptr;
    return a;
}

int pf_relabel_begin(pf_handle* h, int t, uint64_t* host_counts, const void** dev_send, uint64_t* n_send,
                     uint64_t* n_recv) {
    if (!h || !host_counts || !dev_send || !n_send || !n_recv) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (t < 1 || (uint32_t)t > h->L) return fail(h, PF_EINVAL, "cross stage out of range");
    if (!h->top_done) return fail(h, PF_ESTATE, "pf_step_top must run first");
    RelabelArgs a = relabel_args(h, t);
    h->mark(PF_KERNEL_CROSS, true);
    launch_relabel_plan(h->stream, a);
    uint32_t tot[2] = {0u, 0u};
    cudaError_t e = cudaMemcpyAsync(tot, a.off + 2ull * a.nchunks, sizeof(tot), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_relabel_begin: ") + cudaGetErrorString(e));
    launch_relabel_lists(h->stream, a);
    const uint64_t no = tot[0], np = tot[1], kmin = no < np ? no : np;
    a.kmin = kmin;
    a.nsend = np - kmin;  // the partner's surplus outputs read these states of this shard
    launch_relabel_move(h->stream, (int)h->plan.D, a, true, 0, false);
    h->mark(PF_KERNEL_CROSS, false);
    h->rl_t = t;
    h->rl_own = no;
    h->rl_kmin = kmin;
    host_counts[0] = no;
    host_counts[1] = np;
    *dev_send = a.send;
    *n_send = np - kmin;
    *n_recv = no - kmin;
    return check_cuda(h, "pf_relabel_begin");
}

int pf_relabel_end(pf_handle* h, int t, const void* dev_recv) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (t != h->rl_t) return fail(h, PF_ESTATE, "pf_relabel_begin(t) must run first");
    if (!dev_recv && h->rl_own > h->rl_kmin) return fail(h, PF_EINVAL, "NULL receive buffer");
    RelabelArgs a = relabel_args(h, t);
    a.kmin = h->rl_kmin;
    a.recv = dev_recv;
    h->mark(PF_KERNEL_CROSS, true);
    launch_relabel_move(h->stream, (int)h->plan.D, a, false, h->rl_own, (h->flags & PF_FLAG_DEBUG) != 0);
    h->mark(PF_KERNEL_CROSS, false);
    h->cur ^= 1;
    h->rl_t = 0;
    return check_cuda(h, "pf_relabel_end");
}

// ---- sharded AIRPF: the cross island stages (include/pf.h; reading R27) ------
int pf_island_map(pf_handle* h, const int32_t** dev_map) {
    if (!h || !dev_map) return fail(h, PF_EINVAL, "NULL argument");
    if (!h->airpf || !h->isl_valid) return fail(h, PF_ESTATE, "no AIRPF step");
    *dev_map = h->at<int32_t>(h->lay.isl_A);
    return PF_OK;
}

int pf_island_cross(pf_handle* h, int t, const int32_t* dev_partner_map) {
    if (!h || !dev_partner_map) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world < 2) return fail(h, PF_ESTATE, "not a sharded handle");
    if (!h->airpf || !h->isl_valid) return fail(h, PF_ESTATE, "no AIRPF step");
    if (t < 1 || (uint32_t)t > h->L) return fail(h, PF_EINVAL, "cross stage out of range");
    if (!h->top_done) return fail(h, PF_ESTATE, "pf_step_top must run first");
    IslandCrossArgs c{};
    c.key = make_key(h->seed);
    c.n = h->step_n;
    c.s = h->S + (uint32_t)t;
    c.m = h->m;
    c.island0 = h->pos0 >> h->b;
    c.rank = h->rank;
    c.t = (uint32_t)t;
    c.modified = h->airpf == 1;
    c.thr = h->at<uint32_t>(h->lay.top_thr) + (h->world - (h->world >> (t - 1))) + (h->rank >> t);
    c.A = h->at<int32_t>(h->lay.isl_A);
    c.Apar = dev_partner_map;
    c.choice = h->at<uint8_t>(h->lay.isl_choice) + (size_t)(c.s - 1) * ((h->m + 3) / 4);
    h->mark(PF_KERNEL_CROSS, true);
    launch_island_cross(h->stream, c);
    h->mark(PF_KERNEL_CROSS, false);
    return check_cuda(h, "pf_island_cross");
}

int pf_guard_check(pf_handle* h, unsigned char fill, uint64_t* bad_bytes) {
    if (!h || !bad_bytes) return fail(h, PF_EINVAL, "NULL argument");
    if (!(h->flags & PF_FLAG_GUARD)) return fail(h, PF_ESTATE, "handle not created with PF_FLAG_GUARD");
    unsigned long long* cnt = h->at<unsigned long long>(h->lay.guard_count);
    cudaMemsetAsync(cnt, 0, 8, h->stream);
    for (size_t g : h->lay.gaps) launch_guard_check(h->stream, h->ws + g, PF_GUARD_BYTES, fill, cnt);
    unsigned long long bad = 0;
    cudaError_t e = cudaMemcpyAsync(&bad, cnt, 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_guard_check: ") + cudaGetErrorString(e));
    *bad_bytes = bad;
    return check_cuda(h, "pf_guard_check");
}

int pf_step(pf_handle* h, const float* y_host) {
    if (!h || !y_host) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world > 1) return fail(h, PF_ESTATE, "sharded handle: use pf_step_local / pf_step_top / pf_cross_stage");
    for (int k = 0; k < h->mp.dy; ++k)
        if (!std::isfinite(y_host[k])) return fail(h, PF_EOBS, "non-finite observation");
    return dispatch_step(h, y_host, nullptr);
}

int pf_step_dev(pf_handle* h, const float* y_dev) {
    if (!h || !y_dev) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world > 1) return fail(h, PF_ESTATE, "sharded handle: use pf_step_local / pf_step_top / pf_cross_stage");
    return dispatch_step(h, nullptr, y_dev);
}

int pf_run_dev(pf_handle* h, const float* y_dev, uint32_t T, double* est_dev) {
    if (!h || (T && !y_dev)) return fail(h, PF_EINVAL, "NULL argument");
    if (h->world > 1) return fail(h, PF_ESTATE, "sharded handle: use pf_step_local / pf_step_top / pf_cross_stage");
    const int d = h->mp.d, D = h->plan.D;
    for (uint32_t k = 0; k < T; ++k) {
        const int rc = dispatch_step(h, nullptr, y_dev + (size_t)k * h->mp.dy);
        if (rc != PF_OK) return rc;
        if (est_dev) {  // rows: filter x, filter x^2, predict x, predict x^2 (d doubles each)
            // a kernel, not a 2-D memcpy: capturable into pf_graph_capture's graph
            launch_rows_copy(h->stream, h->at<double>(h->lay.est), (uint32_t)D, est_dev + (size_t)k * 4 * d, (uint32_t)d, 4u);
            const int rc2 = check_cuda(h, "pf_run_dev");
            if (rc2 != PF_OK) return rc2;
        }
    }
    return PF_OK;
}

// T steps captured into one CUDA graph (launched by pf_graph_launch): for small problems
// whose step is a few short kernels, the inter-kernel gaps of stream launches dominate.
int pf_graph_capture(pf_handle* h, const float* y_dev, uint32_t T, double* est_dev) {
    if (!h || !T || !y_dev) return fail(h, PF_EINVAL, "NULL argument or T = 0");
    if (h->world > 1) return fail(h, PF_ESTATE, "sharded handle");
    if (h->theta > 0.0) return fail(h, PF_ESTATE, "the fully adapted step synchronises (S*): not capturable");
    if (h->gexec) return fail(h, PF_ESTATE, "a captured graph is pending: pf_graph_launch first");
    if (h->stream == nullptr) return fail(h, PF_ESTATE, "stream capture needs a non-default stream");
    const bool timing = h->timing;
    h->timing = false;  // no event records inside the graph
    cudaError_t e = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        h->timing = timing;
        return fail(h, PF_ECUDA, std::string("pf_graph_capture: ") + cudaGetErrorString(e));
    }
    const int rc = pf_run_dev(h, y_dev, T, est_dev);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(h->stream, &g);
    h->timing = timing;
    if (rc != PF_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&h->gexec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        h->gexec = nullptr;
        return fail(h, PF_ECUDA, std::string("pf_graph_capture: ") + cudaGetErrorString(e));
    }
    h->last_launches *= (int)T;  // kernels in the graph (pf_run_dev's last step x T)
    return PF_OK;
}

int pf_graph_launch(pf_handle* h) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (!h->gexec) return fail(h, PF_ESTATE, "no captured graph");
    const cudaError_t e = cudaGraphLaunch(h->gexec, h->stream);
    cudaGraphExecDestroy(h->gexec);  // freed once the launch completes
    h->gexec = nullptr;
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_graph_launch: ") + cudaGetErrorString(e));
    return PF_OK;
}

int pf_estimate(pf_handle* h, int phi, int kind, double* out) {
    if (!h || !out) return fail(h, PF_EINVAL, "NULL argument");
    if (!h->have_step) return fail(h, PF_ESTATE, "no completed step");
    if ((phi != PF_PHI_X && phi != PF_PHI_X2) ||
        (kind != PF_EST_FILTER && kind != PF_EST_PREDICT && kind != PF_EST_RESAMPLED))
        return fail(h, PF_EINVAL, "bad phi / kind");
    const int D = h->plan.D;
    const double* src;
    if (kind == PF_EST_RESAMPLED) {  // x_hat of the last step: X(cur) (through the island map after AIRPF)
        double* part = h->at<double>(h->lay.mom_part);
        double* res = h->at<double>(h->lay.mom_out);
        const int32_t* isl = (h->airpf && h->isl_valid) ? h->at<int32_t>(h->lay.isl_A) : nullptr;
        const float* xs = h->X(h->cur);
        if (isl && h->world > 1) {  // sharded AIRPF: the blocks live on their owners (R27)
            void* xm = nullptr;
            const int rc = pf_debug_ptr(h, PF_DBG_XHAT, 0, &xm);
            if (rc != PF_OK) return rc;
            xs = static_cast<const float*>(xm);
            isl = nullptr;
        }
        launch_moments(h->stream, D, xs, isl, h->b, h->N, part, res);
        const int rc = check_cuda(h, "pf_estimate (resampled)");
        if (rc != PF_OK) return rc;
        src = res + (phi == PF_PHI_X ? 0 : D);
    } else {
        src = h->at<double>(h->lay.est) + (size_t)((kind == PF_EST_FILTER ? 0 : 2) + (phi == PF_PHI_X ? 0 : 1)) * D;
    }
    cudaError_t e = cudaMemcpyAsync(out, src, sizeof(double) * D, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_estimate: ") + cudaGetErrorString(e));
    return PF_OK;
}

void pf_destroy(pf_handle* h) { delete h; }

const char* pf_last_error(const pf_handle* h) { return h ? h->err.c_str() : g_init_error.c_str(); }

int pf_last_step_launches(const pf_handle* h) { return h ? h->last_launches : 0; }

int pf_timing_enable(pf_handle* h, int on) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    h->timing = on != 0;
    h->recs.clear();
    h->used = 0;
    return PF_OK;
}

int pf_timing_read(pf_handle* h, double* ms, int* launches) {
    if (!h || !ms) return fail(h, PF_EINVAL, "NULL argument");
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_timing_read: ") + cudaGetErrorString(e));
    for (int k = 0; k < PF_KERNEL_KINDS; ++k) {
        ms[k] = 0.0;
        if (launches) launches[k] = 0;
    }
    for (const auto& r : h->recs) {
        float t = 0.0f;
        e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess) return fail(h, PF_ECUDA, std::string("pf_timing_read: ") + cudaGetErrorString(e));
        ms[r.kind] += (double)t;
        if (launches) launches[r.kind] += 1;
    }
    h->recs.clear();
    h->used = 0;
    return PF_OK;
}

int pf_debug_ptr(pf_handle* h, int what, int stage, void** dev_out) {
    if (!h || !dev_out) return fail(h, PF_EINVAL, "NULL argument");
    // before the first step X(cur) holds x_0 (k_init): PF_DBG_XHAT reads it (A0 parity)
    if (!h->have_step && !(what == PF_DBG_XHAT && h->n == 0 && !h->isl_valid))
        return fail(h, PF_ESTATE, "no completed step");
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
            if (stage < 1 || stage > (int)h->Sglobal) return fail(h, PF_EINVAL, "stage out of range");
            *dev_out = h->at<int32_t>(h->lay.dbg_anc) + (size_t)(stage - 1) * h->N;
            return PF_OK;
        case PF_DBG_ANC_FINAL: {
            if (h->world > 1) return fail(h, PF_ESTATE, "composed ancestors span shards: use the stage tables");
            if (h->multinomial && h->anc_ready) {  // Alg. 2: the draws are the ancestors
                *dev_out = h->at<int32_t>(h->lay.dbg_A);
                return PF_OK;
            }
            int32_t* A = h->at<int32_t>(h->lay.dbg_A);
            const uint32_t sc = h->sstar_last >= 0 ? (uint32_t)h->sstar_last : h->S;  // stages run
            launch_debug_compose(LaunchCfg{1024u, 256u, 0u, h->stream}, h->at<int32_t>(h->lay.dbg_anc), h->N, sc, A);
            *dev_out = A;
            return check_cuda(h, "pf_debug_ptr");
        }
        case PF_DBG_XHAT:
            if (h->airpf && h->isl_valid) {  // materialise x_hat = the island blocks (into the free buffer)
                if (h->world > 1) {  // sharded (R27): blocks from their owners
                    if (h->peer_ws.size() != h->world) return fail(h, PF_ESTATE, "no peer mapping");
                    PeerArgs pa{};
                    const size_t xoff = h->cur ? h->lay.X1 : h->lay.X0;
                    for (uint32_t r = 0; r < h->world; ++r) pa.x[r] = reinterpret_cast<const float*>(h->peer_ws[r] + xoff);
                    launch_block_gather_peer(h->stream, pa, h->X(h->cur ^ 1), h->at<int32_t>(h->lay.isl_A), h->N, h->b,
                                             (uint32_t)D, h->S);
                } else {
                    launch_block_gather(h->stream, h->X(h->cur), h->X(h->cur ^ 1), h->at<int32_t>(h->lay.isl_A), h->N,
                                        h->b, (uint32_t)D);
                }
                *dev_out = h->X(h->cur ^ 1);
                return check_cuda(h, "pf_debug_ptr");
            }
            *dev_out = h->X(h->cur);
            return PF_OK;
        case PF_DBG_ISLAND_A:
        case PF_DBG_ISLAND_CHOICE:
        case PF_DBG_ISLAND_LOGW:
            if (!(h->flags & PF_FLAG_AIRPF) || !h->isl_valid) return fail(h, PF_ESTATE, "no AIRPF step");
            if (what == PF_DBG_ISLAND_A) *dev_out = h->at<int32_t>(h->lay.isl_A);
            else if (what == PF_DBG_ISLAND_LOGW) *dev_out = h->at<double>(h->lay.isl_logW);
            else {
                if (stage < 1 || stage > (int)h->Sglobal) return fail(h, PF_EINVAL, "stage out of range");
                *dev_out = h->at<uint8_t>(h->lay.isl_choice) + (size_t)(stage - 1) * ((h->m + 3) / 4);
            }
            return PF_OK;
        case PF_DBG_LOGV: *dev_out = h->at<double>(h->lay.logV); return PF_OK;
        case PF_DBG_THRESH: *dev_out = h->at<uint32_t>(h->lay.thr); return PF_OK;
        case PF_DBG_ESS:
            if (!(h->flags & PF_FLAG_ADAPTIVE)) return fail(h, PF_ESTATE, "handle not created with PF_FLAG_ADAPTIVE");
            *dev_out = h->at<double>(h->lay.ess_out);
            return PF_OK;
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
        case PF_DBG_ESS: need = (size_t)(h->S + 1) * 8; break;
        case PF_DBG_ISLAND_A: need = (size_t)h->m * 4; break;
        case PF_DBG_ISLAND_CHOICE: need = (size_t)(h->m + 3) / 4; break;
        case PF_DBG_ISLAND_LOGW: need = (size_t)h->m * 8; break;
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
    h->n = n;
    h->carry_mode = 0;  // the given state is unweighted
    h->isl_valid = false;  // and holds x_hat itself
    h->rho = 0;            // in the natural group layout
    return PF_OK;
}

int pf_set_airpf(pf_handle* h, int mode) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (mode < 0 || mode > 2) return fail(h, PF_EINVAL, "mode must be 0 (off), 1 (Alg. 7) or 2 (Alg. 6)");
    if (mode && !(h->flags & PF_FLAG_AIRPF)) return fail(h, PF_EINVAL, "handle not created with PF_FLAG_AIRPF");
    if (mode && (h->multinomial || h->rotate)) return fail(h, PF_EINVAL, "one resampling scheme at a time");
    if (h->airpf != mode && h->carry_mode != 0)  // carried weights belong to the scheme that made them
        return fail(h, PF_ESTATE, "particles carry weights of an early-stopped step: run one step with theta = 1 first");
    if (!mode && h->isl_valid) {  // back to augmented resampling: materialise x_hat first
        void* xm = nullptr;
        const int rc = pf_debug_ptr(h, PF_DBG_XHAT, 0, &xm);  // into X(cur ^ 1), from the owners when sharded
        if (rc != PF_OK) return rc;
        h->cur ^= 1;
        h->isl_valid = false;
    }
    h->airpf = mode;
    return check_cuda(h, "pf_set_airpf");
}

int pf_set_adaptive(pf_handle* h, double theta) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (!(theta >= 0.0 && theta <= 1.0)) return fail(h, PF_EINVAL, "theta must lie in [0, 1]");
    if (theta > 0.0 && !(h->flags & PF_FLAG_ADAPTIVE))
        return fail(h, PF_EINVAL, "handle not created with PF_FLAG_ADAPTIVE");
    if (theta > 0.0 && h->world != 1) return fail(h, PF_EINVAL, "the fully adapted scheme needs world = 1");
    if (theta > 0.0 && (h->multinomial || (h->airpf && h->rotate)))
        return fail(h, PF_EINVAL, "one resampling scheme at a time");
    // an early-stopped step leaves weighted particles (R18): a plain step would treat them as
    // equally weighted, so switching off is refused until a step has run all S stages
    if (theta == 0.0 && h->carry_mode != 0)
        return fail(h, PF_ESTATE, "particles carry weights of an early-stopped step: run one step with theta = 1 first");
    h->theta = theta;
    if (theta > 0.0) {  // truncated passes run the runtime-plan stage kernels: load them now
        for (const StagePass& sp : h->plan.passes) preload_stages(h->plan.D, (int)sp.tb, (h->flags & PF_FLAG_DEBUG) != 0);
    }
    return PF_OK;
}

int pf_last_stages(const pf_handle* h) { return h ? h->sstar_last : -1; }

int pf_set_rotation(pf_handle* h, int on) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (on && (!(h->flags & PF_FLAG_ADAPTIVE) || h->M < 4u))
        return fail(h, PF_EINVAL, "stage rotation needs PF_FLAG_ADAPTIVE and M >= 4");
    h->rotate = on != 0;
    return PF_OK;
}

int pf_rotation_offset(const pf_handle* h) { return h ? (int)h->rho : -1; }

int pf_set_multinomial(pf_handle* h, int on) {
    if (!h) return fail(h, PF_EINVAL, "NULL handle");
    if (on && !(h->flags & PF_FLAG_MULTINOMIAL)) return fail(h, PF_EINVAL, "handle not created with PF_FLAG_MULTINOMIAL");
    if (on && (h->theta > 0.0 || h->airpf)) return fail(h, PF_EINVAL, "one resampling scheme at a time");
    h->multinomial = on != 0;
    h->anc_ready = false;
    return PF_OK;
}

}  // extern "C"
