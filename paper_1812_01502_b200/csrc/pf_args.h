// pf_args.h -- argument blocks, shared-memory layouts and constants of the step kernels
// (host + device).  The launchers (pf_launch.h) and the host orchestration (pf_api.cu) see
// only this header, so a kernel edit rebuilds only the units that instantiate it.
#pragma once
#include <cstdint>
#include <cstring>

#include "pf_device.cuh"

namespace pfk {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kPass1MaxGroups = 64;  // T1 <= 64: the V tree of a tile fits one warp's lanes

struct Pass1Smem {
    uint32_t xs, w, qe, ey, L1, tab, chunk, lv1, red, ess, thr, total;
};
__host__ __device__ inline Pass1Smem pass1_smem(int D, uint32_t P1, uint32_t M, uint32_t k1, uint32_t threads,
                                                uint32_t tb) {
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
    s.qe = take(P1);  // quad ends of the CDF (P1 / 4 floats): the first search level
    s.ey = take(M > 64u ? P1 : 0u);  // the same in BFS (Eytzinger) order per pool, pools of > 32 quads
    s.L1 = take(P1 * tb);
    s.tab = take(k1 >= 2 ? (k1 - 1u) * P1 * tb : 0u);
    s.chunk = take(M > 64 ? (P1 / 128u) * 4u : 0u);  // per-warp-chunk maxima / totals
    s.lv1 = take(T1 * 8u);  // pair (or, AIRPF, island) log-means
    s.red = take((threads / 32u) * (2u + 4u * (uint32_t)D) * 4u);
    s.ess = take((threads / 32u) * 4u);  // per-warp sum of squared weights (kPass1Weigh)
    s.thr = take(k1 >= 2 ? (k1 - 1u) * (T1 / 4u) * 4u : 0u);  // k_pass1c: stage 2..k1 thresholds from warp 0
    s.total = off;
    return s;
}

struct Pass1Args {
    ModelParams mp;
    Key key;
    uint32_t n;
    int do_mutate;
    const float* y_dev;  // if non-null, y is read from device memory
    float y[8];
    uint64_t N;           // particles of this shard
    uint32_t pos0;        // global index of the shard's first particle (RNG counters)
    uint32_t m, M, b, S, k1, P1, T1;
    uint32_t probe;       // cost probes of experiment builds (-DPF_PROBES), else unused
    uint32_t spec;        // 1: a compile-time (B, K1, QPT) instance of the fused pass may run (k_pass1c)
    Pass1Smem sl;         // shared-memory layout (pass1_smem)
    const float* x_in;    // xhat_{n-1} (or x_0)
    // sharded AIRPF (R27): island g reads global block isl_src[g] from its owner's state
    // buffer, owner = block >> peer_shift (peer-mapped pointers, kPass1PeerMax ranks);
    // xpeer[0] == nullptr: one GPU (x_in)
    const float* xpeer[64];
    uint32_t peer_shift;
    float* x_out;         // particles moved to their stage-k1 positions
    double* logV;         // level table (m - 1)
    uint32_t* thr;        // threshold table (m - 1)
    double* part;         // per-tile estimate partials, (2 + 4D) doubles each
    float* dbg_x;
    float* dbg_lw;
    int32_t* dbg_anc;
    // fully adapted scheme (R17/R18; modes below)
    float* lw_out;          // kPass1Weigh: log-weights lw = carry + log g (N fp32)
    const float* lw_in;     // kPass1Resample: the same log-weights, read back
    int carry_mode;         // 0 none, 1 particle carry lw_prev[i] - c, 2 block carry lvl[g >> shift] - c
    const float* carry_lw;  // previous step's lw (carry_mode 1)
    const double* carry_lv; // previous step's level-S* values (carry_mode 2)
    uint32_t carry_shift;   // block index of group g: (g >> carry_shift) & carry_mask (carry_mode 2)
    uint32_t carry_mask;
    uint32_t out_rot;       // stage rotation (R23): the tile is written to the next layout,
                            // group g -> rotr_S(g, out_rot); 0 = no move (needs M >= 4)
    double carry_c;         // log V_S of the previous step
    double* ess_part;       // kPass1Weigh: per tile {max lw, sum e^{lw-max}, sum e^{2(lw-max)}}
    unsigned int* ess_lmax; // kPass1Weigh: running max of lw (order-preserving float bits)
    // AIRPF (kPass1Airpf; R19-R21)
    const int32_t* isl_src; // previous step's island map A_isl (group g reads block isl_src[g]); null = identity
    double* logW;           // log island means (m)
};

// Order-preserving map of float bits to unsigned (atomicMax of floats).
__host__ __device__ inline unsigned int float_order_bits(float f) {
#ifdef __CUDA_ARCH__
    const unsigned int u = __float_as_uint(f);
#else
    unsigned int u;
    memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// k_pass1 modes: the fused step (mutate, weight, stages 1..k1, tile written moved) or the
// two halves of a fully adapted step, which must know every ESS before its first draw:
//   kPass1Weigh    mutate, weight (+ carried weight), V levels 1..k1 and thresholds,
//                  estimate and ESS partials; writes x_n (natural order) and lw
//   kPass1Resample stage 1 and stages 2..k1 from x_n and lw (no mutation, no weighting)
constexpr int kPass1Fused = 0;
constexpr int kPass1Weigh = 1;
constexpr int kPass1Resample = 2;
//   kPass1Airpf    AIRPF (Alg. 4): mutate the island blocks named by the previous island
//                  map, weight, within-island resample (Alg. 5: pool = the island's M
//                  particles, WITHIN draws), island log-means, island levels 1..k1 and the
//                  island side thresholds (31-bit, R20); writes the within-resampled
//                  sample in natural order (the island stages run in k_island_*)
constexpr int kPass1Airpf = 3;


// ---- k_stages (pf_stages.cuh)
struct StageArgs {
    Key key;
    uint32_t n;
    uint64_t N;     // particles of this shard
    uint32_t pos0;  // global index of the shard's first particle (RNG counters)
    uint32_t m, M, b, s0, k, P, lowbits;
    uint32_t kd;          // stages drawn, s0 .. s0+kd-1 (<= k, the tile depth; < k for a pass an
                          // early-stopped adaptive step truncates: the tile keeps the plan's depth)
    uint32_t pipe;        // 2: warp-specialised (k_stages_ws); 1: software-pipelined (two buffers
                          // of everything); 0: one buffer
    uint32_t out_rot;     // stage rotation (R23): outputs go to group rotr_S(g, out_rot)
    uint32_t out_S;       //   of the next layout (0: no move; needs M >= 4)
    uint32_t ws_walkers;  // k_stages_ws: walker threads (the rest of the CTA draws)
    uint32_t spec;        // 1: a compile-time (k, b) instance of k_stages_ws may run (k_stages_wsc)
    const void* pin;      // states at stage s0-1 (packed AoS, shard-local)
    void* pout;           // states at stage s0+k-1
    const uint32_t* thr;  // side thresholds, level-table layout (level_offset)
    int32_t* dbg_anc;     // per-stage ancestor tables (debug) or nullptr
};

// Shared memory: two tile-state buffers, two table sets (tile t-1 is walked while tile t
// is drawn), two threshold copies, two mbarriers; one of each when not pipelined.
__host__ __device__ inline uint32_t stages_smem(uint32_t P, uint32_t state_bytes, uint32_t k, uint32_t tb,
                                                uint32_t pipe = 1u) {
    const uint32_t st = (P * state_bytes + 15u) & ~15u;
    const uint32_t tab = (k * P * tb + 15u) & ~15u;
    const uint32_t nb = pipe ? 2u : 1u;
    return nb * (st + tab + 4u * (1u << k)) + (pipe == 2u ? 64u : 16u);
}


// ---- k_init, k_cascade, next rows, sharded runs (pf_kernels.cuh, pf_inst_misc.cu)
constexpr int kCascadeThreads = 1024;

struct InitArgs {
    ModelParams mp;
    Key key;
    uint64_t N;     // particles of this shard
    uint32_t pos0;  // global index of its first particle (multiple of 4)
    float* x;
};

struct CascadeArgs {
    double* logV;
    uint32_t* thr;
    const double* part;  // NT tile partials
    double* scratch;     // >= NT + 2 partials (tree levels)
    double* est;         // outputs: filter[2D], predict[2D] (single shard)
    double* shard_rec;   // sharded runs: {log V at level S (= S_loc), root partial[2+4D]}
    uint32_t* ticket;
    uint64_t N;
    uint32_t m, S, k1, b, NT, LPC;
};

constexpr uint32_t kEssChunk = 4096;
constexpr int kEssThreads = 256;

struct EssArgs {
    const double* lv0;       // AIRPF2: level 0 = the m island log-weights (R26); null: the tile partials
    const double* ess_part;  // NT x 3
    const double* logV;      // level table (m - 1)
    unsigned int* lmax;      // running max of lw (float_order_bits), reset by k_ess_final
    double* chunks;          // 2 per chunk
    double* out;             // E_0..E_S, S*, log V_S
    uint64_t N;
    uint32_t NT, m, S;
    double theta;
};

__host__ __device__ inline uint32_t ess_level_count(const EssArgs& a, uint32_t s) {
    return s == 0 ? (a.lv0 ? a.m : a.NT) : (a.m >> s);
}
__host__ __device__ inline uint32_t ess_chunks_total(const EssArgs& a) {
    uint32_t t = 0;
    for (uint32_t s = 0; s <= a.S; ++s) t += (ess_level_count(a, s) + kEssChunk - 1) / kEssChunk;
    return t;
}

struct IslandArgs {
    Key key;
    uint32_t n, m, S;      // m: islands of this shard; S: the stages to draw (local ones when sharded)
    uint32_t island0;      // global index of the shard's first island (draw counters, map values)
    int modified;
    const uint32_t* thr;   // side thresholds, level-table layout (stage s at level_offset(m, s))
    uint8_t* choice;       // S x nq nibbles (nq = ceil(m / 4))
    int32_t* A;            // m: island map
};

// Cross island stage t of a sharded AIRPF step (R27): island i of this shard (global
// island0 + i) and island i of the partner shard rank ^ 2^{t-1} draw their sides with the
// top threshold; Alg. 7's rule sees both draws; A_own[i] <- A_par[i] when i takes.
struct IslandCrossArgs {
    Key key;
    uint32_t n, s, m, island0, rank, t;
    int modified;
    const uint32_t* thr;   // the stage's top threshold (31-bit, R20)
    int32_t* A;            // this shard's island map (global block ids), updated in place
    const int32_t* Apar;   // the partner's map
    uint8_t* choice;       // the stage's choice nibbles (debug table row) or nullptr
};

constexpr uint32_t kMnTile = 1024;  // particles per CDF tile (one CTA of 1024 threads)

struct MultinomialArgs {
    Key key;
    uint32_t n, NT;              // NT: CDF tiles of kMnTile particles
    uint64_t N;
    float* cdf;                  // N: per-tile local CDFs
    float* cdf32;                // N / 32: the local CDF at every 32nd particle (chunk ends)
    double* trec;                // NT x {tile max, tile total}
    double* off;                 // NT + 1: tile offsets in the global CDF, off[NT] = C
    const unsigned int* lmax;    // max lw (order-preserving bits; from the weigh pass)
    const float* x;              // x_n (N x d)
    float* xhat;                 // x_hat_n (N x d)
    int32_t* dbg_anc;            // ancestors (debug) or nullptr
};

struct TopArgs {
    const double* recs;  // G x (1 + PS)
    double* top_logV;    // G - 1
    uint32_t* top_thr;   // G - 1
    double* est;
    double* scratch;     // >= 2 G partials
    uint64_t Nglobal;
    uint32_t G, L, b;
};

struct CrossArgs {
    Key key;
    uint32_t n, s, t, rank, b, M;
    uint64_t Nloc;
    uint32_t pos0, pos0_partner;
    const uint32_t* thr;    // the stage threshold (device): top_thr entry of block rank >> t
    const void* own_in;
    const void* partner_in;
    void* out;
    int32_t* dbg_anc;       // this shard's stage tables (global source positions)
};

struct PullArgs {
    Key key;
    uint32_t n, S_loc, L, rank, b, M;
    uint64_t Nloc;
    const uint32_t* top_thr;  // G - 1 top thresholds (top level t at G - (G >> (t-1)))
    uint32_t G;
    uint32_t* src_local;      // Nloc: local position of the source on its owner
    uint32_t* src_rank;       // Nloc: owner rank
    unsigned long long* counts;  // G: requests per owner rank
    uint32_t* fill;           // G: slots used (pack)
    const unsigned long long* offsets;  // G: start of each owner's requests (pack)
    uint32_t* req;            // Nloc: requests grouped by owner rank
    uint32_t* outpos;         // Nloc: request slot of output l (where its state arrives)
    int32_t* dbg_anc;         // stage tables (debug) or nullptr
};

// Relabelled exchange of one cross stage (pf_relabel_begin / pf_relabel_end; DESIGN.md
// reading R24).  Shard r pairs with r' = r ^ 2^{t-1} at stage s = S_loc + t;
// both ranks evaluate both shards' counter-based draws, so each knows the two ordered lists
//   own  = this shard's outputs whose draw lies in r'      (positions, increasing)
//   par  = r''s outputs whose draw lies in r               (their sources in r, in order)
// without communication; the k-th entries of the lists swap draws for k < min, and only the
// surplus crosses the pair.
constexpr uint32_t kRlChunk = 2048;   // positions per counting chunk (512 quads, one CTA)
struct RelabelArgs {
    Key key;
    uint32_t n, s, b, M;
    uint64_t Nloc;
    uint32_t rank, partner, own_is_low;
    const uint32_t* thr;         // the stage's side threshold (top_thr entry of block rank >> t)
    uint32_t nchunks;
    uint32_t* cnt;               // 2 x nchunks: per chunk {own wanting r', r' wanting own}
    uint32_t* off;               // 2 x nchunks + 2: exclusive offsets, then the totals
    uint32_t* own;               // Nloc: list own
    uint32_t* par;               // Nloc: list par (local source index in this shard)
    uint32_t* kidx;              // Nloc: the rank of an own output in list own (valid where it wants r')
    const void* x;               // stage s-1 states of this shard (Nloc x d)
    void* out;                   // stage s states
    void* send;                  // packed surplus this rank sends (par[k], k >= kmin)
    const void* recv;            // surplus received (own[k], k >= kmin)
    uint64_t kmin, nsend;
    int32_t* dbg_anc;            // this stage's table (global source positions) or nullptr
};

// Peer-memory exchange (pf_cross_peer): every rank's stage-S_loc state buffer, mapped into
// this process (CUDA IPC over NVLink, or local pointers for shards on one GPU).
constexpr uint32_t kPeerMaxG = 64;
struct PeerArgs {
    const float* x[kPeerMaxG];  // x[r] = rank r's X(cur), Nloc x d fp32
    float* out;                 // this shard's x_hat (X(cur ^ 1))
};

}  // namespace pfk
