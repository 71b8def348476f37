/*
 * pf.h -- C-ABI of the B200-native bootstrap particle filter step with augmented
 * resampling (arXiv 1812.01502, Heine, Whiteley and Cemgil).
 *
 * The method (PAPER.md line numbers; DESIGN.md §1-§3 for the readings):
 *   - HMM  X_0 ~ pi_0, X_n | X_{n-1} ~ f, Y_n | X_n ~ g            (eq. HMM)
 *   - Alg. 1 (BPF): mutate, then RESAMPLE with potentials g_n(.) = g(., y_n)
 *
 *   - Alg. 3 (augmented resampling) with A_s of eq. `A matrices`: N = m M particles in
 *     m = 2^S groups of M; at stage s = 1..S group g is paired with g XOR 2^{s-1}
 *     and each particle redraws its ancestor from the pair's 2M particles with
 *     probability A_s^{ij} V_{s-1}^j / V_s^i
 *
 * One pf_step(y_n) = [mutate x_hat_{n-1} -> x_n (n >= 1)] + weight g_n + S butterfly
 * stages + composition of the stage ancestors, leaving x_hat_n on the device.
 *
 * Conventions (all calls):
 *   - Return value: PF_OK (0) or a negative PF_E* code; pf_last_error() describes it.
 *     No C++ exception crosses this ABI.
 *   - "host" pointers are read (or written) before the call returns; "device"
 *     pointers must stay valid until the work enqueued on the handle's stream is done.
 *   - The library never allocates device memory: the caller passes one device
 *     workspace of pf_workspace_bytes() bytes (256-byte aligned), and a CUDA stream.
 *   - Determinism: the same (model, N, M, seed, flags, y_0..y_n) give bitwise
 *     identical results (counter-based RNG, fixed reduction trees).
 */
#ifndef PF_H_
#define PF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PF_OK 0
#define PF_EINVAL (-1)     /* bad topology / model / argument */
#define PF_EWORKSPACE (-2) /* workspace too small or misaligned */
#define PF_ECUDA (-3)      /* a CUDA runtime error (message in pf_last_error) */
#define PF_EOBS (-4)       /* non-finite observation */
#define PF_ESTATE (-5)     /* call not valid in the current state (e.g. no step yet) */

/* model kinds */
#define PF_LG 1 /* x_n = A x_{n-1} + LQ z,  y_n = H x_n + N(0, R),  x_0 = m0 + L0 z */
#define PF_SV 2 /* x_n = phi x_{n-1} + sigma z, y_n = beta exp(x_n/2) N(0,1), x_0 = sv_m0 + sv_s0 z */

/* Model description (HOST pointers, copied by pf_init; the caller keeps ownership).
 * All matrices row-major fp32: A, LQ, L0 are d x d (LQ, L0 lower Cholesky factors of
 * Q and P0), H is dy x d, Rinv is dy x dy (R^{-1}), m0 has d entries.  d, dy in 1..8.
 * PF_SV uses only the sv_* scalars (d = dy = 1).  The oracle widens the same fp32
 * values to fp64. */
typedef struct pf_model {
    int kind;
    int d, dy;
    const float *A, *LQ, *H, *Rinv, *m0, *L0;
    float sv_phi, sv_sigma, sv_beta, sv_m0, sv_s0;
} pf_model;

typedef struct pf_handle pf_handle;

/* pf_init flags */
#define PF_FLAG_DEBUG 1u /* keep x_n, log-weights and every stage's ancestor table
                            (S x N int32) for pf_debug_get; test-only, costs HBM */
#define PF_FLAG_ADAPTIVE 2u /* reserve the buffers of the fully adapted scheme
                               (pf_set_adaptive; one GPU only): 8 N + 4 N/M + O(N/1024) bytes */

#define PF_FLAG_MULTINOMIAL 8u /* reserve the buffers of multinomial resampling (pf_set_multinomial;
                                   one GPU): 8 N bytes + O(N/1024) */
#define PF_FLAG_AIRPF 4u /* reserve the island buffers of AIRPF (pf_set_airpf; one GPU, M >= 4):
                            13 N/M + S N/(4M) bytes */
#define PF_FLAG_GUARD 16u /* checking aid: a PF_GUARD_BYTES gap after every workspace region
                            (fill the workspace before pf_init; pf_guard_check counts the gap
                            bytes a step overwrote) */
#define PF_GUARD_BYTES 4096

/* Bytes of device workspace pf_init needs for this problem (0 if invalid). */
size_t pf_workspace_bytes(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags);

/* Validate and set up one filter on the current CUDA device, and enqueue the draw of
 * x_0^i ~ pi_0 (Alg. 1 l.1-3) on `cuda_stream` (a cudaStream_t; NULL
 * = legacy default stream).
 * Topology (Assumption A1; reading R5): m = N/M must be an
 * integer power of two with m >= 2 (S = log2 m >= 1); M must be a power of two in
 * [2, 8192] and a stage-1 pool of 2M particles must fit one SM's shared memory
 * (2M (4d + 5) bytes <= 227 KB: M <= 8192 for d = 1, M <= 4096 for d = 4);
 * N < 2^31; d in {1, 2, 4, 8}.  Errors: PF_EINVAL, PF_EWORKSPACE, PF_ECUDA.
 * dev_ws: DEVICE pointer, >= pf_workspace_bytes(), 256-byte aligned, owned by the
 * caller and not touched by anyone else until pf_destroy. */
int pf_init(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags,
            void* dev_ws, size_t ws_bytes, void* cuda_stream, pf_handle** out);

/* Enqueue one time step n (n = 0, 1, 2, ... counted by the handle) with observation
 * y_n (HOST pointer, dy floats, copied into the launch parameters before return).
 * n = 0 weights and resamples x_0 (no mutation); n >= 1 first mutates x_hat_{n-1}
 * (reading R7).  Asynchronous.  Errors: PF_EOBS (non-finite y), PF_ECUDA. */
int pf_step(pf_handle* h, const float* y_host);

/* Same as pf_step with y_n read by the kernels from DEVICE memory (dy floats), so a
 * caller can keep the whole observation sequence resident in HBM.  Non-finite
 * device observations are not detected. */
int pf_step_dev(pf_handle* h, const float* y_dev);

/* T consecutive steps in one call (no per-step host round trip through the binding):
 * step k reads observation k from y_dev (DEVICE, T x dy fp32, contiguous).  est_dev
 * (DEVICE, T x 4 x d fp64, or NULL) receives after step k the rows filter x, filter x^2,
 * predictive x, predictive x^2 of that step.  Asynchronous on
 * the handle's stream except where a step itself synchronises (the fully adapted
 * scheme reads S* back).  Errors as pf_step_dev; steps before a failing one stay done. */
int pf_run_dev(pf_handle* h, const float* y_dev, uint32_t T, double* est_dev);

/* The same T steps captured into one CUDA graph, launched later by pf_graph_launch (one
 * launch; the graph is freed after it).  The handle's state advances at capture (as if
 * the steps had run), so pf_graph_launch must follow before any other step, estimate or
 * debug read.  For small problems whose step is a few microsecond-long kernels, the graph
 * removes the per-launch gaps.  Not for the fully adapted scheme (it synchronises) or
 * sharded handles; the handle's stream must not be the legacy default stream (capture).
 * Errors: PF_EINVAL, PF_ESTATE (adaptive, sharded, graph pending, default stream),
 * PF_ECUDA. */
int pf_graph_capture(pf_handle* h, const float* y_dev, uint32_t T, double* est_dev);
int pf_graph_launch(pf_handle* h);

/* --- fully adapted augmented resampling (AIRPF2) ---
 * With theta in (0, 1], every later pf_step evaluates the ESS of the stage weights
 *   E_s = (N^-1 sum_i V_s^i)^2 / (N^-1 sum_i (V_s^i)^2),  s = 0 (V_0 = the weights), 1..S
 * (reading R17) after weighting -- every V_s is known then --
 * and runs stages 1..S* only, S* = min{s : E_s >= theta} (stage s+1 runs iff E_s < theta;
 * S* <= S since E_S = 1).  The particles then carry the weights V_{S*} into the next
 * step (reading R18); with S* = S nothing is carried and the step equals pf_step's.
 * theta = 0 switches back to the plain step (the carried weights are dropped).
 * Needs a handle created with PF_FLAG_ADAPTIVE and world = 1.  pf_step synchronises the
 * stream once per step (the host reads S* to launch only the passes it needs).
 * Errors: PF_EINVAL (theta outside [0, 1], no PF_FLAG_ADAPTIVE, sharded handle). */
int pf_set_adaptive(pf_handle* h, double theta);

/* S* of the last completed step (S for a plain step), or -1 before the first step. */
int pf_last_stages(const pf_handle* h);

/* Stage rotation with the fully adapted scheme: on != 0 makes every later
 * adaptive step start at the stage after the last one executed.  Realised as a group
 * relabelling (reading R23): the states live in a layout whose group index is
 * rotr_S(g, rho); a step that ran S* >= 1 stages writes its outputs to the next layout
 * (rho += S*).  Estimates are unaffected; debug tables of a step are in its own layout and
 * x_hat in the next one.  Needs PF_FLAG_ADAPTIVE and M >= 4.  Errors: PF_EINVAL. */
int pf_set_rotation(pf_handle* h, int on);

/* Current rotation offset rho (0 without rotation), or -1 for NULL. */
int pf_rotation_offset(const pf_handle* h);

/* --- AIRPF: augmented island resampling particle filter (Alg. 4) ---
 * mode 1: Alg. 4 with the within-island resample (Alg. 5) and the modified augmented
 * island resampling (Alg. 7: pure pairwise exchanges undone); mode 2: with Alg. 6; 0: back
 * to Alg. 1 + Alg. 3 (pf_step).  Each later pf_step mutates the island blocks named by the
 * previous step's island map, weights, resamples every island within itself (pool of M,
 * R19) and composes the S island stages over whole blocks of M (R20, R21); pf_estimate
 * gives the same estimates as for pf_step (before resampling).  Needs a handle created
 * with PF_FLAG_AIRPF, world = 1, M >= 4.
 * AIRPF2 ("AIRPF with the fully adapted resampling scheme"; DESIGN.md
 * reading R26): with pf_set_adaptive(theta > 0) as well (handle created with
 * PF_FLAG_AIRPF | PF_FLAG_ADAPTIVE), the within-island resample runs every step and the
 * island stages run only up to S* = min{s : E_s >= theta}, E_0 the ESS of the m island
 * weights, E_s of the level-s island block weights; the islands then carry V_bar_{S*}
 * (S* = 0: their own island weight) into the next step.  pf_step synchronises once (S*).
 * Errors: PF_EINVAL; PF_ESTATE when switching while weights are carried. */
int pf_set_airpf(pf_handle* h, int mode);

/* --- plain BPF: multinomial resampling (Alg. 2) -------------------
 * on != 0: every later pf_step resamples the N particles multinomially over the whole
 * population (reading R22: inverse CDF in ascending order, MULTI draws) instead of running
 * the butterfly stages -- the paper's baseline, for comparison.  The draw searches a global
 * CDF (fp32 per 1024-particle tile, fp64 tile offsets) and gathers the states at random.
 * Needs PF_FLAG_MULTINOMIAL, world = 1; exclusive with the other schemes.  PF_DBG_ANC_FINAL
 * returns the drawn ancestors (debug handles).  Errors: PF_EINVAL. */
int pf_set_multinomial(pf_handle* h, int on);

/* estimates (phi) */
#define PF_PHI_X 1  /* phi(x) = x_k, k = 0..d-1 */
#define PF_PHI_X2 2 /* phi(x) = x_k^2 */
/* estimate kinds (reading R8) */
#define PF_EST_FILTER 1  /* sum_i g_n(x^i) phi(x^i) / sum_i g_n(x^i): pi_hat_n */
#define PF_EST_PREDICT 2 /* N^-1 sum_i phi(x^i): pi_n^N */
#define PF_EST_RESAMPLED 3 /* N^-1 sum_i phi(x_hat^i): the empirical measure of the resampled
                              sample, pi_hat_n^N; evaluated on demand from the
                              step's output (through the island map after an AIRPF step; after
                              an early-stopped adaptive step, of the S*-stage sample).  Sharded
                              handles: the mean over THIS shard's N/G particles (shards are
                              equally sized; dist.py averages them in rank order) */

/* Synchronise the handle's stream and write the d estimates of the last completed
 * step into out (HOST, d doubles).  FILTER and PREDICT are computed by the step itself;
 * RESAMPLED launches k_moments + k_moments_final over x_hat first (fixed order,
 * deterministic).  Errors: PF_ESTATE before the first step, PF_EINVAL, PF_ECUDA. */
int pf_estimate(pf_handle* h, int phi, int kind, double* out);

/* Release the handle (not the workspace, not the stream). NULL is a no-op. */
void pf_destroy(pf_handle* h);

/* Human-readable description of the last error on h (or of the last failed pf_init
 * when h is NULL).  Valid until the next call on h. */
const char* pf_last_error(const pf_handle* h);

/* --- sharded step over G GPUs -------------------
 * Shard r of G (G a power of two) owns particles [r N/G, (r+1) N/G), i.e. groups
 * [r m/G, (r+1) m/G); every RNG counter uses the GLOBAL particle index, so a sharded run
 * draws exactly the numbers of a single-GPU run.  One time step is the collective sequence
 *   pf_step_local        mutate, weight, stages 1..S - log2 G (all local), shard record
 *   <allgather the G shard records, rank order>          (caller's transport, e.g. NCCL)
 *   pf_step_top          top V levels, cross thresholds, global estimate (same on all)
 *   for t = 1..log2 G:   <exchange pf_cross_buffer with partner rank ^ 2^(t-1)>
 *                        pf_cross_stage(t, partner's buffer)   (stage S - log2 G + t)
 * Every call is stream-ordered on the handle's stream; the caller's transport must order
 * its copies on (or after) that stream. */
#define PF_SHARD_REC_DOUBLES(d) (3 + 4 * (d)) /* {log V_{S_loc}, partial[2 + 4d]} */

/* Workspace bytes for one shard (0 if invalid). */
size_t pf_workspace_bytes_sharded(const pf_model* model, uint64_t N, uint32_t M, uint32_t flags, int world);

/* Like pf_init for shard `rank` of `world`; N is the GLOBAL particle count.  Needs m/world
 * >= 2.  Errors as pf_init.  Sharded handles use the state-moving passes (no gather). */
int pf_init_sharded(const pf_model* model, uint64_t N, uint32_t M, uint64_t seed, uint32_t flags, int rank,
                    int world, void* dev_ws, size_t ws_bytes, void* cuda_stream, pf_handle** out);

/* Local phase of one step; y as in pf_step (y_host) or pf_step_dev (y_dev): give one. */
int pf_step_local(pf_handle* h, const float* y_host, const float* y_dev);

/* pf_step_local in two halves, so that the records' all-gather overlaps the local stage
 * passes: _begin enqueues k_pass1 + k_cascade (after which this shard's record and every
 * local V level are final: each V_s is sigma(xi_0)-measurable, Lemma facts_about_Vs (a),
 * PAPER.md:645); _end enqueues the k_stages passes.  pf_shard_record is valid after
 * _begin; pf_step_top may run before or after _end (it touches only the top tables);
 * the cross exchange must follow _end.  Sharded handles, plain scheme only.
 * Errors: PF_EINVAL, PF_EOBS, PF_ESTATE (not sharded; _end without _begin; _begin twice). */
int pf_step_local_begin(pf_handle* h, const float* y_host, const float* y_dev);
int pf_step_local_end(pf_handle* h);

/* DEVICE pointer of this shard's record (PF_SHARD_REC_DOUBLES(d) doubles), valid after
 * pf_step_local has run on the stream. */
int pf_shard_record(pf_handle* h, const double** dev_rec);

/* Top levels from all G records (DEVICE, G * PF_SHARD_REC_DOUBLES(d), rank order).
 * Afterwards pf_estimate returns the global estimate. */
int pf_step_top(pf_handle* h, const double* dev_all_recs);

/* DEVICE pointer and size of this shard's current state buffer (send it to the partner
 * of the next cross stage).  Valid until the next pf_cross_stage on this handle. */
int pf_cross_buffer(pf_handle* h, const void** dev_states, size_t* bytes);

/* Cross stage t (1..log2 G): assemble this shard's stage-(S_loc + t) states from its own
 * and the partner's (DEVICE, pf_cross_buffer of rank ^ 2^(t-1)) stage-(S_loc + t - 1)
 * states.  Asynchronous. */
int pf_cross_stage(pf_handle* h, int t, const void* dev_partner_states);

/* Pull exchange: the L cross stages in one all-to-all instead of L pairwise rounds.
 * Every output composes its L cross-stage draws (counter-based; the thresholds are known
 * after pf_step_top) into the (owner rank, local position) of its stage-S_loc source.
 * Sequence on every rank, after pf_step_top:
 *   pf_cross_pull_plan(h, counts)        counts[r] = how many of my outputs read rank r
 *                                        (HOST, G uint64; synchronises)
 *   <exchange counts: all-to-all>        -> how many of my states each rank requests
 *   pf_cross_pull_pack(h, offsets, &req) offsets = exclusive prefix of counts (HOST);
 *                                        req = DEVICE uint32 local positions grouped by owner
 *   <all-to-all of req with splits counts / received counts>
 *   pf_cross_pull_serve(h, req_in, n, &states)  gathers the n requested stage-S_loc states
 *                                        (DEVICE, n x d fp32, request order); n <= N
 *   <all-to-all of states back>          -> N/G states grouped by owner, in my request order
 *   pf_cross_pull_finish(h, states_in)   scatters them to their outputs: x_hat of the shard
 * Gives bitwise the x_hat of the pairwise rounds (pf_cross_stage).  Errors: PF_EINVAL,
 * PF_ESTATE (not sharded / before pf_step_top), PF_ECUDA. */
int pf_cross_pull_plan(pf_handle* h, uint64_t* host_counts);
int pf_cross_pull_pack(pf_handle* h, const uint64_t* host_offsets, const uint32_t** dev_requests);
int pf_cross_pull_serve(pf_handle* h, const uint32_t* dev_requests_in, uint64_t n, const void** dev_states);
int pf_cross_pull_finish(pf_handle* h, const void* dev_states_in);

/* Peer-memory exchange: the L cross stages as ONE kernel that composes every output's
 * (owner rank, local position) as the pull exchange does and reads that state straight
 * from the owner's workspace over NVLink (P2P loads through CUDA IPC mappings) into this
 * shard's x_hat.  No request/reply round, no host synchronisation.
 *   pf_peer_export(h, handle, &offset)  handle: HOST, PF_IPC_HANDLE_BYTES bytes (the CUDA
 *                                       IPC handle of the allocation that holds this
 *                                       workspace); offset: the workspace's offset in it
 *   <all-gather of (handle, offset)>    (once, at set-up)
 *   pf_peer_open(h, handles, offsets)   HOST, world x PF_IPC_HANDLE_BYTES / world uint64
 *                                       in rank order; maps every other rank's workspace
 *                                       (closed by pf_destroy)
 *   pf_peer_set(h, workspaces)          instead of export/open when every rank's workspace
 *                                       is already addressable here (shards on one GPU):
 *                                       HOST, world uint64 DEVICE addresses, [rank] = own
 *   per step, after pf_step_top:  pf_cross_peer(h)  <device barrier>
 * Ordering is the caller's: every rank's stage-S_loc states must be complete before any
 * rank reads them (the all-gather of the shard records that precedes pf_step_top gives
 * this when it is stream-ordered, as NCCL's is), and no rank may start its next step
 * before every rank has read them (the barrier: e.g. a 1-element NCCL all-reduce
 * enqueued on the handle's stream).
 * Gives bitwise the x_hat of the pull exchange and of the pairwise rounds.
 * Errors: PF_EINVAL, PF_ESTATE (not sharded, before pf_step_top, no mapping), PF_ECUDA. */
#define PF_IPC_HANDLE_BYTES 64
int pf_peer_export(pf_handle* h, void* ipc_handle, uint64_t* offset);
int pf_peer_open(pf_handle* h, const void* ipc_handles, const uint64_t* offsets);
int pf_peer_set(pf_handle* h, const uint64_t* dev_workspaces);
int pf_cross_peer(pf_handle* h);

/* Sharded AIRPF (Alg. 4 over G GPUs with whole-block moves; reading R27): a
 * handle created with PF_FLAG_AIRPF on world > 1 (m / world a multiple of 4) runs, in
 * pf_step_local, the AIRPF pass (its island blocks read from their owners through the
 * peer mapping: pf_peer_open / pf_peer_set first), the cascade and the local island
 * stages; after pf_step_top (31-bit island thresholds), every cross island stage t = 1..L
 * exchanges the island maps with partner rank ^ 2^{t-1}:
 *   pf_island_map(h, &map)           DEVICE, m / world int32: this shard's island map
 *                                    (global block ids; send it to the partner)
 *   pf_island_cross(h, t, partner)   DEVICE, the partner's map: island i takes the partner
 *                                    island's entry when it draws the partner's side, except
 *                                    a pure exchange under Alg. 7 (mode 1)
 * Only block ids move; the states cross NVLink once, when the next step reads a remote
 * block (a contiguous M x d run).  Bitwise the one-GPU AIRPF step (global counters and
 * the one-GPU operand order).  Errors: PF_EINVAL, PF_ESTATE (not sharded, no AIRPF step,
 * before pf_step_top), PF_ECUDA. */
int pf_island_map(pf_handle* h, const int32_t** dev_map);
int pf_island_cross(pf_handle* h, int t, const int32_t* dev_partner_map);

/* Relabelled exchange of cross stage t (1..L), the BPF variant of SURVEY.md §8(f)3 (the
 * count-imbalance / surplus sketch of PAPER.md:826-850; reading R24).  Every
 * output first takes its Alg. 3 draw of stage s = S_loc + t (pairing shard r with
 * r' = r ^ 2^{t-1}); the k-th output of r that drew from r' and the k-th output of r'
 * that drew from r (both in increasing position) exchange draws for k < min of the two
 * counts, so each reads its own shard, and only the surplus crosses the pair.  Both
 * ranks evaluate both shards' counter-based draws, so the lists need no communication;
 * the output is NOT bitwise the plain exchange's (a permutation within the pair block,
 * on which V_s is constant: Prop. 1 unbiasedness is kept, pinned by the oracle's
 * orc_relabel_stage).  Per stage, on every rank of the pair, after pf_step_top:
 *   pf_relabel_begin(h, t, counts, &send, &n_send, &n_recv)
 *       counts: HOST uint64[2] = {own outputs drawing from r', r' outputs drawing from r};
 *       send: DEVICE, n_send states (n_send x d fp32, the handle's workspace, valid until
 *       the next call) this rank sends to r'; n_recv: states to receive from r'.
 *       Synchronises once (the counts size the transfer).
 *   <send n_send states to r', receive n_recv from r' into a DEVICE buffer>
 *   pf_relabel_end(h, t, recv)   recv: DEVICE, n_recv x d fp32 (NULL if n_recv = 0)
 * Errors: PF_EINVAL (t out of range, NULL), PF_ESTATE (not sharded, before pf_step_top,
 * end without begin), PF_ECUDA. */
int pf_relabel_begin(pf_handle* h, int t, uint64_t* host_counts, const void** dev_send, uint64_t* n_send,
                     uint64_t* n_recv);
int pf_relabel_end(pf_handle* h, int t, const void* dev_recv);

/* PF_FLAG_GUARD handles: count the bytes of the inter-region gaps that differ from
 * `fill` (the byte the caller filled the workspace with before pf_init).  A nonzero
 * count means some kernel wrote outside its region.  Synchronises.  Errors: PF_EINVAL,
 * PF_ESTATE (no PF_FLAG_GUARD), PF_ECUDA. */
int pf_guard_check(pf_handle* h, unsigned char fill, uint64_t* bad_bytes);

/* --- debug / test exports (parity harness) ------------------------------------ */
#define PF_DBG_X 1         /* x_n before resampling, N x d fp32 (needs PF_FLAG_DEBUG) */
#define PF_DBG_LOGW 2      /* log g_n(x_n^i), N fp32 (needs PF_FLAG_DEBUG) */
#define PF_DBG_ANC_STAGE 3 /* a_s(i), N int32, stage = s in 1..S (needs PF_FLAG_DEBUG) */
#define PF_DBG_ANC_FINAL 4 /* A(i) = a_1(...a_S(i)), N int32 (needs PF_FLAG_DEBUG) */
#define PF_DBG_XHAT 5      /* x_hat_n = x_n[A(i)], N x d fp32; before the first step: x_0 of
                              pf_init (Alg. 1 l.1-3) */
#define PF_DBG_LOGV 6      /* log V_s per block, all levels s = 1..S, m-1 fp64
                              (level s at offset m - m/2^{s-1}, m/2^s entries) */
#define PF_DBG_ESS 8       /* E_0..E_S of the last adaptive step, S+1 fp64 (PF_FLAG_ADAPTIVE) */
#define PF_DBG_ISLAND_A 9  /* AIRPF island map A_isl (block held by island g), m int32 */
#define PF_DBG_ISLAND_CHOICE 10 /* AIRPF stage-s choices: ceil(m/4) bytes, bit e of byte q set =
                                   island 4q+e took its partner's block (after Alg. 7's rule) */
#define PF_DBG_ISLAND_LOGW 11   /* AIRPF log island means (W_out of Alg. 5), m fp64 */
#define PF_DBG_THRESH 7    /* stage s >= 2 side thresholds floor(p 2^{32-b}), m-1 uint32,
                              same layout (stage s at offset m - m/2^{s-1}); entry 0.. of
                              level 1 unused */

/* Copy one debug table of the last completed step to HOST memory (bytes = capacity of
 * host_out).  Synchronises.  Errors: PF_ESTATE (no step / not in debug mode), PF_EINVAL. */
int pf_debug_get(pf_handle* h, int what, int stage, void* host_out, size_t bytes);

/* DEVICE pointer of a debug table (same `what`/`stage`), for on-device sampling of
 * large tables; valid until the next pf_step.  PF_DBG_XHAT is materialised on demand. */
int pf_debug_ptr(pf_handle* h, int what, int stage, void** dev_out);

/* Replace the filter state: the next pf_step is time step n and starts from
 * x_hat_{n-1} = host_xhat (N x d fp32, HOST) -- or from x_0 = host_xhat when n = 0.
 * Used by single-step parity tests with seeded synthetic particle clouds. */
int pf_debug_set_state(pf_handle* h, const float* host_xhat, uint32_t n);

/* Number of kernel launches the last pf_step enqueued (bench accounting). */
int pf_last_step_launches(const pf_handle* h);

/* --- kernel timing (bench accounting) ------------------------------------------ */
#define PF_KERNEL_PASS1 0   /* k_pass1: mutate + weight + stages 1..k1 */
#define PF_KERNEL_CASCADE 1 /* k_cascade: V levels, thresholds, estimates */
#define PF_KERNEL_STAGES 2 /* k_stages: stages k1+1..S (S_loc when sharded) */
#define PF_KERNEL_TOP 3     /* k_top: cross-shard V levels and estimate (sharded) */
#define PF_KERNEL_CROSS 4   /* k_cross: one cross-shard stage (sharded) */
#define PF_KERNEL_KINDS 5
/* When on, every pf_step records a CUDA event pair around each of its kernels on the
 * handle's stream.  pf_timing_read synchronises the stream and returns, per kernel kind,
 * the summed device milliseconds (ms[PF_KERNEL_KINDS], HOST) and launch counts
 * (launches[PF_KERNEL_KINDS], HOST, may be NULL) since the last enable or read, then
 * resets them.  Errors: PF_EINVAL, PF_ECUDA. */
int pf_timing_enable(pf_handle* h, int on);
int pf_timing_read(pf_handle* h, double* ms, int* launches);

#ifdef __cplusplus
}
#endif
#endif /* PF_H_ */
