// pf_launch.h -- typed launchers of the step kernels.  Each kernel family is
// instantiated in its own translation unit (pf_inst_*.cu) so the build runs in parallel;
// pf_api.cu (host orchestration) only sees these plain functions.
#pragma once
#include <cuda_runtime.h>

#include "pf_args.h"

namespace pfk {

struct LaunchCfg {
    uint32_t grid, threads, smem;
    cudaStream_t stream;
};

enum StatePayload { kPayloadF1 = 2, kPayloadF2 = 3, kPayloadF4 = 4, kPayloadF8 = 5 };

// 8-float particle state moved as one payload element (d = 8).
struct __align__(16) State8 {
    float4 a, b;
};

void launch_pass1_d1(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d2(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d4(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d8(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_ad_d1(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_ad_d2(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_ad_d4(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_ad_d8(int kind, int tb, bool dbg, int qpt, int mode, const LaunchCfg& c, const Pass1Args& a);
void launch_stages_f1(int tb, bool dbg, int qpt, const LaunchCfg& c, const StageArgs& a);
void launch_stages_f2(int tb, bool dbg, int qpt, const LaunchCfg& c, const StageArgs& a);
void launch_stages_f4(int tb, bool dbg, int qpt, const LaunchCfg& c, const StageArgs& a);
void launch_stages_f8(int tb, bool dbg, int qpt, const LaunchCfg& c, const StageArgs& a);
// Force the (lazily loaded) runtime-plan stage kernels of a payload into the context, so a
// pass the fully adapted scheme truncates (drawn by k_stages_ws / k_stages, not by the
// compile-time instance the full pass uses) does not pay the module load inside a step.
void preload_stages_f1(int tb, bool dbg);
void preload_stages_f2(int tb, bool dbg);
void preload_stages_f4(int tb, bool dbg);
void preload_stages_f8(int tb, bool dbg);
inline void preload_stages(int D, int tb, bool dbg) {
    switch (D) {
        case 1: preload_stages_f1(tb, dbg); break;
        case 2: preload_stages_f2(tb, dbg); break;
        case 4: preload_stages_f4(tb, dbg); break;
        default: preload_stages_f8(tb, dbg); break;
    }
}
inline void launch_stages(int D, int tb, bool dbg, int qpt, const LaunchCfg& c, const StageArgs& a) {
    switch (D) {
        case 1: launch_stages_f1(tb, dbg, qpt, c, a); break;
        case 2: launch_stages_f2(tb, dbg, qpt, c, a); break;
        case 4: launch_stages_f4(tb, dbg, qpt, c, a); break;
        default: launch_stages_f8(tb, dbg, qpt, c, a); break;
    }
}
void launch_cascade(int D, const LaunchCfg& c, const CascadeArgs& a);
void launch_ess(const LaunchCfg& chunks, const EssArgs& a);
void launch_island(cudaStream_t st, const IslandArgs& a);
void launch_pull_compose(cudaStream_t st, const PullArgs& a, bool debug);
void launch_pull_pack(cudaStream_t st, const PullArgs& a);
void launch_guard_check(cudaStream_t st, const unsigned char* p, size_t n, unsigned char fill, unsigned long long* bad);
void launch_peer_gather(cudaStream_t st, int D, const PullArgs& a, const PeerArgs& p, bool debug);
void launch_pull_move(cudaStream_t st, int D, bool gather, const float* src, const uint32_t* idx, float* dst,
                      uint64_t n);
void launch_multinomial(int D, cudaStream_t st, const MultinomialArgs& a, const float* lw);
void launch_block_gather(cudaStream_t st, const float* in, float* out, const int32_t* A, uint64_t N, uint32_t b,
                         uint32_t D);
void launch_init(int D, int kind, const LaunchCfg& c, const InitArgs& a);
void launch_top(int D, const LaunchCfg& c, const TopArgs& a);
void launch_cross(int payload, bool dbg, const LaunchCfg& c, const CrossArgs& a);
constexpr uint32_t kMomPartDoubles = 592u * 2u * 8u;  // k_moments CTA partials (grid x 2 D, D <= 8)
void launch_moments(cudaStream_t st, int D, const float* x, const int32_t* isl, uint32_t b, uint64_t N, double* part,
                    double* out);
void launch_relabel_plan(cudaStream_t st, const RelabelArgs& a);
void launch_relabel_lists(cudaStream_t st, const RelabelArgs& a);
// pack = true: the surplus this rank sends; false: assemble the stage's outputs (nown = |own|)
void launch_relabel_move(cudaStream_t st, int D, const RelabelArgs& a, bool pack, uint64_t nown, bool dbg);
void launch_island_cross(cudaStream_t st, const IslandCrossArgs& a);
void launch_block_gather_peer(cudaStream_t st, const PeerArgs& p, float* out, const int32_t* A, uint64_t N, uint32_t b,
                              uint32_t D, uint32_t shift);
void launch_rows_copy(cudaStream_t st, const double* src, uint32_t sp, double* dst, uint32_t dp, uint32_t rows);
void launch_debug_compose(const LaunchCfg& c, const int32_t* anc, uint64_t N, uint32_t S, int32_t* A);

}  // namespace pfk
