// pf_launch.h -- typed launchers of the step kernels.  Each kernel family is
// instantiated in its own translation unit (pf_inst_*.cu) so the build runs in parallel;
// pf_api.cu (host orchestration) only sees these plain functions.
#pragma once
#include <cuda_runtime.h>

#include "pf_kernels.cuh"

namespace pfk {

struct LaunchCfg {
    uint32_t grid, threads, smem;
    cudaStream_t stream;
};

enum ComposePayload { kPayloadIdent = 0, kPayloadIndex = 1, kPayloadF1 = 2, kPayloadF2 = 3, kPayloadF4 = 4, kPayloadF8 = 5 };

// 8-float particle state moved as one payload element (d = 8).
struct __align__(16) State8 {
    float4 a, b;
};

void launch_pass1_d1(int kind, bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d2(int kind, bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d4(int kind, bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a);
void launch_pass1_d8(int kind, bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a);
void launch_compose_nodbg(int payload, int qpt, const LaunchCfg& c, const ComposeArgs& a);
void launch_compose_dbg(int payload, int qpt, const LaunchCfg& c, const ComposeArgs& a);
void launch_move(int payload, bool dbg, int qpt, const LaunchCfg& c, const ComposeArgs& a);
void launch_cascade(int D, const LaunchCfg& c, const CascadeArgs& a);
void launch_init(int D, int kind, const LaunchCfg& c, const InitArgs& a);
void launch_top(int D, const LaunchCfg& c, const TopArgs& a);
void launch_cross(int payload, bool dbg, const LaunchCfg& c, const CrossArgs& a);
void launch_debug_compose(const LaunchCfg& c, const int32_t* anc, uint64_t N, uint32_t S, int32_t* A);
void launch_gather(int D, const LaunchCfg& c, const float* x, const int32_t* A, uint64_t N, float* out);

}  // namespace pfk
