// Instantiations of k_pass1 for d = 2 (see pf_kernels.cuh).
#include "pf_launch.h"

namespace pfk {
namespace {
template <int KIND, bool GATHER, bool DBG, int QPT>
void go(const LaunchCfg& c, const Pass1Args& a) {
    auto k = k_pass1<2, KIND, GATHER, DBG, QPT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
    k<<<c.grid, c.threads, c.smem, c.stream>>>(a);
}
template <int KIND, bool GATHER, bool DBG>
void by_qpt(int qpt, const LaunchCfg& c, const Pass1Args& a) {
    switch (qpt) {
        case 1: go<KIND, GATHER, DBG, 1>(c, a); break;
        case 2: go<KIND, GATHER, DBG, 2>(c, a); break;
        case 4: go<KIND, GATHER, DBG, 4>(c, a); break;
        default: go<KIND, GATHER, DBG, 8>(c, a); break;
    }
}
template <int KIND>
void by_flags(bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a) {
    (void)gather;  // d <= 2 moves states, never gathers
    if (dbg) by_qpt<KIND, false, true>(qpt, c, a);
    else by_qpt<KIND, false, false>(qpt, c, a);
}
}  // namespace

void launch_pass1_d2(int kind, bool gather, bool dbg, int qpt, const LaunchCfg& c, const Pass1Args& a) {
    (void)kind;
    by_flags<1>(gather, dbg, qpt, c, a);
}

}  // namespace pfk
