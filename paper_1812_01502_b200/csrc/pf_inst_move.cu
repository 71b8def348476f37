// Instantiations of k_move (state-moving compose passes).
#include "pf_launch.h"

namespace pfk {
namespace {
template <typename T, bool DBG, int QPT>
void go(const LaunchCfg& c, const ComposeArgs& a) {
    auto k = k_move<T, DBG, QPT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
    k<<<c.grid, c.threads, c.smem, c.stream>>>(a);
}
template <typename T, bool DBG>
void by_qpt(int qpt, const LaunchCfg& c, const ComposeArgs& a) {
    switch (qpt) {
        case 1: go<T, DBG, 1>(c, a); break;
        case 2: go<T, DBG, 2>(c, a); break;
        case 4: go<T, DBG, 4>(c, a); break;
        default: go<T, DBG, 8>(c, a); break;
    }
}
template <typename T>
void by_dbg(bool dbg, int qpt, const LaunchCfg& c, const ComposeArgs& a) {
    if (dbg) by_qpt<T, true>(qpt, c, a);
    else by_qpt<T, false>(qpt, c, a);
}
}  // namespace

void launch_move(int payload, bool dbg, int qpt, const LaunchCfg& c, const ComposeArgs& a) {
    switch (payload) {
        case kPayloadF1: by_dbg<float>(dbg, qpt, c, a); break;
        case kPayloadF2: by_dbg<float2>(dbg, qpt, c, a); break;
        case kPayloadF4: by_dbg<float4>(dbg, qpt, c, a); break;
        default: by_dbg<State8>(dbg, qpt, c, a); break;
    }
}

}  // namespace pfk
