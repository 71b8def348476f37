// Instantiations of k_compose (DBG = true).
#include "pf_launch.h"

namespace pfk {
namespace {
template <typename T, bool IDENT, int QPT>
void go(const LaunchCfg& c, const ComposeArgs& a) {
    auto k = k_compose<T, IDENT, true, QPT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
    k<<<c.grid, c.threads, c.smem, c.stream>>>(a);
}
template <typename T, bool IDENT>
void by_qpt(int qpt, const LaunchCfg& c, const ComposeArgs& a) {
    switch (qpt) {
        case 1: go<T, IDENT, 1>(c, a); break;
        case 2: go<T, IDENT, 2>(c, a); break;
        case 4: go<T, IDENT, 4>(c, a); break;
        default: go<T, IDENT, 8>(c, a); break;
    }
}
}  // namespace

void launch_compose_dbg(int payload, int qpt, const LaunchCfg& c, const ComposeArgs& a) {
    switch (payload) {
        case kPayloadIdent: by_qpt<int32_t, true>(qpt, c, a); break;
        case kPayloadIndex: by_qpt<int32_t, false>(qpt, c, a); break;
        case kPayloadF1: by_qpt<float, false>(qpt, c, a); break;
        case kPayloadF2: by_qpt<float2, false>(qpt, c, a); break;
        case kPayloadF4: by_qpt<float4, false>(qpt, c, a); break;
        default: by_qpt<State8, false>(qpt, c, a); break;
    }
}

}  // namespace pfk
