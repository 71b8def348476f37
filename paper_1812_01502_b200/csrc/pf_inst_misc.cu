// Instantiations of k_init, k_cascade and the debug kernels.
#include "pf_launch.h"

namespace pfk {

void launch_cascade(int D, const LaunchCfg& c, const CascadeArgs& a) {
    switch (D) {
        case 1: k_cascade<1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_cascade<2><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_cascade<4><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_cascade<8><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

void launch_init(int D, int kind, const LaunchCfg& c, const InitArgs& a) {
    if (kind == 2) {
        k_init<1, 2><<<c.grid, c.threads, 0, c.stream>>>(a);
        return;
    }
    switch (D) {
        case 1: k_init<1, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_init<2, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_init<4, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_init<8, 1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

void launch_top(int D, const LaunchCfg& c, const TopArgs& a) {
    switch (D) {
        case 1: k_top<1><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 2: k_top<2><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        case 4: k_top<4><<<c.grid, c.threads, 0, c.stream>>>(a); break;
        default: k_top<8><<<c.grid, c.threads, 0, c.stream>>>(a); break;
    }
}

template <typename T>
static void cross_t(bool dbg, const LaunchCfg& c, const CrossArgs& a) {
    if (dbg) k_cross<T, true><<<c.grid, c.threads, 0, c.stream>>>(a);
    else k_cross<T, false><<<c.grid, c.threads, 0, c.stream>>>(a);
}

void launch_cross(int payload, bool dbg, const LaunchCfg& c, const CrossArgs& a) {
    switch (payload) {
        case kPayloadF1: cross_t<float>(dbg, c, a); break;
        case kPayloadF2: cross_t<float2>(dbg, c, a); break;
        case kPayloadF4: cross_t<float4>(dbg, c, a); break;
        default: cross_t<State8>(dbg, c, a); break;
    }
}

void launch_debug_compose(const LaunchCfg& c, const int32_t* anc, uint64_t N, uint32_t S, int32_t* A) {
    k_debug_compose<0><<<c.grid, c.threads, 0, c.stream>>>(anc, N, S, A);
}

}  // namespace pfk
