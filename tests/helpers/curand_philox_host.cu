// Test-only helper: exposes cuRAND's own Philox4x32-10 block function on the HOST
// (curand_philox4x32_x.h has an NV_IS_HOST branch) so CPU tests can pin the
// oracle's independent Philox against the library routine.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

extern "C" void curand_philox_blocks(const unsigned* ctrs, const unsigned* keys, unsigned* out, long n) {
    for (long i = 0; i < n; ++i) {
        uint4 c = make_uint4(ctrs[4 * i], ctrs[4 * i + 1], ctrs[4 * i + 2], ctrs[4 * i + 3]);
        uint2 k = make_uint2(keys[2 * i], keys[2 * i + 1]);
        uint4 r = curand_Philox4x32_10(c, k);
        out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
    }
}
