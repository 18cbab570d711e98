// Serial single-stream kernels (no skip-ahead) and the x256 jump setup.
#define RS_KERNELS_MISC
#include "rs_kernels.cuh"

namespace {
template <int E>
const void *serial_e(int fam, int fixed_mode) {
    if (fixed_mode >= 0) return (const void *)k_serial<-1, E>;
    switch (fam) {
    case FAM_NORM: return (const void *)k_serial<FAM_NORM, E>;
    case FAM_EXP: return (const void *)k_serial<FAM_EXP, E>;
    case FAM_GAMMA: return (const void *)k_serial<FAM_GAMMA, E>;
    case FAM_F32: return (const void *)k_serial<FAM_F32, E>;
    case FAM_U32: return (const void *)k_serial<FAM_U32, E>;
    default: return (const void *)k_serial<FAM_LEMIRE, E>;
    }
}
}  // namespace

const void *rsk::serial_kernel(int engine, int fam, int fixed_mode) {
    if (engine == RS_ENG_CWG128) return serial_e<RS_ENG_CWG128>(fam, fixed_mode);
    return engine == RS_ENG_SFC64_SIMD ? serial_e<RS_ENG_SFC64_SIMD>(fam, fixed_mode)
                                       : serial_e<RS_ENG_SFC64>(fam, fixed_mode);
}
const void *rsk::setup_kernel() { return (const void *)k_x256_setup; }
