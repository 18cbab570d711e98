// Per-stream mode kernels (k_streams), the registry's other engines.
#include "rs_kernels.cuh"

namespace {
template <int E>
const void *streams_e(int fam) {
    switch (fam) {
    case FAM_NORM: return (const void *)k_streams<E, FAM_NORM>;
    case FAM_EXP: return (const void *)k_streams<E, FAM_EXP>;
    case FAM_GAMMA: return (const void *)k_streams<E, FAM_GAMMA>;
    case FAM_F32: return (const void *)k_streams<E, FAM_F32>;
    case FAM_U32: return (const void *)k_streams<E, FAM_U32>;
    case FAM_FIXED: return (const void *)k_streams<E, FAM_FIXED>;
    case FAM_LEMIRE_RING: return (const void *)k_streams<E, FAM_LEMIRE_RING>;
    default: return (const void *)k_streams<E, FAM_LEMIRE>;
    }
}
}  // namespace

const void *rsk::streams_kernel_b(int e, int fam) {
    switch (e) {
    case RS_ENG_X128P: return streams_e<RS_ENG_X128P>(fam);
    case RS_ENG_XORO: return streams_e<RS_ENG_XORO>(fam);
    case RS_ENG_SQUARES: return streams_e<RS_ENG_SQUARES>(fam);
    case RS_ENG_CHACHA20: return streams_e<RS_ENG_CHACHA20>(fam);
    default: return streams_e<RS_ENG_CWG128>(fam);
    }
}
