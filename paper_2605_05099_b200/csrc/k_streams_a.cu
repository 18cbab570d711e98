// Per-stream mode kernels (k_streams), north-star engines.
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

const void *rsk::streams_kernel(int e, int fam) {
    switch (e) {
    case RS_ENG_SFC64: return streams_e<RS_ENG_SFC64>(fam);
    case RS_ENG_PCG64: return streams_e<RS_ENG_PCG64>(fam);
    case RS_ENG_PHILOX: return streams_e<RS_ENG_PHILOX>(fam);
    case RS_ENG_X256SS: return streams_e<RS_ENG_X256SS>(fam);
    case RS_ENG_X256PP: return streams_e<RS_ENG_X256PP>(fam);
    default: return rsk::streams_kernel_b(e, fam);
    }
}
