// Fixed-consumption fills: k_fixed per engine and map, the counter-based Philox
// kernel, and the interleaved-engine kernel.
#include <cstdlib>

#include "rs_kernels.cuh"

namespace {
template <int E>
const void *fixed_e(int mode) {
    switch (mode) {
    case FX_RAW: return (const void *)k_fixed<E, FX_RAW>;
    case FX_U01: return (const void *)k_fixed<E, FX_U01>;
    case FX_POW2: return (const void *)k_fixed<E, FX_POW2>;
    case FX_WMAP: return (const void *)k_fixed<E, FX_WMAP>;
    case FX_HMAP: return (const void *)k_fixed<E, FX_HMAP>;
    default: return (const void *)k_fixed<E, FX_U01F>;
    }
}
template <int V>
const void *philox_v(int mode) {
    switch (mode) {
    case FX_RAW: return (const void *)k_philox_fixed<FX_RAW, V>;
    case FX_U01: return (const void *)k_philox_fixed<FX_U01, V>;
    case FX_POW2: return (const void *)k_philox_fixed<FX_POW2, V>;
    case FX_WMAP: return (const void *)k_philox_fixed<FX_WMAP, V>;
    case FX_HMAP: return (const void *)k_philox_fixed<FX_HMAP, V>;
    default: return (const void *)k_philox_fixed<FX_U01F, V>;
    }
}
template <int MODE>
const void *simd_m(int e) {
    return e == RS_ENG_X256SS_SIMD ? (const void *)k_simd_fixed<RS_ENG_X256SS_SIMD, MODE>
                                   : (const void *)k_simd_fixed<RS_ENG_X256PP_SIMD, MODE>;
}
}  // namespace

const void *rsk::fixed_kernel(int e, int mode) {
    switch (e) {
    case RS_ENG_X256SS: return fixed_e<RS_ENG_X256SS>(mode);
    case RS_ENG_X256PP: return fixed_e<RS_ENG_X256PP>(mode);
    case RS_ENG_PCG64: return fixed_e<RS_ENG_PCG64>(mode);
    case RS_ENG_PHILOX: return fixed_e<RS_ENG_PHILOX>(mode);
    case RS_ENG_X128P: return fixed_e<RS_ENG_X128P>(mode);
    case RS_ENG_XORO: return fixed_e<RS_ENG_XORO>(mode);
    case RS_ENG_SQUARES: return fixed_e<RS_ENG_SQUARES>(mode);
    case RS_ENG_CHACHA20: return fixed_e<RS_ENG_CHACHA20>(mode);
    default: return fixed_e<RS_ENG_RANLUX>(mode);
    }
}
const void *rsk::philox_kernel(int mode) {
    // V = 0: mul64x64 (default); RS_PHILOX_VARIANT=1 selects the mad.cc-chain product
    static int variant = getenv("RS_PHILOX_VARIANT") ? atoi(getenv("RS_PHILOX_VARIANT")) : 0;
    return variant == 1 ? philox_v<1>(mode) : philox_v<0>(mode);
}
const void *rsk::simd_kernel(int e, int mode) {
    switch (mode) {
    case FX_RAW: return simd_m<FX_RAW>(e);
    case FX_U01: return simd_m<FX_U01>(e);
    case FX_POW2: return simd_m<FX_POW2>(e);
    case FX_WMAP: return simd_m<FX_WMAP>(e);
    case FX_HMAP: return simd_m<FX_HMAP>(e);
    default: return simd_m<FX_U01F>(e);
    }
}
