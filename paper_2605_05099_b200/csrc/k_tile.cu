// Single-pass tile parse kernels (rs_tile.cuh): ziggurat normal / exponential over PCG64-DXSM and Philox.
#include "rs_tile.cuh"

const void *rsk::tile_kernel(int engine, int fam) {
    if (engine == RS_ENG_PCG64) {
        if (fam == FAM_NORM) return (const void *)k_tile<RS_ENG_PCG64, FAM_NORM>;
        if (fam == FAM_EXP) return (const void *)k_tile<RS_ENG_PCG64, FAM_EXP>;
    } else if (engine == RS_ENG_PHILOX) {
        if (fam == FAM_NORM) return (const void *)k_tile<RS_ENG_PHILOX, FAM_NORM>;
        if (fam == FAM_EXP) return (const void *)k_tile<RS_ENG_PHILOX, FAM_EXP>;
    }
    return nullptr;
}
