// parse kernels over materialized words (RS_ENG_MEM): k_count / k_fixup / k_emit for every sampler family.
#include "rs_kernels.cuh"

namespace {
template <int D>
rsk::VarKernels vk() {
    return rsk::VarKernels{(const void *)k_count<RS_ENG_MEM, D>, (const void *)k_fixup<RS_ENG_MEM, D>, (const void *)k_emit<RS_ENG_MEM, D>};
}
}  // namespace

rsk::VarKernels rsk::var_kernels_mem(int fam) {
    switch (fam) {
    // the word-level 8-word batch parses read a whole batch ahead (EngMemB)
    case FAM_NORM: return rsk::VarKernels{(const void *)k_count<RS_ENG_MEMB, FAM_NORM>, (const void *)k_fixup<RS_ENG_MEMB, FAM_NORM>, (const void *)k_emit<RS_ENG_MEMB, FAM_NORM>};
    case FAM_EXP: return rsk::VarKernels{(const void *)k_count<RS_ENG_MEMB, FAM_EXP>, (const void *)k_fixup<RS_ENG_MEMB, FAM_EXP>, (const void *)k_emit<RS_ENG_MEMB, FAM_EXP>};
    case FAM_GAMMA: return vk<FAM_GAMMA>();
    case FAM_F32: return vk<FAM_F32>();
    case FAM_U32: return vk<FAM_U32>();
    default: return vk<FAM_LEMIRE>();
    }
}
