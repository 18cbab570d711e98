// Ziggurat slow-path data as laid out on the device (read through the
// read-only cache; the 16-byte fast-path strips {K, W} are staged in shared
// memory by each block -- SURVEY 8(a) A21). Built on the host from rs_tables.h.
#pragma once
#include <cstdint>
#include <cstring>

#include "rs_tables.h"

struct RsZigSlow {
    uint64_t k[256];
    double f[256];
    uint64_t ta_lo[256], ta_hi[256], tr_lo[256], tr_hi[256];
};

struct RsZigFastHost {
    uint64_t k;
    uint64_t wbits;
};

static inline void rs_build_zig(int exp_tables, RsZigSlow *z, RsZigFastHost *fast) {
    for (int i = 0; i < 256; i++) {
        uint64_t fb = exp_tables ? RS_FE_BITS[i] : RS_FI_BITS[i];
        z->k[i] = exp_tables ? RS_KE[i] : RS_KI[i];
        std::memcpy(&z->f[i], &fb, 8);
        z->ta_lo[i] = exp_tables ? RS_TA_EXP_LO[i] : RS_TA_NORM_LO[i];
        z->ta_hi[i] = exp_tables ? RS_TA_EXP_HI[i] : RS_TA_NORM_HI[i];
        z->tr_lo[i] = exp_tables ? RS_TR_EXP_LO[i] : RS_TR_NORM_LO[i];
        z->tr_hi[i] = exp_tables ? RS_TR_EXP_HI[i] : RS_TR_NORM_HI[i];
        fast[i].k = z->k[i];
        fast[i].wbits = exp_tables ? RS_WE_BITS[i] : RS_WI_BITS[i];
    }
}
