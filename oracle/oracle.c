/*
 * oracle.c -- CPU restatement of the reference's bulk stream-fill path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2605_05099_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product never links, calls or falls back to it.
 *
 * It restates, sequentially and word for word, the pure-Python reference
 * `randstream` (/root/reference/pkg/src/randstream/, "src/" below):
 *   engines  src/engines/{xorfam,pcg,counter,sfc,ranlux}.py
 *   buffer   src/buffer.py          (144-word refill, u32 halves low first)
 *   uniforms src/rng.py:98-115
 *   seeding  src/seeding.py:48-116  (SeedSequenceFE128)
 *   detmath  src/detmath.py:59-163  (fdlibm exp/log in strict IEEE steps)
 *   samplers src/continuous.py:40-93,157-218 ; src/discrete.py:20-39
 *   jumps    src/jumps.py:55-126, src/engines/pcg.py:41-55,
 *            src/engines/ranlux.py:90-93
 * Pinned against tests/golden/ (vectors produced by importing the reference;
 * see tests/golden/make_golden.py).  Compile with -ffp-contract=off: Python
 * evaluates doubles left to right with no fused multiply-add.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define RS_TABLE_QUAL static const
#include "../paper_2605_05099_b200/csrc/rs_tables.h"

typedef unsigned __int128 u128;
#define CAP 144
#define M64 0xFFFFFFFFFFFFFFFFULL

/* engine ids follow the reference registry order, src/engines/__init__.py:11-26 */
enum { E_X256PP = 1, E_X256SS = 2, E_PCG64 = 5, E_PHILOX = 6, E_SFC64 = 8, E_RANLUX = 10, E_X128P = 3, E_XORO = 4, E_SQUARES = 7, E_CWG128 = 9, E_CHACHA20 = 11,
       E_X256PP_SIMD = 12, E_X256SS_SIMD = 13, E_SFC64_SIMD = 14 };

/* distribution ids, shared with include/randstream_b200.h */
enum { D_UINT64 = 1, D_U01 = 2, D_U01F = 3, D_NORM = 4, D_EXP = 5, D_GAMMA = 6, D_BETA = 7,
       D_STDNORM = 8, D_UNIF = 9, D_UNIFF = 10, D_NORMF = 11, D_EXPF = 12, D_LOGNORMAL = 13, D_CHI2 = 14,
       D_T = 15, D_F = 16, D_GUMBEL = 17, D_PARETO = 18, D_GPD = 19, D_WEIBULL = 20, D_SKEW_NORMAL = 21,
       D_UINT32 = 22, D_INT32 = 23, D_INT64 = 24 };

typedef struct orc_rng {
    int eid;
    int full_mantissa;
    uint64_t st[32];           /* engine state, get_state() order (32 words for the 8-lane engines) */
    uint64_t buf[CAP];
    int fill, cursor;
    int has_pending;
    uint64_t pending;
    /* tallies: norm attempts/pdf, exp attempts/pdf, gamma attempts/pdf */
    uint64_t tally[6];
    int tally_seen[3];
} orc_rng;

static double d_from_bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t bits_of(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* ---------------------------------------------------------------- engines */

/* xoshiro256 linear step, src/engines/xorfam.py:16-26 */
static void x256_step(uint64_t *s) {
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = rotl(s[3], 45);
}

/* src/engines/xorfam.py:111-124 (x256**) and :88-98 (x256++) */
static void gen_x256(uint64_t *s, uint64_t *out, int n, int starstar) {
    for (int i = 0; i < n; i++) {
        out[i] = starstar ? rotl(s[1] * 5, 7) * 9 : rotl(s[0] + s[3], 23) + s[0];
        x256_step(s);
    }
}

/* PCG64-DXSM, src/engines/pcg.py:6-39: output of the pre-step state */
#define PCG_MULT 0xDA942042E4DD58B5ULL
static void gen_pcg(uint64_t *s, uint64_t *out, int n) {
    u128 state = ((u128)s[1] << 64) | s[0];
    u128 inc = ((u128)s[3] << 64) | s[2];
    for (int i = 0; i < n; i++) {
        uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state | 1;
        hi ^= hi >> 32; hi *= PCG_MULT; hi ^= hi >> 48;
        out[i] = hi * lo;
        state = state * PCG_MULT + inc;
    }
    s[0] = (uint64_t)state; s[1] = (uint64_t)(state >> 64);
}

/* src/engines/pcg.py:41-55, Brown's O(log n) advance */
static void pcg_advance(uint64_t *s, u128 delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT;
    u128 cur_plus = ((u128)s[3] << 64) | s[2];
    while (delta > 0) {
        if (delta & 1) { acc_mult *= cur_mult; acc_plus = acc_plus * cur_mult + cur_plus; }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    u128 state = ((u128)s[1] << 64) | s[0];
    state = state * acc_mult + acc_plus;
    s[0] = (uint64_t)state; s[1] = (uint64_t)(state >> 64);
}

/* Philox-4x64-10, src/engines/counter.py:67-121 */
static void philox_block(const uint64_t *ctr, const uint64_t *key, uint64_t *o) {
    uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        u128 p0 = (u128)0xD2E7470EE14C6C93ULL * x0;
        u128 p1 = (u128)0xCA5A826395121157ULL * x2;
        uint64_t n0 = (uint64_t)(p1 >> 64) ^ x1 ^ k0, n1 = (uint64_t)p1;
        uint64_t n2 = (uint64_t)(p0 >> 64) ^ x3 ^ k1, n3 = (uint64_t)p0;
        x0 = n0; x1 = n1; x2 = n2; x3 = n3;
        k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL;
    }
    o[0] = x0; o[1] = x1; o[2] = x2; o[3] = x3;
}
static void gen_philox(uint64_t *s, uint64_t *out, int n) {
    for (int b = 0; b < n / 4; b++) {
        philox_block(s, s + 4, out + 4 * b);
        for (int i = 0; i < 4; i++) { s[i] += 1; if (s[i] != 0) break; }
    }
}

/* sfc64, src/engines/sfc.py:25-36 */
static void gen_sfc(uint64_t *s, uint64_t *out, int n) {
    uint64_t a = s[0], b = s[1], c = s[2], w = s[3];
    for (int i = 0; i < n; i++) {
        uint64_t r = a + b + w;
        w += 1; a = b ^ (b >> 11); b = c + (c << 3); c = rotl(c, 24) + r;
        out[i] = r;
    }
    s[0] = a; s[1] = b; s[2] = c; s[3] = w;
}

/* xorshift128+, src/engines/xorfam.py:127-146 (state a, b; word a + b) */
static void gen_x128p(uint64_t *s, uint64_t *out, int n) {
    for (int i = 0; i < n; i++) {
        uint64_t s1 = s[0], s0 = s[1];
        out[i] = s0 + s1;
        s1 ^= s1 << 23;
        s[0] = s0;
        s[1] = s1 ^ s0 ^ (s1 >> 18) ^ (s0 >> 5);
    }
}
/* xoroshiro128++, src/engines/xorfam.py:149-168 */
static void gen_xoro(uint64_t *s, uint64_t *out, int n) {
    for (int i = 0; i < n; i++) {
        uint64_t s0 = s[0], s1 = s[1];
        out[i] = rotl(s0 + s1, 17) + s0;
        s1 ^= s0;
        s[0] = rotl(s0, 49) ^ s1 ^ (s1 << 21);
        s[1] = rotl(s1, 28);
    }
}
/* squares64, src/engines/counter.py:27-45 (state counter, key) */
static uint64_t sq_rot32(uint64_t x) { return (x >> 32) | (x << 32); }
static void gen_squares(uint64_t *s, uint64_t *out, int n) {
    for (int i = 0; i < n; i++) {
        uint64_t key = s[1], y = s[0] * key, x = y, z = y + key;
        x = x * x + y; x = sq_rot32(x);
        x = x * x + z; x = sq_rot32(x);
        x = x * x + y; x = sq_rot32(x);
        x = x * x + z;
        uint64_t t = x;
        x = sq_rot32(x);
        out[i] = t ^ ((x * x + y) >> 32);
        s[0] += 1;
    }
}
/* ChaCha20 keystream, src/engines/counter.py:170-216 (state: key[4], nonce0|nonce1<<32,
 * nonce2|counter<<32); the caller keeps the 32-bit counter in range */
static uint32_t rl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
static void gen_chacha(uint64_t *s, uint64_t *out, int n) {
    static const int q[8][4] = {{0, 4, 8, 12}, {1, 5, 9, 13}, {2, 6, 10, 14}, {3, 7, 11, 15},
                                {0, 5, 10, 15}, {1, 6, 11, 12}, {2, 7, 8, 13}, {3, 4, 9, 14}};
    for (int b = 0; b < n / 8; b++) {
        uint32_t in[16], x[16];
        in[0] = 0x61707865u; in[1] = 0x3320646Eu; in[2] = 0x79622D32u; in[3] = 0x6B206574u;
        for (int i = 0; i < 4; i++) { in[4 + 2 * i] = (uint32_t)s[i]; in[5 + 2 * i] = (uint32_t)(s[i] >> 32); }
        in[12] = (uint32_t)(s[5] >> 32);
        in[13] = (uint32_t)s[4]; in[14] = (uint32_t)(s[4] >> 32); in[15] = (uint32_t)s[5];
        memcpy(x, in, sizeof x);
        for (int dr = 0; dr < 10; dr++)
            for (int k = 0; k < 8; k++) {
                int a = q[k][0], bb = q[k][1], c = q[k][2], d = q[k][3];
                x[a] += x[bb]; x[d] = rl32(x[d] ^ x[a], 16);
                x[c] += x[d]; x[bb] = rl32(x[bb] ^ x[c], 12);
                x[a] += x[bb]; x[d] = rl32(x[d] ^ x[a], 8);
                x[c] += x[d]; x[bb] = rl32(x[bb] ^ x[c], 7);
            }
        for (int i = 0; i < 8; i++)
            out[8 * b + i] = (uint64_t)(uint32_t)(x[2 * i] + in[2 * i]) |
                             ((uint64_t)(uint32_t)(x[2 * i + 1] + in[2 * i + 1]) << 32);
        s[5] = (s[5] & 0xFFFFFFFFULL) | ((uint64_t)(uint32_t)(in[12] + 1) << 32);
    }
}
/* cwg128, src/engines/cwg.py:28-36 (x, weyl, extra, inc as lo/hi word pairs) */
static void gen_cwg(uint64_t *s, uint64_t *out, int n) {
    typedef unsigned __int128 w128;
    w128 x = ((w128)s[1] << 64) | s[0], weyl = ((w128)s[3] << 64) | s[2];
    w128 extra = ((w128)s[5] << 64) | s[4], inc = ((w128)s[7] << 64) | s[6];
    for (int i = 0; i < n; i++) {
        weyl += x;
        extra += inc;
        x = ((x >> 1) * (weyl | 1)) ^ extra;
        out[i] = (uint64_t)(weyl >> 96) ^ (uint64_t)x;
    }
    s[0] = (uint64_t)x; s[1] = (uint64_t)(x >> 64); s[2] = (uint64_t)weyl; s[3] = (uint64_t)(weyl >> 64);
    s[4] = (uint64_t)extra; s[5] = (uint64_t)(extra >> 64);
}

/* ranlux++: 576-bit residue times A mod m = 2^576 - 2^240 + 1,
 * src/engines/ranlux.py:16-61.  Any exact reduction gives the same residue. */
static const uint64_t RLX_M[9] = {1, 0, 0, 0xFFFF000000000000ULL, M64, M64, M64, M64, M64};
static uint64_t RLX_A[9];
static int rlx_ready = 0;

static int geq9(const uint64_t *a, const uint64_t *b) {
    for (int i = 8; i >= 0; i--) { if (a[i] != b[i]) return a[i] > b[i]; }
    return 1;
}
static void sub9(uint64_t *a, const uint64_t *b) {
    uint64_t br = 0;
    for (int i = 0; i < 9; i++) {
        u128 d = (u128)a[i] - b[i] - br;
        a[i] = (uint64_t)d; br = (uint64_t)(d >> 64) ? 1 : 0;
    }
}
/* r (10 limbs, value < 2^640) += v << (64*limb + bit) ... helper: add shifted 9/10-limb */
static void add_shifted(uint64_t *r, int rl, const uint64_t *v, int vl, int shift) {
    int ls = shift / 64, bs = shift % 64;
    uint64_t t[16] = {0};
    for (int i = 0; i < vl; i++) {
        if (i + ls < rl) t[i + ls] |= v[i] << bs;
        if (bs && i + ls + 1 < rl) t[i + ls + 1] |= v[i] >> (64 - bs);
    }
    u128 carry = 0;
    for (int i = 0; i < rl; i++) {
        u128 s = (u128)r[i] + t[i] + carry;
        r[i] = (uint64_t)s; carry = s >> 64;
    }
}
static void sub_from(uint64_t *r, int rl, const uint64_t *v, int vl) {
    uint64_t br = 0;
    for (int i = 0; i < rl; i++) {
        uint64_t x = i < vl ? v[i] : 0;
        u128 d = (u128)r[i] - x - br;
        r[i] = (uint64_t)d; br = (uint64_t)(d >> 64) ? 1 : 0;
    }
}
static void rlx_mulmod(const uint64_t *x, const uint64_t *y, uint64_t *res) {
    uint64_t prod[18] = {0};
    for (int i = 0; i < 9; i++) {
        u128 carry = 0;
        for (int j = 0; j < 9; j++) {
            u128 t = (u128)x[i] * y[j] + prod[i + j] + carry;
            prod[i + j] = (uint64_t)t; carry = t >> 64;
        }
        prod[i + 9] = (uint64_t)carry;
    }
    /* r = lo + hi*2^240 - hi   (hi = prod[9..17]) ; r < 2^817 fits 13 limbs */
    uint64_t r[13] = {0};
    memcpy(r, prod, 9 * 8);
    add_shifted(r, 13, prod + 9, 9, 240);
    sub_from(r, 13, prod + 9, 9);
    /* fold again: hi2 = r >> 576 */
    uint64_t hi2[4] = {r[9], r[10], r[11], r[12]};
    uint64_t r2[10] = {0};
    memcpy(r2, r, 9 * 8);
    add_shifted(r2, 10, hi2, 4, 240);
    sub_from(r2, 10, hi2, 4);
    /* r2 < 2^576 + 2^496: subtract m while >= m */
    while (r2[9] != 0 || geq9(r2, RLX_M)) {
        uint64_t mm[10]; memcpy(mm, RLX_M, 9 * 8); mm[9] = 0;
        sub_from(r2, 10, mm, 10);
    }
    memcpy(res, r2, 9 * 8);
}
static void rlx_powmod(const uint64_t *base, u128 e, uint64_t *out) {
    uint64_t r[9] = {1, 0, 0, 0, 0, 0, 0, 0, 0}, b[9];
    memcpy(b, base, 72);
    while (e) {
        if (e & 1) rlx_mulmod(r, b, r);
        rlx_mulmod(b, b, b);
        e >>= 1;
    }
    memcpy(out, r, 72);
}
/* A = (b^-1 mod m)^2048, b = 2^24: b^-1 = m - (m-1)/2^24 (src/engines/ranlux.py:16-19) */
static void rlx_init(void) {
    if (rlx_ready) return;
    /* (m-1)/2^24 = (2^576 - 2^240) / 2^24 = 2^552 - 2^216 */
    uint64_t q[9] = {0};
    q[8] = 1ULL << (552 - 512);          /* 2^552 */
    uint64_t t[9] = {0}; t[3] = 1ULL << (216 - 192); /* 2^216 */
    sub9(q, t);
    uint64_t a1[9]; memcpy(a1, RLX_M, 72); sub9(a1, q);
    rlx_powmod(a1, 2048, RLX_A);
    rlx_ready = 1;
}
static void gen_ranlux(uint64_t *s, uint64_t *out, int n) {
    for (int c = 0; c < n / 9; c++) {
        rlx_mulmod(s, RLX_A, s);
        memcpy(out + 9 * c, s, 72);
    }
}

static int engine_state_words(int eid) {
    switch (eid) {
    case E_PHILOX: case E_CHACHA20: return 6;
    case E_RANLUX: return 9;
    case E_X128P: case E_XORO: case E_SQUARES: return 2;
    case E_CWG128: return 8;
    case E_X256PP_SIMD: case E_X256SS_SIMD: case E_SFC64_SIMD: return 32;
    default: return 4;
    }
}
static int engine_seed_words(int eid) {
    switch (eid) {
    case E_PHILOX: case E_X128P: case E_XORO: return 2;
    case E_SQUARES: return 1;
    case E_SFC64: case E_SFC64_SIMD: return 3;
    case E_CHACHA20: return 6;
    case E_CWG128: return 8;
    case E_RANLUX: return 9;
    default: return 4;
    }
}

/* 8-lane interleaved engines, src/engines/interleave.py:71-76: word i from lane i mod 8 */
static void gen_simd(int base, uint64_t *s, uint64_t *out, int n) {
    for (int i = 0; i < n; i++) {
        uint64_t *l = s + 4 * (i & 7);
        if (base == E_SFC64) gen_sfc(l, out + i, 1);
        else gen_x256(l, out + i, 1, base == E_X256SS);
    }
}

static void engine_generate(int eid, uint64_t *s, uint64_t *out, int n) {
    switch (eid) {
    case E_X256PP_SIMD: gen_simd(E_X256PP, s, out, n); break;
    case E_X256SS_SIMD: gen_simd(E_X256SS, s, out, n); break;
    case E_SFC64_SIMD: gen_simd(E_SFC64, s, out, n); break;
    case E_X256PP: gen_x256(s, out, n, 0); break;
    case E_X256SS: gen_x256(s, out, n, 1); break;
    case E_PCG64: gen_pcg(s, out, n); break;
    case E_PHILOX: gen_philox(s, out, n); break;
    case E_SFC64: gen_sfc(s, out, n); break;
    case E_RANLUX: rlx_init(); gen_ranlux(s, out, n); break;
    case E_X128P: gen_x128p(s, out, n); break;
    case E_XORO: gen_xoro(s, out, n); break;
    case E_SQUARES: gen_squares(s, out, n); break;
    case E_CHACHA20: gen_chacha(s, out, n); break;
    case E_CWG128: gen_cwg(s, out, n); break;
    }
}

/* ---------------------------------------------------------------- seeding */
/* SeedSequenceFE128, src/seeding.py:21-116 (numpy SeedSequence pool_size=4) */
#define INIT_A 0x43B0D7E5u
#define MULT_A 0x931E8875u
#define INIT_B 0x8B51F9DDu
#define MULT_B 0x58F38DEDu
#define MIX_L 0xCA01F9DDu
#define MIX_R 0x4973F715u

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = x * MIX_L - y * MIX_R;
    return r ^ (r >> 16);
}
static uint32_t ss_hash(uint32_t v, uint32_t *hc) {
    v ^= *hc; *hc *= MULT_A; v *= *hc; v ^= v >> 16; return v;
}
void orc_seed_words(const uint64_t *ent, int nent, const uint64_t *spawn, int nspawn,
                    uint64_t *out, int nout) {
    uint32_t a[512]; int na = 0;
    for (int i = 0; i < nent; i++) { a[na++] = (uint32_t)ent[i]; a[na++] = (uint32_t)(ent[i] >> 32); }
    if (nspawn > 0) while (na < 4) a[na++] = 0;
    for (int i = 0; i < nspawn; i++) { a[na++] = (uint32_t)spawn[i]; a[na++] = (uint32_t)(spawn[i] >> 32); }
    uint32_t pool[4], hc = INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hash(i < na ? a[i] : 0, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hash(pool[s], &hc));
    for (int s = 4; s < na; s++)
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hash(a[s], &hc));
    uint32_t hb = INIT_B;
    for (int i = 0; i < nout; i++) {
        uint32_t w[2];
        for (int h = 0; h < 2; h++) {
            uint32_t v = pool[(2 * i + h) % 4] ^ hb;
            hb *= MULT_B; v *= hb; v ^= v >> 16; w[h] = v;
        }
        out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    }
}

void orc_x256_charpoly(uint64_t *out5);
void orc_x_pow2k_mod(int k, const uint64_t *c5, uint64_t *out5);
void orc_x256_apply_poly(uint64_t *s, const uint64_t *poly5);

/* seed_from for each engine: xorfam.py:66-70, pcg.py:81-84, counter.py:139-141,
 * sfc.py:53-55, ranlux.py:106-110, interleave.py:127-130,212-215 */
static void engine_seed_from(int eid, uint64_t *s, const uint64_t *w) {
    switch (eid) {
    case E_X256PP_SIMD: case E_X256SS_SIMD: {
        uint64_t base[4];
        memcpy(base, w, 32);
        if (!(base[0] | base[1] | base[2] | base[3])) base[0] = 1;
        uint64_t p[5], poly[5];
        orc_x256_charpoly(p);
        orc_x_pow2k_mod(253, p, poly);   /* lanes 2^253 steps apart (interleave.py:201-208) */
        memcpy(s, base, 32);
        for (int k = 1; k < 8; k++) { memcpy(s + 4 * k, s + 4 * (k - 1), 32); orc_x256_apply_poly(s + 4 * k, poly); }
        break;
    }
    case E_SFC64_SIMD:
        for (int k = 0; k < 8; k++) {
            s[4 * k] = w[0]; s[4 * k + 1] = w[1]; s[4 * k + 2] = w[2];
            s[4 * k + 3] = 1 + (uint64_t)k * (1ULL << 61);
        }
        break;
    case E_X256PP: case E_X256SS:
        memcpy(s, w, 32);
        if (!(s[0] | s[1] | s[2] | s[3])) s[0] = 1;
        break;
    case E_PCG64: s[0] = w[0]; s[1] = w[1]; s[2] = w[2] | 1; s[3] = w[3]; break;
    case E_X128P: case E_XORO:  /* xorfam.py:66-70 */
        s[0] = w[0]; s[1] = w[1];
        if (!(s[0] | s[1])) s[0] = 1;
        break;
    case E_SQUARES: s[0] = 0; s[1] = w[0]; break;                         /* counter.py:63-65 */
    case E_CHACHA20: memcpy(s, w, 40); s[5] = w[5] & 0xFFFFFFFFULL; break;  /* counter.py:228-233 */
    case E_CWG128: memcpy(s, w, 64); s[6] |= 1; break;                     /* cwg.py:62-67 */
    case E_PHILOX: s[0] = s[1] = s[2] = s[3] = 0; s[4] = w[0]; s[5] = w[1]; break;
    case E_SFC64: s[0] = w[0]; s[1] = w[1]; s[2] = w[2]; s[3] = 1; break;
    case E_RANLUX: {
        uint64_t x[9]; memcpy(x, w, 72);
        rlx_init();
        while (geq9(x, RLX_M)) sub9(x, RLX_M);   /* w < 2^576 < 2m */
        int zero = 1; for (int i = 0; i < 9; i++) zero &= x[i] == 0;
        if (zero) x[0] = 1;
        memcpy(s, x, 72);
        break;
    }
    }
}

int orc_create(orc_rng *r, int eid, const uint64_t *seed, int nseed, const uint64_t *spawn, int nspawn) {
    memset(r, 0, sizeof *r);
    r->eid = eid;
    uint64_t w[16];
    orc_seed_words(seed, nseed, spawn, nspawn, w, engine_seed_words(eid));
    engine_seed_from(eid, r->st, w);
    return 0;
}

void orc_set_state(orc_rng *r, int eid, const uint64_t *words) {
    int fm = r->full_mantissa;
    memset(r, 0, sizeof *r);
    r->eid = eid; r->full_mantissa = fm;
    memcpy(r->st, words, 8 * engine_state_words(eid));
}

/* ---------------------------------------------------------------- buffer */
/* WordBuffer.take_u64 / take_u32, src/buffer.py:29-49 */
static uint64_t take_u64(orc_rng *r) {
    r->has_pending = 0;
    if (r->cursor >= r->fill) { engine_generate(r->eid, r->st, r->buf, CAP); r->fill = CAP; r->cursor = 0; }
    return r->buf[r->cursor++];
}
static uint32_t take_u32(orc_rng *r) {
    if (r->has_pending) { r->has_pending = 0; return (uint32_t)r->pending; }
    if (r->cursor >= r->fill) { engine_generate(r->eid, r->st, r->buf, CAP); r->fill = CAP; r->cursor = 0; }
    uint64_t w = r->buf[r->cursor++];
    r->pending = w >> 32; r->has_pending = 1;
    return (uint32_t)w;
}
uint64_t orc_next_u64(orc_rng *r) { return take_u64(r); }
uint32_t orc_next_u32(orc_rng *r) { return take_u32(r); }

/* Rng.u01 / u01f, src/rng.py:98-115 */
static double u01(orc_rng *r) {
    uint64_t w = take_u64(r);
    if (r->full_mantissa) return (double)(w >> 11) * 1.1102230246251565e-16;
    return d_from_bits((w >> 12) | 0x3FF0000000000000ULL) - 1.0;
}
static double u01f(orc_rng *r) {
    uint32_t w = take_u32(r);
    if (r->full_mantissa) return (double)(w >> 8) * 5.9604644775390625e-08;
    uint32_t fb = (w >> 9) | 0x3F800000u; float f; memcpy(&f, &fb, 4);
    return (double)f - 1.0;
}

/* ---------------------------------------------------------------- detmath */
/* fdlibm exp/log restated in strict IEEE steps, src/detmath.py:59-163 */
static uint32_t hi_of(double x) { return (uint32_t)(bits_of(x) >> 32); }
static double with_hi(double x, uint32_t hi) {
    return d_from_bits(((uint64_t)hi << 32) | (bits_of(x) & 0xFFFFFFFFULL));
}
double orc_det_exp(double x) {
    const double huge = 1.0e300, twom1000 = 9.33263618503218878990e-302;
    const double o_thr = 7.09782712893383973096e+02, u_thr = -7.45133219101941108420e+02;
    const double invln2 = 1.44269504088896338700e+00, ln2hi = 6.93147180369123816490e-01,
                 ln2lo = 1.90821492927058770002e-10;
    const double P1 = 1.66666666666666019037e-01, P2 = -2.77777777770155933842e-03,
                 P3 = 6.61375632143793436117e-05, P4 = -1.65339022054652515390e-06,
                 P5 = 4.13813679705723846039e-08;
    uint32_t hx = hi_of(x);
    int xsb = (hx >> 31) & 1;
    hx &= 0x7FFFFFFFu;
    if (hx >= 0x40862E42u) {
        if (hx >= 0x7FF00000u) {
            if (((hx & 0xFFFFFu) | (uint32_t)bits_of(x)) != 0) return x + x;
            return xsb == 0 ? x : 0.0;
        }
        if (x > o_thr) return huge * huge;
        if (x < u_thr) return twom1000 * twom1000;
    }
    int k = 0;
    double hi = 0.0, lo = 0.0;
    if (hx > 0x3FD62E42u) {
        if (hx < 0x3FF0A2E4u) {
            if (xsb == 0) { hi = x - ln2hi; lo = ln2lo; k = 1; }
            else { hi = x + ln2hi; lo = -ln2lo; k = -1; }
        } else {
            double kd = invln2 * x + (xsb == 0 ? 0.5 : -0.5);
            k = (int)kd;               /* Python int() truncates toward zero */
            double t = (double)k;
            hi = x - t * ln2hi;
            lo = t * ln2lo;
        }
        x = hi - lo;
    } else if (hx < 0x3E300000u) {
        if (huge + x > 1.0) return 1.0 + x;
    }
    double t = x * x;
    double c = x - t * (P1 + t * (P2 + t * (P3 + t * (P4 + t * P5))));
    if (k == 0) return 1.0 - ((x * c / (c - 2.0)) - x);
    double y = 1.0 - ((lo - (x * c) / (2.0 - c)) - hi);
    if (k >= -1021) return with_hi(y, hi_of(y) + ((uint32_t)k << 20));
    return with_hi(y, hi_of(y) + ((uint32_t)(k + 1000) << 20)) * twom1000;
}

double orc_det_log(double x) {
    const double ln2hi = 6.93147180369123816490e-01, ln2lo = 1.90821492927058770002e-10;
    const double two54 = 1.80143985094819840000e+16;
    const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                 Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                 Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                 Lg7 = 1.479819860511658591e-01;
    uint64_t u = bits_of(x);
    int32_t hx = (int32_t)(u >> 32);
    uint32_t lx = (uint32_t)u;
    int k = 0;
    if (hx < 0) {
        if (((hx & 0x7FFFFFFF) | lx) == 0) return -INFINITY;
        return NAN;
    }
    if (hx < 0x00100000) {
        if ((hx | lx) == 0) return -INFINITY;
        k -= 54; x *= two54; hx = (int32_t)hi_of(x);
    }
    if (hx >= 0x7FF00000) return x + x;
    k += (hx >> 20) - 1023;
    hx &= 0x000FFFFF;
    int32_t i = (hx + 0x95F64) & 0x100000;
    x = with_hi(x, (uint32_t)(hx | (i ^ 0x3FF00000)));
    k += i >> 20;
    double f = x - 1.0;
    if ((0x000FFFFF & (2 + hx)) < 3) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            double dk = (double)k;
            return dk * ln2hi + dk * ln2lo;
        }
        double R = f * f * (0.5 - 0.33333333333333333 * f);
        if (k == 0) return f - R;
        double dk = (double)k;
        return dk * ln2hi - ((R - dk * ln2lo) - f);
    }
    double s = f / (2.0 + f);
    double dk = (double)k;
    double z = s * s;
    int32_t ii = hx - 0x6147A;
    double w = z * z;
    int32_t j = 0x6B851 - hx;
    double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
    double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
    ii |= j;
    double R = t2 + t1;
    if (ii > 0) {
        double hfsq = 0.5 * f * f;
        if (k == 0) return f - (hfsq - s * (hfsq + R));
        return dk * ln2hi - ((hfsq - (s * (hfsq + R) + dk * ln2lo)) - f);
    }
    if (k == 0) return f - s * (f - R);
    return dk * ln2hi - ((s * (f - R) - dk * ln2lo) - f);
}

/* ---------------------------------------------------------------- samplers */
static int lt128(uint64_t alo, uint64_t ahi, uint64_t blo, uint64_t bhi) {
    return ahi < bhi || (ahi == bhi && alo < blo);
}
/* lhs = yv*d + (rabs-K)*2^52 as a 128-bit integer (src/continuous.py:59-61) */
static void zig_lhs(uint64_t yv, uint64_t d, uint64_t rk, uint64_t *lo, uint64_t *hi) {
    u128 v = (u128)yv * d + ((u128)rk << 52);
    *lo = (uint64_t)v; *hi = (uint64_t)(v >> 64);
}

/* std_norm, src/continuous.py:40-68 */
static double std_norm(orc_rng *r) {
    r->tally_seen[0] = 1;
    const double nor_r = d_from_bits(RS_NOR_R_BITS), nor_inv_r = d_from_bits(RS_NOR_INV_R_BITS);
    for (;;) {
        r->tally[0]++;
        uint64_t w = take_u64(r);
        int idx = (int)(w & 0xFF);
        int sign = (int)((w >> 8) & 1);
        uint64_t rabs = (w >> 9) & ((1ULL << 52) - 1);
        double x = (double)rabs * d_from_bits(RS_WI_BITS[idx]);
        if (rabs < RS_KI[idx]) return sign ? -x : x;
        if (idx == 0) {
            for (;;) {
                double xx = -nor_inv_r * orc_det_log(1.0 - u01(r));
                double yy = -orc_det_log(1.0 - u01(r));
                if (yy + yy > xx * xx) { double t = nor_r + xx; return sign ? -t : t; }
            }
        }
        uint64_t yv = take_u64(r) >> 12;
        uint64_t lo, hi;
        zig_lhs(yv, (1ULL << 52) - RS_KI[idx], rabs - RS_KI[idx], &lo, &hi);
        if (lt128(lo, hi, RS_TA_NORM_LO[idx], RS_TA_NORM_HI[idx])) return sign ? -x : x;
        if (!lt128(RS_TR_NORM_LO[idx], RS_TR_NORM_HI[idx], lo, hi)) {   /* lhs <= TR */
            r->tally[1]++;
            double fi = d_from_bits(RS_FI_BITS[idx]), fim1 = d_from_bits(RS_FI_BITS[idx - 1]);
            double y = fi + ((double)yv * 2.220446049250313e-16) * (fim1 - fi);
            if (y < orc_det_exp(-0.5 * x * x)) return sign ? -x : x;
        }
    }
}

/* std_exp, src/continuous.py:71-93 */
static double std_exp(orc_rng *r) {
    r->tally_seen[1] = 1;
    const double exp_r = d_from_bits(RS_EXP_R_BITS);
    for (;;) {
        r->tally[2]++;
        uint64_t w = take_u64(r);
        int idx = (int)(w & 0xFF);
        uint64_t rabs = (w >> 8) & ((1ULL << 53) - 1);
        double x = (double)rabs * d_from_bits(RS_WE_BITS[idx]);
        if (rabs < RS_KE[idx]) return x;
        if (idx == 0) return exp_r - orc_det_log(1.0 - u01(r));
        uint64_t yv = take_u64(r) >> 12;
        uint64_t lo, hi;
        zig_lhs(yv, (1ULL << 53) - RS_KE[idx], rabs - RS_KE[idx], &lo, &hi);
        if (lt128(lo, hi, RS_TA_EXP_LO[idx], RS_TA_EXP_HI[idx])) return x;
        if (!lt128(RS_TR_EXP_LO[idx], RS_TR_EXP_HI[idx], lo, hi)) {
            r->tally[3]++;
            double fe = d_from_bits(RS_FE_BITS[idx]), fem1 = d_from_bits(RS_FE_BITS[idx - 1]);
            double y = fe + ((double)yv * 2.220446049250313e-16) * (fem1 - fe);
            if (y < orc_det_exp(-x)) return x;
        }
    }
}

/* gamma, src/continuous.py:183-212 (validation done by the caller) */
static double gamma_s(orc_rng *r, double alpha, double theta) {
    if (alpha < 1.0) {
        double base = gamma_s(r, alpha + 1.0, 1.0);
        double u = u01(r);
        return theta * base * orc_det_exp(orc_det_log(u) / alpha);
    }
    r->tally_seen[2] = 1;
    double d = alpha - 1.0 / 3.0;
    double cc = 1.0 / sqrt(9.0 * d);
    for (;;) {
        r->tally[4]++;
        double z, t;
        for (;;) { z = std_norm(r); t = 1.0 + cc * z; if (t > 0.0) break; }
        double v = t * t * t;
        double u = u01(r);
        double zz = z * z;
        if (u < 1.0 - 0.0331 * zz * zz) return theta * d * v;
        if (orc_det_log(u) < 0.5 * zz + d - d * v + d * orc_det_log(v)) return theta * d * v;
    }
}


static double to_f32(double x) { return (double)(float)x; }  /* numpy float32 rounding (_f32) */

/* std_norm_f, src/continuous.py:96-115 (32-bit halves, f32 tables) */
static double std_norm_f(orc_rng *r) {
    const double nor_r = d_from_bits(RS_NOR_R_BITS), nor_inv_r = d_from_bits(RS_NOR_INV_R_BITS);
    for (;;) {
        uint32_t w = take_u32(r);
        int idx = (int)(w & 0xFF);
        int sign = (int)((w >> 8) & 1);
        uint32_t rabs = (w >> 9) & 0x7FFFFF;
        float wf; memcpy(&wf, &RS_WI_F_BITS[idx], 4);
        double x = to_f32((double)rabs * (double)wf);
        if (rabs < RS_KI_F[idx]) return sign ? -x : x;
        if (idx == 0) {
            for (;;) {
                double xx = -nor_inv_r * orc_det_log(1.0 - u01f(r));
                double yy = -orc_det_log(1.0 - u01f(r));
                if (yy + yy > xx * xx) { double t = to_f32(nor_r + xx); return sign ? -t : t; }
            }
        }
        double u = (double)(take_u32(r) >> 8) * 5.9604644775390625e-08;
        float fi, fim1; memcpy(&fi, &RS_FI_F_BITS[idx], 4); memcpy(&fim1, &RS_FI_F_BITS[idx - 1], 4);
        double y = (double)fi + u * ((double)fim1 - (double)fi);
        if (y < orc_det_exp(-0.5 * x * x)) return sign ? -x : x;
    }
}
/* std_exp_f, src/continuous.py:118-133 */
static double std_exp_f(orc_rng *r) {
    const double exp_r = d_from_bits(RS_EXP_R_BITS);
    for (;;) {
        uint32_t w = take_u32(r);
        int idx = (int)(w & 0xFF);
        uint32_t rabs = (w >> 8) & 0xFFFFFF;
        float wf; memcpy(&wf, &RS_WE_F_BITS[idx], 4);
        double x = to_f32((double)rabs * (double)wf);
        if (rabs < RS_KE_F[idx]) return x;
        if (idx == 0) return to_f32(exp_r - orc_det_log(1.0 - u01f(r)));
        double u = (double)(take_u32(r) >> 8) * 5.9604644775390625e-08;
        float fe, fem1; memcpy(&fe, &RS_FE_F_BITS[idx], 4); memcpy(&fem1, &RS_FE_F_BITS[idx - 1], 4);
        double y = (double)fe + u * ((double)fem1 - (double)fe);
        if (y < orc_det_exp(-x)) return x;
    }
}

/* bounded_uint for widths 8/16/32 on 32-bit halves, src/discrete.py:14-39 */
static uint64_t bounded32(orc_rng *r, uint64_t b, int width) {
    uint64_t mask = (width == 32) ? 0xFFFFFFFFULL : ((1ULL << width) - 1);
    uint64_t x = take_u32(r) & mask;
    if (b == 0) return x;
    uint64_t m = x * b;
    uint64_t low = m & mask;
    if (low < b) {
        uint64_t thr = ((1ULL << width) - b) % b;
        while (low < thr) { x = take_u32(r) & mask; m = x * b; low = m & mask; }
    }
    return m >> width;
}

/* bounded_uint width 64, src/discrete.py:20-39; b_is_2p64 covers b == 2^64 */
static uint64_t bounded64(orc_rng *r, uint64_t b, int b_is_2p64) {
    uint64_t x = take_u64(r);
    if (b == 0 || b_is_2p64) return x;
    u128 m = (u128)x * b;
    uint64_t low = (uint64_t)m;
    if (low < b) {
        uint64_t thr = (0 - b) % b;
        while (low < thr) { x = take_u64(r); m = (u128)x * b; low = (uint64_t)m; }
    }
    return (uint64_t)(m >> 64);
}

/* Bulk fill: Rng.fill -> continuous.fill / discrete.fill (src/rng.py:223-241,
 * src/continuous.py:413-431, src/discrete.py:103-111).  Parameters are already
 * validated by the caller.  out is u64[n] / f64[n] / f32[n] (u01f). */
int orc_fill(orc_rng *r, int dist, const double *fp, const uint64_t *ip, uint64_t n, void *out) {
    uint64_t *o64 = (uint64_t *)out;
    double *od = (double *)out;
    float *of = (float *)out;
    switch (dist) {
    case D_UINT64:
        for (uint64_t i = 0; i < n; i++) o64[i] = bounded64(r, ip[0], (int)ip[1]);
        return 0;
    case D_U01:
        for (uint64_t i = 0; i < n; i++) od[i] = u01(r);
        return 0;
    case D_U01F:
        for (uint64_t i = 0; i < n; i++) of[i] = (float)u01f(r);
        return 0;
    case D_NORM: {
        double mu = fp[0], sd = sqrt(fp[1]);
        for (uint64_t i = 0; i < n; i++) od[i] = mu + sd * std_norm(r);
        return 0;
    }
    case D_STDNORM:
        for (uint64_t i = 0; i < n; i++) od[i] = std_norm(r);
        return 0;
    case D_EXP:
        for (uint64_t i = 0; i < n; i++) od[i] = fp[0] * std_exp(r);
        return 0;
    case D_GAMMA:
        for (uint64_t i = 0; i < n; i++) od[i] = gamma_s(r, fp[0], fp[1]);
        return 0;
    case D_BETA:
        for (uint64_t i = 0; i < n; i++) {
            double x = gamma_s(r, fp[0], 1.0);
            double y = gamma_s(r, fp[1], 1.0);
            od[i] = x / (x + y);
        }
        return 0;
    /* derived laws and transforms, src/continuous.py:136-290 (bitexact forms) */
    case D_UNIF: for (uint64_t i = 0; i < n; i++) od[i] = fp[0] + u01(r) * (fp[1] - fp[0]); return 0;
    case D_UNIFF: for (uint64_t i = 0; i < n; i++) of[i] = (float)(fp[0] + u01f(r) * (fp[1] - fp[0])); return 0;
    case D_NORMF: {
        double sd = sqrt(fp[1]);
        for (uint64_t i = 0; i < n; i++) of[i] = (float)(fp[0] + sd * std_norm_f(r));
        return 0;
    }
    case D_EXPF: for (uint64_t i = 0; i < n; i++) of[i] = (float)(fp[0] * std_exp_f(r)); return 0;
    case D_LOGNORMAL: {
        double sd = sqrt(fp[1]);
        for (uint64_t i = 0; i < n; i++) od[i] = orc_det_exp(fp[0] + sd * std_norm(r));
        return 0;
    }
    case D_CHI2: for (uint64_t i = 0; i < n; i++) od[i] = gamma_s(r, fp[0] / 2.0, 2.0); return 0;
    case D_T:
        for (uint64_t i = 0; i < n; i++) {
            double z = std_norm(r);
            double v = gamma_s(r, fp[0] / 2.0, 2.0);
            od[i] = z / sqrt(v / fp[0]);
        }
        return 0;
    case D_F:
        for (uint64_t i = 0; i < n; i++) {
            double x = gamma_s(r, fp[0] / 2.0, 1.0);
            double y = gamma_s(r, fp[1] / 2.0, 1.0);
            od[i] = (x / fp[0]) / (y / fp[1]);
        }
        return 0;
    case D_GUMBEL:
        for (uint64_t i = 0; i < n; i++) od[i] = fp[0] - fp[1] * orc_det_log(-orc_det_log(u01(r)));
        return 0;
    case D_PARETO: for (uint64_t i = 0; i < n; i++) od[i] = fp[1] * orc_det_exp(std_exp(r) / fp[0]); return 0;
    case D_GPD:
        for (uint64_t i = 0; i < n; i++) {
            double xi = fp[0], mu = fp[1], sigma = fp[2];
            if (xi == 0.0) { od[i] = mu + sigma * std_exp(r); continue; }
            double pp = orc_det_exp(std_exp(r) * fabs(xi));
            od[i] = xi > 0.0 ? mu + sigma * (pp - 1.0) / xi : mu - sigma * (1.0 - 1.0 / pp) / xi;
        }
        return 0;
    case D_WEIBULL:
        for (uint64_t i = 0; i < n; i++) od[i] = fp[1] * orc_det_exp(orc_det_log(std_exp(r)) / fp[0]);
        return 0;
    case D_SKEW_NORMAL: {
        double alpha = fp[0], mu = fp[1], sigma = fp[2];
        double delta = alpha / sqrt(1.0 + alpha * alpha);
        double cd = sqrt(1.0 - delta * delta);
        for (uint64_t i = 0; i < n; i++) {
            double z1 = std_norm(r);
            double z2 = std_norm(r);
            od[i] = mu + sigma * (delta * fabs(z1) + cd * z2);
        }
        return 0;
    }
    /* bounded integers on halves / signed ranges, src/discrete.py:20-55,103-118.
       ip = {b or span, width, m (two's complement), full_span_flag} */
    case D_UINT32: {
        uint32_t *o32 = (uint32_t *)out;
        for (uint64_t i = 0; i < n; i++) o32[i] = (uint32_t)bounded32(r, ip[0], (int)ip[1]);
        return 0;
    }
    case D_INT32: {
        int32_t *o = (int32_t *)out;
        for (uint64_t i = 0; i < n; i++) {
            uint64_t v = ip[3] ? (uint64_t)take_u32(r) : bounded32(r, ip[0], 32);
            o[i] = (int32_t)(uint32_t)((uint32_t)ip[2] + (uint32_t)v);
        }
        return 0;
    }
    case D_INT64: {
        for (uint64_t i = 0; i < n; i++) {
            uint64_t v = ip[3] ? take_u64(r) : bounded64(r, ip[0], 0);
            o64[i] = ip[2] + v;
        }
        return 0;
    }
    }
    return -1;
}

/* ---------------------------------------------------------------- jumps */
/* GF(2) polynomials of degree <= 256 as 5 x u64 (bit i = coeff of x^i). */
typedef struct { uint64_t w[9]; } poly_t;   /* room for squaring (<= 512 bits) */

static int pdeg(const poly_t *p) {
    for (int i = 8; i >= 0; i--) if (p->w[i]) return i * 64 + 63 - __builtin_clzll(p->w[i]);
    return -1;
}
static void pmod(poly_t *r, const poly_t *c) {
    int n = pdeg(c);
    for (;;) {
        int d = pdeg(r);
        if (d < n) return;
        int sh = d - n;
        int ws = sh / 64, bs = sh % 64;
        for (int i = 8; i >= 0; i--) {
            uint64_t v = 0;
            if (i - ws >= 0) v = c->w[i - ws] << bs;
            if (bs && i - ws - 1 >= 0) v |= c->w[i - ws - 1] >> (64 - bs);
            r->w[i] ^= v;
        }
    }
}
static void psquare(poly_t *r, const poly_t *a) {
    poly_t t; memset(&t, 0, sizeof t);
    for (int i = 0; i < 256; i++)
        if ((a->w[i / 64] >> (i % 64)) & 1) t.w[(2 * i) / 64] |= 1ULL << ((2 * i) % 64);
    *r = t;
}
/* x^n mod c, src/jumps.py:55-64 */
void orc_x_pow_mod(uint64_t nlo, uint64_t nhi, const uint64_t *c5, uint64_t *out5) {
    poly_t c; memset(&c, 0, sizeof c); memcpy(c.w, c5, 40);
    poly_t r; memset(&r, 0, sizeof r); r.w[0] = 1;
    u128 n = ((u128)nhi << 64) | nlo;
    int nb = 0; for (u128 t = n; t; t >>= 1) nb++;
    for (int s = nb - 1; s >= 0; s--) {
        psquare(&r, &r); pmod(&r, &c);
        if ((n >> s) & 1) {
            for (int i = 8; i > 0; i--) r.w[i] = (r.w[i] << 1) | (r.w[i - 1] >> 63);
            r.w[0] <<= 1;
            pmod(&r, &c);
        }
    }
    memcpy(out5, r.w, 40);
}
/* characteristic polynomial of the xoshiro256 step via Berlekamp-Massey,
 * src/jumps.py:67-113 (degree 256, so 5 words) */
void orc_x256_charpoly(uint64_t *out5) {
    uint64_t s[4] = {1, 0, 0, 0};
    static uint8_t bits[512];
    for (int i = 0; i < 512; i++) { bits[i] = s[0] & 1; x256_step(s); }
    /* connection polynomial c, b as bit arrays (degree <= 512) */
    static uint8_t c[520], b[520], old[520];
    memset(c, 0, sizeof c); memset(b, 0, sizeof b);
    c[0] = 1; b[0] = 1;
    int L = 0, m = 1;
    for (int i = 0; i < 512; i++) {
        int d = bits[i];
        for (int j = 1; j <= L; j++) if (c[j]) d ^= bits[i - j];
        if (d) {
            memcpy(old, c, sizeof c);
            for (int j = 0; j + m < 520; j++) c[j + m] ^= b[j];
            if (2 * L <= i) { L = i + 1 - L; memcpy(b, old, sizeof b); m = 1; }
            else m++;
        } else m++;
    }
    memset(out5, 0, 40);
    for (int j = 0; j <= L; j++) if (c[j]) out5[(L - j) / 64] |= 1ULL << ((L - j) % 64);
}
/* apply_polynomial, src/jumps.py:116-126 */
void orc_x256_apply_poly(uint64_t *s, const uint64_t *poly5) {
    uint64_t acc[4] = {0}, cur[4];
    memcpy(cur, s, 32);
    for (int i = 0; i < 257; i++) {
        if ((poly5[i / 64] >> (i % 64)) & 1) for (int k = 0; k < 4; k++) acc[k] ^= cur[k];
        x256_step(cur);
    }
    memcpy(s, acc, 32);
}
void orc_pcg_advance(uint64_t *s, uint64_t dlo, uint64_t dhi) { pcg_advance(s, ((u128)dhi << 64) | dlo); }
/* RanluxPP.jump: x <- x * A^(2^k) (src/engines/ranlux.py:90-93); generalised to N chunks */
void orc_ranlux_advance_chunks(uint64_t *s, uint64_t nlo, uint64_t nhi) {
    rlx_init();
    uint64_t p[9];
    rlx_powmod(RLX_A, ((u128)nhi << 64) | nlo, p);
    rlx_mulmod(s, p, s);
}
void orc_ranlux_mulmod(const uint64_t *x, const uint64_t *y, uint64_t *out) { rlx_init(); rlx_mulmod(x, y, out); }
void orc_engine_generate(int eid, uint64_t *s, uint64_t *out, int n) { engine_generate(eid, s, out, n); }

/* 2^k steps of xorshift128+ / xoroshiro128 (src/jumps.py: T^N = (x^N mod p)(T), so the
 * same map as the matrix T^(2^k)); T by unit vectors, then k squarings */
typedef struct { uint64_t c[128][2]; } m128;
static void m128_vec(const m128 *m, const uint64_t v[2], uint64_t o[2]) {
    uint64_t a = 0, b = 0;
    for (int j = 0; j < 128; j++)
        if ((v[j >> 6] >> (j & 63)) & 1) { a ^= m->c[j][0]; b ^= m->c[j][1]; }
    o[0] = a; o[1] = b;
}
void orc_x128_jump_pow2k(int eid, uint64_t *s, int k) {
    static m128 t, sq;
    for (int j = 0; j < 128; j++) {
        uint64_t v[2] = {0, 0}, w[2];
        v[j >> 6] = 1ULL << (j & 63);
        uint64_t tmp[2] = {v[0], v[1]};
        if (eid == E_X128P) gen_x128p(tmp, w, 1); else gen_xoro(tmp, w, 1);
        t.c[j][0] = tmp[0]; t.c[j][1] = tmp[1];
    }
    for (int i = 0; i < k; i++) {
        for (int j = 0; j < 128; j++) m128_vec(&t, t.c[j], sq.c[j]);
        t = sq;
    }
    uint64_t o[2];
    m128_vec(&t, s, o);
    s[0] = o[0]; s[1] = o[1];
}

/* ---------------------------------------------------------------- threaded CPU baseline */
/* The --impl reference / cpu_baseline leg: P host threads, each running this
 * sequential restatement on its own disjoint substream (jumped / advanced /
 * counter-offset exactly as the GPU partitions), timed by the caller. */
typedef struct { orc_rng r; int dist; double fp[4]; uint64_t ip[4]; uint64_t n; void *out; } job_t;
static void *job_run(void *a) { job_t *j = (job_t *)a; orc_fill(&j->r, j->dist, j->fp, j->ip, j->n, j->out); return 0; }
int orc_fill_threads(orc_rng *rs, int nthreads, int dist, const double *fp, const uint64_t *ip,
                     uint64_t n_per_thread, void **outs) {
    pthread_t *th = (pthread_t *)calloc(nthreads, sizeof(pthread_t));
    job_t *jobs = (job_t *)calloc(nthreads, sizeof(job_t));
    for (int t = 0; t < nthreads; t++) {
        jobs[t].r = rs[t]; jobs[t].dist = dist; jobs[t].n = n_per_thread; jobs[t].out = outs[t];
        memcpy(jobs[t].fp, fp, 4 * sizeof(double)); memcpy(jobs[t].ip, ip, 4 * sizeof(uint64_t));
        pthread_create(&th[t], 0, job_run, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) { pthread_join(th[t], 0); rs[t] = jobs[t].r; }
    free(jobs);
    free(th);
    return 0;
}
size_t orc_sizeof_rng(void) { return sizeof(orc_rng); }
/* x^(2^k) mod c by k squarings (the jump-table entries, src/jumps.py:141-147) */
void orc_x_pow2k_mod(int k, const uint64_t *c5, uint64_t *out5) {
    poly_t c; memset(&c, 0, sizeof c); memcpy(c.w, c5, 40);
    poly_t r; memset(&r, 0, sizeof r); r.w[0] = 2;
    pmod(&r, &c);
    for (int i = 0; i < k; i++) { psquare(&r, &r); pmod(&r, &c); }
    memcpy(out5, r.w, 40);
}
/* RanluxPP.jump(k): x <- x * A^(2^k) mod m, src/engines/ranlux.py:90-93 */
void orc_ranlux_jump_pow2k(uint64_t *s, int k) {
    rlx_init();
    uint64_t p[9]; memcpy(p, RLX_A, 72);
    for (int i = 0; i < k; i++) rlx_mulmod(p, p, p);
    rlx_mulmod(s, p, s);
}
