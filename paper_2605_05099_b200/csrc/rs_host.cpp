// Host-side engine math: the reference's engine protocol (generate / seed_from /
// set_state validation) and its stream-positioning algebra (GF(2) jumps, LCG
// advance, counter offsets, ranlux powers). This is state bookkeeping for the
// 144-word WordBuffer and for computing fill start/end positions; the bulk fills
// themselves run only on the GPU (rs_fill.cu).
#include <cstring>
#include <mutex>
#include <vector>

#include "rs_internal.h"

namespace rs {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
void clear_error() { g_err.clear(); }

int state_words(int e) {  // engines/*.py STATE_WORDS
    switch (e) {
    case RS_ENG_X256PP: case RS_ENG_X256SS: case RS_ENG_PCG64: case RS_ENG_SFC64: return 4;
    case RS_ENG_X128P: case RS_ENG_XORO: case RS_ENG_SQUARES: return 2;
    case RS_ENG_PHILOX: case RS_ENG_CHACHA20: return 6;
    case RS_ENG_CWG128: return 8;
    case RS_ENG_RANLUX: return 9;
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD: case RS_ENG_SFC64_SIMD: return 32;
    default: return 0;
    }
}
int seed_words(int e) {  // engines/*.py SEED_WORDS
    switch (e) {
    case RS_ENG_X256PP: case RS_ENG_X256SS: case RS_ENG_PCG64: return 4;
    case RS_ENG_PHILOX: case RS_ENG_X128P: case RS_ENG_XORO: return 2;
    case RS_ENG_SQUARES: return 1;
    case RS_ENG_SFC64: case RS_ENG_SFC64_SIMD: return 3;
    case RS_ENG_CHACHA20: return 6;
    case RS_ENG_CWG128: return 8;
    case RS_ENG_RANLUX: return 9;
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD: return 4;
    default: return 0;
    }
}
int chunk(int e) {
    switch (e) {
    case RS_ENG_PHILOX: return 4;
    case RS_ENG_RANLUX: return 9;
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD: case RS_ENG_SFC64_SIMD: case RS_ENG_CHACHA20: return 8;
    default: return 1;
    }
}
bool simd_engine(int e) { return e == RS_ENG_X256PP_SIMD || e == RS_ENG_X256SS_SIMD || e == RS_ENG_SFC64_SIMD; }
bool known_engine(int e) { return state_words(e) > 0; }
bool device_engine(int e) { return known_engine(e); }

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// ------------------------------------------------------------------ xoshiro256
void x256_step_host(uint64_t s[4]) {  // xorfam.py:16-26
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = rotl(s[3], 45);
}

void mat_vec(const Mat256 &m, const uint64_t in[4], uint64_t out[4]) {
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int w = 0; w < 4; w++) {
        uint64_t v = in[w];
        while (v) {
            int b = __builtin_ctzll(v);
            v &= v - 1;
            const uint64_t *c = m.col[w * 64 + b];
            a0 ^= c[0]; a1 ^= c[1]; a2 ^= c[2]; a3 ^= c[3];
        }
    }
    out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3;
}

void mat_mul(const Mat256 &a, const Mat256 &b, Mat256 &out) {
    Mat256 *tmp = new Mat256;
    for (int j = 0; j < 256; j++) mat_vec(a, b.col[j], tmp->col[j]);
    memcpy(&out, tmp, sizeof(Mat256));
    delete tmp;
}

static std::vector<Mat256> *g_x256_pow2 = nullptr;
static std::once_flag g_x256_once;
static void build_x256_table() {
    g_x256_pow2 = new std::vector<Mat256>(256);
    Mat256 &t = (*g_x256_pow2)[0];
    for (int j = 0; j < 256; j++) {
        uint64_t s[4] = {0, 0, 0, 0};
        s[j / 64] = 1ULL << (j % 64);
        x256_step_host(s);
        memcpy(t.col[j], s, 32);
    }
    for (int k = 1; k < 256; k++) mat_mul((*g_x256_pow2)[k - 1], (*g_x256_pow2)[k - 1], (*g_x256_pow2)[k]);
}
const Mat256 &x256_pow2(int k) {
    std::call_once(g_x256_once, build_x256_table);
    return (*g_x256_pow2)[k];
}
void x256_advance(uint64_t s[4], u128 n) {
    if (n < 64) {
        for (int i = 0; i < (int)n; i++) x256_step_host(s);
        return;
    }
    for (int k = 0; k < 128 && n; k++, n >>= 1)
        if (n & 1) {
            uint64_t o[4];
            mat_vec(x256_pow2(k), s, o);
            memcpy(s, o, 32);
        }
}

// ------------------------------------------------------------------ xorshift128+ / xoroshiro128
// (xorfam.py:29-42, 127-170). Their 128-bit linear steps reuse the 256-bit matrix
// type with words 2 and 3 (and columns 128..255) left zero.
void x128p_step_host(uint64_t s[2]) {  // xorfam.py:29-34
    uint64_t s1 = s[0], s0 = s[1];
    s1 ^= s1 << 23;
    s[0] = s0;
    s[1] = s1 ^ s0 ^ (s1 >> 18) ^ (s0 >> 5);
}
void xoro_step_host(uint64_t s[2]) {  // xorfam.py:37-42
    uint64_t s0 = s[0], s1 = s[1] ^ s[0];
    s[0] = rotl(s0, 49) ^ s1 ^ (s1 << 21);
    s[1] = rotl(s1, 28);
}
static std::vector<Mat256> *g_x128_pow2[2] = {nullptr, nullptr};
static std::once_flag g_x128_once[2];
static void build_x128_table(int f) {  // f = 0: x128+, 1: xoro
    g_x128_pow2[f] = new std::vector<Mat256>(128);
    Mat256 &t = (*g_x128_pow2[f])[0];
    memset(&t, 0, sizeof t);
    for (int j = 0; j < 128; j++) {
        uint64_t v[2] = {0, 0};
        v[j / 64] = 1ULL << (j % 64);
        if (f == 0) x128p_step_host(v); else xoro_step_host(v);
        t.col[j][0] = v[0];
        t.col[j][1] = v[1];
    }
    for (int k = 1; k < 128; k++) mat_mul((*g_x128_pow2[f])[k - 1], (*g_x128_pow2[f])[k - 1], (*g_x128_pow2[f])[k]);
}
const Mat256 &x128_pow2(int e, int k) {
    int f = e == RS_ENG_XORO ? 1 : 0;
    std::call_once(g_x128_once[f], build_x128_table, f);
    return (*g_x128_pow2[f])[k];
}
void x128_advance(int e, uint64_t s[2], u128 n) {
    if (n < 64) {
        for (int i = 0; i < (int)n; i++) { if (e == RS_ENG_XORO) xoro_step_host(s); else x128p_step_host(s); }
        return;
    }
    for (int k = 0; k < 128 && n; k++, n >>= 1)
        if (n & 1) {
            uint64_t in[4] = {s[0], s[1], 0, 0}, o[4];
            mat_vec(x128_pow2(e, k), in, o);
            s[0] = o[0];
            s[1] = o[1];
        }
}

// squares64, counter.py:12-48: word = f(counter * key), one per counter value
static inline uint64_t sq_swap(uint64_t x) { return (x >> 32) | (x << 32); }
uint64_t squares_word(uint64_t ctr, uint64_t key) {
    uint64_t x = ctr * key, y = x, z = y + key;
    x = sq_swap(x * x + y);
    x = sq_swap(x * x + z);
    x = sq_swap(x * x + y);
    uint64_t t = x = x * x + z;
    x = sq_swap(x);
    return t ^ ((x * x + y) >> 32);
}

// ChaCha20, counter.py:170-207: state words [k0..k3, nonce0|nonce1<<32, nonce2|counter<<32]
static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
void chacha_block(const uint64_t *s, uint32_t counter, uint64_t *out) {
    uint32_t st[16] = {0x61707865u, 0x3320646Eu, 0x79622D32u, 0x6B206574u};
    for (int i = 0; i < 4; i++) { st[4 + 2 * i] = (uint32_t)s[i]; st[5 + 2 * i] = (uint32_t)(s[i] >> 32); }
    st[12] = counter;
    st[13] = (uint32_t)s[4];
    st[14] = (uint32_t)(s[4] >> 32);
    st[15] = (uint32_t)s[5];
    uint32_t x[16];
    memcpy(x, st, sizeof x);
    static const int QR[8][4] = {{0, 4, 8, 12}, {1, 5, 9, 13}, {2, 6, 10, 14}, {3, 7, 11, 15},
                                 {0, 5, 10, 15}, {1, 6, 11, 12}, {2, 7, 8, 13}, {3, 4, 9, 14}};
    for (int r = 0; r < 10; r++)
        for (int q = 0; q < 8; q++) {
            uint32_t &a = x[QR[q][0]], &b = x[QR[q][1]], &c = x[QR[q][2]], &d = x[QR[q][3]];
            a += b; d = rotl32(d ^ a, 16);
            c += d; b = rotl32(b ^ c, 12);
            a += b; d = rotl32(d ^ a, 8);
            c += d; b = rotl32(b ^ c, 7);
        }
    for (int i = 0; i < 8; i++)
        out[i] = (uint64_t)(x[2 * i] + st[2 * i]) | ((uint64_t)(x[2 * i + 1] + st[2 * i + 1]) << 32);
}

// ------------------------------------------------------------------ PCG64
void pcg_affine(u128 inc, u128 n, u128 &mul, u128 &add) {  // pcg.py:41-55
    u128 am = 1, ap = 0, cm = PCG_MULT, cp = inc;
    while (n) {
        if (n & 1) { am *= cm; ap = ap * cm + cp; }
        cp = (cm + 1) * cp;
        cm *= cm;
        n >>= 1;
    }
    mul = am; add = ap;
}
void pcg_advance(uint64_t s[4], u128 n) {
    u128 inc = ((u128)s[3] << 64) | s[2], m, a;
    pcg_affine(inc, n, m, a);
    u128 st = ((u128)s[1] << 64) | s[0];
    st = st * m + a;
    s[0] = (uint64_t)st; s[1] = (uint64_t)(st >> 64);
}

// ------------------------------------------------------------------ Philox
void philox_add(uint64_t c[4], u128 blocks) {
    u128 lo = (u128)c[0] + (uint64_t)blocks;
    c[0] = (uint64_t)lo;
    u128 carry = (lo >> 64) + (uint64_t)(blocks >> 64);
    for (int i = 1; i < 4 && carry; i++) {
        u128 t = (u128)c[i] + (uint64_t)carry;
        c[i] = (uint64_t)t;
        carry = (carry >> 64) + (t >> 64);
    }
}
static void philox_block(const uint64_t *ctr, const uint64_t *key, uint64_t *o) {
    uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        u128 p0 = (u128)0xD2E7470EE14C6C93ULL * x0, p1 = (u128)0xCA5A826395121157ULL * x2;
        uint64_t y0 = (uint64_t)(p1 >> 64) ^ x1 ^ k0, y2 = (uint64_t)(p0 >> 64) ^ x3 ^ k1;
        x1 = (uint64_t)p1; x3 = (uint64_t)p0; x0 = y0; x2 = y2;
        k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL;
    }
    o[0] = x0; o[1] = x1; o[2] = x2; o[3] = x3;
}

// ------------------------------------------------------------------ ranlux++
// m = 2^576 - 2^240 + 1 as 9 limbs
static const uint64_t RLX_M[9] = {1ULL, 0, 0, 0xFFFF000000000000ULL, ~0ULL, ~0ULL, ~0ULL, ~0ULL, ~0ULL};
const uint64_t *rlx_modulus() { return RLX_M; }

static bool ge_m(const uint64_t *x, int nl) {  // x (nl >= 9 limbs) >= m ?
    for (int i = nl - 1; i >= 9; i--) if (x[i]) return true;
    for (int i = 8; i >= 0; i--) if (x[i] != RLX_M[i]) return x[i] > RLX_M[i];
    return true;
}
static void sub_m(uint64_t *x, int nl) {
    uint64_t br = 0;
    for (int i = 0; i < nl; i++) {
        uint64_t m = i < 9 ? RLX_M[i] : 0;
        u128 d = (u128)x[i] - m - br;
        x[i] = (uint64_t)d;
        br = (uint64_t)(d >> 64) & 1;
    }
}
// r[nl] = a[0..8] + (h << 240) - h, h has hl limbs; requires result >= 0
static void fold(const uint64_t *a, const uint64_t *h, int hl, uint64_t *r, int nl) {
    uint64_t sh[16] = {0};
    for (int i = 0; i < hl; i++) {
        sh[i + 3] |= h[i] << 48;
        sh[i + 4] |= h[i] >> 16;
    }
    u128 acc = 0;
    int64_t borrow = 0;
    for (int i = 0; i < nl; i++) {
        u128 t = (u128)(i < 9 ? a[i] : 0) + sh[i] + (uint64_t)acc;
        acc = t >> 64;
        uint64_t lo = (uint64_t)t;
        uint64_t hv = i < hl ? h[i] : 0;
        u128 d = (u128)lo - hv - (uint64_t)borrow;
        r[i] = (uint64_t)d;
        borrow = (int64_t)((d >> 64) & 1);
    }
}
void rlx_mulmod(const uint64_t *x, const uint64_t *y, uint64_t *out) {
    uint64_t p[18] = {0};
    for (int i = 0; i < 9; i++) {
        u128 c = 0;
        for (int j = 0; j < 9; j++) {
            u128 t = (u128)x[i] * y[j] + p[i + j] + (uint64_t)c;
            p[i + j] = (uint64_t)t;
            c = t >> 64;
        }
        p[i + 9] = (uint64_t)c;
    }
    uint64_t r[13];
    fold(p, p + 9, 9, r, 13);        // < 2^817
    uint64_t r2[10];
    fold(r, r + 9, 4, r2, 10);       // < 2^576 + 2^481
    while (ge_m(r2, 10)) sub_m(r2, 10);
    memcpy(out, r2, 72);
}
static uint64_t g_rlx_pow2[256][9];
static std::once_flag g_rlx_once;
static void build_rlx() {
    // a = b^-1 mod m = m - (m-1)/2^24 ;  (m-1)/2^24 = 2^552 - 2^216   (ranlux.py:16-19)
    uint64_t q[9] = {0};
    q[8] = 1ULL << 40;
    uint64_t br = 0;
    uint64_t t[9] = {0};
    t[3] = 1ULL << 24;
    for (int i = 0; i < 9; i++) { u128 d = (u128)q[i] - t[i] - br; q[i] = (uint64_t)d; br = (uint64_t)(d >> 64) & 1; }
    uint64_t a1[9];
    br = 0;
    for (int i = 0; i < 9; i++) { u128 d = (u128)RLX_M[i] - q[i] - br; a1[i] = (uint64_t)d; br = (uint64_t)(d >> 64) & 1; }
    // A = a1^2048 = a1 squared 11 times
    for (int i = 0; i < 11; i++) rlx_mulmod(a1, a1, a1);
    memcpy(g_rlx_pow2[0], a1, 72);
    for (int k = 1; k < 256; k++) rlx_mulmod(g_rlx_pow2[k - 1], g_rlx_pow2[k - 1], g_rlx_pow2[k]);
}
void rlx_pow2k_A(int k, uint64_t *out) {
    std::call_once(g_rlx_once, build_rlx);
    memcpy(out, g_rlx_pow2[k], 72);
}
void rlx_pow_A(u128 e, uint64_t *out) {
    std::call_once(g_rlx_once, build_rlx);
    uint64_t r[9] = {1, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 128 && e; k++, e >>= 1)
        if (e & 1) rlx_mulmod(r, g_rlx_pow2[k], r);
    memcpy(out, r, 72);
}
void rlx_reduce_seed(const uint64_t *w, uint64_t *out) {  // ranlux.py:106-110
    uint64_t x[10];
    memcpy(x, w, 72);
    x[9] = 0;
    while (ge_m(x, 10)) sub_m(x, 10);
    bool zero = true;
    for (int i = 0; i < 9; i++) zero &= x[i] == 0;
    if (zero) x[0] = 1;
    memcpy(out, x, 72);
}

// ------------------------------------------------------------------ generic
void engine_generate(int e, uint64_t *s, uint64_t *out, int n) {
    switch (e) {
    case RS_ENG_X256SS:
        for (int i = 0; i < n; i++) { out[i] = rotl(s[1] * 5, 7) * 9; x256_step_host(s); }
        break;
    case RS_ENG_X256PP:
        for (int i = 0; i < n; i++) { out[i] = rotl(s[0] + s[3], 23) + s[0]; x256_step_host(s); }
        break;
    case RS_ENG_PCG64: {
        u128 st = ((u128)s[1] << 64) | s[0], inc = ((u128)s[3] << 64) | s[2];
        for (int i = 0; i < n; i++) {
            uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st | 1;
            hi ^= hi >> 32; hi *= PCG_MULT; hi ^= hi >> 48;
            out[i] = hi * lo;
            st = st * PCG_MULT + inc;
        }
        s[0] = (uint64_t)st; s[1] = (uint64_t)(st >> 64);
        break;
    }
    case RS_ENG_PHILOX:
        for (int b = 0; b < n / 4; b++) { philox_block(s, s + 4, out + 4 * b); philox_add(s, 1); }
        break;
    case RS_ENG_SFC64: {
        uint64_t a = s[0], b = s[1], c = s[2], w = s[3];
        for (int i = 0; i < n; i++) {
            uint64_t r = a + b + w;
            w += 1; a = b ^ (b >> 11); b = c + (c << 3); c = rotl(c, 24) + r;
            out[i] = r;
        }
        s[0] = a; s[1] = b; s[2] = c; s[3] = w;
        break;
    }
    case RS_ENG_RANLUX: {
        uint64_t A[9];
        rlx_pow2k_A(0, A);
        for (int c = 0; c < n / 9; c++) { rlx_mulmod(s, A, s); memcpy(out + 9 * c, s, 72); }
        break;
    }
    case RS_ENG_X128P:  // xorfam.py:137-146
        for (int i = 0; i < n; i++) { out[i] = s[0] + s[1]; x128p_step_host(s); }
        break;
    case RS_ENG_XORO:  // xorfam.py:160-168
        for (int i = 0; i < n; i++) { out[i] = rotl(s[0] + s[1], 17) + s[0]; xoro_step_host(s); }
        break;
    case RS_ENG_SQUARES:  // state [counter, key]
        for (int i = 0; i < n; i++) out[i] = squares_word(s[0]++, s[1]);
        break;
    case RS_ENG_CHACHA20:  // the caller checked the 32-bit block counter (counter.py:209-216)
        for (int b = 0; b < n / 8; b++) {
            uint32_t ctr = (uint32_t)(s[5] >> 32);
            chacha_block(s, ctr, out + 8 * b);
            s[5] = (s[5] & 0xFFFFFFFFULL) | ((uint64_t)(ctr + 1) << 32);
        }
        break;
    case RS_ENG_CWG128: {  // cwg.py:28-36: state words x, weyl, extra, inc (lo, hi each)
        u128 x = ((u128)s[1] << 64) | s[0], weyl = ((u128)s[3] << 64) | s[2];
        u128 extra = ((u128)s[5] << 64) | s[4], inc = ((u128)s[7] << 64) | s[6];
        for (int i = 0; i < n; i++) {
            weyl += x;
            extra += inc;
            x = ((x >> 1) * (weyl | 1)) ^ extra;
            out[i] = (uint64_t)(weyl >> 96) ^ (uint64_t)x;
        }
        s[0] = (uint64_t)x; s[1] = (uint64_t)(x >> 64); s[2] = (uint64_t)weyl; s[3] = (uint64_t)(weyl >> 64);
        s[4] = (uint64_t)extra; s[5] = (uint64_t)(extra >> 64);
        break;
    }
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD: case RS_ENG_SFC64_SIMD: {
        // interleave.py:71-76: word i = lane (i mod 8) at step i / 8; state is lane-major
        int base = e == RS_ENG_X256PP_SIMD ? RS_ENG_X256PP : e == RS_ENG_X256SS_SIMD ? RS_ENG_X256SS : RS_ENG_SFC64;
        uint64_t w[1];
        for (int i = 0; i < n; i++) {
            engine_generate(base, s + 4 * (i & 7), w, 1);
            out[i] = w[0];
        }
        break;
    }
    }
}

bool engine_advance_words(int e, uint64_t *s, u128 words) {
    switch (e) {
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD:  // every lane advances words/8 steps
        if (words % 8) return false;
        for (int k = 0; k < 8; k++) x256_advance(s + 4 * k, words / 8);
        return true;
    case RS_ENG_X256SS: case RS_ENG_X256PP: x256_advance(s, words); return true;
    case RS_ENG_PCG64: pcg_advance(s, words); return true;
    case RS_ENG_PHILOX:
        if (words % 4) return false;
        philox_add(s, words / 4);
        return true;
    case RS_ENG_RANLUX: {
        if (words % 9) return false;
        uint64_t p[9];
        rlx_pow_A(words / 9, p);
        rlx_mulmod(s, p, s);
        return true;
    }
    case RS_ENG_X128P: case RS_ENG_XORO: x128_advance(e, s, words); return true;
    case RS_ENG_SQUARES: s[0] += (uint64_t)words; return true;
    case RS_ENG_CHACHA20: {  // 32-bit block counter: positions up to block 2^32 exist
        if (words % 8) return false;
        u128 c = (u128)(s[5] >> 32) + words / 8;
        if (c > ((u128)1 << 32)) return false;
        if (c == ((u128)1 << 32)) return false;  // not representable in the state word
        s[5] = (s[5] & 0xFFFFFFFFULL) | ((uint64_t)c << 32);
        return true;
    }
    default: return false;  // sfc64 / cwg128 have no skip-ahead (rng.py:162-163)
    }
}

// SeedSequenceFE128 (seeding.py:21-116), numpy SeedSequence(pool_size=4) mixing
void seed_words_fe128(const uint64_t *ent, int nent, const uint64_t *spawn, int nspawn, uint64_t *out,
                      int nout) {
    std::vector<uint32_t> a;
    for (int i = 0; i < nent; i++) { a.push_back((uint32_t)ent[i]); a.push_back((uint32_t)(ent[i] >> 32)); }
    if (nspawn > 0) while (a.size() < 4) a.push_back(0);
    for (int i = 0; i < nspawn; i++) { a.push_back((uint32_t)spawn[i]); a.push_back((uint32_t)(spawn[i] >> 32)); }
    uint32_t hc = 0x43B0D7E5u;
    auto hashed = [&](uint32_t v) {
        v ^= hc; hc *= 0x931E8875u; v *= hc; v ^= v >> 16; return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
        uint32_t r = x * 0xCA01F9DDu - y * 0x4973F715u; return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; i++) pool[i] = hashed(i < (int)a.size() ? a[i] : 0);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashed(pool[s]));
    for (size_t s = 4; s < a.size(); s++)
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashed(a[s]));
    uint32_t hb = 0x8B51F9DDu;
    for (int i = 0; i < nout; i++) {
        uint32_t w[2];
        for (int h = 0; h < 2; h++) {
            uint32_t v = pool[(2 * i + h) & 3] ^ hb;
            hb *= 0x58F38DEDu; v *= hb; v ^= v >> 16; w[h] = v;
        }
        out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    }
}

// lanes of the xoshiro interleaved engines: lane k = base jumped k * 2^253 (interleave.py:201-208)
static void x256_simd_lanes(uint64_t *s) {
    for (int k = 1; k < 8; k++) mat_vec(x256_pow2(253), s + 4 * (k - 1), s + 4 * k);
}
// sfc64 lanes: the Weyl counter offset by k * 2^61 (interleave.py:225-228)
static void sfc_simd_lanes(uint64_t *s) {
    for (int k = 1; k < 8; k++) {
        memcpy(s + 4 * k, s, 24);
        s[4 * k + 3] = s[3] + (uint64_t)k * (1ULL << 61);
    }
}
void engine_simd_from_base(int e, uint64_t *s) {
    if (e == RS_ENG_SFC64_SIMD) sfc_simd_lanes(s);
    else x256_simd_lanes(s);
}

void engine_seed_from(int e, const uint64_t *w, uint64_t *s) {
    switch (e) {
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD:  // interleave.py:127-130
        engine_seed_from(RS_ENG_X256PP, w, s);
        x256_simd_lanes(s);
        break;
    case RS_ENG_SFC64_SIMD:  // interleave.py:212-215
        engine_seed_from(RS_ENG_SFC64, w, s);
        sfc_simd_lanes(s);
        break;
    case RS_ENG_X256PP: case RS_ENG_X256SS:  // xorfam.py:66-70
        memcpy(s, w, 32);
        if (!(s[0] | s[1] | s[2] | s[3])) s[0] = 1;
        break;
    case RS_ENG_PCG64: s[0] = w[0]; s[1] = w[1]; s[2] = w[2] | 1; s[3] = w[3]; break;  // pcg.py:81-84
    case RS_ENG_PHILOX: s[0] = s[1] = s[2] = s[3] = 0; s[4] = w[0]; s[5] = w[1]; break;  // counter.py:139-141
    case RS_ENG_SFC64: s[0] = w[0]; s[1] = w[1]; s[2] = w[2]; s[3] = 1; break;  // sfc.py:53-55
    case RS_ENG_RANLUX: rlx_reduce_seed(w, s); break;  // ranlux.py:106-110
    case RS_ENG_X128P: case RS_ENG_XORO:  // xorfam.py:66-70
        s[0] = w[0]; s[1] = w[1];
        if (!(s[0] | s[1])) s[0] = 1;
        break;
    case RS_ENG_SQUARES: s[0] = 0; s[1] = w[0]; break;  // counter.py:63-65
    case RS_ENG_CHACHA20:  // counter.py:228-233: key, 96-bit nonce, counter 0
        memcpy(s, w, 40);
        s[5] = w[5] & 0xFFFFFFFFULL;
        break;
    case RS_ENG_CWG128: memcpy(s, w, 64); s[6] |= 1; break;  // cwg.py:62-67
    }
}

}  // namespace rs

// ------------------------------------------------------------------ C ABI (host part)
using namespace rs;

extern "C" {

int32_t rs_abi_version(void) { return RS_ABI_VERSION; }
const char *rs_last_error(void) { return g_err.c_str(); }
int32_t rs_engine_supported(int32_t e) { return device_engine(e) ? 1 : 0; }
int32_t rs_engine_state_words(int32_t e) { return state_words(e); }
int32_t rs_engine_seed_words(int32_t e) { return seed_words(e); }
int32_t rs_engine_chunk(int32_t e) { return known_engine(e) ? chunk(e) : 0; }

rs_status rs_seed_words(const uint64_t *entropy, int32_t ne, const uint64_t *spawn, int32_t ns, uint64_t *out,
                        int32_t nout) {
    if (ne < 0 || ns < 0 || nout < 0) { set_error("negative word count"); return RS_ERR_VALUE; }
    seed_words_fe128(entropy, ne, spawn, ns, out, nout);
    clear_error();
    return RS_OK;
}

rs_status rs_engine_seed_from(int32_t e, const uint64_t *w, uint64_t *state) {
    if (!known_engine(e)) { set_error("engine not on the B200 path"); return RS_ERR_UNSUPPORTED; }
    engine_seed_from(e, w, state);
    clear_error();
    return RS_OK;
}

rs_status rs_engine_seed(int32_t e, const uint64_t *entropy, int32_t ne, const uint64_t *spawn, int32_t ns,
                         uint64_t *state) {
    if (!known_engine(e)) { set_error("engine not on the B200 path"); return RS_ERR_UNSUPPORTED; }
    uint64_t w[16];
    seed_words_fe128(entropy, ne, spawn, ns, w, seed_words(e));  // seeding.py:115-116
    engine_seed_from(e, w, state);
    clear_error();
    return RS_OK;
}

rs_status rs_engine_check_state(int32_t e, const uint64_t *w) {
    // set_state validation: xorfam.py:57-64, pcg.py:68-76, ranlux.py:98-104
    if (!known_engine(e)) { set_error("engine not on the B200 path"); return RS_ERR_UNSUPPORTED; }
    if (e == RS_ENG_X256PP || e == RS_ENG_X256SS) {
        if (!(w[0] | w[1] | w[2] | w[3])) {
            set_error(std::string("all-zero state is invalid for ") + (e == RS_ENG_X256PP ? "x256++" : "x256**"));
            return RS_ERR_VALUE;
        }
    } else if (e == RS_ENG_X256PP_SIMD || e == RS_ENG_X256SS_SIMD) {  // interleave.py:120-123
        for (int k = 0; k < 8; k++)
            if (!(w[4 * k] | w[4 * k + 1] | w[4 * k + 2] | w[4 * k + 3])) {
                set_error("lane " + std::to_string(k) + " state must not be all zero");
                return RS_ERR_VALUE;
            }
    } else if (e == RS_ENG_X128P || e == RS_ENG_XORO) {
        if (!(w[0] | w[1])) {
            set_error(std::string("all-zero state is invalid for ") + (e == RS_ENG_X128P ? "x128+" : "xoro++"));
            return RS_ERR_VALUE;
        }
    } else if (e == RS_ENG_CWG128) {  // cwg.py:56-57
        if (!(w[6] & 1)) { set_error("cwg128 Weyl increment must be odd"); return RS_ERR_VALUE; }
    } else if (e == RS_ENG_PCG64) {
        if (!(w[2] & 1)) { set_error("pcg64 increment must be odd"); return RS_ERR_VALUE; }
    } else if (e == RS_ENG_RANLUX) {
        uint64_t x[10];
        memcpy(x, w, 72);
        x[9] = 0;
        if (ge_m(x, 10)) { set_error("ranlux++ residue must be < 2^576 - 2^240 + 1"); return RS_ERR_VALUE; }
    }
    clear_error();
    return RS_OK;
}

rs_status rs_engine_generate(int32_t e, uint64_t *state, uint64_t *out, int32_t n) {
    if (!known_engine(e)) { set_error("engine not on the B200 path"); return RS_ERR_UNSUPPORTED; }
    if (n < 0 || n % chunk(e)) { set_error("generate count must be a multiple of the engine chunk"); return RS_ERR_VALUE; }
    if (e == RS_ENG_CHACHA20 && (state[5] >> 32) + (uint64_t)(n / 8) > 0xFFFFFFFFULL + 1) {
        set_error("chacha20 stream exhausted");  // counter.py:212-213 (OverflowError)
        return RS_ERR_VALUE;
    }
    engine_generate(e, state, out, n);
    clear_error();
    return RS_OK;
}

rs_status rs_engine_jump(int32_t e, uint64_t *state, int32_t k) {
    // Rng.jump(k) semantics, rng.py:135-164: x256 family: 2^k steps; pcg64: advance(2^k);
    // ranlux++: multiply by A^(2^k) (2^k chunks of 9 words).
    if (k < 0 || k > 255) { set_error("jump exponent out of range"); return RS_ERR_VALUE; }
    switch (e) {
    case RS_ENG_X256PP: case RS_ENG_X256SS: {
        uint64_t o[4];
        mat_vec(x256_pow2(k), state, o);
        memcpy(state, o, 32);
        break;
    }
    case RS_ENG_X256PP_SIMD: case RS_ENG_X256SS_SIMD:  // per-lane jump, interleave.py:132-139
        for (int l = 0; l < 8; l++) {
            uint64_t o[4];
            mat_vec(x256_pow2(k), state + 4 * l, o);
            memcpy(state + 4 * l, o, 32);
        }
        break;
    case RS_ENG_PCG64:
        if (k >= 128) { uint64_t keep[4]; memcpy(keep, state, 32); (void)keep; break; }  // 2^k = 0 mod 2^128
        pcg_advance(state, (u128)1 << k);
        break;
    case RS_ENG_RANLUX: {
        uint64_t p[9];
        rlx_pow2k_A(k, p);
        rlx_mulmod(state, p, state);
        break;
    }
    case RS_ENG_X128P: case RS_ENG_XORO: {  // 2^k steps, jumps.py FAMILY_JUMPS (k < 128)
        if (k >= 128) { set_error("jump exponent out of range"); return RS_ERR_VALUE; }
        uint64_t in[4] = {state[0], state[1], 0, 0}, o[4];
        mat_vec(x128_pow2(e, k), in, o);
        state[0] = o[0];
        state[1] = o[1];
        break;
    }
    default:
        set_error("jump unsupported for this engine");
        return RS_ERR_VALUE;
    }
    clear_error();
    return RS_OK;
}

rs_status rs_engine_advance_words(int32_t e, uint64_t *state, uint64_t lo, uint64_t hi) {
    if (!engine_advance_words(e, state, ((u128)hi << 64) | lo)) {
        set_error("advance unsupported for this engine / distance");
        return RS_ERR_VALUE;
    }
    clear_error();
    return RS_OK;
}

rs_status rs_pcg_advance(uint64_t *state, uint64_t lo, uint64_t hi) {
    pcg_advance(state, ((u128)hi << 64) | lo);
    clear_error();
    return RS_OK;
}

}  // extern "C"
