// Device building blocks for the bulk stream-fill kernels (sm_100a).
//
//  * engines: xoshiro256**/++, PCG64-DXSM, Philox-4x64-10, sfc64, ranlux++ --
//    one 64-bit word per next(), same words as the reference generate()
//    (engines/xorfam.py:88-124, pcg.py:25-39, counter.py:98-121, sfc.py:25-36,
//    ranlux.py:36-88);
//  * det_exp / det_log: fdlibm kernels op for op (detmath.py:59-163). The whole
//    library is compiled with -fmad=false so no multiply-add is contracted:
//    results are bit-identical to CPython's IEEE doubles;
//  * parsers: the reference samplers restated as word-at-a-time state machines
//    (continuous.py:40-93 ziggurats, :183-218 gamma/beta, discrete.py:20-39 Lemire)
//    so a segment of the word stream can be parsed by one thread. A "boundary"
//    is the position right after an emitted sample -- the only point where the
//    reference's call stack carries no state;
//  * VecWriter: per-lane contiguous runs written with 256-bit stores (STG.256).
#pragma once
#include <cstdint>

#include "rs_tables_dev.cuh"

typedef uint64_t u64;
typedef unsigned int u32;

#define RS_DEV __device__ __forceinline__

RS_DEV u64 rotl64(u64 x, int k) { return (x << k) | (x >> (64 - k)); }

// ----------------------------------------------------------------------------- engines

// 32-bit halves of a 64-bit register, and funnel-shift rotates (one SHF per half)
RS_DEV void split64(u64 x, u32 &lo, u32 &hi) { asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(x)); }
RS_DEV u64 join64(u32 lo, u32 hi) {
    u64 x;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(lo), "r"(hi));
    return x;
}
RS_DEV u32 shfl_l(u32 a, u32 b, int k) {  // high word of (b:a) << k
    u32 r;
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(k));
    return r;
}
// x * c for a small constant c on the FMA pipe: IMAD.WIDE.U32 + IMAD (ptxas turns a
// C-level x*5 into three wide multiplies, or into LEAs that load the ALU pipe)
RS_DEV void mulc_fma(u32 lo, u32 hi, u32 c, u32 &rlo, u32 &rhi) {
    asm("{\n\t.reg .u64 w;\n\t.reg .u32 wl, wh;\n\t"
        "mul.wide.u32 w, %2, %4;\n\tmov.b64 {wl, wh}, w;\n\t"
        "mad.lo.u32 %1, %3, %4, wh;\n\tmov.b32 %0, wl;\n\t}"
        : "=r"(rlo), "=r"(rhi) : "r"(lo), "r"(hi), "r"(c));
}

template <bool SS>
struct EngX256 {  // xorfam.py:88-124
    u64 s0, s1, s2, s3;
    RS_DEV void load(const u64 *p) { s0 = p[0]; s1 = p[1]; s2 = p[2]; s3 = p[3]; }
#ifndef RS_X256_C
    // Per 32-bit halves, so the step costs 13 ALU instructions (8 LOP3, 5 SHF) and
    // the multiplies (x256**) or adds (x256++) go to the FMA pipe: the two pipes
    // each take one warp instruction per 2 cycles, and the C form put ~20 on ALU.
    RS_DEV u64 next() {
        u32 a0, b0, a1, b1, a2, b2, a3, b3;
        split64(s0, a0, b0);
        split64(s1, a1, b1);
        split64(s2, a2, b2);
        split64(s3, a3, b3);
        u32 rl, rh;
        if (SS) {  // rotl(s1 * 5, 7) * 9
            u32 ml, mh;
            mulc_fma(a1, b1, 5u, ml, mh);
            u32 ql = shfl_l(mh, ml, 7), qh = shfl_l(ml, mh, 7);
            mulc_fma(ql, qh, 9u, rl, rh);
        } else {   // rotl(s0 + s3, 23) + s0
            u64 p = s0 + s3;
            u32 pl, ph;
            split64(p, pl, ph);
            u32 ql = shfl_l(ph, pl, 23), qh = shfl_l(pl, ph, 23);
            split64(join64(ql, qh) + s0, rl, rh);
        }
        u32 tl = a1 << 17, th = shfl_l(a1, b1, 17);           // t = s1 << 17
        u32 n2l = a2 ^ a0 ^ tl, n2h = b2 ^ b0 ^ th;           // s2 ^= s0; ... s2 ^= t
        u32 n1l = a1 ^ a2 ^ a0, n1h = b1 ^ b2 ^ b0;           // s1 ^= s2 (new s2 without t)
        u32 x3l = a3 ^ a1, x3h = b3 ^ b1;                     // s3 ^= s1
        u32 n0l = a0 ^ x3l, n0h = b0 ^ x3h;                   // s0 ^= s3
        u32 n3l = shfl_l(x3l, x3h, 45 - 32), n3h = shfl_l(x3h, x3l, 45 - 32);  // rotl(s3, 45)
        s0 = join64(n0l, n0h);
        s1 = join64(n1l, n1h);
        s2 = join64(n2l, n2h);
        s3 = join64(n3l, n3h);
        return join64(rl, rh);
    }
#else
    RS_DEV u64 next() {
        u64 r = SS ? rotl64(s1 * 5ULL, 7) * 9ULL : rotl64(s0 + s3, 23) + s0;
        u64 t = s1 << 17;
        s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t;
        s3 = rotl64(s3, 45);
        return r;
    }
#endif
};

#define RS_PCG_MULT 0xDA942042E4DD58B5ULL
struct EngPcg {  // pcg.py:25-39 (DXSM of the pre-step state; 64-bit "cheap" multiplier)
    u64 slo, shi, ilo, ihi;
    RS_DEV u64 next() {
        u64 hi = shi, lo = slo | 1ULL;
        hi ^= hi >> 32;
        hi *= RS_PCG_MULT;
        hi ^= hi >> 48;
        u64 r = hi * lo;
        // state * M + inc as one 128-bit expression: the carry into the high word rides the
        // add chain (IADD3.X) instead of a compare + select (pcg64 raw 2^30 1.71 -> 1.61 ms,
        // normals 2^28 2.01 -> 1.95 ms)
        typedef unsigned __int128 U;
        const U st = (((U)shi << 64) | slo) * (U)RS_PCG_MULT + (((U)ihi << 64) | ilo);
        slo = (u64)st; shi = (u64)(st >> 64);
        return r;
    }
    // state <- mul*state + add (mod 2^128)
    RS_DEV void affine(u64 mlo, u64 mhi, u64 alo, u64 ahi) {
        u64 plo = slo * mlo;
        u64 phi = __umul64hi(slo, mlo) + slo * mhi + shi * mlo;
        u64 r = plo + alo;
        phi += ahi + (r < plo ? 1ULL : 0ULL);
        slo = r; shi = phi;
    }
};

// the same product as a 32-bit multiply-add carry chain (IMAD / IMAD.HI with .X)
RS_DEV void mul64x64_cc(u64 a, u64 b, u64 &lo, u64 &hi) {
    u32 a0 = (u32)a, a1 = (u32)(a >> 32), b0 = (u32)b, b1 = (u32)(b >> 32);
    u32 r0, r1, r2, r3;
    asm("{\n\t"
        "mul.lo.u32 %0, %4, %6;\n\t"
        "mul.hi.u32 %1, %4, %6;\n\t"
        "mad.lo.cc.u32 %1, %5, %6, %1;\n\t"
        "madc.hi.u32 %2, %5, %6, 0;\n\t"
        "mad.lo.cc.u32 %1, %4, %7, %1;\n\t"
        "madc.hi.cc.u32 %2, %4, %7, %2;\n\t"
        "madc.hi.u32 %3, %5, %7, 0;\n\t"
        "mad.lo.cc.u32 %2, %5, %7, %2;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "}"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    lo = ((u64)r1 << 32) | r0;
    hi = ((u64)r3 << 32) | r2;
}

RS_DEV u64 mulw(u32 a, u32 b) {
    u64 r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
// 64x64 -> 128 product: four 32x32->64 products (IMAD.WIDE.U32, 4 cycles each on the
// fmaheavy pipe -- 16 cycles per product is the floor) and the column sums as 64-bit
// adds of zero-extended halves, which ptxas splits between the ALU pipe (IADD3 with
// two carries) and the FMA pipe. Measured the fastest of five formulations on B200
// (profiles/README.md, round 1: Philox u01 2^30 3.82 -> 3.69 ms).
RS_DEV void mul64x64(u64 a, u64 b, u64 &lo, u64 &hi) {
    u32 a0 = (u32)a, a1 = (u32)(a >> 32), b0 = (u32)b, b1 = (u32)(b >> 32);
    u64 p00 = mulw(a0, b0), p01 = mulw(a0, b1), p10 = mulw(a1, b0), p11 = mulw(a1, b1);
    u64 mid = (p00 >> 32) + (u64)(u32)p01 + (u64)(u32)p10;
    lo = (mid << 32) | (u64)(u32)p00;
    hi = p11 + (p01 >> 32) + (p10 >> 32) + (mid >> 32);
}

RS_DEV void philox4x64_10(u64 c0, u64 c1, u64 c2, u64 c3, u64 k0, u64 k1, u64 &o0, u64 &o1, u64 &o2, u64 &o3) {
    // counter.py:83-96
#pragma unroll
    for (int r = 0; r < 10; r++) {
        u64 lo0, hi0, lo1, hi1;
        mul64x64(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
        mul64x64(0xCA5A826395121157ULL, c2, lo1, hi1);
        u64 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// same bijection with the 10 round keys precomputed (read from the constant bank)
// V = 0: mul64x64 (default); V = 1: the mad.cc-chain form (RS_PHILOX_VARIANT=1)
template <int V = 0>
RS_DEV void philox4x64_10_rk(u64 c0, u64 c1, u64 c2, u64 c3, const u64 *rk0, const u64 *rk1, u64 &o0, u64 &o1,
                             u64 &o2, u64 &o3) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        u64 lo0, hi0, lo1, hi1;
        if constexpr (V == 0) {
            mul64x64(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
            mul64x64(0xCA5A826395121157ULL, c2, lo1, hi1);
        } else {
            mul64x64_cc(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
            mul64x64_cc(0xCA5A826395121157ULL, c2, lo1, hi1);
        }
        u64 n0 = hi1 ^ c1 ^ rk0[r], n2 = hi0 ^ c3 ^ rk1[r];
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// The same bijection when counter words 1-3 are launch constants (no carry out of
// word 0 anywhere in the launch). Round 0's c2 product and round 1's c0 product then
// depend only on words 1-3 and the keys, so they are folded into four per-thread
// constants (philox_fold) and each block costs 18 products instead of 20.
struct PhiloxFold { u64 ka, kb, kc, kd; };
RS_DEV PhiloxFold philox_fold(u64 c1, u64 c2, u64 c3, const u64 *rk0, const u64 *rk1) {
    u64 lo1, hi1, lo0, hi0;
    mul64x64(0xCA5A826395121157ULL, c2, lo1, hi1);        // round 0, c2 product
    u64 n0 = hi1 ^ c1 ^ rk0[0];                            // round-1 c0
    mul64x64(0xD2E7470EE14C6C93ULL, n0, lo0, hi0);         // round 1, c0 product
    return PhiloxFold{c3 ^ rk1[0], lo1 ^ rk0[1], hi0 ^ rk1[1], lo0};
}
template <int V = 0>
RS_DEV void philox4x64_10_folded(u64 c0, const PhiloxFold &f, const u64 *rk0, const u64 *rk1, u64 &o0, u64 &o1,
                                 u64 &o2, u64 &o3) {
    u64 lo0, hi0, lo1, hi1;
    mul64x64(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);         // round 0, c0 product
    mul64x64(0xCA5A826395121157ULL, hi0 ^ f.ka, lo1, hi1);  // round 1, c2 product
    u64 c1 = lo1, c2 = lo0 ^ f.kc, c3 = f.kd;
    c0 = hi1 ^ f.kb;
#pragma unroll
    for (int r = 2; r < 10; r++) {
        if constexpr (V == 0) {
            mul64x64(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
            mul64x64(0xCA5A826395121157ULL, c2, lo1, hi1);
        } else {
            mul64x64_cc(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
            mul64x64_cc(0xCA5A826395121157ULL, c2, lo1, hi1);
        }
        u64 n0 = hi1 ^ c1 ^ rk0[r], n2 = hi0 ^ c3 ^ rk1[r];
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

struct EngPhilox {  // counter.py:98-121; words of a block are served x0..x3
    u64 c0, c1, c2, c3, k0, k1;
    u64 b0, b1, b2, b3;
    int left;
    RS_DEV void bump() {
        c0 += 1;
        if (c0 == 0) { c1 += 1; if (c1 == 0) { c2 += 1; if (c2 == 0) c3 += 1; } }
    }
    RS_DEV void add(u64 blocks) {
        u64 o = c0;
        c0 += blocks;
        if (c0 < o) { c1 += 1; if (c1 == 0) { c2 += 1; if (c2 == 0) c3 += 1; } }
    }
    RS_DEV u64 next() {
        if (left == 0) {
            philox4x64_10(c0, c1, c2, c3, k0, k1, b0, b1, b2, b3);
            bump();
            left = 4;
        }
        u64 r = b0;
        b0 = b1; b1 = b2; b2 = b3;
        left--;
        return r;
    }
};

struct EngSfc {  // sfc.py:25-36
    u64 a, b, c, w;
    RS_DEV u64 next() {
        u64 r = a + b + w;
        w += 1;
        a = b ^ (b >> 11);
        b = c + (c << 3);
        c = rotl64(c, 24) + r;
        return r;
    }
};

// xorshift128+ (xorfam.py:127-146): state [a, b], word a + b
struct EngX128p {
    u64 a, b;
    RS_DEV void load(const u64 *p) { a = p[0]; b = p[1]; }
    RS_DEV u64 next() {
        u64 r = a + b, s1 = a, s0 = b;
        s1 ^= s1 << 23;
        a = s0;
        b = s1 ^ s0 ^ (s1 >> 18) ^ (s0 >> 5);
        return r;
    }
};
// xoroshiro128++ (xorfam.py:149-168)
struct EngXoro {
    u64 s0, s1;
    RS_DEV void load(const u64 *p) { s0 = p[0]; s1 = p[1]; }
    RS_DEV u64 next() {
        u64 r = rotl64(s0 + s1, 17) + s0, t = s1 ^ s0;
        s0 = rotl64(s0, 49) ^ t ^ (t << 21);
        s1 = rotl64(t, 28);
        return r;
    }
};
// squares64 (counter.py:12-48): word i = f(counter + i, key)
RS_DEV u64 sq_swap(u64 x) { return (x >> 32) | (x << 32); }
struct EngSquares {
    u64 ctr, key;
    RS_DEV u64 next() {
        u64 x = ctr++ * key, y = x, z = y + key;
        x = sq_swap(x * x + y);
        x = sq_swap(x * x + z);
        x = sq_swap(x * x + y);
        u64 t = x = x * x + z;
        x = sq_swap(x);
        return t ^ ((x * x + y) >> 32);
    }
};
// ChaCha20 (counter.py:144-216): 64-byte blocks of the 32-bit block counter, served as
// eight little-endian words
RS_DEV u32 rotl32d(u32 x, int r) { return __funnelshift_l(x, x, r); }
#define RS_CHACHA_QR(a, b, c, d)                                   \
    a += b; d = rotl32d(d ^ a, 16); c += d; b = rotl32d(b ^ c, 12); \
    a += b; d = rotl32d(d ^ a, 8); c += d; b = rotl32d(b ^ c, 7);
struct EngChacha {
    u32 k[8], n0, n1, n2, ctr;
    u64 o[8];
    int left;
    RS_DEV void block() {
        const u32 c0 = 0x61707865u, c1 = 0x3320646Eu, c2 = 0x79622D32u, c3 = 0x6B206574u;
        u32 x0 = c0, x1 = c1, x2 = c2, x3 = c3, x4 = k[0], x5 = k[1], x6 = k[2], x7 = k[3];
        u32 x8 = k[4], x9 = k[5], x10 = k[6], x11 = k[7], x12 = ctr, x13 = n0, x14 = n1, x15 = n2;
#pragma unroll 2
        for (int r = 0; r < 10; r++) {
            RS_CHACHA_QR(x0, x4, x8, x12) RS_CHACHA_QR(x1, x5, x9, x13)
            RS_CHACHA_QR(x2, x6, x10, x14) RS_CHACHA_QR(x3, x7, x11, x15)
            RS_CHACHA_QR(x0, x5, x10, x15) RS_CHACHA_QR(x1, x6, x11, x12)
            RS_CHACHA_QR(x2, x7, x8, x13) RS_CHACHA_QR(x3, x4, x9, x14)
        }
        o[0] = (u64)(x0 + c0) | ((u64)(x1 + c1) << 32);
        o[1] = (u64)(x2 + c2) | ((u64)(x3 + c3) << 32);
        o[2] = (u64)(x4 + k[0]) | ((u64)(x5 + k[1]) << 32);
        o[3] = (u64)(x6 + k[2]) | ((u64)(x7 + k[3]) << 32);
        o[4] = (u64)(x8 + k[4]) | ((u64)(x9 + k[5]) << 32);
        o[5] = (u64)(x10 + k[6]) | ((u64)(x11 + k[7]) << 32);
        o[6] = (u64)(x12 + ctr) | ((u64)(x13 + n0) << 32);
        o[7] = (u64)(x14 + n1) | ((u64)(x15 + n2) << 32);
        ctr++;
    }
    RS_DEV u64 next() {
        if (left == 0) {
            block();
            left = 8;
        }
        u64 r = o[0];
#pragma unroll
        for (int i = 0; i < 7; i++) o[i] = o[i + 1];
        left--;
        return r;
    }
};
#undef RS_CHACHA_QR
// cwg128 (cwg.py:28-36): 128-bit x, Weyl state, additive state, odd increment
struct EngCwg {
    unsigned __int128 x, weyl, extra, inc;
    RS_DEV u64 next() {
        weyl += x;
        extra += inc;
        x = ((x >> 1) * (weyl | 1)) ^ extra;
        return (u64)(weyl >> 96) ^ (u64)x;
    }
};

// sfc64simd (interleave.py:172-187): 8 sfc64 lanes, word i from lane i mod 8
struct EngSfcSimd {
    EngSfc l[8];
    int k;
    RS_DEV u64 next() {
        u64 r;
        switch (k) {  // constant-indexed registers (no local-memory array)
        case 0: r = l[0].next(); break;
        case 1: r = l[1].next(); break;
        case 2: r = l[2].next(); break;
        case 3: r = l[3].next(); break;
        case 4: r = l[4].next(); break;
        case 5: r = l[5].next(); break;
        case 6: r = l[6].next(); break;
        default: r = l[7].next(); break;
        }
        k = (k + 1) & 7;
        return r;
    }
};

// ranlux++: x <- x*A mod m, m = 2^576 - 2^240 + 1 (ranlux.py:36-61); any exact
// reduction yields the same canonical residue.
RS_DEV void rlx_mulmod_dev(const u64 *x, const u64 *y, u64 *out) {
    u64 p[18];
#pragma unroll
    for (int i = 0; i < 18; i++) p[i] = 0;
#pragma unroll
    for (int i = 0; i < 9; i++) {
        u64 carry = 0;
#pragma unroll
        for (int j = 0; j < 9; j++) {
            u64 lo = x[i] * y[j], hi = __umul64hi(x[i], y[j]);
            u64 s = p[i + j] + lo;
            hi += (s < lo) ? 1ULL : 0ULL;
            u64 s2 = s + carry;
            hi += (s2 < s) ? 1ULL : 0ULL;
            p[i + j] = s2;
            carry = hi;
        }
        p[i + 9] = carry;
    }
    // r = lo + (hi << 240) - hi over 13 limbs (>= 0)
    u64 r[13];
    {
        u64 ca = 0, br = 0;
#pragma unroll
        for (int i = 0; i < 13; i++) {
            u64 a = i < 9 ? p[i] : 0ULL;
            u64 sh = 0;
            if (i >= 3 && i - 3 < 9) sh |= p[9 + i - 3] << 48;
            if (i >= 4 && i - 4 < 9) sh |= p[9 + i - 4] >> 16;
            u64 t = a + sh;
            u64 c1 = t < a ? 1ULL : 0ULL;
            u64 t2 = t + ca;
            c1 += t2 < t ? 1ULL : 0ULL;
            ca = c1;
            u64 h = i < 9 ? p[9 + i] : 0ULL;
            u64 d = t2 - h;
            u64 b1 = t2 < h ? 1ULL : 0ULL;
            u64 d2 = d - br;
            b1 += d < br ? 1ULL : 0ULL;
            br = b1;
            r[i] = d2;
        }
    }
    // fold r[9..12] again into 10 limbs
    u64 q[10];
    {
        u64 ca = 0, br = 0;
#pragma unroll
        for (int i = 0; i < 10; i++) {
            u64 a = i < 9 ? r[i] : 0ULL;
            u64 sh = 0;
            if (i >= 3 && i - 3 < 4) sh |= r[9 + i - 3] << 48;
            if (i >= 4 && i - 4 < 4) sh |= r[9 + i - 4] >> 16;
            u64 t = a + sh;
            u64 c1 = t < a ? 1ULL : 0ULL;
            u64 t2 = t + ca;
            c1 += t2 < t ? 1ULL : 0ULL;
            ca = c1;
            u64 h = i < 4 ? r[9 + i] : 0ULL;
            u64 d = t2 - h;
            u64 b1 = t2 < h ? 1ULL : 0ULL;
            u64 d2 = d - br;
            b1 += d < br ? 1ULL : 0ULL;
            br = b1;
            q[i] = d2;
        }
    }
    // q < 2m: one conditional subtraction of m
    const u64 M[9] = {1ULL, 0ULL, 0ULL, 0xFFFF000000000000ULL, ~0ULL, ~0ULL, ~0ULL, ~0ULL, ~0ULL};
    bool ge = q[9] != 0;
    if (!ge) {
        ge = true;
        bool decided = false;
#pragma unroll
        for (int i = 8; i >= 0; i--) {
            if (!decided && q[i] != M[i]) { ge = q[i] > M[i]; decided = true; }
        }
    }
    if (ge) {
        u64 br = 0;
#pragma unroll
        for (int i = 0; i < 9; i++) {
            u64 d = q[i] - M[i];
            u64 b1 = q[i] < M[i] ? 1ULL : 0ULL;
            u64 d2 = d - br;
            b1 += d < br ? 1ULL : 0ULL;
            br = b1;
            q[i] = d2;
        }
    }
#pragma unroll
    for (int i = 0; i < 9; i++) out[i] = q[i];
}

#include "rs_ranlux_mul.cuh"  // rlx_mul_A: the engine step with the fixed multiplier

struct EngRanlux {  // words of a chunk: the 9 limbs of the new residue, low first
    u64 x[9];
    u64 o[9];
    int left;
    const u64 *A;  // multiplier limbs (global)
    RS_DEV u64 next() {
        if (left == 0) {
            rlx_mul_A(x, x);
#pragma unroll
            for (int i = 0; i < 9; i++) o[i] = x[i];
            left = 9;
        }
        u64 r = o[0];
#pragma unroll
        for (int i = 0; i < 8; i++) o[i] = o[i + 1];
        left--;
        return r;
    }
};

// ----------------------------------------------------------------------------- uniforms
RS_DEV double dbl(u64 b) { return __longlong_as_double((long long)b); }
RS_DEV u64 bits(double d) { return (u64)__double_as_longlong(d); }

// Rng.u01, rng.py:98-106
RS_DEV double u01_of(u64 w, bool fm) {
    if (fm) return (double)(w >> 11) * 1.1102230246251565e-16;
    return dbl((w >> 12) | 0x3FF0000000000000ULL) - 1.0;
}
// Rng.u01f on one u32 half, rng.py:108-115 (exact in f32 either way)
RS_DEV float u01f_of(u32 h, bool fm) {
    if (fm) return (float)((double)(h >> 8) * 5.9604644775390625e-08);
    return (float)((double)__uint_as_float((h >> 9) | 0x3F800000u) - 1.0);
}

// ----------------------------------------------------------------------------- detmath
RS_DEV u32 hiw(double x) { return (u32)(bits(x) >> 32); }
RS_DEV double with_hiw(double x, u32 h) { return dbl(((u64)h << 32) | (bits(x) & 0xFFFFFFFFULL)); }

// det_exp, detmath.py:59-104
static __device__ __noinline__ double det_exp_dev(double x) {
    const double huge = 1.0e300, twom1000 = 9.33263618503218878990e-302;
    const double o_thr = 7.09782712893383973096e+02, u_thr = -7.45133219101941108420e+02;
    const double invln2 = 1.44269504088896338700e+00, ln2hi = 6.93147180369123816490e-01,
                 ln2lo = 1.90821492927058770002e-10;
    const double P1 = 1.66666666666666019037e-01, P2 = -2.77777777770155933842e-03,
                 P3 = 6.61375632143793436117e-05, P4 = -1.65339022054652515390e-06,
                 P5 = 4.13813679705723846039e-08;
    u32 hx = hiw(x);
    int xsb = (hx >> 31) & 1;
    hx &= 0x7FFFFFFFu;
    if (hx >= 0x40862E42u) {
        if (hx >= 0x7FF00000u) {
            if (((hx & 0xFFFFFu) | (u32)bits(x)) != 0) return x + x;
            return xsb == 0 ? x : 0.0;
        }
        if (x > o_thr) return huge * huge;
        if (x < u_thr) return twom1000 * twom1000;  // underflow to +0 (fdlibm)
    }
    int k = 0;
    double hi = 0.0, lo = 0.0;
    if (hx > 0x3FD62E42u) {
        if (hx < 0x3FF0A2E4u) {
            if (xsb == 0) { hi = x - ln2hi; lo = ln2lo; k = 1; }
            else { hi = x + ln2hi; lo = -ln2lo; k = -1; }
        } else {
            double kd = invln2 * x + (xsb == 0 ? 0.5 : -0.5);
            k = __double2int_rz(kd);  // Python int(): truncation toward zero
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
    if (k >= -1021) return with_hiw(y, hiw(y) + ((u32)k << 20));
    return with_hiw(y, hiw(y) + ((u32)(k + 1000) << 20)) * twom1000;
}

// det_log, detmath.py:107-163
static __device__ __noinline__ double det_log_dev(double x) {
    const double ln2hi = 6.93147180369123816490e-01, ln2lo = 1.90821492927058770002e-10;
    const double two54 = 1.80143985094819840000e+16;
    const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                 Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                 Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                 Lg7 = 1.479819860511658591e-01;
    u64 u = bits(x);
    int hx = (int)(u >> 32);
    u32 lx = (u32)u;
    int k = 0;
    if (hx < 0) {
        if (((hx & 0x7FFFFFFF) | (int)lx) == 0) return dbl(0xFFF0000000000000ULL);  // -inf
        return dbl(0x7FF8000000000000ULL);                                          // nan
    }
    if (hx < 0x00100000) {
        if ((hx | (int)lx) == 0) return dbl(0xFFF0000000000000ULL);
        k -= 54;
        x *= two54;
        hx = (int)hiw(x);
    }
    if (hx >= 0x7FF00000) return x + x;
    k += (hx >> 20) - 1023;
    hx &= 0x000FFFFF;
    int i = (hx + 0x95F64) & 0x100000;
    x = with_hiw(x, (u32)(hx | (i ^ 0x3FF00000)));
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
    int ii = hx - 0x6147A;
    double w = z * z;
    int j = 0x6B851 - hx;
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

// ----------------------------------------------------------------------------- samplers
// The reference samplers restated as device functions that pull words from a
// source `S` (anything with `u64 next()`), in exactly the reference's draw order.
// One call = one sample, so the source position after a call is a sample
// boundary -- the only points where the reference's call stack carries no state.
// Tallies (attempts / density evaluations, continuous.py:32-33) accumulate into
// the caller's counters.

struct ZigFast {  // 16-byte fast-path strip {K, W}, staged in shared memory
    u64 k;
    double w;
};

struct Tally {
    u32 norm_att, norm_pdf, exp_att, exp_pdf, gamma_att;
};

RS_DEV bool lt128(u64 alo, u64 ahi, u64 blo, u64 bhi) { return ahi < bhi || (ahi == bhi && alo < blo); }

// lhs = yv*d + (rabs-K)*2^52 exactly (continuous.py:59-61)
RS_DEV void zig_lhs(u64 yv, u64 d, u64 rk, u64 &lo, u64 &hi) {
    u64 plo = yv * d, phi = __umul64hi(yv, d);
    u64 slo = rk << 52, shi = rk >> 12;
    lo = plo + slo;
    hi = phi + shi + (lo < plo ? 1ULL : 0ULL);
}

struct ZigCtx {
    const ZigFast *fast;  // shared memory
    const RsZigSlow *slow;
    bool fm;              // full-mantissa u01 inside tails / gamma (rng.py:98-106)
};

// std_norm, continuous.py:40-68
template <class S>
RS_DEV double std_norm(S &s, const ZigCtx &z, Tally &t) {
    while (true) {
        t.norm_att++;
        u64 w = s.next();
        int idx = (int)(w & 0xFF);
        u64 rabs = (w >> 9) & ((1ULL << 52) - 1);
        ZigFast f = z.fast[idx];
        double x = (double)rabs * f.w;
        bool neg = (w >> 8) & 1;
        if (rabs < f.k) return neg ? -x : x;
        if (idx == 0) {  // Marsaglia tail: pairs of uniforms until accepted
            while (true) {
                double xx = -dbl(RS_NOR_INV_R_BITS) * det_log_dev(1.0 - u01_of(s.next(), z.fm));
                double yy = -det_log_dev(1.0 - u01_of(s.next(), z.fm));
                if (yy + yy > xx * xx) {
                    double r = dbl(RS_NOR_R_BITS) + xx;
                    return neg ? -r : r;
                }
            }
        }
        u64 yv = s.next() >> 12;
        u64 K = __ldg(&z.slow->k[idx]);
        u64 lo, hi;
        zig_lhs(yv, (1ULL << 52) - K, rabs - K, lo, hi);
        if (lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]))) return neg ? -x : x;
        if (!lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) {
            t.norm_pdf++;
            double fi = __ldg(&z.slow->f[idx]), fim1 = __ldg(&z.slow->f[idx - 1]);
            double y = fi + ((double)yv * 2.220446049250313e-16) * (fim1 - fi);
            if (y < det_exp_dev(-0.5 * x * x)) return neg ? -x : x;
        }
    }
}

// std_exp, continuous.py:71-93
template <class S>
RS_DEV double std_exp(S &s, const ZigCtx &z, Tally &t) {
    while (true) {
        t.exp_att++;
        u64 w = s.next();
        int idx = (int)(w & 0xFF);
        u64 rabs = (w >> 8) & ((1ULL << 53) - 1);
        ZigFast f = z.fast[idx];
        double x = (double)rabs * f.w;
        if (rabs < f.k) return x;
        if (idx == 0) return dbl(RS_EXP_R_BITS) - det_log_dev(1.0 - u01_of(s.next(), z.fm));
        u64 yv = s.next() >> 12;
        u64 K = __ldg(&z.slow->k[idx]);
        u64 lo, hi;
        zig_lhs(yv, (1ULL << 53) - K, rabs - K, lo, hi);
        if (lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]))) return x;
        if (!lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) {
            t.exp_pdf++;
            double fe = __ldg(&z.slow->f[idx]), fem1 = __ldg(&z.slow->f[idx - 1]);
            double y = fe + ((double)yv * 2.220446049250313e-16) * (fem1 - fe);
            if (y < det_exp_dev(-x)) return x;
        }
    }
}

// Marsaglia-Tsang gamma with the power-of-uniform boost below 1, continuous.py:183-212.
struct GammaPrm {
    double d, cc, td;  // d = a-1/3, cc = 1/sqrt(9d), td = theta*d (for the alpha >= 1 core)
    double alpha, theta;
    int boost;         // alpha < 1: core runs gamma(alpha+1, 1), then the U^(1/alpha) boost
};

// gamma_core's exact acceptance test after the squeeze fails (continuous.py:199):
//   det_log(u) < 0.5 zz + d - d v + d det_log(v).
// Both sides are first estimated with the MUFU log (__logf: <= 2^-21.4 absolute on
// [0.5, 2], 3 ulp elsewhere; plus 2^-24 from rounding the argument to f32). Outside a
// band of 1e-5 (1 + |log u| + d (1 + |log v|)) -- 25x those bounds, far above the
// double rounding of either side -- the estimate decides exactly as the exact
// expression would; inside it (and for 0, NaN or f32-underflowing arguments, where
// the comparisons fail) the exact det_log expression decides. This keeps the
// ~10 % of attempts that miss the squeeze off the two-det_log divergent path.
// the MUFU-log screen alone: +1 accept, -1 reject, 0 inside the band (the exact test decides)
RS_DEV int gamma_screen(double u, double zz, double v, const GammaPrm &g) {
    double a = (double)__logf((float)u);
    double lv = (double)__logf((float)v);
    double b = 0.5 * zz + g.d - g.d * v + g.d * lv;
    double m = 1e-5 * (1.0 + fabs(a) + g.d * (1.0 + fabs(lv))) + 1e-12 * (zz + g.d * v);
    return a < b - m ? 1 : (a > b + m ? -1 : 0);
}
RS_DEV bool gamma_exact(double u, double zz, double v, const GammaPrm &g) {  // continuous.py:199
    return det_log_dev(u) < 0.5 * zz + g.d - g.d * v + g.d * det_log_dev(v);
}
RS_DEV bool gamma_accept(double u, double zz, double v, const GammaPrm &g) {
    int sc = gamma_screen(u, zz, v, g);
    return sc != 0 ? sc > 0 : gamma_exact(u, zz, v, g);
}

template <class S>
RS_DEV double gamma_core(S &s, const ZigCtx &z, const GammaPrm &g, Tally &t) {
    while (true) {
        t.gamma_att++;
        double zn, tt;
        do {
            zn = std_norm(s, z, t);
            tt = 1.0 + g.cc * zn;
        } while (!(tt > 0.0));
        double v = tt * tt * tt;
        double u = u01_of(s.next(), z.fm);
        double zz = zn * zn;
        if (u < 1.0 - 0.0331 * zz * zz) return g.td * v;
        if (gamma_accept(u, zz, v, g)) return g.td * v;
    }
}

template <class S>
RS_DEV double gamma_sample(S &s, const ZigCtx &z, const GammaPrm &g, Tally &t) {
    double r = gamma_core(s, z, g, t);
    if (!g.boost) return r;
    double u = u01_of(s.next(), z.fm);
    return g.theta * r * det_exp_dev(det_log_dev(u) / g.alpha);
}

// f32 ziggurats on 32-bit halves (continuous.py:96-133): strips {K (u32), W (f32)}
struct ZigFastF {
    u32 k;
    float w;
};
struct RsZigSlowF {
    float f[256];
};
struct ZigCtxF {
    const ZigFastF *fast;  // shared memory
    const RsZigSlowF *slow;
    bool fm;
};
RS_DEV double f32r(double x) { return (double)__double2float_rn(x); }  // numpy float32(), _f32

template <class S>
RS_DEV double std_norm_f(S &s, const ZigCtxF &z) {
    while (true) {
        u32 w = s.next32();
        int idx = (int)(w & 0xFF);
        u32 rabs = (w >> 9) & 0x7FFFFFu;
        ZigFastF f = z.fast[idx];
        double x = f32r((double)rabs * (double)f.w);
        bool neg = (w >> 8) & 1;
        if (rabs < f.k) return neg ? -x : x;
        if (idx == 0) {
            while (true) {
                double xx = -dbl(RS_NOR_INV_R_BITS) * det_log_dev(1.0 - (double)u01f_of(s.next32(), z.fm));
                double yy = -det_log_dev(1.0 - (double)u01f_of(s.next32(), z.fm));
                if (yy + yy > xx * xx) {
                    double t = f32r(dbl(RS_NOR_R_BITS) + xx);
                    return neg ? -t : t;
                }
            }
        }
        double u = (double)(s.next32() >> 8) * 5.9604644775390625e-08;
        double fi = (double)__ldg(&z.slow->f[idx]), fim1 = (double)__ldg(&z.slow->f[idx - 1]);
        double y = fi + u * (fim1 - fi);
        if (y < det_exp_dev(-0.5 * x * x)) return neg ? -x : x;
    }
}

template <class S>
RS_DEV double std_exp_f(S &s, const ZigCtxF &z) {
    while (true) {
        u32 w = s.next32();
        int idx = (int)(w & 0xFF);
        u32 rabs = (w >> 8) & 0xFFFFFFu;
        ZigFastF f = z.fast[idx];
        double x = f32r((double)rabs * (double)f.w);
        if (rabs < f.k) return x;
        if (idx == 0) return f32r(dbl(RS_EXP_R_BITS) - det_log_dev(1.0 - (double)u01f_of(s.next32(), z.fm)));
        double u = (double)(s.next32() >> 8) * 5.9604644775390625e-08;
        double fe = (double)__ldg(&z.slow->f[idx]), fem1 = (double)__ldg(&z.slow->f[idx - 1]);
        double y = fe + u * (fem1 - fe);
        if (y < det_exp_dev(-x)) return x;
    }
}

// ----------------------------------------------------------------------------- word-level machines
// The same ziggurat samplers restated one word at a time (states: 0 start, 1 slow
// second word, 2/3 tail pairs). In a SIMT warp every lane then consumes exactly one
// word per step, so the engine step is never inside a divergent branch -- only the
// rare slow/tail decision is (1.5 % of normal, 2.2 % of exponential words).
struct ZigWM {
    u32 st, idx;
    u64 rabs;
    u32 neg;
    double xx;
};

RS_DEV bool norm_rare(ZigWM &m, u64 w, const ZigCtx &z, Tally &t, double &out) {
    if (m.st == 1) {  // second word of the slow path (continuous.py:59-68)
        m.st = 0;
        u64 yv = w >> 12;
        int idx = (int)m.idx;
        double x = (double)m.rabs * z.fast[idx].w;
        u64 K = __ldg(&z.slow->k[idx]);
        u64 lo, hi;
        zig_lhs(yv, (1ULL << 52) - K, m.rabs - K, lo, hi);
        bool acc = lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]));
        if (!acc && !lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) {
            t.norm_pdf++;
            double fi = __ldg(&z.slow->f[idx]), fim1 = __ldg(&z.slow->f[idx - 1]);
            double y = fi + ((double)yv * 2.220446049250313e-16) * (fim1 - fi);
            acc = y < det_exp_dev(-0.5 * x * x);
        }
        if (acc) out = m.neg ? -x : x;
        return acc;
    }
    if (m.st == 2) {  // tail: xx (continuous.py:52-58)
        m.xx = -dbl(RS_NOR_INV_R_BITS) * det_log_dev(1.0 - u01_of(w, z.fm));
        m.st = 3;
        return false;
    }
    double yy = -det_log_dev(1.0 - u01_of(w, z.fm));
    if (yy + yy > m.xx * m.xx) {
        double r = dbl(RS_NOR_R_BITS) + m.xx;
        out = m.neg ? -r : r;
        m.st = 0;
        return true;
    }
    m.st = 2;
    return false;
}

// std_norm one word at a time; returns true when a sample completes (in out).
// f = z.fast[w & 0xFF], loaded by the caller (batched loads overlap their latency)
RS_DEV bool norm_feed(ZigWM &m, u64 w, ZigFast f, const ZigCtx &z, Tally &t, double &out) {
    if (__builtin_expect(m.st == 0, 1)) {
        t.norm_att++;
        int idx = (int)(w & 0xFF);
        u64 rabs = (w >> 9) & ((1ULL << 52) - 1);
        if (rabs < f.k) {
            double x = (double)rabs * f.w;
            out = (w >> 8) & 1 ? -x : x;
            return true;
        }
        m.idx = idx;
        m.rabs = rabs;
        m.neg = (u32)((w >> 8) & 1);
        m.st = idx == 0 ? 2 : 1;
        return false;
    }
    return norm_rare(m, w, z, t, out);
}

RS_DEV bool exp_rare(ZigWM &m, u64 w, const ZigCtx &z, Tally &t, double &out) {
    if (m.st == 1) {  // continuous.py:83-93
        m.st = 0;
        u64 yv = w >> 12;
        int idx = (int)m.idx;
        double x = (double)m.rabs * z.fast[idx].w;
        u64 K = __ldg(&z.slow->k[idx]);
        u64 lo, hi;
        zig_lhs(yv, (1ULL << 53) - K, m.rabs - K, lo, hi);
        bool acc = lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]));
        if (!acc && !lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) {
            t.exp_pdf++;
            double fe = __ldg(&z.slow->f[idx]), fem1 = __ldg(&z.slow->f[idx - 1]);
            double y = fe + ((double)yv * 2.220446049250313e-16) * (fem1 - fe);
            acc = y < det_exp_dev(-x);
        }
        if (acc) out = x;
        return acc;
    }
    m.st = 0;  // tail (continuous.py:82): one uniform
    out = dbl(RS_EXP_R_BITS) - det_log_dev(1.0 - u01_of(w, z.fm));
    return true;
}

RS_DEV bool exp_feed(ZigWM &m, u64 w, ZigFast f, const ZigCtx &z, Tally &t, double &out) {
    if (__builtin_expect(m.st == 0, 1)) {
        t.exp_att++;
        int idx = (int)(w & 0xFF);
        u64 rabs = (w >> 8) & ((1ULL << 53) - 1);
        if (rabs < f.k) {
            out = (double)rabs * f.w;
            return true;
        }
        m.idx = idx;
        m.rabs = rabs;
        m.st = idx == 0 ? 2 : 1;
        return false;
    }
    return exp_rare(m, w, z, t, out);
}

// The wedge decision alone (accept / reject) of a token whose first word gave (idx, rabs)
// and whose second word is w2: state 1 of norm_rare / exp_rare without the output (the
// batch parse computes the sample value ahead, from the first word).
RS_DEV bool norm_wedge(u32 idx, u64 rabs, u64 w2, const ZigCtx &z, Tally &t) {
    u64 yv = w2 >> 12;
    u64 K = __ldg(&z.slow->k[idx]);
    u64 lo, hi;
    zig_lhs(yv, (1ULL << 52) - K, rabs - K, lo, hi);
    if (lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]))) return true;
    if (lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) return false;
    t.norm_pdf++;
    double x = (double)rabs * z.fast[idx].w;
    double fi = __ldg(&z.slow->f[idx]), fim1 = __ldg(&z.slow->f[idx - 1]);
    double y = fi + ((double)yv * 2.220446049250313e-16) * (fim1 - fi);
    return y < det_exp_dev(-0.5 * x * x);
}
RS_DEV bool exp_wedge(u32 idx, u64 rabs, u64 w2, const ZigCtx &z, Tally &t) {
    u64 yv = w2 >> 12;
    u64 K = __ldg(&z.slow->k[idx]);
    u64 lo, hi;
    zig_lhs(yv, (1ULL << 53) - K, rabs - K, lo, hi);
    if (lt128(lo, hi, __ldg(&z.slow->ta_lo[idx]), __ldg(&z.slow->ta_hi[idx]))) return true;
    if (lt128(__ldg(&z.slow->tr_lo[idx]), __ldg(&z.slow->tr_hi[idx]), lo, hi)) return false;
    t.exp_pdf++;
    double x = (double)rabs * z.fast[idx].w;
    double fe = __ldg(&z.slow->f[idx]), fem1 = __ldg(&z.slow->f[idx - 1]);
    double y = fe + ((double)yv * 2.220446049250313e-16) * (fem1 - fe);
    return y < det_exp_dev(-x);
}

// ----------------------------------------------------------------------------- distributions
// A Dist draws one sample per call to sample(s, t). Families share a kernel and pick
// the law with a (warp-uniform) kind, which keeps the number of kernel instantiations
// small. HALF marks samplers fed by 32-bit halves (stream positions in halves).

enum { NK_NORM = 0, NK_STD = 1, NK_LOGNORMAL = 2, NK_SKEW = 3 };
struct DistNorm {  // continuous.py:157-158 (norm), :176-177 (lognormal), :281-290 (skew_normal), mvn z
    typedef double out_t;
    static constexpr bool HALF = false;
    ZigCtx z;
    double a, b, c, d;  // NORM/LOGNORMAL: mu, sd | SKEW: delta, sqrt(1-delta^2), mu, sigma
    int kind;
    // a skew-normal sample is a pair of normals: the phase-1 parse starts with its second one
    RS_DEV bool paired() const { return kind == NK_SKEW; }
    RS_DEV bool word_level() const { return kind != NK_SKEW; }
    RS_DEV double finish(double v) const {
        if (kind == NK_STD) return v;
        double r = a + b * v;
        return kind == NK_LOGNORMAL ? det_exp_dev(r) : r;
    }
    RS_DEV ZigFast strip(u64 w) const { return z.fast[w & 0xFF]; }
    RS_DEV bool feed(ZigWM &m, u64 w, ZigFast f, Tally &t, double &out) const { return norm_feed(m, w, f, z, t, out); }
    // batch-parse hooks (rs_kernels.cuh zb_*): a word's fast-path test and signed value, the
    // wedge decision of a token (first word w1 or a carried state, second word w2), the
    // state carried into the next batch by a token that starts on its last word
    static RS_DEV u64 zrabs(u64 w) { return (w >> 9) & ((1ULL << 52) - 1); }
    RS_DEV bool zfast(u64 w, ZigFast f) const { return zrabs(w) < f.k; }
    RS_DEV double zval(u64 w, ZigFast f) const {
        double x = (double)zrabs(w) * f.w;
        return (w >> 8) & 1 ? -x : x;
    }
    RS_DEV bool zwedge(u64 w1, u64 w2, Tally &t) const { return norm_wedge((u32)(w1 & 0xFF), zrabs(w1), w2, z, t); }
    RS_DEV bool zwedge_m(const ZigWM &m, u64 w2, Tally &t) const { return norm_wedge(m.idx, m.rabs, w2, z, t); }
    RS_DEV double zval_m(const ZigWM &m) const {
        double x = (double)m.rabs * z.fast[m.idx].w;
        return m.neg ? -x : x;
    }
    RS_DEV void zcarry(ZigWM &m, u64 w) const {
        m.st = 1;
        m.idx = (u32)(w & 0xFF);
        m.rabs = zrabs(w);
        m.neg = (u32)((w >> 8) & 1);
    }
    RS_DEV void zatt(Tally &t, u32 k) const { t.norm_att += k; }
    RS_DEV bool feed(ZigWM &m, u64 w, Tally &t, double &out) const { return norm_feed(m, w, strip(w), z, t, out); }
    template <class S> RS_DEV void skip_second(S &s, Tally &t) const { std_norm(s, z, t); }
    template <class S> RS_DEV double sample(S &s, Tally &t) const {
        double v = std_norm(s, z, t);
        if (kind == NK_STD) return v;
        if (kind == NK_SKEW) {
            double v2 = std_norm(s, z, t);
            return c + d * (a * fabs(v) + b * v2);
        }
        double r = a + b * v;
        return kind == NK_LOGNORMAL ? det_exp_dev(r) : r;
    }
};
enum { EK_EXP = 0, EK_PARETO = 1, EK_GPD = 2, EK_WEIBULL = 3 };
struct DistExp {  // continuous.py:165-169 (exp), :252-254 (pareto), :257-266 (gpd), :269-274 (weibull)
    typedef double out_t;
    static constexpr bool HALF = false;
    ZigCtx z;
    double a, b, c;  // EXP: beta | PARETO: alpha, xm | GPD: xi, mu, sigma | WEIBULL: k, lam
    int kind;
    RS_DEV bool paired() const { return false; }
    template <class S> RS_DEV void skip_second(S &, Tally &) const {}
    RS_DEV bool word_level() const { return true; }
    RS_DEV double finish(double e) const {
        if (kind == EK_EXP) return a * e;
        if (kind == EK_PARETO) return b * det_exp_dev(e / a);
        if (kind == EK_WEIBULL) return b * det_exp_dev(det_log_dev(e) / a);
        if (a == 0.0) return b + c * e;
        double p = det_exp_dev(e * fabs(a));
        return a > 0.0 ? b + c * (p - 1.0) / a : b - c * (1.0 - 1.0 / p) / a;
    }
    RS_DEV ZigFast strip(u64 w) const { return z.fast[w & 0xFF]; }
    RS_DEV bool feed(ZigWM &m, u64 w, ZigFast f, Tally &t, double &out) const { return exp_feed(m, w, f, z, t, out); }
    static RS_DEV u64 zrabs(u64 w) { return (w >> 8) & ((1ULL << 53) - 1); }
    RS_DEV bool zfast(u64 w, ZigFast f) const { return zrabs(w) < f.k; }
    RS_DEV double zval(u64 w, ZigFast f) const { return (double)zrabs(w) * f.w; }
    RS_DEV bool zwedge(u64 w1, u64 w2, Tally &t) const { return exp_wedge((u32)(w1 & 0xFF), zrabs(w1), w2, z, t); }
    RS_DEV bool zwedge_m(const ZigWM &m, u64 w2, Tally &t) const { return exp_wedge(m.idx, m.rabs, w2, z, t); }
    RS_DEV double zval_m(const ZigWM &m) const { return (double)m.rabs * z.fast[m.idx].w; }
    RS_DEV void zcarry(ZigWM &m, u64 w) const {
        m.st = 1;
        m.idx = (u32)(w & 0xFF);
        m.rabs = zrabs(w);
    }
    RS_DEV void zatt(Tally &t, u32 k) const { t.exp_att += k; }
    RS_DEV bool feed(ZigWM &m, u64 w, Tally &t, double &out) const { return exp_feed(m, w, strip(w), z, t, out); }
    template <class S> RS_DEV double sample(S &s, Tally &t) const {
        double e = std_exp(s, z, t);
        if (kind == EK_EXP) return a * e;
        if (kind == EK_PARETO) return b * det_exp_dev(e / a);
        if (kind == EK_WEIBULL) return b * det_exp_dev(det_log_dev(e) / a);
        if (a == 0.0) return b + c * e;  // gpd, xi == 0
        double p = det_exp_dev(e * fabs(a));
        return a > 0.0 ? b + c * (p - 1.0) / a : b - c * (1.0 - 1.0 / p) / a;
    }
};
// ----------------------------------------------------------------------------- attempt-level gamma
// The attempt's first two words, drawn by the caller, then the stream: the source of the
// exact normal draw(s) when the first word is not a fast-path token or t <= 0 (an
// attempt always consumes both: a normal token >= 1 word, then the uniform).
template <class S>
struct PairSrc {
    u64 w1, w2;
    int k;
    S *s;
    RS_DEV u64 next() {
        if (k == 0) { k = 1; return w1; }
        if (k == 1) { k = 2; return w2; }
        return s->next();
    }
};
// Per-lane state of the attempt-level machine: which sub-sample is being drawn (beta / f
// draw x from ga then y from gb, continuous.py:215-218, :237-243), the finished x, and
// whether the parse started with a lone second sub-sample (the phase-1 parse).
struct GammaAM {
    u32 role, lone;
    double x;
};

enum { GK_GAMMA = 0, GK_BETA = 1, GK_T = 2, GK_F = 3 };
struct DistGamma {  // continuous.py:183-212 (gamma, chi2 = gamma(nu/2, 2)), :215-218 beta, :228-234 t, :237-243 f
    typedef double out_t;
    static constexpr bool HALF = false;
    ZigCtx z;
    GammaPrm ga, gb;
    double nu1, nu2;
    int kind;
    // beta / f / t samples are (first, second) pairs of sub-samples
    RS_DEV bool paired() const { return kind != GK_GAMMA; }
    template <class S> RS_DEV void skip_second(S &s, Tally &t) const {
        if (kind == GK_T) gamma_sample(s, z, ga, t);
        else gamma_sample(s, z, gb, t);
    }
    // Attempt-level machine (kinds gamma / beta / f): one Marsaglia-Tsang attempt per call,
    // its two words drawn at one call site, so the lanes of a warp run the engine and the
    // common attempt (fast-path normal, t > 0, squeeze / screened acceptance) in step
    // whatever sample each is in; the sample-level loop ran the normal-word and the
    // uniform-word engine steps as two divergent sites. Returns true when a sample
    // completes (value in out); words, tallies and values equal sample()'s.
    RS_DEV bool am_applies() const { return kind != GK_T; }
    template <class S> RS_DEV bool am_step(GammaAM &m, S &s, Tally &t, double &out) const {
        const bool second = m.role != 0;
        GammaPrm g;
        g.d = second ? gb.d : ga.d;
        g.cc = second ? gb.cc : ga.cc;
        g.td = second ? gb.td : ga.td;
        g.alpha = second ? gb.alpha : ga.alpha;
        g.theta = second ? gb.theta : ga.theta;
        g.boost = second ? gb.boost : ga.boost;
        const u64 w1 = s.next(), w2 = s.next();
        const u32 idx = (u32)(w1 & 0xFF);
        const u64 rabs = (w1 >> 9) & ((1ULL << 52) - 1);
        const ZigFast f = z.fast[idx];
        double zn = (double)rabs * f.w;
        if ((w1 >> 8) & 1) zn = -zn;
        double tt = 1.0 + g.cc * zn;
        t.gamma_att++;
        u64 uw = w2;
        if (__builtin_expect(rabs < f.k && tt > 0.0, 1)) {
            t.norm_att++;
        } else {  // a slow / tail normal token, or t <= 0: the exact normal draw(s) from w1 on
            PairSrc<S> ps{w1, w2, 0, &s};
            do {
                zn = std_norm(ps, z, t);
                tt = 1.0 + g.cc * zn;
            } while (!(tt > 0.0));
            uw = ps.next();
        }
        const double v = tt * tt * tt;
        const double u = u01_of(uw, z.fm);
        const double zz = zn * zn;
        double val = g.td * v;
        // The squeeze misses on ~10 % of attempts, so nearly every warp-step had a lane in
        // the screen branch (and the accepted lanes then finished the step as two groups):
        // the screen runs branch-free on every lane, only the in-band exact test branches.
        const bool sq = u < 1.0 - 0.0331 * zz * zz;
        const int sc = gamma_screen(u, zz, v, g);
        bool acc = sq || sc > 0;
        if (__builtin_expect(!sq && sc == 0, 0)) acc = gamma_exact(u, zz, v, g);
        if (!acc) return false;
        if (g.boost) val = g.theta * val * det_exp_dev(det_log_dev(u01_of(s.next(), z.fm)) / g.alpha);
        if (kind == GK_GAMMA) {
            out = val;
            return true;
        }
        if (!second) {
            m.x = val;
            m.role = 1;
            return false;
        }
        m.role = 0;
        if (m.lone) {  // the phase-1 parse's lone second sub-sample: a boundary, no sample
            m.lone = 0;
            out = 0.0;
            return true;
        }
        out = kind == GK_BETA ? m.x / (m.x + val) : (m.x / nu1) / (val / nu2);
        return true;
    }
    template <class S> RS_DEV double sample(S &s, Tally &t) const {
        if (kind == GK_T) {
            double zn = std_norm(s, z, t);
            double v = gamma_sample(s, z, ga, t);
            return zn / sqrt(v / nu1);
        }
        double x = gamma_sample(s, z, ga, t);
        if (kind == GK_GAMMA) return x;
        double y = gamma_sample(s, z, gb, t);
        return kind == GK_BETA ? x / (x + y) : (x / nu1) / (y / nu2);
    }
};
struct DistLemire {  // bounded_uint(rng, b, 64) discrete.py:20-39 (+ m: bounded_int long_long, :42-55)
    typedef u64 out_t;
    static constexpr bool HALF = false;
    u64 b, thr, m;
    RS_DEV bool paired() const { return false; }
    template <class S> RS_DEV void skip_second(S &, Tally &) const {}
    template <class S> RS_DEV u64 sample(S &s, Tally &) const {
        while (true) {
            u64 w = s.next();
            if (w * b >= thr) return m + __umul64hi(w, b);
        }
    }
    // word-level form: every lane consumes one word per step (no divergent redraw loops).
    // For b < 2^32 the 128-bit product w*b needs two 32x32 products, not four.
    RS_DEV bool accept(u64 w, u64 &o) const {
        if ((b >> 32) == 0) {
            const u64 lo = (u64)(u32)w * b;                 // w_lo * b
            const u64 mid = (w >> 32) * b + (lo >> 32);       // w_hi * b + carry, < 2^64
            o = m + (mid >> 32);                              // high word of w*b
            return ((mid << 32) | (lo & 0xFFFFFFFFULL)) >= thr;  // low word of w*b
        }
        o = m + __umul64hi(w, b);
        return w * b >= thr;
    }
};
enum { FK_NORMF = 0, FK_EXPF = 1 };
struct DistF32 {  // normf / expf, continuous.py:136-154 (32-bit halves, f32 tables)
    typedef float out_t;
    static constexpr bool HALF = true;
    ZigCtxF z;
    double a, b;  // NORMF: mu, sd | EXPF: beta
    int kind;
    RS_DEV bool paired() const { return false; }
    template <class S> RS_DEV void skip_second(S &, Tally &) const {}
    template <class S> RS_DEV float sample(S &s, Tally &) const {
        if (kind == FK_NORMF) return __double2float_rn(a + b * std_norm_f(s, z));
        return __double2float_rn(a * std_exp_f(s, z));
    }
};
struct DistU32 {  // bounded_uint(rng, b, 8|16|32) on halves (+ m: bounded_int int), discrete.py:14-55
    typedef u32 out_t;
    static constexpr bool HALF = true;
    u64 b, thr, mask;
    u32 m;
    int width;
    RS_DEV bool paired() const { return false; }
    template <class S> RS_DEV void skip_second(S &, Tally &) const {}
    template <class S> RS_DEV u32 sample(S &s, Tally &) const {
        while (true) {
            u32 o;
            if (accept(s.next32(), o)) return o;
        }
    }
    RS_DEV bool accept(u32 h, u32 &o) const {
        u64 x = (u64)h & mask;
        u64 mm = x * b;
        o = m + (u32)(mm >> width);
        return (mm & mask) >= thr;
    }
};

// ----------------------------------------------------------------------------- run writers
// Writes a contiguous run of elements starting at element `start` of `out`, in 32-byte
// groups (one STG.256 each); ragged heads/tails (shared with the neighbouring runs) are
// element stores.
//
// Every writer keeps its own per-thread pointer to the current group and advances it,
// never a (uniform base + per-thread index) pair recomputed at the store. Round 1 hit an
// illegal-address fault in k_streams with the ring writer (x256** normals, 64 streams x
// 4096): cuda-gdb put the faulting PC on the flush STG.256, whose address ptxas had built
// as uniform register UR6:UR7 (the 32-byte-aligned output base) + the thread's group
// index, with UR7 reloaded inside the divergent flush branch. The same loop also wrote
// UR7 (shared-memory table base, sampler kind) on the sampler's divergent retry path, and
// at the fault the warp's lanes were spread over the sampler and the flush. Uniform
// registers are one per warp, so a divergent group running the sampler between the
// flush group's reload and its store replaced the address's high word (DESIGN 7,
// profiles/r02_ringwriter/). A per-thread pointer carried across iterations lives in
// vector registers, which divergent groups do not share.
template <class T>
struct VecWriter8 {
    T *gp;         // this thread's current 32-byte group
    int slot, first;
    T v0, v1, v2, v3;
    RS_DEV void init(T *out, u64 start) {
        uintptr_t a = (uintptr_t)out;
        u64 s = start + ((a & 31) >> 3);
        gp = (T *)(a & ~(uintptr_t)31) + (s & ~3ULL);
        slot = (int)(s & 3);
        first = slot;
    }
    RS_DEV void put(T v) {
        switch (slot) {
        case 0: v0 = v; break;
        case 1: v1 = v; break;
        case 2: v2 = v; break;
        default: v3 = v; break;
        }
        if (++slot == 4) flush_full();
    }
    RS_DEV void flush_full() {
        T *p = gp;
        if (first == 0) {
            u64 a = *(u64 *)&v0, b = *(u64 *)&v1, c = *(u64 *)&v2, d = *(u64 *)&v3;
            asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
                         : "memory");
        } else {
            if (first <= 1) p[1] = v1;
            if (first <= 2) p[2] = v2;
            p[3] = v3;
        }
        first = 0;
        slot = 0;
        gp += 4;
    }
    RS_DEV void finish() {
        T *p = gp;
        if (first == 0 && slot > 0) p[0] = v0;
        if (first <= 1 && slot > 1) p[1] = v1;
        if (first <= 2 && slot > 2) p[2] = v2;
    }
};

// The current group is staged in a per-thread shared-memory ring (slot-major with stride
// NT = the launch's block size, so a warp's STS is conflict-free) and leaves as one
// STG.256 once full. Unlike a register array with a dynamic slot index, put() is
// branch-free apart from the flush.
template <class T, int NT>
struct RingWriter {
    static constexpr int G = 32 / (int)sizeof(T);
    T *gp;     // this thread's current 32-byte group
    int slot, first;
    T *ring;   // this thread's slot 0; slot k at ring[k * NT]
    RS_DEV void init(T *out, u64 start, T *ring_) {
        ring = ring_;
        uintptr_t a = (uintptr_t)out;
        u64 s = start + (u64)((a & 31) / sizeof(T));
        gp = (T *)(a & ~(uintptr_t)31) + (s & ~(u64)(G - 1));
        slot = (int)(s & (G - 1));
        first = slot;
    }
    RS_DEV T *at() const { return gp + slot; }  // where the next element goes
    RS_DEV void put(T v) {
        ring[slot * NT] = v;
        if (++slot == G) flush_full();
    }
    RS_DEV void flush_full() {
        T *p = gp;
        if (first == 0) {
            u64 q[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if constexpr (sizeof(T) == 8) {
                    q[k] = *(const u64 *)&ring[k * NT];
                } else {
                    u64 lo = *(const u32 *)&ring[(2 * k) * NT], hi = *(const u32 *)&ring[(2 * k + 1) * NT];
                    q[k] = lo | (hi << 32);
                }
            }
            asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(q[0]), "l"(q[1]), "l"(q[2]),
                         "l"(q[3]) : "memory");
        } else {
            for (int k = first; k < G; k++) p[k] = ring[k * NT];
        }
        first = 0;
        slot = 0;
        gp += G;
    }
    RS_DEV void finish() {
        T *p = gp;
        for (int k = first; k < slot; k++) p[k] = ring[k * NT];
    }
};

// RingWriter with the flush taken off the per-sample path: a ring of two 32-byte groups
// per thread, and tick() -- called by every lane of a warp on the same steps, once per G
// steps of a word-level loop that emits at most one sample per step -- stores at most one
// complete group. A lane's groups then leave on the same steps as its neighbours'
// instead of a divergent flush on nearly every step (some lane of 32 is always at its
// group end). Buffered samples stay below 2G: <= G-1 after a tick, + G before the next.
template <class T, int NT, int GB = 32>  // GB: bytes per group (32: one STG.256)
struct BatchRing {
    static constexpr int G = GB / (int)sizeof(T);
    T *gp;        // this thread's current (unstored) group, 32-byte aligned
    u32 head;     // elements of that group before the run (shared with the previous run)
    u32 npend;    // elements from the group start up to the next sample (head included)
    u32 rbase;    // ring slot of the group's first element (0 or G)
    T *ring;      // this thread's slot 0; slot k at ring[k * NT]
    RS_DEV void init(T *out, u64 start, T *ring_) {
        ring = ring_;
        uintptr_t a = (uintptr_t)out;
        const u64 s = start + (u64)((a & 31) / sizeof(T));
        gp = (T *)(a & ~(uintptr_t)31) + (s & ~(u64)(G - 1));
        head = npend = (u32)(s & (G - 1));
        rbase = (u32)(s & (2 * G - 1)) & ~(u32)(G - 1);
    }
    RS_DEV void put(T v) {
        ring[(int)((rbase + npend) & (2 * G - 1)) * NT] = v;
        npend++;
    }
    // scratch in the free slots: slot_at(free_base() + k) is free until k + 1 more puts
    RS_DEV u32 free_base() const { return rbase + npend; }
    RS_DEV void advance(u32 k) { npend += k; }  // k elements written at the free slots
    RS_DEV u64 *slot_at(u32 i) const {
        static_assert(sizeof(T) == 8, "8-byte slots");
        return (u64 *)&ring[(int)(i & (2 * G - 1)) * NT];
    }
    RS_DEV void tick() {
        if (npend < (u32)G) return;
        T *p = gp;
        const int b = (int)rbase;
        if (head == 0) {
            constexpr int E32 = 32 / (int)sizeof(T);  // elements per 32-byte store
#pragma unroll
            for (int h = 0; h < GB / 32; h++) {
                u64 q[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if constexpr (sizeof(T) == 8) {
                        q[k] = *(const u64 *)&ring[(b + h * E32 + k) * NT];
                    } else {
                        u64 lo = *(const u32 *)&ring[(b + h * E32 + 2 * k) * NT];
                        u64 hi = *(const u32 *)&ring[(b + h * E32 + 2 * k + 1) * NT];
                        q[k] = lo | (hi << 32);
                    }
                }
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p + h * E32), "l"(q[0]), "l"(q[1]),
                             "l"(q[2]), "l"(q[3]) : "memory");
            }
        } else {  // the run's first group is shared with the previous run
            for (int k = (int)head; k < G; k++) p[k] = ring[(b + k) * NT];
        }
        gp += G;
        npend -= G;
        rbase ^= G;
        head = 0;
    }
    RS_DEV void finish() {
        for (u32 k = head; k < npend; k++) gp[k] = ring[(int)((rbase + k) & (2 * G - 1)) * NT];
    }
};

template <class T>
struct ScalarWriter {
    T *ptr;
    RS_DEV void init(T *out, u64 start) { ptr = out + start; }
    RS_DEV void put(T v) { *ptr++ = v; }
    RS_DEV void finish() {}
};

template <class T>
struct VecWriter2 {
    T *ptr;     // next element
    bool head;  // first element is not 16-byte aligned: it goes out alone
    bool have;  // v0 holds the first half of a pair
    T v0;
    RS_DEV void init(T *out, u64 start) {
        ptr = out + start;
        head = ((uintptr_t)ptr & 15) != 0;
        have = false;
    }
    RS_DEV void put(T v) {
        if (head) { *ptr++ = v; head = false; return; }
        if (!have) { v0 = v; have = true; return; }
        u64 a = *(u64 *)&v0, b = *(u64 *)&v;
        asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(ptr), "l"(a), "l"(b) : "memory");
        ptr += 2;
        have = false;
    }
    RS_DEV void finish() {
        if (have) *ptr = v0;
    }
};
