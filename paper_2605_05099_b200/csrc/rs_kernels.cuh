// Device side of the fill path: plan types, engines-as-sources, samplers, and every
// kernel template. Included by the kernel translation units (k_*.cu), which each
// instantiate one group of kernels and hand them out through the rsk:: accessors
// below, and by the host translation unit rs_fill.cu (types only). Split so the
// ~240 kernels compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "rs_device.cuh"
#include "rs_internal.h"

using rs::u128;

namespace {

constexpr int BLOCK = 256;
// Gamma-family parses converge only after ~10^2 words, so the count
// pass records where its parses put sample boundaries, over the whole segment
// (p.bmw 32-unit words per thread); the fixup then re-parses from the true entry alone
// and looks the meeting point up instead of re-running the speculative parses beside
// it. (A 1024-unit window made the rare threads that met later restart both parses
// from the segment start: gamma 2^26 fixup 1.04 ms.)
constexpr int MAXLEV = 24;
constexpr int CAP = RS_BUFFER_CAPACITY;

// ----------------------------------------------------------------------------- plan
struct FillPlan {
    int engine, dist, fm, P;      // P = buffered words ahead of the engine stream
    int pending_used;             // u01f: the buffered high half feeds sample 0
    u32 pending_val;
    u64 lp0;                      // thread 0's first logical position
    u64 n;                        // samples wanted from this chunk
    u64 L;                        // engine words per thread
    u32 T;                        // segments
    u64 weng;                     // fixed fills: engine words needed
    u64 base[9];                  // engine state at this chunk's engine origin
    u64 prefix[CAP];
    u64 pcg_m[MAXLEV][2], pcg_a[MAXLEV][2];
    u64 rlx[MAXLEV][9];
    u64 rk0[10], rk1[10];         // philox round keys (counter.py:95-96)
    u64 lanes[32];                // interleaved engines: the 8 lane states (lane-major)
    u64 G, Gpad;                  // interleaved fixed fills: step groups (real / padded)
    int vec_ok;                   // counter-based fill: outputs 32-byte aligned per block
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int raw_norm;                 // std_norm without the epilogue (mvn z)
    int kind;                     // law within a sampler family (NK_*, EK_*, GK_*, FK_*)
    int unit;                     // 1: positions in 64-bit words, 2: in 32-bit halves
    int fmode;                    // fixed-consumption map (serial kernel)
    const RsZigSlowF *zslowf;
    const ZigFastF *zfastf;
    const u64 *x256_states;
    const u64 *words;             // materialized engine words (RS_ENG_MEM parse source)
    u64 nwords;
    u32 *bm;                      // gamma family: count-pass boundary bitmaps [2][bmw][T]
    u32 bmw;                      // 32-unit bitmap words per thread and phase
    u32 *overrun;                 // RS_ENG_MEM: set when a parse reads past the materialized words
    const RsZigSlow *zslow;
    const ZigFast *zfast;
    const u64 *rlx_A;
    void *out;
    u64 out0;                     // element index in `out` of this chunk's sample 0
    // gamma (GK_GAMMA) speculative store: the count pass keeps its parse's samples (+ a
    // packed per-sample tally word) per segment, the fixup keeps the re-parsed prefix, and
    // the emit pass copies instead of parsing a third time
    double *spec;                 // [T][spec_cap]
    u32 *spec_tal;                // [T][spec_cap]
    u64 spec_cap;
    double *pre;                  // [T][spec_cap]: a prefix is at most a segment's samples
    u32 *pre_tal;                 // [T][spec_cap]
    u32 *cmode;                   // per segment: 1 = copy (pre + spec), 0 = re-parse
    u32 *pre_n;                   // re-parsed prefix samples
    u32 *spec_from;               // speculative sample index where the prefix meets it
    u32 *spec_over;               // device flag: a segment or tally word overflowed (re-parse all)
    // paired laws (beta, F): the phase-1 parse's own samples (before it merges with phase 0)
    double *spec1;                // [T][spec_cap]
    u32 *spec1_tal;               // [T][spec_cap]
    u32 *c1own;                   // phase-1 samples before the merge (all of them if none)
    u32 *mrank0;                  // phase-0 sample index at the merge point
    // counted ranges: the first n_warm segments only resolve the slice's entry (count 0)
    u32 n_warm;
    // single-pass tile parse (rs_tile.cuh): tile records, tiles in the chunk, launch epoch,
    // and PCG64's affine step from one of a CTA's tiles to its next (G tiles on)
    u64 *tile_rec;
    u32 tile_nt, tile_epoch;
    u64 tile_m[2], tile_a[2];
};
// tile geometry of the single-pass parse: threads per CTA, words per thread and tile
constexpr int TL_T = 512, TL_W = 16;
constexpr size_t TL_SMEM = (size_t)(2 * TL_T + 2) * (TL_W + 1) * 8;
// per-sample tally word of the gamma attempt machine: gamma attempts (8 bits), normal
// attempts (12), normal pdf evaluations (12); 0xFFFFFFFF never occurs (flagged instead)
__device__ __forceinline__ bool pack_tally(u32 ga, u32 na, u32 np, u32 &w) {
    if (ga > 0xFF || na > 0xFFF || np > 0xFFF) return false;
    w = ga | (na << 8) | (np << 20);
    return true;
}

struct DevResult {
    u64 end_pos;     // logical position after the word that emitted sample n-1
    u64 total;       // samples available in this chunk
    u64 next_start;  // first boundary after the last segment
    u32 flag;        // entry resolution not at a fixed point
    u32 pad;
    u64 tally[6];
    u64 serial_state[32];
    u64 serial_buf[CAP];
    u64 serial_consumed;
};

// ----------------------------------------------------------------------------- device helpers
// segment bounds in stream units (words, or halves when unit == 2; a pending half
// precedes the buffered words in the half-unit stream of the first chunk)
__device__ __forceinline__ u64 seg_start(const FillPlan &p, u32 t) {
    return t == 0 ? p.lp0 : (u64)p.unit * ((u64)p.P + (u64)t * p.L) + p.pending_used;
}
__device__ __forceinline__ u64 seg_end(const FillPlan &p, u32 t) {
    return (u64)p.unit * ((u64)p.P + (u64)(t + 1) * p.L) + p.pending_used;
}

template <int E>
struct EngOf;
template <> struct EngOf<RS_ENG_X256SS> { typedef EngX256<true> type; };
template <> struct EngOf<RS_ENG_X256PP> { typedef EngX256<false> type; };
template <> struct EngOf<RS_ENG_PCG64> { typedef EngPcg type; };
template <> struct EngOf<RS_ENG_PHILOX> { typedef EngPhilox type; };
template <> struct EngOf<RS_ENG_RANLUX> { typedef EngRanlux type; };
template <> struct EngOf<RS_ENG_SFC64> { typedef EngSfc type; };
template <> struct EngOf<RS_ENG_SFC64_SIMD> { typedef EngSfcSimd type; };
template <> struct EngOf<RS_ENG_X128P> { typedef EngX128p type; };
template <> struct EngOf<RS_ENG_XORO> { typedef EngXoro type; };
template <> struct EngOf<RS_ENG_SQUARES> { typedef EngSquares type; };
template <> struct EngOf<RS_ENG_CHACHA20> { typedef EngChacha type; };
template <> struct EngOf<RS_ENG_CWG128> { typedef EngCwg type; };

// Parse source for engines whose words are expensive (Philox-4x64, ranlux++): the
// chunk's engine words are materialized once by the coalesced fixed-fill kernel and
// both parse passes read them back instead of regenerating them.
constexpr int RS_ENG_MEM = 100;
struct EngMem {  // reads its (per-lane sequential) words 32 bytes at a time, one group ahead
    const u64 *w;
    u32 *overrun;
    u64 idx, nw;   // idx: next word to return
    u64 g;         // word index of the prefetched group n0..n3
    u64 b0, b1, b2, b3, n0, n1, n2, n3;
    int have;      // words left in b (-1: nothing loaded yet)
    __device__ __forceinline__ void load(u64 at, u64 &x0, u64 &x1, u64 &x2, u64 &x3) {
        if (at >= nw) { *overrun = 1; x0 = x1 = x2 = x3 = 0; return; }
        asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(w + at));
    }
    __device__ __forceinline__ u64 next() {
        if (have <= 0) {
            if (have < 0) {  // first use: the group holding idx, then the one after it
                u64 a = idx & ~3ULL;
                load(a, b0, b1, b2, b3);
                have = 4;
                for (u64 j = a; j < idx; j++) { b0 = b1; b1 = b2; b2 = b3; have--; }
                g = a + 4;
            } else {
                b0 = n0; b1 = n1; b2 = n2; b3 = n3;
                have = 4;
                g += 4;
            }
            if (g < nw) load(g, n0, n1, n2, n3);
            // (the next 128-byte line towards L1: philox normals 2^28 3.75 -> 3.50 ms, gamma 3.12 -> 2.93)
            if ((g & 15) == 0 && g + 16 < nw) asm volatile("prefetch.global.L1 [%0];" ::"l"(w + g + 16));
        }
        u64 r = b0;
        b0 = b1; b1 = b2; b2 = b3;
        have--;
        idx++;
        return r;
    }
};
template <> struct EngOf<RS_ENG_MEM> { typedef EngMem type; };

// The same source for the 8-word batch loops (normal / exponential word-level parses): a
// batch is two 32-byte loads, and the line of the batch after next is requested with an L1
// prefetch hint, so the loads hit L1 without holding prefetched words in registers. (EngMem's
// group ahead in registers is consumed 4 words later -- too soon to hide the load latency
// in a batch that draws its 8 words back to back -- and a whole batch ahead in registers
// spilled: emit ran at 34 % issue with 92 M local-memory sectors. Philox normals 2^28
// 3.75 -> 2.80 ms, exponentials 2^26 1.06 -> 0.85 ms.) Single words (preambles, segment
// tails, re-parses) are plain 8-byte loads.
constexpr int RS_ENG_MEMB = 101;
struct EngMemB {
    const u64 *w;
    u32 *overrun;
    u64 idx, nw;  // idx: next word to return
    __device__ __forceinline__ void gen8(u64 *o) {
        if (idx + 8 > nw) { *overrun = 1; for (int k = 0; k < 8; k++) o[k] = 0; idx += 8; return; }
        if ((idx & 3) == 0) {
            asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(w + idx));
            asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(o[4]), "=l"(o[5]), "=l"(o[6]), "=l"(o[7]) : "l"(w + idx + 4));
        } else {
            for (int k = 0; k < 8; k++) o[k] = __ldg(w + idx + k);
        }
        idx += 8;
        if (idx + 8 < nw) asm volatile("prefetch.global.L1 [%0];" ::"l"(w + idx + 8));
    }
    __device__ __forceinline__ u64 next() {
        if (idx >= nw) { *overrun = 1; idx++; return 0; }
        return __ldg(w + idx++);
    }
    __device__ __forceinline__ bool batch_aligned() const { return (idx & 3) == 0; }
};
template <> struct EngOf<RS_ENG_MEMB> { typedef EngMemB type; };
// 8 consecutive words of any engine
template <class EN>
__device__ __forceinline__ void gen_batch(EN &e, u64 *w) {
    if constexpr (std::is_same<EN, EngMemB>::value) {
        e.gen8(w);
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = e.next();
    }
}

// engine positioned at engine word t*L of the chunk (thread t's segment start)
template <int E>
__device__ __forceinline__ void make_engine(const FillPlan &p, u32 t, typename EngOf<E>::type &e) {
    if constexpr (E == RS_ENG_X256SS || E == RS_ENG_X256PP || E == RS_ENG_X128P || E == RS_ENG_XORO) {
        e.load(p.x256_states + 4 * (u64)t);  // 128-bit engines use words 0, 1 of the padded state
    } else if constexpr (E == RS_ENG_SQUARES) {
        e.ctr = p.base[0] + (u64)t * p.L;
        e.key = p.base[1];
    } else if constexpr (E == RS_ENG_CHACHA20) {
#pragma unroll
        for (int i = 0; i < 4; i++) { e.k[2 * i] = (u32)p.base[i]; e.k[2 * i + 1] = (u32)(p.base[i] >> 32); }
        e.n0 = (u32)p.base[4];
        e.n1 = (u32)(p.base[4] >> 32);
        e.n2 = (u32)p.base[5];
        e.ctr = (u32)(p.base[5] >> 32) + (u32)((u64)t * (p.L / 8));  // the host checked 2^32
        e.left = 0;
    } else if constexpr (E == RS_ENG_CWG128) {
        typedef unsigned __int128 U;
        e.x = ((U)p.base[1] << 64) | p.base[0];
        e.weyl = ((U)p.base[3] << 64) | p.base[2];
        e.extra = ((U)p.base[5] << 64) | p.base[4];
        e.inc = ((U)p.base[7] << 64) | p.base[6];
    } else if constexpr (E == RS_ENG_PCG64) {
        e.slo = p.base[0]; e.shi = p.base[1]; e.ilo = p.base[2]; e.ihi = p.base[3];
        for (int j = 0; j < MAXLEV && (t >> j); j++)
            if ((t >> j) & 1) e.affine(p.pcg_m[j][0], p.pcg_m[j][1], p.pcg_a[j][0], p.pcg_a[j][1]);
    } else if constexpr (E == RS_ENG_PHILOX) {
        e.c0 = p.base[0]; e.c1 = p.base[1]; e.c2 = p.base[2]; e.c3 = p.base[3];
        e.k0 = p.base[4]; e.k1 = p.base[5];
        e.add((u64)t * (p.L / 4));
        e.left = 0;
    } else if constexpr (E == RS_ENG_RANLUX) {
#pragma unroll
        for (int i = 0; i < 9; i++) e.x[i] = p.base[i];
        for (int j = 0; j < MAXLEV && (t >> j); j++)
            if ((t >> j) & 1) rlx_mulmod_dev(e.x, p.rlx[j], e.x);
        e.left = 0;
        e.A = p.rlx_A;
    } else if constexpr (E == RS_ENG_SFC64) {
        e.a = p.base[0]; e.b = p.base[1]; e.c = p.base[2]; e.w = p.base[3];
    } else if constexpr (E == RS_ENG_SFC64_SIMD) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            e.l[k].a = p.lanes[4 * k]; e.l[k].b = p.lanes[4 * k + 1];
            e.l[k].c = p.lanes[4 * k + 2]; e.l[k].w = p.lanes[4 * k + 3];
        }
        e.k = 0;
    } else if constexpr (E == RS_ENG_MEM) {
        e.w = p.words;
        e.overrun = p.overrun;
        e.idx = (u64)t * p.L;
        e.nw = p.nwords;
        e.have = -1;
    } else if constexpr (E == RS_ENG_MEMB) {
        e.w = p.words;
        e.overrun = p.overrun;
        e.idx = (u64)t * p.L;
        e.nw = p.nwords;
    }
}

// The logical word stream of one segment: the buffered prefix (thread 0 of the
// first chunk only) then the engine. `pos` is the logical position.
template <int E>
struct Src {
    typename EngOf<E>::type e;
    const u64 *pre;
    int npre;
    u64 pos;
    __device__ __forceinline__ u64 next() {
        pos++;
        if (npre > 0) { npre--; return *pre++; }
        return e.next();
    }
};

// word source positioned at logical WORD position `pos` of segment t
template <int E>
__device__ __forceinline__ void make_wsrc(const FillPlan &p, u32 t, u64 pos, Src<E> &s) {
    make_engine<E>(p, t, s.e);
    s.npre = 0;
    s.pre = p.prefix;
    s.pos = pos;
    u64 skip;
    if (t == 0) {
        if (pos < (u64)p.P) { s.pre = p.prefix + pos; s.npre = p.P - (int)pos; skip = 0; }
        else skip = pos - p.P;
    } else {
        skip = pos - ((u64)p.P + (u64)t * p.L);
    }
    for (u64 i = 0; i < skip; i++) s.e.next();
}
template <int E>
__device__ __forceinline__ void make_src(const FillPlan &p, u32 t, u64 pos, Src<E> &s) { make_wsrc<E>(p, t, pos, s); }

// 32-bit half source (buffer.py:38-49): low half first; the pending half comes first
template <int E>
struct HSrc {
    Src<E> w;
    u64 pos;  // in halves
    u32 hi, pv;
    bool have, pend;
    __device__ __forceinline__ u32 next32() {
        pos++;
        if (pend) { pend = false; return pv; }
        if (have) { have = false; return hi; }
        u64 x = w.next();
        hi = (u32)(x >> 32);
        have = true;
        return (u32)x;
    }
};
template <int E>
__device__ __forceinline__ void make_src(const FillPlan &p, u32 t, u64 hpos, HSrc<E> &s) {
    s.pos = hpos;
    s.have = false;
    s.pend = false;
    s.pv = p.pending_val;
    if (t == 0 && p.pending_used && hpos == 0) {
        s.pend = true;
        make_wsrc<E>(p, t, 0, s.w);
        return;
    }
    u64 rel = hpos - p.pending_used;
    make_wsrc<E>(p, t, rel >> 1, s.w);
    if (rel & 1) {
        u64 x = s.w.next();
        s.hi = (u32)(x >> 32);
        s.have = true;
    }
}

// ---- sampler families (template key) and their construction from the plan
enum { FAM_LEMIRE = RS_DIST_UINT64, FAM_NORM = RS_DIST_NORM, FAM_EXP = RS_DIST_EXP, FAM_GAMMA = RS_DIST_GAMMA,
       FAM_F32 = 11, FAM_U32 = 22, FAM_FIXED = 40 /* per-stream mode: a fixed map of each word */,
       FAM_LEMIRE_RING = 41 /* per-stream mode: Lemire rows through the word-level chunk ring */ };
template <int D> struct DistOf;
template <> struct DistOf<FAM_NORM> { typedef DistNorm type; };
template <> struct DistOf<FAM_EXP> { typedef DistExp type; };
template <> struct DistOf<FAM_GAMMA> { typedef DistGamma type; };
template <> struct DistOf<FAM_LEMIRE> { typedef DistLemire type; };
template <> struct DistOf<FAM_F32> { typedef DistF32 type; };
template <> struct DistOf<FAM_U32> { typedef DistU32 type; };

template <int E, int D>
struct SrcOf {
    typedef typename std::conditional<DistOf<D>::type::HALF, HSrc<E>, Src<E>>::type type;
};

struct DistArgs {  // what a family needs (the plan and the per-stream args both provide it)
    const double *fp;
    const u64 *ip;
    const GammaPrm *ga, *gb;
    int kind, fm;
    const RsZigSlow *zslow;
    const RsZigSlowF *zslowf;
};

template <int D>
__device__ __forceinline__ void make_dist_a(const DistArgs &a, const void *fast, typename DistOf<D>::type &d) {
    if constexpr (D == FAM_LEMIRE) {
        d.b = a.ip[0]; d.thr = a.ip[1]; d.m = a.ip[2];
    } else if constexpr (D == FAM_U32) {
        d.b = a.ip[0]; d.thr = a.ip[1]; d.m = (u32)a.ip[2]; d.width = (int)a.ip[3];
        d.mask = d.width == 32 ? 0xFFFFFFFFULL : ((1ULL << d.width) - 1);
    } else if constexpr (D == FAM_F32) {
        d.z.fast = (const ZigFastF *)fast; d.z.slow = a.zslowf; d.z.fm = a.fm;
        d.a = a.fp[0]; d.b = a.fp[1]; d.kind = a.kind;
    } else {
        d.z.fast = (const ZigFast *)fast; d.z.slow = a.zslow; d.z.fm = a.fm;
        if constexpr (D == FAM_NORM) {
            d.a = a.fp[0]; d.b = a.fp[1]; d.c = a.fp[2]; d.d = a.fp[3]; d.kind = a.kind;
        } else if constexpr (D == FAM_EXP) {
            d.a = a.fp[0]; d.b = a.fp[1]; d.c = a.fp[2]; d.kind = a.kind;
        } else {
            d.ga = *a.ga; d.gb = *a.gb; d.nu1 = a.fp[0]; d.nu2 = a.fp[1]; d.kind = a.kind;
        }
    }
}
template <int D>
__device__ __forceinline__ void make_dist(const FillPlan &p, const void *fast, typename DistOf<D>::type &d) {
    DistArgs a{p.fp, p.ip, &p.ga, &p.gb, p.kind, p.fm, p.zslow, p.zslowf};
    make_dist_a<D>(a, fast, d);
}

__device__ __forceinline__ void stage_tables(const FillPlan &p, ZigFast *sm) {
    if (p.zfast) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = p.zfast[i];
    } else if (p.zfastf) {
        ZigFastF *f = (ZigFastF *)sm;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) f[i] = p.zfastf[i];
    }
    __syncthreads();
}

// ----------------------------------------------------------------------------- x256 jump setup
// Thread t starts at engine word t*L: state = T^(t*L) * base over GF(2) (jumps.py:116-126
// restated as 256x256 bit matrices, column-major, 8 KB each). Warp w first jumps by
// 32*L*w using ML[1 + k] = T^(32*L*2^k) for the set bits k of w; its 32 lane states
// then follow by chained products with ML[0] = T^L. Every product is warp-cooperative:
// lane l owns columns 8l..8l+7 (one coalesced 256-byte read), then a 5-step xor
// butterfly leaves the result in every lane.
// One warp-cooperative product with the state held as one byte per lane (lane l: bits
// 8l..8l+7). Lane l owns columns 8l..8l+7 (one coalesced 256-byte read); the partial sums
// are then reduce-scattered in 5 halving steps (9 32-bit shuffles) so that every lane ends
// with exactly its own byte of the product -- the input of the next product.
__device__ __forceinline__ u32 warp_matvec_rs(const u64 *M, u32 byte) {
    const u32 lane = threadIdx.x & 31;
    u64 a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const ulonglong2 *c = (const ulonglong2 *)(M + (u64)(8 * lane) * 4);
#pragma unroll
    for (int k = 0; k < 8; k++) {
        u64 m = (byte >> k) & 1 ? ~0ULL : 0ULL;
        ulonglong2 x = __ldg(c + 2 * k), y = __ldg(c + 2 * k + 1);
        a0 ^= x.x & m;
        a1 ^= x.y & m;
        a2 ^= y.x & m;
        a3 ^= y.y & m;
    }
    // lane bit 4 picks the 128-bit half (words 0-1 / 2-3), bit 3 the word, bit 2 the 32-bit
    // half, bit 1 the 16-bit quarter, bit 0 the byte
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
    u64 k0 = b4 ? a2 : a0, k1 = b4 ? a3 : a1;
    k0 ^= __shfl_xor_sync(0xFFFFFFFFu, b4 ? a0 : a2, 16);
    k1 ^= __shfl_xor_sync(0xFFFFFFFFu, b4 ? a1 : a3, 16);
    u64 kw = b3 ? k1 : k0;
    kw ^= __shfl_xor_sync(0xFFFFFFFFu, b3 ? k0 : k1, 8);
    const u32 lo = (u32)kw, hi = (u32)(kw >> 32);
    u32 k32 = b2 ? hi : lo;
    k32 ^= __shfl_xor_sync(0xFFFFFFFFu, b2 ? lo : hi, 4);
    u32 k16 = b1 ? (k32 >> 16) : (k32 & 0xFFFFu);
    k16 ^= __shfl_xor_sync(0xFFFFFFFFu, b1 ? (k32 & 0xFFFFu) : (k32 >> 16), 2);
    u32 k8 = b0 ? (k16 >> 8) : (k16 & 0xFFu);
    k8 ^= __shfl_xor_sync(0xFFFFFFFFu, b0 ? (k16 & 0xFFu) : (k16 >> 8), 1);
    return k8;
}

#ifdef RS_KERNELS_MISC
__global__ void __launch_bounds__(BLOCK) k_x256_setup(const __grid_constant__ FillPlan p, const u64 *ML,
                                                      u64 *states) {
    // each lane's byte of its warp's states at steps 0..31 (lane j then reads row j)
    __shared__ __align__(16) unsigned char sb[BLOCK / 32][32][32];
    const u32 lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const u64 w = ((u64)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    // gridDim.y == 8: interleaved engine, one grid row per lane (base = that lane's state)
    const u64 *b0 = gridDim.y > 1 ? p.lanes + 4 * blockIdx.y : p.base;
    states += (u64)blockIdx.y * 4 * ((u64)gridDim.x * BLOCK);
    const u64 vq = __ldg(b0 + (lane >> 3));
    u32 byte = (u32)((vq >> (8 * (lane & 7))) & 0xFF);
    u64 ww = w;
    for (int k = 0; ww; k++, ww >>= 1)
        if (ww & 1) byte = warp_matvec_rs(ML + (u64)(1 + k) * 1024, byte);
    sb[wi][0][lane] = (unsigned char)byte;
    for (u32 j = 1; j < 32; j++) {
        byte = warp_matvec_rs(ML, byte);
        sb[wi][j][lane] = (unsigned char)byte;
    }
    __syncwarp();
    const ulonglong2 *row = (const ulonglong2 *)&sb[wi][lane][0];
    ulonglong2 *d = (ulonglong2 *)(states + 4 * (32 * w + lane));
    d[0] = row[0];
    d[1] = row[1];
}
#endif  // RS_KERNELS_MISC

// bytes per BatchRing group in k_emit (one group leaves per tick as GB/32 STG.256)
constexpr int EMIT_GB = 64;

// resident blocks per SM the parse kernels are compiled for (register budget)
constexpr int minb(int E, int D) {
    return D == FAM_GAMMA ? 2 : (D == FAM_LEMIRE || D == FAM_U32) ? 4 : 3;
}

// ----------------------------------------------------------------------------- word-level drivers
// Samples that start before `end` (count) / the next `kmax` samples (emit). The buffered
// prefix (thread 0 of the first chunk only) is consumed in a preamble so the steady-state
// loop reads the engine directly and tracks its position with 32-bit counters.
//
// Batch parse (the bulk of both passes): every lane takes ZB = 8 words per step. The 8
// fast-path tests and sample values are computed unconditionally (no branch per word);
// a lane whose 8 words are all fast-path samples from a boundary emits them as they are.
// Otherwise the lane walks only its non-fast words: a non-fast start is a wedge token
// (two words, the second one's decision made after the walk) or a tail (the lane then
// runs the exact word machine over the batch, ~0.2 % of lane-batches). The wedge
// consumption is 2 words whatever the decision, so the token structure is known before
// any decision is made, and the decisions of a batch run once per warp for all lanes
// (the per-word machine ran its rare branch on ~37 % of warp-steps, one lane active).
// An accepted wedge's sample takes its first word's slot, so samples stay in order.
constexpr int ZB = 8;

// The batch's token structure in machine state m (0, or 1 = a wedge carried from the
// previous batch whose second word is w[0]). Returns false when the lane must take the
// exact machine (a carried tail, or a tail token in the batch) -- before any side effect.
// Otherwise: O = sample slots (fast starts, accepted wedges at their first word, and bit 0
// for an accepted carried wedge, whose value is xc), att = attempts started in the batch,
// m = the state carried out (1: a wedge starts on the last word), bnd = the batch ends on
// a sample boundary.
// WS: the batch's words staged in shared memory, ws(q) = word q. F: fast-path bits, Z: bits
// of words whose strip index is 0 (a non-fast start there is a tail).
template <class D, class WS>
__device__ __forceinline__ bool zb_tokens(const D &d, ZigWM &m, const WS &ws, u32 F, u32 Z, u32 &O, u32 &att,
                                       bool &bnd, double &xc, Tally &tl) {
    const u32 cin = m.st;
    const u32 N = ~F & 0xFFu;
    // (a non-fast word with index 0 may be a tail start: the exact machine takes the batch;
    // ~0.2 % of lane-batches, some of them a wedge's second word that only looks like one)
    if (cin >= 2 || (N & Z)) return false;
    u32 Wm, starts = cin ? 0xFEu : 0xFFu;
    if ((N & (N >> 1)) == 0) {  // no two non-fast words in a row: each one (but a carried
        Wm = N & starts;        // wedge's second word) starts a wedge
    } else {
        Wm = 0;
        u32 cand = N & starts;
        while (cand) {
            const int q = __ffs(cand) - 1;
            Wm |= 1u << q;
            starts &= ~(2u << q);  // the next word is the wedge's second
            cand = N & starts & ~((2u << q) - 1u);
        }
    }
    starts &= ~(Wm << 1);
    u32 o = F & starts;
    if (cin) {
        xc = d.zval_m(m);
        if (d.zwedge_m(m, ws(0), tl)) o |= 1u;
    }
    u32 dw = Wm & 0x7Fu;
    while (dw) {
        const int q = __ffs(dw) - 1;
        dw &= dw - 1;
        if (d.zwedge(ws(q), ws(q + 1), tl)) o |= 1u << q;
    }
    if (Wm & 0x80u) d.zcarry(m, ws(ZB - 1));
    else m.st = 0;
    bnd = ((o >> 7) & 1) || (((Wm >> 6) & 1) && ((o >> 6) & 1));
    O = o;
    att = __popc(starts);
    return true;
}

template <class D, class SRC>
__device__ __forceinline__ u64 wl_count(const D &d, SRC &s, u64 end, Tally &tl, u64 *wsm) {
    ZigWM m;
    m.st = 0;
    bool bnd = true;
    u64 c = 0;
    while (s.npre > 0 && !(bnd && s.pos >= end)) {
        double z;
        bnd = d.feed(m, s.next(), tl, z);
        c += bnd;
    }
    u32 left = s.pos < end ? (u32)(end - s.pos) : 0u, used = 0, cc = 0;
    // batches that lie inside the segment (no exit is possible inside them)
    auto ws = [wsm](int q) -> u64 { return wsm[q * BLOCK]; };
    while (used + ZB <= left) {
        u64 w[ZB];
        gen_batch(s.e, w);
        u32 F = 0, Z = 0;
#pragma unroll
        for (int h = 0; h < ZB; h += 4) {
            ZigFast f[4];
#pragma unroll
            for (int k = 0; k < 4; k++) f[k] = d.strip(w[h + k]);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                F |= (d.zfast(w[h + k], f[k]) ? 1u : 0u) << (h + k);
                Z |= (((u32)w[h + k] & 0xFFu) == 0 ? 1u : 0u) << (h + k);
            }
        }
        if (F == 0xFFu && m.st == 0) {
            cc += ZB;
            bnd = true;
        } else if constexpr (std::is_same<decltype(s.e), EngMemB>::value) {
            // materialised words are read again where they lie (L1 hits) instead of staged
            const u64 *wp = s.e.w + (s.e.idx - ZB);
            auto wg = [wp](int q) -> u64 { return __ldg(wp + q); };
            u32 O, att;
            double xc;
            if (zb_tokens(d, m, wg, F, Z, O, att, bnd, xc, tl)) {
                cc += __popc(O);
            } else {
                for (int k = 0; k < ZB; k++) {
                    double z;
                    bnd = d.feed(m, wg(k), tl, z);
                    cc += bnd;
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < ZB; k++) wsm[k * BLOCK] = w[k];
            u32 O, att;
            double xc;
            if (zb_tokens(d, m, ws, F, Z, O, att, bnd, xc, tl)) {
                cc += __popc(O);
            } else {  // exact machine over the batch
                for (int k = 0; k < ZB; k++) {
                    double z;
                    bnd = d.feed(m, ws(k), tl, z);
                    cc += bnd;
                }
            }
        }
        used += ZB;
    }
    // the rest of the segment word by word, up to the first boundary past its end (words
    // generated past the exit are dropped: only the position matters)
    while (!(bnd && used >= left)) {
        u64 w[4];
        ZigFast f[4];
#pragma unroll
        for (int k = 0; k < 4; k++) w[k] = s.e.next();
#pragma unroll
        for (int k = 0; k < 4; k++) f[k] = d.strip(w[k]);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (bnd && used >= left) break;
            double z;
            bnd = d.feed(m, w[k], f[k], tl, z);
            used++;
            cc += bnd;
        }
    }
    s.pos += used;
    return c + cc;
}
template <class D, class SRC, class W>
__device__ __forceinline__ void wl_emit(const D &d, SRC &s, u64 kmax, W &wr, Tally &tl) {
    static_assert(W::G == ZB, "one BatchRing group per batch");
    ZigWM m;
    m.st = 0;
    u64 k = 0;
    while (s.npre > 0 && k < kmax) {
        double z;
        if (d.feed(m, s.next(), tl, z)) { wr.put(d.finish(z)); k++; }
        wr.tick();  // (thread 0 only: one sample per tick keeps the ring bound)
    }
    u32 left = (u32)(kmax - k), used = 0;
    // batches while at least ZB samples remain (a batch emits at most ZB). A slow batch
    // stages its words in the ring's free slots (at most G - 1 samples are pending after a
    // tick, so the next ZB slots are free; the batch's own samples overwrite them in order,
    // after the words have been read).
    if constexpr (std::is_same<decltype(s.e), EngMemB>::value) {
        // (word by word up to a 32-byte boundary of the materialised words: the batches'
        // loads are then two aligned 32-byte groups per lane)
        while (!s.e.batch_aligned() && left) {
            double z;
            used++;
            if (d.feed(m, s.e.next(), tl, z)) { wr.put(d.finish(z)); left--; }
            wr.tick();
        }
    }
    while (left >= ZB) {
        u64 w[ZB];
        gen_batch(s.e, w);
        u32 F = 0, Z = 0;
        double x[ZB];
#pragma unroll
        for (int h = 0; h < ZB; h += 4) {
            ZigFast f[4];
#pragma unroll
            for (int q = 0; q < 4; q++) f[q] = d.strip(w[h + q]);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                F |= (d.zfast(w[h + q], f[q]) ? 1u : 0u) << (h + q);
                Z |= (((u32)w[h + q] & 0xFFu) == 0 ? 1u : 0u) << (h + q);
                x[h + q] = d.zval(w[h + q], f[q]);
            }
        }
        u32 O = 0xFFu;
        if (F != 0xFFu || m.st != 0) {
            const u32 fb = wr.free_base();
            const u64 *wp = nullptr;
            if constexpr (std::is_same<decltype(s.e), EngMemB>::value) {
                wp = s.e.w + (s.e.idx - ZB);  // materialised words: read again where they lie
            } else {
#pragma unroll
                for (int q = 0; q < ZB; q++) *wr.slot_at(fb + q) = w[q];
            }
            auto ws = [&wr, fb, wp](int q) -> u64 {
                if constexpr (std::is_same<decltype(s.e), EngMemB>::value) return __ldg(wp + q);
                else return *wr.slot_at(fb + (u32)q);
            };
            u32 att;
            bool bnd;
            double xc = 0.0;
            const u32 cin = m.st;
            if (zb_tokens(d, m, ws, F, Z, O, att, bnd, xc, tl)) {
                d.zatt(tl, att);
                if (cin) x[0] = xc;  // the carried wedge's sample takes slot 0 (its second word)
            } else {  // exact machine over the batch, writing its own samples
                // (the j-th put of the batch lands in staged slot j <= the word being fed)
                O = 0;
                for (int q = 0; q < ZB; q++) {
                    double z;
                    if (d.feed(m, ws(q), tl, z)) { wr.put(d.finish(z)); left--; }
                }
            }
        } else {
            d.zatt(tl, ZB);
        }
        // the batch's samples into the ring without a branch per word: x[q] goes to the slot
        // after the samples of the words before it, so a word without a sample is overwritten
        // by the next sample (or lands in a free slot past them)
        {
            const u32 fb = wr.free_base();
            u32 c = 0;
#pragma unroll
            for (int q = 0; q < ZB; q++) {
                *(double *)wr.slot_at(fb + c) = d.finish(x[q]);
                c += (O >> q) & 1;
            }
            wr.advance(c);
        }
        left -= __popc(O);
        used += ZB;
        wr.tick();
    }
    // the last < ZB samples word by word (one word of software pipelining: the next word is
    // generated and its strip load issued before the current word is fed; the extra word
    // at the end is never fed, the position counts fed words only)
    u64 wn = s.e.next();
    ZigFast fn = d.strip(wn);
    while (left) {
        u64 w = wn;
        ZigFast f = fn;
        wn = s.e.next();
        fn = d.strip(wn);
        double z;
        used++;
        if (d.feed(m, w, f, tl, z)) { wr.put(d.finish(z)); left--; }
        if ((used & (W::G - 1)) == 0) wr.tick();
    }
    s.pos += used;
}

// ----------------------------------------------------------------------------- two-pass parse
// boundary bitmap writer: bit q of the segment's map = a sample starts at start + q
struct BmRec {
    u32 *bm;  // [W][T]
    u32 T, t;
    u64 start;
    u32 W;
    u32 acc = 0, kw = 0;
    __device__ __forceinline__ void put(u64 pos) {
        u64 q = pos - start;
        if (!bm || q >= 32ULL * W) return;
        u32 k = (u32)(q >> 5);
        while (kw < k) { bm[(size_t)kw * T + t] = acc; acc = 0; kw++; }
        acc |= 1u << (q & 31);
    }
    __device__ __forceinline__ void close() {
        if (!bm) return;
        while (kw < W) { bm[(size_t)kw * T + t] = acc; acc = 0; kw++; }
    }
};
// samples of a recorded parse that start before unit q (q < 32 * bmw)
__device__ __forceinline__ u64 bm_rank(const u32 *bm, u32 T, u32 t, u64 q) {
    u32 k = (u32)(q >> 5);
    u64 r = 0;
#pragma unroll 8
    for (u32 j = 0; j < k; j++) r += __popc(__ldg(&bm[(size_t)j * T + t]));
    return r + __popc(bm[(size_t)k * T + t] & ((1u << (q & 31)) - 1u));
}
// unit offset of the j-th recorded boundary (j = 0: the segment start), -1 if not recorded
__device__ __forceinline__ long long bm_select(const u32 *bm, u32 T, u32 t, u32 W, u64 j) {
    u64 r = 0;
    for (u32 k = 0; k < W; k++) {
        u32 w = __ldg(&bm[(size_t)k * T + t]);
        u32 pc = __popc(w);
        if (r + pc > j) {
            for (u64 i = r; i < j; i++) w &= w - 1;  // drop the lower set bits
            return 32LL * k + (__ffs(w) - 1);
        }
        r += pc;
    }
    return -1;
}
// bm_rank over bitmaps the calling thread wrote itself in this kernel (no __ldg)
__device__ __forceinline__ u64 bm_rank_own(const u32 *bm, u32 T, u32 t, u64 q) {
    u32 k = (u32)(q >> 5);
    u64 r = 0;
#pragma unroll 8
    for (u32 j = 0; j < k; j++) r += __popc(bm[(size_t)j * T + t]);
    return r + __popc(bm[(size_t)k * T + t] & ((1u << (q & 31)) - 1u));
}
// The count pass's phase-1 parse of a paired law (kept out of line: its registers and
// its speculative store would otherwise weigh on the phase-0 loop of every gamma law).
template <int E, int D>
__device__ __noinline__ void count_phase1(const FillPlan &p, const typename DistOf<D>::type &d, u32 t, u64 end,
                                          u64 c, u64 spos, Tally &tl, unsigned char *ring_sp, u64 *cnt1,
                                          u32 *ex1) {
        typename SrcOf<E, D>::type s1;
        make_src<E>(p, t, seg_start(p, t), s1);
        u64 c1 = 0;
        BmRec r{p.bm ? p.bm + (size_t)p.bmw * p.T : nullptr, p.T, t, seg_start(p, t), p.bmw};
        bool am = false;
        if constexpr (D == FAM_GAMMA) am = d.am_applies();
        bool merged = false;
        if (am) {
            if constexpr (D == FAM_GAMMA) {
                GammaAM m{1, 1, 0.0};  // a lone second sub-sample first
                double v;
                while (!d.am_step(m, s1, tl, v)) {}
                r.put(s1.pos);  // phase 1's first full sample starts after the lone second
                // speculative store of phase 1's own samples (the rest are phase 0's)
                const bool sp = p.spec != nullptr;
                BatchRing<double, BLOCK> wv;
                BatchRing<u32, BLOCK> wt;
                if (sp) {
                    wv.init(p.spec1, (u64)t * p.spec_cap, (double *)ring_sp + threadIdx.x);
                    wt.init(p.spec1_tal, (u64)t * p.spec_cap, (u32 *)(ring_sp + 64 * BLOCK) + threadIdx.x);
                }
                Tally t0 = tl;
                bool over = false;
                u32 it = 0;
                u64 rk0 = 0;
                // Once phase 1 starts a sample where phase 0 did, the two parses coincide
                // to the segment end: the rest of phase 1's count is phase 0's, read off
                // the phase-0 bitmap this thread just wrote (plain loads: own stores).
                const u32 *b0 = p.bm;
                const u64 st0 = seg_start(p, t);
                while (s1.pos < end) {
                    if (b0) {
                        const u64 q = s1.pos - st0;
                        if ((b0[(size_t)(q >> 5) * p.T + t] >> (q & 31)) & 1) {
                            rk0 = bm_rank_own(b0, p.T, t, q);
                            merged = true;
                            break;
                        }
                    }
                    while (!d.am_step(m, s1, tl, v)) {}
                    c1++;
                    r.put(s1.pos);
                    if (sp) {
                        u32 w;
                        over |= !pack_tally(tl.gamma_att - t0.gamma_att, tl.norm_att - t0.norm_att,
                                            tl.norm_pdf - t0.norm_pdf, w);
                        t0 = tl;
                        if (c1 <= p.spec_cap) { wv.put(v); wt.put(w); }
                        if ((++it & 3) == 0) { wv.tick(); wt.tick(); }
                    }
                }
                if (sp) {
                    wv.finish();
                    wt.finish();
                    if (over || c1 > p.spec_cap) atomicOr(p.spec_over, 1u);
                    p.c1own[t] = (u32)c1;
                    p.mrank0[t] = (u32)rk0;
                }
                if (merged) c1 += c - rk0;
            }
        } else {
            d.skip_second(s1, tl);
            r.put(s1.pos);  // phase 1's first full sample starts after the lone second
            while (s1.pos < end) {
                d.sample(s1, tl);
                c1++;
                r.put(s1.pos);
            }
        }
        r.close();
        cnt1[t] = c1;
        ex1[t] = merged ? (u32)(spos - end) : (u32)(s1.pos - end);
}

// count: samples that START inside [seg_start, seg_end) and the exit (first sample
// boundary at or beyond seg_end), parsing from seg_start as if it were a boundary.
// For paired samplers (beta, f, t, skew_normal: two sub-samples per sample) a parse
// that starts one sub-sample off never realigns at a sample boundary when the two
// sub-grammars coincide, so the count pass also parses phase 1 (starting with a lone
// second sub-sample) into cnt1/ex1; the fixup converges against either phase.
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_count(const __grid_constant__ FillPlan p, u64 *cnt0, u32 *ex0,
                                                            u64 *cnt1, u32 *ex1) {
    __shared__ ZigFast sm[256];
    __shared__ __align__(16) unsigned char ring_sp[D == FAM_GAMMA ? 128 * BLOCK : 16];  // speculative store
    __shared__ u64 zb_sm[(D == FAM_NORM || D == FAM_EXP) ? ZB * BLOCK : 1];              // batch words
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    if (t >= p.T) return;
    const u64 end = seg_end(p, t);
    typename SrcOf<E, D>::type s;
    make_src<E>(p, t, seg_start(p, t), s);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl = {0, 0, 0, 0, 0};
    u64 c = 0;
    if constexpr (D == FAM_LEMIRE || D == FAM_U32) {  // independent one-unit tokens: unit-level loop
        bool bnd = true;
        while (!(bnd && s.pos >= end)) {
            typename DistOf<D>::type::out_t o;
            if constexpr (D == FAM_LEMIRE) bnd = d.accept(s.next(), o);
            else bnd = d.accept(s.next32(), o);
            c += bnd;
        }
    } else {
        bool done = false;
        if constexpr (D == FAM_NORM || D == FAM_EXP) {
            if (d.word_level()) {  // one word per lane per step (uniform engine step)
                c = wl_count(d, s, end, tl, zb_sm + threadIdx.x);
                done = true;
            }
        }
        if (!done) {
            if constexpr (D == FAM_GAMMA) {
                BmRec r{p.bm, p.T, t, seg_start(p, t), p.bmw};
                r.put(r.start);  // phase 0 starts a sample at the segment start
                if (d.am_applies() && p.spec) {  // + speculative store
                    BatchRing<double, BLOCK> wv;
                    BatchRing<u32, BLOCK> wt;
                    wv.init(p.spec, (u64)t * p.spec_cap, (double *)ring_sp + threadIdx.x);
                    wt.init(p.spec_tal, (u64)t * p.spec_cap, (u32 *)(ring_sp + 64 * BLOCK) + threadIdx.x);
                    GammaAM m{0, 0, 0.0};
                    Tally t0 = tl;
                    bool over = false;
                    u32 it = 0;
                    while (true) {
                        double v;
                        if (d.am_step(m, s, tl, v)) {
                            c++;
                            r.put(s.pos);
                            u32 w;
                            over |= !pack_tally(tl.gamma_att - t0.gamma_att, tl.norm_att - t0.norm_att,
                                                tl.norm_pdf - t0.norm_pdf, w);
                            t0 = tl;
                            if (c <= p.spec_cap) { wv.put(v); wt.put(w); }
                            if (s.pos >= end) break;
                        }
                        if ((++it & 3) == 0) { wv.tick(); wt.tick(); }
                    }
                    wv.finish();
                    wt.finish();
                    if (over || c > p.spec_cap) atomicOr(p.spec_over, 1u);
                } else if (d.am_applies()) {  // attempt-level machine (same samples and positions)
                    GammaAM m{0, 0, 0.0};
                    while (true) {
                        double v;
                        if (d.am_step(m, s, tl, v)) {
                            c++;
                            r.put(s.pos);
                            if (s.pos >= end) break;
                        }
                    }
                } else {
                    while (s.pos < end) {
                        d.sample(s, tl);
                        c++;
                        r.put(s.pos);
                    }
                }
                r.close();
            } else {
                while (s.pos < end) {
                    d.sample(s, tl);
                    c++;
                }
            }
        }
        if (d.paired()) count_phase1<E, D>(p, d, t, end, c, s.pos, tl, ring_sp, cnt1, ex1);
    }
    cnt0[t] = c;
    ex0[t] = (u32)(s.pos - end);
}

// The true entry e of segment t is segment t-1's exit. Parse from start+e (B) and
// from start (A) in lockstep, always advancing the one behind by one sample, until
// they meet at a common boundary inside the segment (then counts differ only by
// the samples before the meeting point) or B reaches its own exit.
template <int E, int D>
__device__ void resolve_entry(const FillPlan &p, const ZigFast *sm, u32 t, u32 e, u64 c0, u32 x0, u64 c1, u32 x1,
                              u64 &cnt, u32 &ex) {
    const u64 start = seg_start(p, t), end = seg_end(p, t);
    if constexpr (D == FAM_GAMMA) {
        if (p.bm) {  // B alone, meeting points looked up in the count pass's bitmaps
            typename SrcOf<E, D>::type sb;
            make_src<E>(p, t, start + e, sb);
            typename DistOf<D>::type d;
            make_dist<D>(p, sm, d);
            Tally tl = {0, 0, 0, 0, 0};
            const bool two = d.paired();
            // speculative store (GK_GAMMA): keep the prefix samples for k_emit's copy
            const bool sp = p.spec && d.am_applies();
            bool keep = sp;
            const u32 *bm0 = p.bm, *bm1 = p.bm + (size_t)p.bmw * p.T;
            u64 nb = 0;
            u32 kw = ~0u, wa = 0, wc = 0;
            while (true) {
                if (sb.pos >= end) {
                    cnt = nb;
                    ex = (u32)(sb.pos - end);
                    if (sp) { p.cmode[t] = keep; p.pre_n[t] = (u32)nb; p.spec_from[t] = 0; }
                    return;
                }
                u64 q = sb.pos - start;
                if (q >= 32ULL * p.bmw) break;
                u32 k = (u32)(q >> 5), bit = 1u << (q & 31);
                if (k != kw) {
                    kw = k;
                    wa = bm0[(size_t)k * p.T + t];
                    if (two) wc = bm1[(size_t)k * p.T + t];
                }
                if (wa & bit) {
                    const u64 rk = bm_rank(bm0, p.T, t, q);
                    cnt = c0 - rk + nb;
                    ex = x0;
                    if (sp) { p.cmode[t] = keep; p.pre_n[t] = (u32)nb; p.spec_from[t] = (u32)rk; }
                    return;
                }
                if (two && (wc & bit)) {
                    const u64 rk = bm_rank(bm1, p.T, t, q);
                    cnt = c1 - rk + nb;
                    ex = x1;
                    if (sp) { p.cmode[t] = keep ? 2u : 0u; p.pre_n[t] = (u32)nb; p.spec_from[t] = (u32)rk; }
                    return;
                }
                if (d.am_applies()) {  // one sample through the attempt-level machine
                    GammaAM m{0, 0, 0.0};
                    double v;
                    Tally t0 = tl;
                    while (!d.am_step(m, sb, tl, v)) {}
                    if (keep) {
                        u32 w;
                        if (nb < p.spec_cap && pack_tally(tl.gamma_att - t0.gamma_att, tl.norm_att - t0.norm_att,
                                                       tl.norm_pdf - t0.norm_pdf, w)) {
                            p.pre[(size_t)t * p.spec_cap + nb] = v;
                            p.pre_tal[(size_t)t * p.spec_cap + nb] = w;
                        } else {
                            keep = false;
                        }
                    }
                } else {
                    d.sample(sb, tl);
                }
                nb++;
            }
            if (sp) p.cmode[t] = 0;
        }  // no meeting in the recorded window: the lockstep parse below
    }
    typename SrcOf<E, D>::type sa, sb, sc;
    make_src<E>(p, t, start, sa);
    make_src<E>(p, t, start + e, sb);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl = {0, 0, 0, 0, 0};
    const bool two = d.paired();
    if (two) {  // the phase-1 parse: lone second sub-sample first
        make_src<E>(p, t, start, sc);
        d.skip_second(sc, tl);
    }
    u64 na = 0, nb = 0, nc = 0;
    while (true) {
        if (sb.pos >= end) {  // B reached its exit without meeting A
            cnt = nb;
            ex = (u32)(sb.pos - end);
            return;
        }
        if (sa.pos == sb.pos) {  // converged with the phase-0 parse inside the segment
            cnt = c0 - na + nb;
            ex = x0;
            return;
        }
        if (two && sc.pos == sb.pos) {  // converged with the phase-1 parse
            cnt = c1 - nc + nb;
            ex = x1;
            return;
        }
        // advance the parse that is furthest behind (A parses only inside the segment)
        u64 pa = sa.pos < end ? sa.pos : ~0ULL;
        u64 pc = two && sc.pos < end ? sc.pos : ~0ULL;
        if (pa <= pc && pa < sb.pos) {
            d.sample(sa, tl);
            na++;
        } else if (pc < pa && pc < sb.pos) {
            d.sample(sc, tl);
            nc++;
        } else {
            d.sample(sb, tl);
            nb++;
        }
    }
}

// Output offsets without a scan launch: k_fixup leaves the sum of each block's counts
// (bsum[block]) and their total; an emit block adds the sums of the blocks before it
// (<= T / BLOCK values) to the exclusive scan of its own BLOCK counts.
__device__ __forceinline__ u64 warp_sum64(u64 v) {
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, sh);
    return v;
}
__device__ __forceinline__ u64 block_offset(const u64 *bsum, u64 c) {
    __shared__ u64 wtot[BLOCK / 32], wbase[BLOCK / 32];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u64 b = 0;
    for (u32 i = threadIdx.x; i < blockIdx.x; i += BLOCK) b += bsum[i];
    b = warp_sum64(b);
    u64 inc = c;
#pragma unroll
    for (int sh = 1; sh < 32; sh <<= 1) {
        u64 v = __shfl_up_sync(0xFFFFFFFFu, inc, sh);
        if (lane >= (u32)sh) inc += v;
    }
    if (lane == 31) wtot[wid] = inc;
    if (lane == 0) wbase[wid] = b;
    __syncthreads();
    u64 o = inc - c;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; w++) {
        o += wbase[w];
        if ((u32)w < wid) o += wtot[w];
    }
    return o;
}

// round 0: prev_ex = ex0, every thread; round r>0: only threads whose entry changed
// re-resolve; every thread contributes its count to the block's sum.
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_fixup(const __grid_constant__ FillPlan p, const u64 *cnt0, const u32 *ex0,
                                                 const u64 *cnt1, const u32 *ex1, const u32 *prev_ex, u32 *entry,
                                                 u64 *cnt, u32 *ex, int round, DevResult *res, u64 *bsum) {
    __shared__ ZigFast sm[256];
    __shared__ u64 wsum[BLOCK / 32];
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    u64 c = 0;
    if (t < p.T) {
        u32 e = t == 0 ? 0u : prev_ex[t - 1];
        if (round > 0 && e == entry[t]) {
            ex[t] = prev_ex[t];
            c = cnt[t];
        } else {
            entry[t] = e;
            u32 x;
            if (e == 0) {
                c = cnt0[t];
                x = ex0[t];
                if (p.spec) { p.cmode[t] = 1; p.pre_n[t] = 0; p.spec_from[t] = 0; }
            } else {
                resolve_entry<E, D>(p, sm, t, e, cnt0[t], ex0[t], cnt1[t], ex1[t], c, x);
            }
            if (t < p.n_warm) c = 0;  // a warm-up segment emits nothing
            cnt[t] = c;
            ex[t] = x;
            if (x != prev_ex[t]) atomicOr(&res->flag, 1u);
        }
    }
    c = warp_sum64(c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 tot = 0;
#pragma unroll
        for (int w = 0; w < BLOCK / 32; w++) tot += wsum[w];
        bsum[blockIdx.x] = tot;
        if (tot) atomicAdd((unsigned long long *)&res->total, (unsigned long long)tot);
    }
}

// emit: re-parse from the true entry and write this segment's samples at their
// global offsets (exclusive scan of the counts).
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_emit(const __grid_constant__ FillPlan p, const u32 *entry, const u64 *cnt,
                                                const u64 *bsum, const u32 *ex, DevResult *res) {
    __shared__ ZigFast sm[256];
    __shared__ __align__(16) unsigned char ring_sm[2 * EMIT_GB * BLOCK];  // RingWriter: 32 B, BatchRing: 2 groups per thread
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    const u64 my_cnt = t < p.T ? cnt[t] : 0;
    const u64 my_off = block_offset(bsum, my_cnt);
    Tally tl = {0, 0, 0, 0, 0};
    bool cp = false;
    if constexpr (D == FAM_GAMMA) {
        // Speculative store (GK_GAMMA): a segment whose samples are the count pass's (after
        // the fixup's re-parsed prefix) is copied, not parsed; the one holding sample n-1
        // still re-parses (it reports the end position). The copy is warp-cooperative:
        // the warp walks its lanes' runs with coalesced 256-byte loads and stores.
        if (p.spec && p.kind != GK_T && !*p.spec_over) {
            const u32 lane = threadIdx.x & 31;
            u64 o = 0, c = 0, endp = 0;
            if (t < p.T) {
                o = my_off;
                c = my_cnt;
                cp = o < p.n && c > 0 && p.cmode[t];
                if (cp && o + c >= p.n) {  // holds sample n-1: the position after it
                    if (o + c == p.n) {
                        endp = seg_end(p, t) + ex[t];
                    } else {  // = the start of the next speculative sample, from the boundary bitmaps
                        const u64 kk = p.n - o - 1, pn = p.pre_n[t];
                        long long q = -1;
                        if (kk >= pn) {
                            const u64 i = p.spec_from[t] + (kk - pn);  // speculative index of sample n-1
                            const u32 *bm1 = p.bm + (size_t)p.bmw * p.T;
                            if (p.cmode[t] == 1) {
                                q = bm_select(p.bm, p.T, t, p.bmw, i + 1);
                            } else {
                                const u64 own = p.c1own[t];
                                if (i + 1 < own) q = bm_select(bm1, p.T, t, p.bmw, i + 1);
                                else if (i + 1 == own) q = bm_select(p.bm, p.T, t, p.bmw, p.mrank0[t]);
                                else q = bm_select(p.bm, p.T, t, p.bmw, p.mrank0[t] + (i - own) + 1);
                            }
                        }
                        if (q < 0) cp = false;
                        else endp = seg_start(p, t) + (u64)q;
                    }
                }
            }
            unsigned m = __ballot_sync(0xFFFFFFFFu, cp);
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const u32 tj = t - lane + j;
                const u64 oj = __shfl_sync(0xFFFFFFFFu, o, j), c0j = __shfl_sync(0xFFFFFFFFu, c, j);
                const u64 endj = __shfl_sync(0xFFFFFFFFu, endp, j);
                const u64 cj = c0j < p.n - oj ? c0j : p.n - oj;
                const u64 pn = p.pre_n[tj] < cj ? p.pre_n[tj] : cj;
                const u64 sf = p.spec_from[tj];
                const size_t row = (size_t)tj * p.spec_cap;
                double *dst = (double *)p.out + p.out0 + oj;
                // up to three contiguous pieces: the re-parsed prefix, the speculative run it met
                // (phase 0, or phase 1 up to its merge), then phase 0 from the merge point
                u64 ka = cj;  // end of the second piece
                const double *va = p.spec + row + sf;
                const u32 *wa = p.spec_tal + row + sf;
                const double *vb = nullptr;
                const u32 *wb = nullptr;
                if (p.cmode[tj] == 2) {
                    va = p.spec1 + row + sf;
                    wa = p.spec1_tal + row + sf;
                    const u64 kown = pn + p.c1own[tj] - sf;
                    if (kown < cj) ka = kown;
                    vb = p.spec + row + p.mrank0[tj];
                    wb = p.spec_tal + row + p.mrank0[tj];
                }
                // 8 loads of each array in flight per lane before the stores (the copy is
                // latency-bound: ncu showed 4.4 TB/s at 11 % issue with the plain loop)
                auto piece = [&](const double *v, const u32 *w, u64 k0, u64 k1) {
                    u64 k = k0 + lane;
                    for (; k + 7 * 32 < k1; k += 8 * 32) {
                        double vv[8];
                        u32 ww[8];
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            vv[i] = __ldg(v + (k - k0) + 32 * i);
                            ww[i] = __ldg(w + (k - k0) + 32 * i);
                        }
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            dst[k + 32 * i] = vv[i];
                            tl.gamma_att += ww[i] & 0xFF;
                            tl.norm_att += (ww[i] >> 8) & 0xFFF;
                            tl.norm_pdf += ww[i] >> 20;
                        }
                    }
                    for (; k < k1; k += 32) {
                        const u32 x = __ldg(w + (k - k0));
                        dst[k] = __ldg(v + (k - k0));
                        tl.gamma_att += x & 0xFF;
                        tl.norm_att += (x >> 8) & 0xFFF;
                        tl.norm_pdf += x >> 20;
                    }
                };
                piece(p.pre + row, p.pre_tal + row, 0, pn);
                piece(va, wa, pn, ka);
                if (vb) piece(vb, wb, ka, cj);
                if (lane == 0 && oj + cj == p.n) res->end_pos = endj;
            }
        }
    }
    if (t < p.T) {
        u64 o = my_off, c = my_cnt;
        if (t == p.T - 1) {
            res->total = o + c;
            res->next_start = seg_end(p, t) + ex[t];
        }
        if (o < p.n && c > 0 && !cp) {
            u64 kmax = c < p.n - o ? c : p.n - o;
            typename SrcOf<E, D>::type s;
            make_src<E>(p, t, seg_start(p, t) + entry[t], s);
            typename DistOf<D>::type d;
            make_dist<D>(p, sm, d);
            typedef typename DistOf<D>::type::out_t T;
            T *ring = (T *)ring_sm + threadIdx.x;
            if constexpr (D == FAM_LEMIRE || D == FAM_U32) {  // one unit per step, <= 1 sample
                BatchRing<T, BLOCK, EMIT_GB> wr;
                wr.init((T *)p.out, p.out0 + o, ring);
                u32 it = 0;
                for (u64 k = 0; k < kmax;) {
                    T v;
                    bool ok;
                    if constexpr (D == FAM_LEMIRE) ok = d.accept(s.next(), v);
                    else ok = d.accept(s.next32(), v);
                    if (ok) { wr.put(v); k++; }
                    if ((++it & (BatchRing<T, BLOCK, EMIT_GB>::G - 1)) == 0) wr.tick();
                }
                wr.finish();
            } else {
                bool done = false;
                if constexpr (D == FAM_NORM || D == FAM_EXP) {
                    if (d.word_level()) {
                        BatchRing<T, BLOCK, EMIT_GB> wr;
                        wr.init((T *)p.out, p.out0 + o, ring);
                        wl_emit(d, s, kmax, wr, tl);
                        wr.finish();
                        done = true;
                    }
                }
                if constexpr (D == FAM_GAMMA) {
                    if (d.am_applies()) {  // one attempt per step, <= 1 sample
                        BatchRing<T, BLOCK, EMIT_GB> wr;
                        wr.init((T *)p.out, p.out0 + o, ring);
                        GammaAM m{0, 0, 0.0};
                        u32 it = 0;
                        for (u64 k = 0; k < kmax;) {
                            double v;
                            if (d.am_step(m, s, tl, v)) { wr.put(v); k++; }
                            if ((++it & (BatchRing<T, BLOCK, EMIT_GB>::G - 1)) == 0) wr.tick();
                        }
                        wr.finish();
                        done = true;
                    }
                }
                if (!done) {  // sample-level: lanes out of step, flush when a group is full
                    RingWriter<T, BLOCK> wr;
                    wr.init((T *)p.out, p.out0 + o, ring);
                    for (u64 k = 0; k < kmax; k++) wr.put(d.sample(s, tl));
                    wr.finish();
                }
            }
            if (o + kmax == p.n) res->end_pos = s.pos;
        }
    }
    // tallies: warp reduce then one atomic per warp
    u64 tv[6] = {tl.norm_att, tl.norm_pdf, tl.exp_att, tl.exp_pdf, tl.gamma_att, 0};
#pragma unroll
    for (int i = 0; i < 5; i++) {
        u64 v = tv[i];
        for (int sh = 16; sh > 0; sh >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, sh);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)&res->tally[i], (unsigned long long)v);
    }
}

// ----------------------------------------------------------------------------- fixed-consumption fills
// word modes map one 64-bit word to one 8-byte output; half modes map each 32-bit
// half (low first) to one 4-byte output, packed as a pair into one 8-byte element.
enum { FX_RAW = 0, FX_U01 = 1, FX_POW2 = 2, FX_U01F = 3, FX_WMAP = 4, FX_HMAP = 5 };
enum { WK_UNIF = 0, WK_GUMBEL = 1, WK_I64 = 2 };                  // FX_WMAP kinds
enum { HK_UNIFF = 0, HK_MASK = 1, HK_POW2 = 2, HK_I32 = 3 };       // FX_HMAP kinds
constexpr bool is_half(int mode) { return mode == FX_U01F || mode == FX_HMAP; }

// PL = FillPlan or StreamArgs (both carry fp, ip, fm, kind)
template <class PL>
__device__ __forceinline__ u32 hmap(const PL &p, u32 h) {
    switch (p.kind) {
    case HK_UNIFF:  // _f32(a + u01f * (b - a)), continuous.py:143-147
        return __float_as_uint(__double2float_rn(p.fp[0] + (double)u01f_of(h, p.fm) * (p.fp[1] - p.fp[0])));
    case HK_MASK: return h & (u32)p.ip[3];                                   // b = 0: the masked half
    case HK_POW2: return (u32)((((u64)h & p.ip[3]) * p.ip[0]) >> p.ip[1]);  // b = 2^k: no rejection zone
    default: return (u32)p.ip[2] + h;                                        // int over the full span
    }
}

template <int MODE, class PL>
__device__ __forceinline__ u64 fx_map(const PL &p, u64 w) {
    if constexpr (MODE == FX_RAW) return w;
    else if constexpr (MODE == FX_POW2) return __umul64hi(w, p.ip[0]);
    else if constexpr (MODE == FX_U01) return bits(u01_of(w, p.fm));
    else if constexpr (MODE == FX_WMAP) {
        if (p.kind == WK_UNIF) return bits(p.fp[0] + u01_of(w, p.fm) * (p.fp[1] - p.fp[0]));  // :136-140
        if (p.kind == WK_GUMBEL)  // mu - beta * det_log(-det_log(u)), continuous.py:246-249
            return bits(p.fp[0] - p.fp[1] * det_log_dev(-det_log_dev(u01_of(w, p.fm))));
        return p.ip[2] + w;       // long_long over the full span
    } else if constexpr (MODE == FX_U01F) {
        u32 lo = __float_as_uint(u01f_of((u32)w, p.fm)), hi = __float_as_uint(u01f_of((u32)(w >> 32), p.fm));
        return (u64)lo | ((u64)hi << 32);
    } else {
        return (u64)hmap(p, (u32)w) | ((u64)hmap(p, (u32)(w >> 32)) << 32);
    }
}

// u64/f64 outputs: logical word i -> out[i]. u01f: logical word i -> f32 out[pp + 2i], out[pp + 2i + 1]
// (written as one 8-byte element when that address is 8-byte aligned, else as two scalars).
// out[i] = map(word i) for i in [first, last). Each lane owns a contiguous run,
// so direct stores from a warp would touch 32 different lines. Instead lanes
// write 32-word chunks (256 bytes, two lines) into a padded per-warp shared tile
// (fx_at), and each STG.128 instruction of the warp
// then stores two lanes' chunks, 256 contiguous bytes per half-warp. Measured on
// B200 for 8 GiB of per-lane runs: 5.8 TB/s with 256-byte runs per instruction vs
// 4.6 TB/s with 128-byte ones (exp/wpeak2.cu). The ragged head (up to line
// alignment, and the buffered prefix) and tail are scalar.
constexpr int FX_CH = 32;
constexpr int LR_ROW = 65;  // per-stream Lemire rows: a 64-sample ring per lane (two chunks), padded
// Row stride 33 words: the lanes' row-wise STS.64 are conflict-free and the store
// phase's LDS.64 pairs 2-way conflicted. An XOR-swizzled unpadded layout (conflict-free
// LDS.128) measured slower -- 1.80 vs 1.51 ms for x256** 2^30 -- because its per-word
// address arithmetic lands on the ALU pipe, which the xoshiro step already fills (74 %).
constexpr int FX_ROW = FX_CH + 1;
constexpr size_t FX_SMEM = (size_t)(BLOCK / 32) * 32 * FX_ROW * 8;  // dynamic shared memory of k_fixed
__device__ __forceinline__ u32 fx_at(u32 l, u32 j) { return l * FX_ROW + j; }
template <int E, int MODE>
__device__ __forceinline__ void write_run(const FillPlan &p, Src<E> &s, u64 *out, u64 first, u64 last,
                                          u64 *tile, bool active) {
    const u32 lane = threadIdx.x & 31;
    u64 i = first;
    if (active)
        while (i < last && ((((uintptr_t)(out + i)) & 127) != 0 || s.npre > 0)) out[i++] = fx_map<MODE>(p, s.next());
    u64 nchunk = active && last > i ? (last - i) / FX_CH : 0;
    u64 maxc = nchunk;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        u64 v = __shfl_xor_sync(0xFFFFFFFFu, maxc, o);
        maxc = v > maxc ? v : maxc;
    }
    for (u64 k = 0; k < maxc; k++) {
        bool has = k < nchunk;
        if (has) {
            if constexpr (E == RS_ENG_RANLUX) {  // keep the 9x9-limb mulmod out of an unrolled body (I-cache)
#pragma unroll 1
                for (int j = 0; j < FX_CH; j++) tile[fx_at(lane, j)] = fx_map<MODE>(p, s.e.next());
            } else {
#pragma unroll
                for (int j = 0; j < FX_CH; j++) tile[fx_at(lane, j)] = fx_map<MODE>(p, s.e.next());
            }
        }
        u64 dst = has ? (u64)(uintptr_t)(out + i) : 0;
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 16; g++) {  // 2 rows (chunks) per instruction, 16 lanes x 16 B per row
            u32 r = 2 * g + (lane >> 4), c = lane & 15;
            u64 d = __shfl_sync(0xFFFFFFFFu, dst, r);
            if (d) {
                u64 x = tile[fx_at(r, 2 * c)], y = tile[fx_at(r, 2 * c + 1)];
                asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(d + 16 * c), "l"(x), "l"(y) : "memory");
            }
        }
        __syncwarp();
        if (has) i += FX_CH;
    }
    if (active)
        for (; i < last; i++) out[i] = fx_map<MODE>(p, s.e.next());
}

template <int E, int MODE>
__global__ void __launch_bounds__(BLOCK) k_fixed(const __grid_constant__ FillPlan p) {
    extern __shared__ __align__(16) u64 fx_dyn[];  // FX_SMEM
    u64 *tile = fx_dyn + (threadIdx.x >> 5) * 32 * FX_ROW;
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    // every lane of a warp takes part in the tile stores; idle lanes just contribute nothing
    bool active = t < p.T && ((u64)t * p.L < p.weng || t == 0);
    u64 j0 = (u64)t * p.L;
    u64 j1 = j0 + p.L < p.weng ? j0 + p.L : p.weng;
    if (j1 < j0) j1 = j0;
    u64 first = t == 0 ? 0 : (u64)p.P + j0;       // first logical word
    u64 last = (u64)p.P + j1;                     // one past
    Src<E> s;
    if (t < p.T) make_engine<E>(p, t, s.e);
    s.pre = p.prefix;
    s.npre = t == 0 ? p.P : 0;
    if constexpr (!is_half(MODE)) {
        u64 *out = (u64 *)p.out;
        if (t == 0 && last > p.n) last = p.n;  // n < P: prefix only
        write_run<E, MODE>(p, s, out, first, last, tile, active);
    } else {
        u32 *out = (u32 *)p.out;
        u64 halves = p.n - p.pending_used;  // halves to emit
        if (t == 0 && p.pending_used) out[0] = (u32)fx_map<MODE>(p, p.pending_val);
        u64 full_words = halves / 2;        // words whose both halves are emitted
        u64 lim = last < full_words ? last : full_words;
        u32 *o2 = out + p.pending_used;
        if ((((uintptr_t)o2) & 7) == 0) {  // warp-uniform: the whole grid shares o2
            write_run<E, MODE>(p, s, (u64 *)o2, first, lim > first ? lim : first, tile, active);
        } else if (active) {
            for (u64 i = first; i < lim; i++) {
                u64 q = fx_map<MODE>(p, s.next());
                o2[2 * i] = (u32)q;
                o2[2 * i + 1] = (u32)(q >> 32);
            }
        }
        if (active && (halves & 1) && full_words >= first && full_words < last) {  // trailing low half
            u64 w = 0;
            for (u64 i = lim; i <= full_words; i++) w = s.next();
            o2[2 * full_words] = (u32)fx_map<MODE>(p, w);
        }
    }
}

// Counter-based fixed fills (Philox-4x64-10, counter.py:98-121): word w of the
// stream is block(ctr0 + w/4)[w % 4], so threads take lane-consecutive blocks in
// a grid-stride loop and each warp store is one contiguous 1 KB (STG.256 per lane).
#ifndef RS_PHILOX_ILP
#define RS_PHILOX_ILP 1  // blocks per thread and iteration: 1 (32 registers) beat 2/3/4 on B200, DESIGN 4.1
#endif
template <int MODE, int V, bool FOLD>
__device__ __forceinline__ void philox_fixed_loop(const FillPlan &p, const PhiloxFold &f, u64 b, u64 nblk,
                                                  u64 stride);
template <int MODE, int V = 0>
__global__ void __launch_bounds__(BLOCK) k_philox_fixed(const __grid_constant__ FillPlan p) {
    const u64 nblk = (p.weng + 3) / 4;
    const u64 stride = (u64)gridDim.x * BLOCK;
    u64 b = (u64)blockIdx.x * BLOCK + threadIdx.x;
    if (b == 0) {  // the buffered prefix and a pending half (thread 0)
        if constexpr (is_half(MODE)) {
            u32 *out = (u32 *)p.out;
            if (p.pending_used) out[0] = (u32)fx_map<MODE>(p, p.pending_val);
            for (int i = 0; i < p.P; i++) {
                u64 f = (u64)p.pending_used + 2ULL * i;
                u64 q = fx_map<MODE>(p, p.prefix[i]);
                if (f < p.n) out[f] = (u32)q;
                if (f + 1 < p.n) out[f + 1] = (u32)(q >> 32);
            }
        } else {
            u64 *out = (u64 *)p.out;
            for (int i = 0; i < p.P && (u64)i < p.n; i++) out[i] = fx_map<MODE>(p, p.prefix[i]);
        }
    }
    // No carry out of counter word 0 over the launch's blocks (launch-uniform): words
    // 1-3 are constants and the first two rounds fold (philox4x64_10_folded). Blocks
    // at bb >= nblk are computed but never stored, so they need not satisfy it.
    if (nblk > 0 && p.base[0] + (nblk - 1) >= p.base[0]) {
        const PhiloxFold f = philox_fold(p.base[1], p.base[2], p.base[3], p.rk0, p.rk1);
        philox_fixed_loop<MODE, V, true>(p, f, b, nblk, stride);
    } else {
        philox_fixed_loop<MODE, V, false>(p, PhiloxFold{}, b, nblk, stride);
    }
}

template <int MODE, int V, bool FOLD>
__device__ __forceinline__ void philox_fixed_loop(const FillPlan &p, const PhiloxFold &f, u64 b, u64 nblk,
                                                  u64 stride) {
    // RS_PHILOX_ILP blocks per iteration (higher ILP measured slower: more registers, fewer warps)
    for (; b < nblk; b += RS_PHILOX_ILP * stride) {
        u64 w[RS_PHILOX_ILP][4];
#pragma unroll
        for (int h = 0; h < RS_PHILOX_ILP; h++) {
            u64 bb = b + h * stride;
            if constexpr (FOLD) {
                philox4x64_10_folded<V>(p.base[0] + bb, f, p.rk0, p.rk1, w[h][0], w[h][1], w[h][2], w[h][3]);
            } else {
                u64 c0 = p.base[0] + bb, c1 = p.base[1], c2 = p.base[2], c3 = p.base[3];
                if (c0 < bb) { if (++c1 == 0) { if (++c2 == 0) ++c3; } }
                philox4x64_10_rk<V>(c0, c1, c2, c3, p.rk0, p.rk1, w[h][0], w[h][1], w[h][2], w[h][3]);
            }
        }
#pragma unroll
        for (int h = 0; h < RS_PHILOX_ILP; h++) {
            u64 bb = b + h * stride;
            if (bb >= nblk) break;
            u64 q0 = fx_map<MODE>(p, w[h][0]), q1 = fx_map<MODE>(p, w[h][1]);
            u64 q2 = fx_map<MODE>(p, w[h][2]), q3 = fx_map<MODE>(p, w[h][3]);
            if constexpr (is_half(MODE)) {
                u64 f = (u64)p.pending_used + 2ULL * ((u64)p.P + 4 * bb);  // first 32-bit index of this block
                float *out = (float *)p.out;
                if (p.vec_ok && f + 8 <= p.n) {
                    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + f), "l"(q0), "l"(q1),
                                 "l"(q2), "l"(q3) : "memory");
                } else {
                    u64 q[4] = {q0, q1, q2, q3};
#pragma unroll
                    for (int i = 0; i < 8; i++)
                        if (f + i < p.n) out[f + i] = __uint_as_float((u32)(q[i >> 1] >> (32 * (i & 1))));
                }
            } else {
                u64 e = (u64)p.P + 4 * bb;
                u64 *out = (u64 *)p.out;
                if (p.vec_ok && e + 4 <= p.n) {
                    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + e), "l"(q0), "l"(q1),
                                 "l"(q2), "l"(q3) : "memory");
                } else {
                    if (e < p.n) out[e] = q0;
                    if (e + 1 < p.n) out[e + 1] = q1;
                    if (e + 2 < p.n) out[e + 2] = q2;
                    if (e + 3 < p.n) out[e + 3] = q3;
                }
            }
        }
    }
}

// Interleaved xoshiro engines (interleave.py:94-166): word j of the stream is lane
// j mod 8 at step j / 8. Thread t = 8 g + k runs lane k over steps
// [g Ls, (g+1) Ls) from its own GF(2)-jumped state, so the 8 threads of a group emit
// 8 consecutive words per step (64 contiguous bytes per group and step).
template <int E, int MODE>
__global__ void __launch_bounds__(BLOCK) k_simd_fixed(const __grid_constant__ FillPlan p) {
    const u64 t = (u64)blockIdx.x * BLOCK + threadIdx.x;
    const u64 g = t >> 3, k = t & 7;
    if (t == 0) {  // the buffered prefix and a pending half
        if constexpr (is_half(MODE)) {
            u32 *out = (u32 *)p.out;
            if (p.pending_used) out[0] = (u32)fx_map<MODE>(p, p.pending_val);
            for (int i = 0; i < p.P; i++) {
                u64 f = (u64)p.pending_used + 2ULL * i;
                u64 q = fx_map<MODE>(p, p.prefix[i]);
                if (f < p.n) out[f] = (u32)q;
                if (f + 1 < p.n) out[f + 1] = (u32)(q >> 32);
            }
        } else {
            u64 *out = (u64 *)p.out;
            for (int i = 0; i < p.P && (u64)i < p.n; i++) out[i] = fx_map<MODE>(p, p.prefix[i]);
        }
    }
    if (g >= p.G) return;
    EngX256<E == RS_ENG_X256SS_SIMD> e;
    e.load(p.x256_states + 4 * (k * p.Gpad + g));
    const u64 steps = (p.weng + 7) / 8;
    u64 s0 = g * p.L, s1 = s0 + p.L < steps ? s0 + p.L : steps;
    // A group's 8 threads emit 64 contiguous bytes per step and consecutive steps are adjacent,
    // so 4 steps staged in shared memory leave as one 256-byte run per group: each thread
    // stores 32 bytes of it (a store-only probe: 64-byte runs 4.5 TB/s, 256-byte runs 5.8,
    // DESIGN 4.3). Needs 32-byte aligned runs (p.vec_ok) and whole steps; the rest goes word by word.
    if (p.vec_ok) {
        __shared__ __align__(16) u64 stg[BLOCK / 8][34];
        u64 *row = stg[threadIdx.x >> 3];
        u64 *out = (u64 *)p.out;
        const unsigned gmask = 0xFFu << (threadIdx.x & 24);  // my group's 8 lanes (groups differ in trip count)
        const u64 whole = p.weng / 8;  // steps whose 8 words all exist
        const u64 sv = s1 < whole ? s1 : whole;
        for (; s0 + 4 <= sv; s0 += 4) {
#pragma unroll
            for (int i = 0; i < 4; i++) row[8 * i + k] = fx_map<MODE>(p, e.next());
            __syncwarp(gmask);
            const ulonglong2 a = *(const ulonglong2 *)&row[4 * k], b = *(const ulonglong2 *)&row[4 * k + 2];
            u64 *dst;
            if constexpr (is_half(MODE)) dst = (u64 *)((u32 *)out + p.pending_used) + (u64)p.P + 8 * s0 + 4 * k;
            else dst = out + (u64)p.P + 8 * s0 + 4 * k;
            asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(a.x), "l"(a.y), "l"(b.x), "l"(b.y)
                         : "memory");
            __syncwarp(gmask);
        }
    }
    for (u64 st = s0; st < s1; st++) {
        u64 q = fx_map<MODE>(p, e.next());
        u64 j = 8 * st + k;
        if (j >= p.weng) break;
        if constexpr (is_half(MODE)) {
            u32 *out = (u32 *)p.out;
            u64 f = (u64)p.pending_used + 2ULL * ((u64)p.P + j);
            if (f < p.n) out[f] = (u32)q;
            if (f + 1 < p.n) out[f + 1] = (u32)(q >> 32);
        } else {
            ((u64 *)p.out)[(u64)p.P + j] = q;
        }
    }
}

// ----------------------------------------------------------------------------- serial (sfc64 single stream)
// sfc64 has no skip-ahead (rng.py:162-163): a single stream is parsed by one
// thread; per-stream mode (k_streams) is the parallel path for sfc64. The
// thread also rebuilds the reference's post-fill WordBuffer: it snapshots the
// engine at every 144-word refill boundary and replays the last refill.
template <class EN>
struct SerialSrc {
    EN e, snap;
    const u64 *pre;
    int npre;
    u64 eng, pos;
    __device__ __forceinline__ u64 next() {
        pos++;
        if (npre > 0) { npre--; return *pre++; }
        if (eng % CAP == 0) snap = e;
        eng++;
        return e.next();
    }
};

template <class EN>
struct SerialHSrc {
    SerialSrc<EN> *w;
    u64 pos;
    u32 hi, pv;
    bool have, pend;
    __device__ __forceinline__ u32 next32() {
        pos++;
        if (pend) { pend = false; return pv; }
        if (have) { have = false; return hi; }
        u64 x = w->next();
        hi = (u32)(x >> 32);
        have = true;
        return (u32)x;
    }
};

template <class PL>
__device__ u64 fx_map_rt(const PL &p, u64 w) {
    switch (p.fmode) {
    case FX_RAW: return fx_map<FX_RAW>(p, w);
    case FX_POW2: return fx_map<FX_POW2>(p, w);
    case FX_U01: return fx_map<FX_U01>(p, w);
    case FX_WMAP: return fx_map<FX_WMAP>(p, w);
    case FX_U01F: return fx_map<FX_U01F>(p, w);
    default: return fx_map<FX_HMAP>(p, w);
    }
}

// D < 0: fixed-consumption map p.fmode; otherwise a sampler family. end_pos is in the
// family's stream units (halves for u32-fed samplers and half modes).
template <int D, int E>
__global__ void k_serial(const __grid_constant__ FillPlan p, DevResult *res) {
    __shared__ ZigFast sm[256];
    stage_tables(p, sm);
    if (threadIdx.x != 0) return;
    typedef typename EngOf<E>::type EN;
    SerialSrc<EN> s;
    make_engine<E>(p, 0, s.e);
    s.snap = s.e;
    s.pre = p.prefix;
    s.npre = p.P;
    s.eng = 0;
    s.pos = 0;
    Tally tl = {0, 0, 0, 0, 0};
    if constexpr (D < 0) {
        if (is_half(p.fmode)) {
            u32 *out = (u32 *)p.out;
            u64 i = 0;
            if (p.pending_used) out[i++] = (u32)fx_map_rt(p, p.pending_val);
            while (i < p.n) {
                u64 q = fx_map_rt(p, s.next());
                out[i++] = (u32)q;
                if (i < p.n) out[i++] = (u32)(q >> 32);
            }
            res->end_pos = p.n;
        } else {
            u64 *out = (u64 *)p.out;
            for (u64 i = 0; i < p.n; i++) out[i] = fx_map_rt(p, s.next());
            res->end_pos = s.pos;
        }
    } else {
        typename DistOf<D>::type d;
        make_dist<D>(p, sm, d);
        typedef typename DistOf<D>::type::out_t T;
        T *out = (T *)p.out;
        if constexpr (DistOf<D>::type::HALF) {
            SerialHSrc<EN> h{&s, 0, 0, p.pending_val, false, p.pending_used != 0};
            for (u64 i = 0; i < p.n; i++) out[i] = d.sample(h, tl);
            res->end_pos = h.pos;
        } else {
            for (u64 i = 0; i < p.n; i++) out[i] = d.sample(s, tl);
            res->end_pos = s.pos;
        }
    }
    res->tally[0] = tl.norm_att; res->tally[1] = tl.norm_pdf; res->tally[2] = tl.exp_att;
    res->tally[3] = tl.exp_pdf; res->tally[4] = tl.gamma_att; res->tally[5] = 0;
    res->serial_consumed = s.eng;
    EN f = s.snap;
    if (s.eng > 0)
        for (int i = 0; i < CAP; i++) res->serial_buf[i] = f.next();
    if constexpr (E == RS_ENG_SFC64_SIMD) {
        for (int k = 0; k < 8; k++) {
            res->serial_state[4 * k] = f.l[k].a; res->serial_state[4 * k + 1] = f.l[k].b;
            res->serial_state[4 * k + 2] = f.l[k].c; res->serial_state[4 * k + 3] = f.l[k].w;
        }
    } else if constexpr (E == RS_ENG_CWG128) {
        res->serial_state[0] = (u64)f.x; res->serial_state[1] = (u64)(f.x >> 64);
        res->serial_state[2] = (u64)f.weyl; res->serial_state[3] = (u64)(f.weyl >> 64);
        res->serial_state[4] = (u64)f.extra; res->serial_state[5] = (u64)(f.extra >> 64);
        res->serial_state[6] = (u64)f.inc; res->serial_state[7] = (u64)(f.inc >> 64);
    } else {
        res->serial_state[0] = f.a; res->serial_state[1] = f.b;
        res->serial_state[2] = f.c; res->serial_state[3] = f.w;
    }
}

// ----------------------------------------------------------------------------- per-stream mode
// SeedSequenceFE128 on the device (seeding.py:48-116): stream j's state from
// entropy (ip words in `seedw`) + spawn key prefix + (j0 + j).
struct StreamArgs {
    int engine, nseed, nprefix, dist, fm, fmode;
    u64 seed[16];
    u64 prefix[8];
    u64 j0, nstreams, nper;
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int kind;
    const RsZigSlow *zslow;
    const ZigFast *zfast;
    const RsZigSlowF *zslowf;
    const ZigFastF *zfastf;
    const u64 *rlx_A;
    void *out;
};

template <class EN>
struct EngHalves {  // 32-bit halves of a bare engine (a fresh stream has no buffer / pending)
    EN *e;
    u32 hi;
    bool have;
    __device__ __forceinline__ u32 next32() {
        if (have) { have = false; return hi; }
        u64 x = e->next();
        hi = (u32)(x >> 32);
        have = true;
        return (u32)x;
    }
};

__device__ void seed_fe128(const StreamArgs &a, u64 j, u64 *out, int nout) {
    u32 words[48];
    int na = 0;
    for (int i = 0; i < a.nseed; i++) { words[na++] = (u32)a.seed[i]; words[na++] = (u32)(a.seed[i] >> 32); }
    while (na < 4) words[na++] = 0;  // a spawn key is always present here
    for (int i = 0; i < a.nprefix; i++) { words[na++] = (u32)a.prefix[i]; words[na++] = (u32)(a.prefix[i] >> 32); }
    words[na++] = (u32)j;
    words[na++] = (u32)(j >> 32);
    u32 hc = 0x43B0D7E5u;
    u32 pool[4];
#define RS_HASH(v) ([&](u32 x) { x ^= hc; hc *= 0x931E8875u; x *= hc; x ^= x >> 16; return x; })(v)
#define RS_MIX(x, y) ([](u32 aa, u32 bb) { u32 r = aa * 0xCA01F9DDu - bb * 0x4973F715u; return r ^ (r >> 16); })(x, y)
    for (int i = 0; i < 4; i++) pool[i] = RS_HASH(words[i]);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = RS_MIX(pool[d], RS_HASH(pool[s]));
    for (int s = 4; s < na; s++)
        for (int d = 0; d < 4; d++) pool[d] = RS_MIX(pool[d], RS_HASH(words[s]));
#undef RS_HASH
#undef RS_MIX
    u32 hb = 0x8B51F9DDu;
    for (int i = 0; i < nout; i++) {
        u32 w2[2];
        for (int h = 0; h < 2; h++) {
            u32 v = pool[(2 * i + h) & 3] ^ hb;
            hb *= 0x58F38DEDu;
            v *= hb;
            v ^= v >> 16;
            w2[h] = v;
        }
        out[i] = (u64)w2[0] | ((u64)w2[1] << 32);
    }
}

// Per-stream rows of 8-byte outputs (row j = [j * nper, (j + 1) * nper), every row the
// same length): each lane fills 32 outputs of its row into its row of the warp tile,
// then the warp stores two lanes' 256-byte chunks per STG.128 instruction (the fixed
// fills' pattern, write_run). produce() returns the lane's next output as bits.
template <class F>
__device__ __forceinline__ void stream_rows8(u64 *out, u64 j, u64 nper, bool valid, u64 *tile, F produce) {
    const u32 lane = threadIdx.x & 31;
    const u64 nch = nper / FX_CH;
    const u64 row = (u64)(uintptr_t)(out + j * nper);
    for (u64 k = 0; k < nch; k++) {
        if (valid) {
            // a per-lane pointer bound, not a uniform counter (see k_streams' row loop)
            u64 *q = tile + fx_at(lane, 0), *const qe = q + FX_CH;
#pragma unroll 4
            while (q < qe) *q++ = produce();
        }
        __syncwarp();
        const u64 dst = valid ? row + k * FX_CH * 8 : 0;
#pragma unroll
        for (int g = 0; g < 16; g++) {
            u32 r = 2 * g + (lane >> 4), c = lane & 15;
            u64 d = __shfl_sync(0xFFFFFFFFu, dst, r);
            if (d) {
                u64 x = tile[fx_at(r, 2 * c)], y = tile[fx_at(r, 2 * c + 1)];
                asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(d + 16 * c), "l"(x), "l"(y) : "memory");
            }
        }
        __syncwarp();
    }
    if (valid)
        for (u64 i = nch * FX_CH; i < nper; i++) out[j * nper + i] = produce();
}

// Per-stream Lemire rows (rejections: a lane needs a variable number of words per
// sample): every lane consumes one word per step and appends accepted samples to a
// 64-slot ring (its tile row); every 32 steps the warp stores the rows that hold a full
// 32-sample chunk, two lanes' 256-byte chunks per STG.128 instruction (rows without one
// sit the store out). A lane adds <= 32 samples between stores, so the ring never holds
// more than 63. The per-sample redraw loop instead kept every lane waiting for the
// warp's slowest sample (m = 2^63 + 1 rejects half of the words).
// Lemire rows whose bound rejects (almost) never (threshold <= 2^44: a rejection rate of at
// most 2^-20; larger thresholds keep the redraw loops or the ring form below): a chunk takes one word per sample with no redraw
// loop -- straight-line code the compiler schedules across samples -- and a chunk that did
// see a rejected word (b = 6: 2^-62 per word) is redone from the saved engine with the
// exact loop.
template <class D, class EN>
__device__ __forceinline__ void stream_rows_lemire_spec(u64 *out, u64 j, u64 nper, bool valid, u64 *tile, const D &d,
                                                        EN &e) {
    const u32 lane = threadIdx.x & 31;
    const u64 nch = nper / FX_CH;
    const u64 row = (u64)(uintptr_t)(out + j * nper);
    for (u64 k = 0; k < nch; k++) {
        if (valid) {
            const EN e0 = e;
            u64 *q = tile + fx_at(lane, 0), *const qe = q + FX_CH;
            bool ok = true;
#pragma unroll 8
            while (q < qe) {
                u64 o;
                ok &= d.accept(e.next(), o);
                *q++ = o;
            }
            if (!ok) {
                e = e0;
                q = tile + fx_at(lane, 0);
                while (q < qe) {
                    u64 o;
                    while (!d.accept(e.next(), o)) {}
                    *q++ = o;
                }
            }
        }
        __syncwarp();
        const u64 dst = valid ? row + k * FX_CH * 8 : 0;
#pragma unroll
        for (int g = 0; g < 16; g++) {
            u32 r = 2 * g + (lane >> 4), c = lane & 15;
            u64 dd = __shfl_sync(0xFFFFFFFFu, dst, r);
            if (dd) {
                u64 x = tile[fx_at(r, 2 * c)], y = tile[fx_at(r, 2 * c + 1)];
                asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(dd + 16 * c), "l"(x), "l"(y) : "memory");
            }
        }
        __syncwarp();
    }
    if (valid)
        for (u64 i = nch * FX_CH; i < nper; i++) {
            u64 o;
            while (!d.accept(e.next(), o)) {}
            out[j * nper + i] = o;
        }
}

template <class D, class EN>
__device__ __forceinline__ void stream_rows_lemire(u64 *out, u64 j, u64 nper, bool valid, u64 *tile, const D &d,
                                                   EN &e) {
    const u32 lane = threadIdx.x & 31;
    u64 *ring = tile + lane * LR_ROW;
    u64 k = 0, stored = 0;  // samples produced / stored (stored: whole chunks)
    const u64 nch = nper / FX_CH;
    const u64 row = (u64)(uintptr_t)(out + j * nper);
    for (;;) {
        // 32 words per flush check, unrolled so the next words' engine steps overlap the
        // current word's 64x64 product and compare (one stream per thread: ILP is the only
        // latency hiding at 2^16 streams, ~3.5 warps per SMSP)
        if (valid && k + 32 <= nper) {
#pragma unroll 8
            for (int i = 0; i < 32; i++) {
                u64 o;
                const bool ok = d.accept(e.next(), o);
                ring[k & 63] = o;  // a rejected word's slot is overwritten by the next sample
                k += ok;
            }
        } else {
            for (int i = 0; i < 32; i++) {
                if (valid && k < nper) {
                    u64 o;
                    if (d.accept(e.next(), o)) {
                        ring[k & 63] = o;
                        k++;
                    }
                }
            }
        }
        {
            const bool ready = valid && k - stored >= FX_CH && stored < nch * FX_CH;
            const u64 dst = ready ? row + stored * 8 : 0;
            const u32 base = (u32)(stored & 63);
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 16; g++) {
                u32 r = 2 * g + (lane >> 4), c = lane & 15;
                u64 dd = __shfl_sync(0xFFFFFFFFu, dst, r);
                u32 bb = __shfl_sync(0xFFFFFFFFu, base, r);
                if (dd) {
                    u64 x = tile[r * LR_ROW + bb + 2 * c], y = tile[r * LR_ROW + bb + 2 * c + 1];
                    asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(dd + 16 * c), "l"(x), "l"(y) : "memory");
                }
            }
            __syncwarp();
            if (ready) stored += FX_CH;
            const bool more = valid && (k < nper || stored < nch * FX_CH);
            if (!__any_sync(0xFFFFFFFFu, more)) break;
        }
    }
    if (valid)
        for (u64 i = stored; i < nper; i++) out[j * nper + i] = ring[i & 63];  // the tail (< 32)
}

// 64-thread blocks: one thread per stream cannot be split (sfc64 has no skip-ahead), so
// small blocks spread the few warps evenly over the SMs (2^16 streams: 13.8 warps/SM)
constexpr int STR_BLOCK = 64;
constexpr size_t ST_SMEM = (size_t)(STR_BLOCK / 32) * 32 * FX_ROW * 8;   // dynamic shared memory of k_streams
constexpr size_t ST_SMEM_RING = (size_t)(STR_BLOCK / 32) * 32 * LR_ROW * 8;  // ... with a.ring
template <int E, int D>
__global__ void __launch_bounds__(STR_BLOCK) k_streams(const __grid_constant__ StreamArgs a) {
    __shared__ ZigFast sm[256];
    if (a.zfast) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = a.zfast[i];
    } else if (a.zfastf) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) ((ZigFastF *)sm)[i] = a.zfastf[i];
    }
    __syncthreads();
    u64 j = (u64)blockIdx.x * STR_BLOCK + threadIdx.x;
    // 8-byte rows through the warp tile (whole warps: no early exit) when every row
    // start is 16-byte aligned; otherwise the per-thread writers below
    extern __shared__ __align__(16) u64 st_dyn[];  // ST_SMEM
    constexpr bool W8 = sizeof(typename DistOf<(D == FAM_FIXED || D == FAM_LEMIRE_RING) ? FAM_LEMIRE : D>::type::out_t) == 8;
    const bool tiled = W8 && !(D == FAM_FIXED && is_half(a.fmode)) && a.nper % 2 == 0 &&
                       (((uintptr_t)a.out) & 15) == 0;
    if (!tiled && j >= a.nstreams) return;
    const bool valid = j < a.nstreams;
    u64 *tile = st_dyn + (threadIdx.x >> 5) * 32 * (D == FAM_LEMIRE_RING ? LR_ROW : FX_ROW);
    u64 w[9];
    typename EngOf<E>::type e;
    if (valid) {
    if constexpr (E == RS_ENG_SFC64) {
        seed_fe128(a, a.j0 + j, w, 3);
        e.a = w[0]; e.b = w[1]; e.c = w[2]; e.w = 1;  // sfc.py:53-55
    } else if constexpr (E == RS_ENG_PCG64) {
        seed_fe128(a, a.j0 + j, w, 4);
        e.slo = w[0]; e.shi = w[1]; e.ilo = w[2] | 1ULL; e.ihi = w[3];
    } else if constexpr (E == RS_ENG_PHILOX) {
        seed_fe128(a, a.j0 + j, w, 2);
        e.c0 = e.c1 = e.c2 = e.c3 = 0; e.k0 = w[0]; e.k1 = w[1]; e.left = 0;
    } else if constexpr (E == RS_ENG_X128P || E == RS_ENG_XORO) {  // xorfam.py:66-70
        seed_fe128(a, a.j0 + j, w, 2);
        if (!(w[0] | w[1])) w[0] = 1;
        e.load(w);
    } else if constexpr (E == RS_ENG_SQUARES) {  // counter.py:63-65
        seed_fe128(a, a.j0 + j, w, 1);
        e.ctr = 0;
        e.key = w[0];
    } else if constexpr (E == RS_ENG_CHACHA20) {  // counter.py:228-233
        seed_fe128(a, a.j0 + j, w, 6);
#pragma unroll
        for (int i = 0; i < 4; i++) { e.k[2 * i] = (u32)w[i]; e.k[2 * i + 1] = (u32)(w[i] >> 32); }
        e.n0 = (u32)w[4]; e.n1 = (u32)(w[4] >> 32); e.n2 = (u32)w[5];
        e.ctr = 0;
        e.left = 0;
    } else if constexpr (E == RS_ENG_CWG128) {  // cwg.py:62-67
        seed_fe128(a, a.j0 + j, w, 8);
        typedef unsigned __int128 U;
        e.x = ((U)w[1] << 64) | w[0];
        e.weyl = ((U)w[3] << 64) | w[2];
        e.extra = ((U)w[5] << 64) | w[4];
        e.inc = (((U)w[7] << 64) | w[6]) | 1;
    } else {  // x256
        seed_fe128(a, a.j0 + j, w, 4);
        if (!(w[0] | w[1] | w[2] | w[3])) w[0] = 1;
        e.s0 = w[0]; e.s1 = w[1]; e.s2 = w[2]; e.s3 = w[3];
    }
    }  // valid
    // Rows that cannot take the warp tile go out through the shared-memory RingWriter (one
    // STG.256 per 32-byte group). Its round-1 fault here was a uniform-register hazard in
    // the writer's address arithmetic under divergence, not the ring (rs_device.cuh run
    // writers, DESIGN 7); the writers now carry per-thread group pointers.
    if constexpr (D == FAM_FIXED) {  // raw / uniform / masked laws: a fresh stream, no pending half
        if (tiled) {
            stream_rows8((u64 *)a.out, j, a.nper, valid, tile, [&]() { return fx_map_rt(a, e.next()); });
            return;
        }
        if (is_half(a.fmode)) {  // low half first, a trailing high half dropped
            RingWriter<u32, STR_BLOCK> wr;
            wr.init((u32 *)a.out, j * a.nper, (u32 *)st_dyn + threadIdx.x);
            for (u64 i = 0; i < a.nper; i += 2) {
                u64 q = fx_map_rt(a, e.next());
                wr.put((u32)q);
                if (i + 1 < a.nper) wr.put((u32)(q >> 32));
            }
            wr.finish();
        } else {
            RingWriter<u64, STR_BLOCK> wr;
            wr.init((u64 *)a.out, j * a.nper, st_dyn + threadIdx.x);
            for (u64 i = 0; i < a.nper; i++) wr.put(fx_map_rt(a, e.next()));
            wr.finish();
        }
        return;
    }
    typedef typename DistOf<(D == FAM_FIXED || D == FAM_LEMIRE_RING) ? FAM_LEMIRE : D>::type DT;
    DT d;
    DistArgs da{a.fp, a.ip, &a.ga, &a.gb, a.kind, a.fm, a.zslow, a.zslowf};
    make_dist_a<(D == FAM_FIXED || D == FAM_LEMIRE_RING) ? FAM_LEMIRE : D>(da, sm, d);
    typedef typename DT::out_t T;
    Tally tl = {0, 0, 0, 0, 0};
    if constexpr (sizeof(T) == 8) {
        if (tiled) {
            if constexpr (D == FAM_LEMIRE_RING) {
                stream_rows_lemire((u64 *)a.out, j, a.nper, valid, tile, d, e);
            } else if constexpr (D == FAM_LEMIRE) {
                if (d.thr <= (1ULL << 44)) {  // rejection rate <= 2^-20: speculative 32-sample chunks
                    stream_rows_lemire_spec((u64 *)a.out, j, a.nper, valid, tile, d, e);
                } else {  // up to 1/16 (above that the host picks the ring form): redraw loops
                    auto prod = [&]() {
                        u64 o;
                        while (!d.accept(e.next(), o)) {}
                        return o;
                    };
                    stream_rows8((u64 *)a.out, j, a.nper, valid, tile, prod);
                }
            } else {  // 8-byte samplers are word-fed
                auto prod = [&]() {
                    T v = d.sample(e, tl);
                    return *(u64 *)&v;
                };
                stream_rows8((u64 *)a.out, j, a.nper, valid, tile, prod);
            }
            return;
        }
    }
    RingWriter<T, STR_BLOCK> wr;
    wr.init((T *)a.out, j * a.nper, (T *)st_dyn + threadIdx.x);
    if constexpr (D == FAM_LEMIRE) {
        for (u64 i = 0; i < a.nper;) {
            u64 o;
            if (d.accept(e.next(), o)) { wr.put(o); i++; }
        }
    } else if constexpr (D == FAM_U32) {
        EngHalves<typename EngOf<E>::type> h{&e, 0, false};
        for (u64 i = 0; i < a.nper;) {
            u32 o;
            if (d.accept(h.next32(), o)) { wr.put(o); i++; }
        }
    } else {
        // The loop runs to this row's end pointer, not to a sample counter: every lane has the
        // same trip count nper, so ptxas kept such a counter in a uniform register, and it
        // merged the sampler's rejection retry into this loop's back edge -- the lanes that
        // produced a sample advanced the one warp-wide counter for the lanes that had
        // rejected (rows ended short; DESIGN 7). A per-lane bound cannot be uniform.
        T *const rend = (T *)a.out + (j + 1) * a.nper;
        if constexpr (DT::HALF) {
            EngHalves<typename EngOf<E>::type> h{&e, 0, false};
            while (wr.at() < rend) wr.put(d.sample(h, tl));
        } else {
            while (wr.at() < rend) wr.put(d.sample(e, tl));
        }
    }
    wr.finish();
}


}  // namespace

// kernel accessors (one definition each, in the k_*.cu unit named beside it)
namespace rsk {
struct VarKernels {
    const void *count, *fixup, *emit;
};
VarKernels var_kernels_x256ss(int fam);  // k_var_x256ss.cu
VarKernels var_kernels_x256pp(int fam);  // k_var_x256pp.cu
VarKernels var_kernels_pcg(int fam);     // k_var_pcg.cu
VarKernels var_kernels_mem(int fam);     // k_var_mem.cu
const void *tile_kernel(int engine, int fam);    // k_tile.cu: single-pass normal / exponential (pcg64, philox), else null
const void *fixed_kernel(int engine, int mode);  // k_fixed.cu
const void *philox_kernel(int mode);             // k_fixed.cu
const void *simd_kernel(int engine, int mode);   // k_fixed.cu
const void *streams_kernel(int engine, int fam); // k_streams_a.cu (dispatch), k_streams_b.cu
const void *streams_kernel_b(int engine, int fam);
const void *serial_kernel(int engine, int fam, int fixed_mode);  // k_misc.cu
const void *setup_kernel();     // k_misc.cu: k_x256_setup
struct MvnLaunch {  // k_mvn.cu: the FP64 tensor-core contraction X = mean + z L^T
    const void *fn;
    size_t smem;
    int threads, bm, bn;
};
MvnLaunch mvn_kernel(int vec16, int layout);
}  // namespace rsk
