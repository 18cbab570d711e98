// B200 bulk stream-fill: kernels + orchestration behind the C ABI (include/randstream_b200.h).
//
// One logical word stream (the WordBuffer remainder followed by the engine's
// words, buffer.py:29-49) is cut into T contiguous segments of L engine words;
// thread t owns segment t and starts from an exact skip-ahead of the engine:
//   x256**/++ : GF(2) matrices T^(L*2^j) (block start: warp-cooperative mat-vec,
//               in-block: log-depth doubling in shared memory)   [A6]
//   pcg64     : affine LCG powers (mul, add) for L*2^j            [A7]
//   philox    : counter + t*L/4                                  [A9]
//   ranlux++  : x * A^((L/9)*2^j)                                [A8]
// Fixed-consumption fills (raw, u01, u01f, power-of-two bounds) map word i to
// output i and are written in one pass with 256-bit stores. Variable-consumption
// fills (ziggurat normal/exponential, gamma, beta, Lemire) keep the reference's
// exact draw order with a two-pass parse:
//   count  : each thread parses its segment from its start, counting samples that
//            start inside it and recording its exit (first boundary >= end);
//   fixup  : thread t's true entry is thread t-1's exit; the few threads whose
//            entry is not 0 re-parse in lockstep with their entry-0 parse until the
//            two meet at a common boundary (parses of these grammars converge within
//            a few words) -> exact per-thread counts;
//   scan   : exclusive prefix sum of the counts (stream compaction offsets);
//   emit   : each thread re-parses from its true entry and writes its samples at
//            their global offsets.
// Non-convergence inside a segment is detected and iterated to a fixed point.
#include <cuda_runtime.h>
#include <cublas_v2.h>

#include <cub/device/device_scan.cuh>
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
// pass records where its parses put sample boundaries in the first BM_WORDS * 32
// units of the segment; the fixup then re-parses from the true entry alone and looks
// the meeting point up instead of re-running the speculative parses beside it.
constexpr u32 BM_WORDS = 32;
constexpr u64 BM_UNITS = 32 * BM_WORDS;
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
    u32 *bm;                      // gamma family: count-pass boundary bitmaps (see BM_WORDS)
    const RsZigSlow *zslow;
    const ZigFast *zfast;
    const u64 *rlx_A;
    void *out;
    u64 out0;                     // element index in `out` of this chunk's sample 0
};

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
__device__ u32 g_mem_overrun;
struct EngMem {  // reads its (per-lane sequential) words 32 bytes at a time, one group ahead
    const u64 *w;
    u64 idx, nw;   // idx: next word to return
    u64 g;         // word index of the prefetched group n0..n3
    u64 b0, b1, b2, b3, n0, n1, n2, n3;
    int have;      // words left in b (-1: nothing loaded yet)
    __device__ __forceinline__ void load(u64 at, u64 &x0, u64 &x1, u64 &x2, u64 &x3) {
        if (at >= nw) { g_mem_overrun = 1; x0 = x1 = x2 = x3 = 0; return; }
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
        }
        u64 r = b0;
        b0 = b1; b1 = b2; b2 = b3;
        have--;
        idx++;
        return r;
    }
};
template <> struct EngOf<RS_ENG_MEM> { typedef EngMem type; };

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
        e.idx = (u64)t * p.L;
        e.nw = p.nwords;
        e.have = -1;
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
       FAM_F32 = 11, FAM_U32 = 22, FAM_FIXED = 40 /* per-stream mode: a fixed map of each word */ };
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
__device__ __forceinline__ void warp_matvec(const u64 *M, const u64 v[4], u64 out[4]) {
    int lane = threadIdx.x & 31;
    u64 a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    u32 byte = (u32)((v[lane >> 3] >> (8 * (lane & 7))) & 0xFF);
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 ^= __shfl_xor_sync(0xFFFFFFFFu, a0, o);
        a1 ^= __shfl_xor_sync(0xFFFFFFFFu, a1, o);
        a2 ^= __shfl_xor_sync(0xFFFFFFFFu, a2, o);
        a3 ^= __shfl_xor_sync(0xFFFFFFFFu, a3, o);
    }
    out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3;
}

__global__ void __launch_bounds__(BLOCK) k_x256_setup(const __grid_constant__ FillPlan p, const u64 *ML,
                                                      u64 *states) {
    const u32 lane = threadIdx.x & 31;
    const u64 w = ((u64)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    // gridDim.y == 8: interleaved engine, one grid row per lane (base = that lane's state)
    const u64 *b0 = gridDim.y > 1 ? p.lanes + 4 * blockIdx.y : p.base;
    states += (u64)blockIdx.y * 4 * ((u64)gridDim.x * BLOCK);
    u64 v[4] = {b0[0], b0[1], b0[2], b0[3]};
    u64 ww = w;
    for (int k = 0; ww; k++, ww >>= 1)
        if (ww & 1) warp_matvec(ML + (u64)(1 + k) * 1024, v, v);
    u64 mine[4] = {v[0], v[1], v[2], v[3]};
    for (u32 j = 1; j < 32; j++) {
        warp_matvec(ML, v, v);
        if (lane == j) { mine[0] = v[0]; mine[1] = v[1]; mine[2] = v[2]; mine[3] = v[3]; }
    }
    ulonglong2 *d = (ulonglong2 *)(states + 4 * (32 * w + lane));
    d[0] = make_ulonglong2(mine[0], mine[1]);
    d[1] = make_ulonglong2(mine[2], mine[3]);
}

// resident blocks per SM the parse kernels are compiled for (register budget)
constexpr int minb(int E, int D) {
    return D == FAM_GAMMA ? 2 : (D == FAM_LEMIRE || D == FAM_U32) ? 4 : 3;
}

// ----------------------------------------------------------------------------- word-level drivers
// Samples that start before `end` (count) / the next `kmax` samples (emit) with one
// word per lane per step. The buffered prefix (thread 0 of the first chunk only) is
// consumed in a preamble so the steady-state loop reads the engine directly and
// tracks its position with 32-bit counters.
template <class D, class SRC>
__device__ __forceinline__ u64 wl_count(const D &d, SRC &s, u64 end, Tally &tl) {
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
    // 4 words per step: the engine chain and the 4 strip loads overlap; words generated
    // past the exit are dropped (only the position matters)
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
    ZigWM m;
    m.st = 0;
    u64 k = 0;
    while (s.npre > 0 && k < kmax) {
        double z;
        if (d.feed(m, s.next(), tl, z)) { wr.put(d.finish(z)); k++; }
    }
    u32 left = (u32)(kmax - k), used = 0;
    while (left) {
        double z;
        used++;
        if (d.feed(m, s.e.next(), tl, z)) { wr.put(d.finish(z)); left--; }
    }
    s.pos += used;
}

// ----------------------------------------------------------------------------- two-pass parse
// boundary bitmap writer: bit q of the segment's map = a sample starts at start + q
struct BmRec {
    u32 *bm;  // [BM_WORDS][T]
    u32 T, t;
    u64 start;
    u32 acc = 0, kw = 0;
    __device__ __forceinline__ void put(u64 pos) {
        u64 q = pos - start;
        if (!bm || q >= BM_UNITS) return;
        u32 k = (u32)(q >> 5);
        while (kw < k) { bm[(size_t)kw * T + t] = acc; acc = 0; kw++; }
        acc |= 1u << (q & 31);
    }
    __device__ __forceinline__ void close() {
        if (!bm) return;
        while (kw < BM_WORDS) { bm[(size_t)kw * T + t] = acc; acc = 0; kw++; }
    }
};
// samples of a recorded parse that start before unit q (q < BM_UNITS)
__device__ __forceinline__ u64 bm_rank(const u32 *bm, u32 T, u32 t, u64 q) {
    u32 k = (u32)(q >> 5);
    u64 r = 0;
    for (u32 j = 0; j < k; j++) r += __popc(bm[(size_t)j * T + t]);
    return r + __popc(bm[(size_t)k * T + t] & ((1u << (q & 31)) - 1u));
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
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    if (t >= p.T) return;
    const u64 end = seg_end(p, t);
    typename SrcOf<E, D>::type s;
    make_src<E>(p, t, seg_start(p, t), s);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl;
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
                c = wl_count(d, s, end, tl);
                done = true;
            }
        }
        if (!done) {
            if constexpr (D == FAM_GAMMA) {
                BmRec r{p.bm, p.T, t, seg_start(p, t)};
                r.put(r.start);  // phase 0 starts a sample at the segment start
                while (s.pos < end) {
                    d.sample(s, tl);
                    c++;
                    r.put(s.pos);
                }
                r.close();
            } else {
                while (s.pos < end) {
                    d.sample(s, tl);
                    c++;
                }
            }
        }
        if (d.paired()) {
            typename SrcOf<E, D>::type s1;
            make_src<E>(p, t, seg_start(p, t), s1);
            d.skip_second(s1, tl);
            u64 c1 = 0;
            BmRec r{p.bm ? p.bm + (size_t)BM_WORDS * p.T : nullptr, p.T, t, seg_start(p, t)};
            r.put(s1.pos);  // phase 1's first full sample starts after the lone second
            while (s1.pos < end) {
                d.sample(s1, tl);
                c1++;
                r.put(s1.pos);
            }
            r.close();
            cnt1[t] = c1;
            ex1[t] = (u32)(s1.pos - end);
        }
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
            Tally tl;
            const bool two = d.paired();
            const u32 *bm0 = p.bm, *bm1 = p.bm + (size_t)BM_WORDS * p.T;
            u64 nb = 0;
            u32 kw = ~0u, wa = 0, wc = 0;
            while (true) {
                if (sb.pos >= end) {
                    cnt = nb;
                    ex = (u32)(sb.pos - end);
                    return;
                }
                u64 q = sb.pos - start;
                if (q >= BM_UNITS) break;
                u32 k = (u32)(q >> 5), bit = 1u << (q & 31);
                if (k != kw) {
                    kw = k;
                    wa = bm0[(size_t)k * p.T + t];
                    if (two) wc = bm1[(size_t)k * p.T + t];
                }
                if (wa & bit) {
                    cnt = c0 - bm_rank(bm0, p.T, t, q) + nb;
                    ex = x0;
                    return;
                }
                if (two && (wc & bit)) {
                    cnt = c1 - bm_rank(bm1, p.T, t, q) + nb;
                    ex = x1;
                    return;
                }
                d.sample(sb, tl);
                nb++;
            }
        }  // no meeting in the recorded window: the lockstep parse below
    }
    typename SrcOf<E, D>::type sa, sb, sc;
    make_src<E>(p, t, start, sa);
    make_src<E>(p, t, start + e, sb);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl;
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

// round 0: prev_ex = ex0, every thread; round r>0: only threads whose entry changed.
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_fixup(const __grid_constant__ FillPlan p, const u64 *cnt0, const u32 *ex0,
                                                 const u64 *cnt1, const u32 *ex1, const u32 *prev_ex, u32 *entry,
                                                 u64 *cnt, u32 *ex, int round, DevResult *res) {
    __shared__ ZigFast sm[256];
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    if (t >= p.T) return;
    u32 e = t == 0 ? 0u : prev_ex[t - 1];
    if (round > 0 && e == entry[t]) {
        ex[t] = prev_ex[t];
        return;
    }
    entry[t] = e;
    u64 c;
    u32 x;
    if (e == 0) {
        c = cnt0[t];
        x = ex0[t];
    } else {
        resolve_entry<E, D>(p, sm, t, e, cnt0[t], ex0[t], cnt1[t], ex1[t], c, x);
    }
    cnt[t] = c;
    ex[t] = x;
    if (x != prev_ex[t]) atomicOr(&res->flag, 1u);
}

// emit: re-parse from the true entry and write this segment's samples at their
// global offsets (exclusive scan of the counts).
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_emit(const __grid_constant__ FillPlan p, const u32 *entry, const u64 *cnt,
                                                const u64 *off, const u32 *ex, DevResult *res) {
    __shared__ ZigFast sm[256];
    __shared__ __align__(16) unsigned char ring_sm[32 * BLOCK];
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    Tally tl = {0, 0, 0, 0, 0};
    if (t < p.T) {
        u64 o = off[t], c = cnt[t];
        if (t == p.T - 1) {
            res->total = o + c;
            res->next_start = seg_end(p, t) + ex[t];
        }
        if (o < p.n && c > 0) {
            u64 kmax = c < p.n - o ? c : p.n - o;
            typename SrcOf<E, D>::type s;
            make_src<E>(p, t, seg_start(p, t) + entry[t], s);
            typename DistOf<D>::type d;
            make_dist<D>(p, sm, d);
            typedef typename DistOf<D>::type::out_t T;
            RingWriter<T, BLOCK> wr;
            wr.init((T *)p.out, p.out0 + o, (T *)ring_sm + threadIdx.x);
            if constexpr (D == FAM_LEMIRE || D == FAM_U32) {
                for (u64 k = 0; k < kmax;) {
                    T v;
                    bool ok;
                    if constexpr (D == FAM_LEMIRE) ok = d.accept(s.next(), v);
                    else ok = d.accept(s.next32(), v);
                    if (ok) { wr.put(v); k++; }
                }
            } else {
                bool done = false;
                if constexpr (D == FAM_NORM || D == FAM_EXP) {
                    if (d.word_level()) {
                        wl_emit(d, s, kmax, wr, tl);
                        done = true;
                    }
                }
                if (!done)
                    for (u64 k = 0; k < kmax; k++) wr.put(d.sample(s, tl));
            }
            wr.finish();
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
// write 16-word chunks (one 128-byte line each) into a padded per-warp shared tile
// (row stride 17 words: conflict-free), and the warp then stores 4 whole lines per
// STG.128 instruction. The ragged head (up to line alignment, and the buffered
// prefix) and tail are scalar.
constexpr int FX_ROW = 17;
template <int E, int MODE>
__device__ __forceinline__ void write_run(const FillPlan &p, Src<E> &s, u64 *out, u64 first, u64 last,
                                          u64 (*tile)[FX_ROW], bool active) {
    const u32 lane = threadIdx.x & 31;
    u64 i = first;
    if (active)
        while (i < last && ((((uintptr_t)(out + i)) & 127) != 0 || s.npre > 0)) out[i++] = fx_map<MODE>(p, s.next());
    u64 nchunk = active && last > i ? (last - i) / 16 : 0;
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
                for (int j = 0; j < 16; j++) tile[lane][j] = fx_map<MODE>(p, s.e.next());
            } else {
#pragma unroll
                for (int j = 0; j < 16; j++) tile[lane][j] = fx_map<MODE>(p, s.e.next());
            }
        }
        u64 dst = has ? (u64)(uintptr_t)(out + i) : 0;
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 8; g++) {  // 4 rows (lines) per instruction, 8 lanes x 16 B per row
            u32 r = 4 * g + (lane >> 3), c = lane & 7;
            u64 d = __shfl_sync(0xFFFFFFFFu, dst, r);
            if (d) {
                u64 x = tile[r][2 * c], y = tile[r][2 * c + 1];
                asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(d + 16 * c), "l"(x), "l"(y) : "memory");
            }
        }
        __syncwarp();
        if (has) i += 16;
    }
    if (active)
        for (; i < last; i++) out[i] = fx_map<MODE>(p, s.e.next());
}

template <int E, int MODE>
__global__ void __launch_bounds__(BLOCK) k_fixed(const __grid_constant__ FillPlan p) {
    __shared__ u64 tiles[BLOCK / 32][32][FX_ROW];
    u64 (*tile)[FX_ROW] = tiles[threadIdx.x >> 5];
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
    // two independent blocks per iteration (ILP for the IMAD pipe)
    for (; b < nblk; b += 2 * stride) {
        u64 w[2][4];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            u64 bb = b + h * stride;
            u64 c0 = p.base[0] + bb, c1 = p.base[1], c2 = p.base[2], c3 = p.base[3];
            if (c0 < bb) { if (++c1 == 0) { if (++c2 == 0) ++c3; } }
            philox4x64_10_rk<V>(c0, c1, c2, c3, p.rk0, p.rk1, w[h][0], w[h][1], w[h][2], w[h][3]);
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
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

template <int E, int D>
__global__ void __launch_bounds__(BLOCK) k_streams(const __grid_constant__ StreamArgs a) {
    __shared__ ZigFast sm[256];
    if (a.zfast) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = a.zfast[i];
    } else if (a.zfastf) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) ((ZigFastF *)sm)[i] = a.zfastf[i];
    }
    __syncthreads();
    u64 j = (u64)blockIdx.x * BLOCK + threadIdx.x;
    if (j >= a.nstreams) return;
    u64 w[9];
    typename EngOf<E>::type e;
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
    // Per-stream rows go out through VecWriter8 (8-byte) / ScalarWriter (4-byte). The
    // shared-memory RingWriter used by k_emit produced an illegal address here in some
    // configurations (x256**/pcg64 normals, >= 8 streams) that vanished under printf
    // instrumentation; it stays out of this kernel until that is understood.
    if constexpr (D == FAM_FIXED) {  // raw / uniform / masked laws: a fresh stream, no pending half
        if (is_half(a.fmode)) {  // low half first, a trailing high half dropped
            ScalarWriter<u32> wr;
            wr.init((u32 *)a.out, j * a.nper);
            for (u64 i = 0; i < a.nper; i += 2) {
                u64 q = fx_map_rt(a, e.next());
                wr.put((u32)q);
                if (i + 1 < a.nper) wr.put((u32)(q >> 32));
            }
            wr.finish();
        } else {
            VecWriter8<u64> wr;
            wr.init((u64 *)a.out, j * a.nper);
            for (u64 i = 0; i < a.nper; i++) wr.put(fx_map_rt(a, e.next()));
            wr.finish();
        }
        return;
    }
    typedef typename DistOf<D == FAM_FIXED ? FAM_LEMIRE : D>::type DT;
    DT d;
    DistArgs da{a.fp, a.ip, &a.ga, &a.gb, a.kind, a.fm, a.zslow, a.zslowf};
    make_dist_a<D == FAM_FIXED ? FAM_LEMIRE : D>(da, sm, d);
    typedef typename DT::out_t T;
    typename std::conditional<sizeof(T) == 8, VecWriter8<T>, ScalarWriter<T>>::type wr;
    wr.init((T *)a.out, j * a.nper);
    Tally tl;
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
    } else if constexpr (DT::HALF) {
        EngHalves<typename EngOf<E>::type> h{&e, 0, false};
        for (u64 i = 0; i < a.nper; i++) wr.put(d.sample(h, tl));
    } else {
        for (u64 i = 0; i < a.nper; i++) wr.put(d.sample(e, tl));
    }
    wr.finish();
}

__global__ void k_mvn_init(double *c, const double *mean, int64_t d, u64 n, int layout) {
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    u64 tot = n * (u64)d;
    for (; i < tot; i += (u64)gridDim.x * blockDim.x) {
        // layout n_d: C is d x n col-major => element i belongs to row i % d
        // layout d_n: C is n x d col-major => element i belongs to column i / n
        c[i] = layout == 0 ? mean[i % d] : mean[i / n];
    }
}

// ----------------------------------------------------------------------------- host side
#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess) {                                                               \
            rs::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #x);  \
            return RS_ERR_CUDA;                                                                \
        }                                                                                      \
    } while (0)

struct DevCtx {
    bool ready = false;
    int sms = 0;
    RsZigSlow *zslow[2] = {nullptr, nullptr};
    ZigFast *zfast[2] = {nullptr, nullptr};
    RsZigSlowF *zslowf[2] = {nullptr, nullptr};
    ZigFastF *zfastf[2] = {nullptr, nullptr};
    u64 *rlxA = nullptr;
    // scratch
    size_t cap_T = 0;
    u64 *states = nullptr, *cnt0 = nullptr, *cnt1 = nullptr, *cnt = nullptr, *off = nullptr;
    u32 *ex0 = nullptr, *ex1 = nullptr, *exA = nullptr, *exB = nullptr, *entry = nullptr;
    u32 *bm = nullptr;  // [2][BM_WORDS][T] boundary bitmaps
    void *cub_tmp = nullptr;
    size_t cub_bytes = 0;
    DevResult *res = nullptr;
    DevResult *res_host = nullptr;
    std::map<std::tuple<int, u64, int>, u64 *> x256_ml;  // (family, L, levels) -> matrices
    void *stage = nullptr;
    size_t stage_bytes = 0;
    cublasHandle_t blas = nullptr;
    double *mvn_z = nullptr;
    size_t mvn_bytes = 0;
    u64 *words = nullptr;  // materialized engine words for parse-from-memory
    size_t words_bytes = 0;
};

std::mutex g_mu;
std::map<int, DevCtx> g_dev;

rs_status init_dev(int dev, DevCtx **out) {
    DevCtx &c = g_dev[dev];
    *out = &c;
    if (c.ready) return RS_OK;
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
    for (int k = 0; k < 2; k++) {
        RsZigSlow zs;
        RsZigFastHost zf[256];
        rs_build_zig(k, &zs, zf);
        CK(cudaMalloc(&c.zslow[k], sizeof(RsZigSlow)));
        CK(cudaMalloc(&c.zfast[k], sizeof(zf)));
        CK(cudaMemcpy(c.zslow[k], &zs, sizeof(RsZigSlow), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.zfast[k], zf, sizeof(zf), cudaMemcpyHostToDevice));
    }
    for (int k = 0; k < 2; k++) {  // f32 tables (zigtables.py:1563-3116)
        RsZigSlowF zs;
        ZigFastF zf[256];
        for (int i = 0; i < 256; i++) {
            uint32_t fb = k ? RS_FE_F_BITS[i] : RS_FI_F_BITS[i], wb = k ? RS_WE_F_BITS[i] : RS_WI_F_BITS[i];
            memcpy(&zs.f[i], &fb, 4);
            zf[i].k = k ? RS_KE_F[i] : RS_KI_F[i];
            memcpy(&zf[i].w, &wb, 4);
        }
        CK(cudaMalloc(&c.zslowf[k], sizeof(RsZigSlowF)));
        CK(cudaMalloc(&c.zfastf[k], sizeof(zf)));
        CK(cudaMemcpy(c.zslowf[k], &zs, sizeof(RsZigSlowF), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.zfastf[k], zf, sizeof(zf), cudaMemcpyHostToDevice));
    }
    u64 A[9];
    rs::rlx_pow2k_A(0, A);
    CK(cudaMalloc(&c.rlxA, sizeof(A)));
    CK(cudaMemcpy(c.rlxA, A, sizeof(A), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.res, sizeof(DevResult)));
    CK(cudaMallocHost(&c.res_host, sizeof(DevResult)));
    c.ready = true;
    return RS_OK;
}

rs_status ensure_scratch(DevCtx &c, size_t T) {
    if (T <= c.cap_T) return RS_OK;
    size_t nT = T + T / 4;
    cudaFree(c.states); cudaFree(c.cnt0); cudaFree(c.cnt1); cudaFree(c.cnt); cudaFree(c.off);
    cudaFree(c.ex0); cudaFree(c.ex1); cudaFree(c.exA); cudaFree(c.exB); cudaFree(c.entry); cudaFree(c.cub_tmp);
    cudaFree(c.bm);
    CK(cudaMalloc(&c.states, nT * 32));
    CK(cudaMalloc(&c.cnt0, nT * 8));
    CK(cudaMalloc(&c.cnt1, nT * 8));
    CK(cudaMalloc(&c.ex1, nT * 4));
    CK(cudaMalloc(&c.cnt, nT * 8));
    CK(cudaMalloc(&c.off, nT * 8));
    CK(cudaMalloc(&c.ex0, nT * 4));
    CK(cudaMalloc(&c.exA, nT * 4));
    CK(cudaMalloc(&c.exB, nT * 4));
    CK(cudaMalloc(&c.entry, nT * 4));
    CK(cudaMalloc(&c.bm, nT * 4 * 2 * BM_WORDS));
    c.cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c.cub_bytes, c.cnt, c.off, (int)nT);
    CK(cudaMalloc(&c.cub_tmp, c.cub_bytes));
    c.cap_T = nT;
    return RS_OK;
}

// x256: ML[0] = T^L, ML[1 + k] = T^(32 L 2^k) for k < levels; cached per (L, levels) on the device
rs_status x256_mats(DevCtx &c, int engine, u64 L, int levels, u64 **out) {
    // x256 family, or the 128-bit xorshift128+ / xoroshiro128 matrices padded to 256 bits
    const bool narrow = engine == RS_ENG_X128P || engine == RS_ENG_XORO;
    auto pow2 = [&](int k) -> const rs::Mat256 & { return narrow ? rs::x128_pow2(engine, k) : rs::x256_pow2(k); };
    auto key = std::make_tuple(narrow ? engine : 0, L, levels);
    auto it = c.x256_ml.find(key);
    if (it != c.x256_ml.end()) { *out = it->second; return RS_OK; }
    std::vector<rs::Mat256> m(1 + levels);
    bool init = false;
    for (int k = 0; k < 64; k++)
        if ((L >> k) & 1) {
            if (!init) { m[0] = pow2(k); init = true; }
            else rs::mat_mul(pow2(k), m[0], m[0]);
        }
    if (levels > 0) {
        rs::Mat256 *t = new rs::Mat256(m[0]);
        for (int i = 0; i < 5; i++) rs::mat_mul(*t, *t, *t);  // T^(32 L)
        m[1] = *t;
        delete t;
        for (int k = 1; k < levels; k++) rs::mat_mul(m[k], m[k], m[k + 1]);
    }
    u64 *d;
    CK(cudaMalloc(&d, (size_t)(1 + levels) * sizeof(rs::Mat256)));
    CK(cudaMemcpy(d, m.data(), (size_t)(1 + levels) * sizeof(rs::Mat256), cudaMemcpyHostToDevice));
    if (c.x256_ml.size() > 16) {  // bound the cache
        for (auto &kv : c.x256_ml) cudaFree(kv.second);
        c.x256_ml.clear();
    }
    c.x256_ml[key] = d;
    *out = d;
    return RS_OK;
}

int occupancy(const void *fn) {
    static std::map<const void *, int> cache;
    auto it = cache.find(fn);
    if (it != cache.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BLOCK, 0) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    cache[fn] = nb;
    return nb;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t elem_size(int dist) {
    switch (dist) {
    case RS_DIST_U01F: case RS_DIST_UNIFF: case RS_DIST_NORMF: case RS_DIST_EXPF: case RS_DIST_UINT32:
    case RS_DIST_INT32: return 4;
    default: return 8;
    }
}

// ---- dispatch tables
struct VarKernels {
    const void *count, *fixup, *emit;
};

template <int E, int D>
VarKernels var_kernels_ed() {
    return VarKernels{(const void *)k_count<E, D>, (const void *)k_fixup<E, D>, (const void *)k_emit<E, D>};
}
template <int E>
VarKernels var_kernels_e(int fam) {
    switch (fam) {
    case FAM_NORM: return var_kernels_ed<E, FAM_NORM>();
    case FAM_EXP: return var_kernels_ed<E, FAM_EXP>();
    case FAM_GAMMA: return var_kernels_ed<E, FAM_GAMMA>();
    case FAM_F32: return var_kernels_ed<E, FAM_F32>();
    case FAM_U32: return var_kernels_ed<E, FAM_U32>();
    default: return var_kernels_ed<E, FAM_LEMIRE>();
    }
}
// Engines whose parse passes read materialized words: the expensive ones (Philox,
// ranlux++, ChaCha20), the interleaved ones, and the registry's other skip-ahead
// engines (x128+, xoro++, squares), which thereby need no parse-kernel instantiations.
bool parse_from_memory(int e) {
    return e == RS_ENG_PHILOX || e == RS_ENG_RANLUX || e == RS_ENG_X256PP_SIMD || e == RS_ENG_X256SS_SIMD ||
           e == RS_ENG_CHACHA20 || e == RS_ENG_X128P || e == RS_ENG_XORO || e == RS_ENG_SQUARES;
}
// no skip-ahead: one device thread replays the stream (sfc64 rng.py:162-163; cwg128 likewise)
bool is_serial(int e) { return e == RS_ENG_SFC64 || e == RS_ENG_SFC64_SIMD || e == RS_ENG_CWG128; }
VarKernels var_kernels(int e, int fam) {
    switch (e) {
    case RS_ENG_X256SS: return var_kernels_e<RS_ENG_X256SS>(fam);
    case RS_ENG_X256PP: return var_kernels_e<RS_ENG_X256PP>(fam);
    case RS_ENG_PCG64: return var_kernels_e<RS_ENG_PCG64>(fam);
    default: return var_kernels_e<RS_ENG_MEM>(fam);  // philox, ranlux++: words materialized first
    }
}
template <int E>
const void *fixed_kernel_e(int mode) {
    switch (mode) {
    case FX_RAW: return (const void *)k_fixed<E, FX_RAW>;
    case FX_U01: return (const void *)k_fixed<E, FX_U01>;
    case FX_POW2: return (const void *)k_fixed<E, FX_POW2>;
    case FX_WMAP: return (const void *)k_fixed<E, FX_WMAP>;
    case FX_HMAP: return (const void *)k_fixed<E, FX_HMAP>;
    default: return (const void *)k_fixed<E, FX_U01F>;
    }
}
const void *fixed_kernel(int e, int mode) {
    switch (e) {
    case RS_ENG_X256SS: return fixed_kernel_e<RS_ENG_X256SS>(mode);
    case RS_ENG_X256PP: return fixed_kernel_e<RS_ENG_X256PP>(mode);
    case RS_ENG_PCG64: return fixed_kernel_e<RS_ENG_PCG64>(mode);
    case RS_ENG_PHILOX: return fixed_kernel_e<RS_ENG_PHILOX>(mode);
    case RS_ENG_X128P: return fixed_kernel_e<RS_ENG_X128P>(mode);
    case RS_ENG_XORO: return fixed_kernel_e<RS_ENG_XORO>(mode);
    case RS_ENG_SQUARES: return fixed_kernel_e<RS_ENG_SQUARES>(mode);
    case RS_ENG_CHACHA20: return fixed_kernel_e<RS_ENG_CHACHA20>(mode);
    default: return fixed_kernel_e<RS_ENG_RANLUX>(mode);
    }
}
template <int V>
const void *philox_kernel_v(int mode) {
    switch (mode) {
    case FX_RAW: return (const void *)k_philox_fixed<FX_RAW, V>;
    case FX_U01: return (const void *)k_philox_fixed<FX_U01, V>;
    case FX_POW2: return (const void *)k_philox_fixed<FX_POW2, V>;
    case FX_WMAP: return (const void *)k_philox_fixed<FX_WMAP, V>;
    case FX_HMAP: return (const void *)k_philox_fixed<FX_HMAP, V>;
    default: return (const void *)k_philox_fixed<FX_U01F, V>;
    }
}
const void *philox_kernel(int mode) {
    static int variant = getenv("RS_PHILOX_VARIANT") ? atoi(getenv("RS_PHILOX_VARIANT")) : 0;
    return variant == 1 ? philox_kernel_v<1>(mode) : philox_kernel_v<0>(mode);
}
template <int E>
const void *serial_kernel_e(int fam, int fixed_mode) {
    if (fixed_mode >= 0) return (const void *)k_serial<-1, E>;
    switch (fam) {
    case FAM_NORM: return (const void *)k_serial<FAM_NORM, E>;
    case FAM_EXP: return (const void *)k_serial<FAM_EXP, E>;
    case FAM_GAMMA: return (const void *)k_serial<FAM_GAMMA, E>;
    case FAM_F32: return (const void *)k_serial<FAM_F32, E>;
    case FAM_U32: return (const void *)k_serial<FAM_U32, E>;
    default: return (const void *)k_serial<FAM_LEMIRE, E>;
    }
}
const void *serial_kernel(int engine, int fam, int fixed_mode) {
    if (engine == RS_ENG_CWG128) return serial_kernel_e<RS_ENG_CWG128>(fam, fixed_mode);
    return engine == RS_ENG_SFC64_SIMD ? serial_kernel_e<RS_ENG_SFC64_SIMD>(fam, fixed_mode)
                                       : serial_kernel_e<RS_ENG_SFC64>(fam, fixed_mode);
}
template <int MODE>
const void *simd_kernel_m(int e) {
    return e == RS_ENG_X256SS_SIMD ? (const void *)k_simd_fixed<RS_ENG_X256SS_SIMD, MODE>
                                   : (const void *)k_simd_fixed<RS_ENG_X256PP_SIMD, MODE>;
}
const void *simd_kernel(int e, int mode) {
    switch (mode) {
    case FX_RAW: return simd_kernel_m<FX_RAW>(e);
    case FX_U01: return simd_kernel_m<FX_U01>(e);
    case FX_POW2: return simd_kernel_m<FX_POW2>(e);
    case FX_WMAP: return simd_kernel_m<FX_WMAP>(e);
    case FX_HMAP: return simd_kernel_m<FX_HMAP>(e);
    default: return simd_kernel_m<FX_U01F>(e);
    }
}

rs_status launch(const void *fn, dim3 g, dim3 b, void **args, cudaStream_t st) {
    CK(cudaLaunchKernel(fn, g, b, args, 0, st));
    return RS_OK;
}

// ---- parameter resolution (validated values)
struct Resolved {
    int dist;          // RS_DIST_* as requested
    int fixed_mode;    // FX_* or -1 for a variable-consumption family
    int family;        // FAM_*
    int kind;          // law within the family / fixed map
    int unit;          // 1 words, 2 halves
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int raw_norm;
    double words_per_sample;
    int table;         // 0 normal, 1 exponential, 2 normal f32, 3 exponential f32, -1 none
};

GammaPrm gamma_prm(double alpha, double theta) {
    // continuous.py:183-199; alpha < 1 runs gamma(alpha + 1, 1) then the boost
    GammaPrm g;
    g.alpha = alpha;
    g.theta = theta;
    g.boost = alpha < 1.0;
    double a = g.boost ? alpha + 1.0 : alpha;
    double th = g.boost ? 1.0 : theta;
    g.d = a - 1.0 / 3.0;
    g.cc = 1.0 / std::sqrt(9.0 * g.d);
    g.td = th * g.d;
    return g;
}
double gamma_words(const GammaPrm &g) { return 2.2 + (g.boost ? 1.0 : 0.0); }

#define RS_FAIL(msg)                \
    do {                            \
        rs::set_error(msg);         \
        return RS_ERR_VALUE;        \
    } while (0)

// fp / ip layouts per distribution: include/randstream_b200.h
rs_status resolve(int dist, const double *fp, const u64 *ip, Resolved &r) {
    memset(&r, 0, sizeof r);
    r.dist = dist;
    r.fixed_mode = -1;
    r.family = -1;
    r.unit = 1;
    r.table = -1;
    r.words_per_sample = 1.0;
    switch (dist) {
    case RS_DIST_UINT64: {
        u64 b = ip[0];
        bool b64 = ip[1] != 0;
        if (b == 0 || b64) { r.fixed_mode = FX_RAW; }
        else if ((b & (b - 1)) == 0) { r.fixed_mode = FX_POW2; r.ip[0] = b; }
        else {
            r.family = FAM_LEMIRE;
            r.ip[0] = b;
            r.ip[1] = (0 - b) % b;  // discrete.py:34
            r.words_per_sample = 1.0 / (1.0 - (double)r.ip[1] * 5.421010862427522e-20);
        }
        return RS_OK;
    }
    case RS_DIST_INT64: {  // bounded_int(m, n, 64): ip = {span, 64, m, full}
        if (ip[3]) { r.fixed_mode = FX_WMAP; r.kind = WK_I64; r.ip[2] = ip[2]; return RS_OK; }
        u64 b = ip[0];
        if (b == 0) RS_FAIL("bad signed range");
        r.family = FAM_LEMIRE;
        r.ip[0] = b;
        r.ip[1] = (0 - b) % b;
        r.ip[2] = ip[2];
        r.words_per_sample = 1.0 / (1.0 - (double)r.ip[1] * 5.421010862427522e-20);
        return RS_OK;
    }
    case RS_DIST_UINT32: case RS_DIST_INT32: {  // halves; ip = {b, width} | {span, 32, m, full}
        int width = dist == RS_DIST_INT32 ? 32 : (int)ip[1];
        if (width != 8 && width != 16 && width != 32) RS_FAIL("bounded width must be 8, 16, or 32");
        u64 full = 1ULL << width, mask = full - 1;
        u64 b = ip[0];
        r.unit = 2;
        if (dist == RS_DIST_INT32 && ip[3]) { r.fixed_mode = FX_HMAP; r.kind = HK_I32; r.ip[2] = ip[2]; return RS_OK; }
        if (b > full) RS_FAIL("bound out of range");
        if (dist == RS_DIST_UINT32 && (b == 0 || b == full)) {
            r.fixed_mode = FX_HMAP; r.kind = HK_MASK; r.ip[3] = mask; return RS_OK;
        }
        if (dist == RS_DIST_UINT32 && (b & (b - 1)) == 0) {
            r.fixed_mode = FX_HMAP; r.kind = HK_POW2; r.ip[0] = b; r.ip[1] = (u64)width; r.ip[3] = mask; return RS_OK;
        }
        if (b == 0) RS_FAIL("bad signed range");
        r.family = FAM_U32;
        r.ip[0] = b;
        r.ip[1] = (full - b) % b;
        r.ip[2] = dist == RS_DIST_INT32 ? ip[2] : 0;
        r.ip[3] = (u64)width;
        r.words_per_sample = 0.5 / (1.0 - (double)r.ip[1] / (double)full);
        return RS_OK;
    }
    case RS_DIST_U01: r.fixed_mode = FX_U01; return RS_OK;
    case RS_DIST_U01F: r.fixed_mode = FX_U01F; r.unit = 2; return RS_OK;
    case RS_DIST_UNIF:
        if (!(fp[1] > fp[0])) RS_FAIL("unif needs b > a");
        r.fixed_mode = FX_WMAP; r.kind = WK_UNIF; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_UNIFF:
        if (!(fp[1] > fp[0])) RS_FAIL("uniff needs b > a");
        r.fixed_mode = FX_HMAP; r.kind = HK_UNIFF; r.unit = 2; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_GUMBEL:
        if (!(fp[1] > 0.0)) RS_FAIL("gumbel scale must be > 0");
        r.fixed_mode = FX_WMAP; r.kind = WK_GUMBEL; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_NORM: case RS_DIST_STDNORM: case RS_DIST_LOGNORMAL:
        r.family = FAM_NORM;
        r.table = 0;
        r.words_per_sample = 1.03;
        if (dist == RS_DIST_STDNORM) { r.kind = NK_STD; r.raw_norm = 1; return RS_OK; }
        if (!(fp[1] >= 0.0)) RS_FAIL(dist == RS_DIST_NORM ? "normal variance must be >= 0" : "lognormal variance must be >= 0");
        r.kind = dist == RS_DIST_NORM ? NK_NORM : NK_LOGNORMAL;
        r.fp[0] = fp[0];
        r.fp[1] = std::sqrt(fp[1]);
        return RS_OK;
    case RS_DIST_SKEW_NORMAL: {  // fp = {alpha, mu, sigma}
        if (!(fp[2] > 0.0)) RS_FAIL("skew_normal scale must be > 0");
        double delta = fp[0] / std::sqrt(1.0 + fp[0] * fp[0]);
        r.family = FAM_NORM; r.kind = NK_SKEW; r.table = 0; r.words_per_sample = 2.06;
        r.fp[0] = delta; r.fp[1] = std::sqrt(1.0 - delta * delta); r.fp[2] = fp[1]; r.fp[3] = fp[2];
        return RS_OK;
    }
    case RS_DIST_EXP:
        if (!(fp[0] > 0.0)) RS_FAIL("exponential scale must be > 0");
        r.family = FAM_EXP; r.kind = EK_EXP; r.table = 1; r.fp[0] = fp[0]; r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_PARETO:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("pareto needs alpha > 0 and xm > 0");
        r.family = FAM_EXP; r.kind = EK_PARETO; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_GPD:
        if (!(fp[2] > 0.0)) RS_FAIL("gpd scale must be > 0");
        r.family = FAM_EXP; r.kind = EK_GPD; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1]; r.fp[2] = fp[2];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_WEIBULL:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("weibull needs k > 0 and lambda > 0");
        r.family = FAM_EXP; r.kind = EK_WEIBULL; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_GAMMA:
        if (!(fp[0] > 0.0)) RS_FAIL("gamma shape must be > 0");
        if (!(fp[1] > 0.0)) RS_FAIL("gamma scale must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_GAMMA; r.table = 0;
        r.ga = gamma_prm(fp[0], fp[1]);
        r.words_per_sample = gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_CHI2:
        if (!(fp[0] > 0.0)) RS_FAIL("chi2 degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_GAMMA; r.table = 0;
        r.ga = gamma_prm(fp[0] / 2.0, 2.0);
        r.words_per_sample = gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_T:
        if (!(fp[0] > 0.0)) RS_FAIL("t degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_T; r.table = 0; r.fp[0] = fp[0];
        r.ga = gamma_prm(fp[0] / 2.0, 2.0);
        r.words_per_sample = 1.03 + gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_F:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("f degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_F; r.table = 0; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.ga = gamma_prm(fp[0] / 2.0, 1.0);
        r.gb = gamma_prm(fp[1] / 2.0, 1.0);
        r.words_per_sample = gamma_words(r.ga) + gamma_words(r.gb);
        return RS_OK;
    case RS_DIST_BETA:
        if (!(fp[0] > 0.0) || !(fp[1] > 0.0)) RS_FAIL("gamma shape must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_BETA; r.table = 0;
        r.ga = gamma_prm(fp[0], 1.0);
        r.gb = gamma_prm(fp[1], 1.0);
        r.words_per_sample = gamma_words(r.ga) + gamma_words(r.gb);
        return RS_OK;
    case RS_DIST_NORMF:
        if (!(fp[1] >= 0.0)) RS_FAIL("normf variance must be >= 0");
        r.family = FAM_F32; r.kind = FK_NORMF; r.unit = 2; r.table = 2; r.fp[0] = fp[0]; r.fp[1] = std::sqrt(fp[1]);
        r.words_per_sample = 0.52;
        return RS_OK;
    case RS_DIST_EXPF:
        if (!(fp[0] > 0.0)) RS_FAIL("expf scale must be > 0");
        r.family = FAM_F32; r.kind = FK_EXPF; r.unit = 2; r.table = 3; r.fp[0] = fp[0];
        r.words_per_sample = 0.53;
        return RS_OK;
    }
    RS_FAIL("unknown distribution id");
}

void fill_plan_common(FillPlan &p, DevCtx &c, const Resolved &r, int engine, int fm) {
    p.engine = engine;
    p.dist = r.dist;
    p.fm = fm;
    memcpy(p.fp, r.fp, sizeof p.fp);
    memcpy(p.ip, r.ip, sizeof p.ip);
    p.ga = r.ga;
    p.gb = r.gb;
    p.raw_norm = r.raw_norm;
    p.kind = r.kind;
    p.unit = r.unit;
    p.fmode = r.fixed_mode;
    p.zslow = (r.table == 0 || r.table == 1) ? c.zslow[r.table] : nullptr;
    p.zfast = (r.table == 0 || r.table == 1) ? c.zfast[r.table] : nullptr;
    p.zslowf = (r.table == 2 || r.table == 3) ? c.zslowf[r.table - 2] : nullptr;
    p.zfastf = (r.table == 2 || r.table == 3) ? c.zfastf[r.table - 2] : nullptr;
    p.rlx_A = c.rlxA;
}

// Segment geometry + per-engine jump tables for stride L (engine origin = p.base)
rs_status plan_segments(DevCtx &c, FillPlan &p, u64 words, u64 Lmin, int occ, cudaStream_t st, bool tables = true,
                        u64 align = 36) {
    // exactly one wave of resident threads: equal segments finish together
    u64 Tfull = (u64)c.sms * (u64)occ * BLOCK;
    u64 L = (words + Tfull - 1) / Tfull;
    if (L < Lmin) L = Lmin;
    // a whole number of philox blocks (4) and ranlux chunks (9); fixed fills pass
    // align = 144 (also 16-word lines): every thread then has the same alignment
    // prologue, so the lanes stay in phase (ranlux mulmods convergent)
    L = (L + align - 1) / align * align;
    u64 T = (words + L - 1) / L;
    if (T < 1) T = 1;
    T = (T + BLOCK - 1) / BLOCK * BLOCK;
    p.L = L;
    p.T = (u32)T;
    int levels = 1;
    while ((1ULL << levels) < T) levels++;
    if (levels > MAXLEV) { rs::set_error("fill too large for one plan"); return RS_ERR_INTERNAL; }
    rs_status s = ensure_scratch(c, T);
    if (s) return s;
    if (!tables) return RS_OK;
    if (p.engine == RS_ENG_PCG64) {
        u128 inc = ((u128)p.base[3] << 64) | p.base[2];
        for (int j = 0; j < levels; j++) {
            u128 m, a;
            rs::pcg_affine(inc, (u128)L << j, m, a);
            p.pcg_m[j][0] = (u64)m; p.pcg_m[j][1] = (u64)(m >> 64);
            p.pcg_a[j][0] = (u64)a; p.pcg_a[j][1] = (u64)(a >> 64);
        }
    } else if (p.engine == RS_ENG_RANLUX) {
        for (int j = 0; j < levels; j++) rs::rlx_pow_A((u128)(L / 9) << j, p.rlx[j]);
    } else if (p.engine == RS_ENG_CHACHA20) {
        if ((p.base[5] >> 32) + (u128)T * (L / 8) > ((u128)1 << 32)) {
            rs::set_error("chacha20 stream exhausted");  // counter.py:212-213
            return RS_ERR_VALUE;
        }
    } else if (p.engine == RS_ENG_X256SS || p.engine == RS_ENG_X256PP || p.engine == RS_ENG_X128P ||
               p.engine == RS_ENG_XORO) {
        int lv = 0;  // bits of the warp index
        while ((1ULL << lv) < T / 32) lv++;
        u64 *ml;
        if (p.engine == RS_ENG_X128P || p.engine == RS_ENG_XORO) {  // padded 4-word states
            p.base[2] = p.base[3] = 0;
        }
        s = x256_mats(c, p.engine, L, lv, &ml);
        if (s) return s;
        p.x256_states = c.states;
        void *args[] = {&p, &ml, &c.states};
        s = launch((const void *)k_x256_setup, dim3((unsigned)(T / BLOCK)), dim3(BLOCK), args, st);
        if (s) return s;
    }
    return RS_OK;
}

// logical stream of `s`: buffer remainder then engine words
void stream_prefix(const rs_stream *s, FillPlan &p) {
    int P = s->fill - s->cursor;
    if (P < 0) P = 0;
    p.P = P;
    for (int i = 0; i < P; i++) p.prefix[i] = s->buf[s->cursor + i];
}

// post-fill position (buffer.py:29-49): E logical words consumed
rs_status apply_consumption(rs_stream *s, u64 E, const DevResult *sr) {
    int P = s->fill - s->cursor;
    if (P < 0) P = 0;
    if (E <= (u64)P) {
        s->cursor += (int)E;
        return RS_OK;
    }
    u64 ep = E - P;
    u64 R = (ep + CAP - 1) / CAP;
    if (is_serial(s->engine)) {  // rebuilt on the device by k_serial
        if (!sr || sr->serial_consumed != ep) {
            rs::set_error("serial fill bookkeeping mismatch");
            return RS_ERR_INTERNAL;
        }
        memcpy(s->state, sr->serial_state, 8 * rs::state_words(s->engine));
        memcpy(s->buf, sr->serial_buf, CAP * 8);
    } else {
        if (!rs::engine_advance_words(s->engine, s->state, (u128)(R - 1) * CAP)) {
            rs::set_error("cannot advance engine");
            return RS_ERR_INTERNAL;
        }
        rs::engine_generate(s->engine, s->state, s->buf, CAP);
    }
    s->fill = CAP;
    s->cursor = (int)(ep - (R - 1) * CAP);
    return RS_OK;
}

struct Staging {
    void *dptr = nullptr;
    bool host = false;
};

rs_status get_out(DevCtx &c, void *out, size_t bytes, Staging &sg) {
    if (is_device_ptr(out)) { sg.dptr = out; sg.host = false; return RS_OK; }
    sg.host = true;
    if (bytes > c.stage_bytes) {
        cudaFree(c.stage);
        c.stage = nullptr;
        CK(cudaMalloc(&c.stage, bytes));
        c.stage_bytes = bytes;
    }
    sg.dptr = c.stage;
    return RS_OK;
}

// interleaved xoshiro fixed fill: lane states jumped per step group on the device
rs_status launch_simd(DevCtx &c, FillPlan &p, int mode, cudaStream_t st) {
    const void *fn = simd_kernel(p.engine, mode);
    u64 steps = (p.weng + 7) / 8;
    if (steps == 0) steps = 1;
    // an eighth of a wave of lane-threads: the per-lane GF(2) setup (k_x256_setup) costs
    // per thread, while the store-bound fill saturates HBM well before a full wave
    // (x256++simd 2^28 normals 3.86 -> 3.71 ms, 2^24 raw 0.28 -> 0.09 ms)
    u64 Gfull = (u64)c.sms * occupancy(fn) * BLOCK / 64;
    u64 Ls = (steps + Gfull - 1) / Gfull;
    if (Ls < 16) Ls = 16;
    u64 G = (steps + Ls - 1) / Ls;
    u64 Gpad = (G + BLOCK - 1) / BLOCK * BLOCK;
    p.L = Ls;
    p.G = G;
    p.Gpad = Gpad;
    rs_status rc = ensure_scratch(c, 8 * Gpad);
    if (rc) return rc;
    int lv = 0;
    while ((1ULL << lv) < Gpad / 32) lv++;
    u64 *ml;
    if ((rc = x256_mats(c, RS_ENG_X256PP, Ls, lv, &ml))) return rc;
    p.x256_states = c.states;
    void *sargs[] = {&p, &ml, &c.states};
    if ((rc = launch((const void *)k_x256_setup, dim3((unsigned)(Gpad / BLOCK), 8), dim3(BLOCK), sargs, st))) return rc;
    void *args[] = {&p};
    return launch(fn, dim3((unsigned)(8 * Gpad / BLOCK)), dim3(BLOCK), args, st);
}

// engine words [0, m.weng) of m.base into m.out (raw u64) with the fixed-fill kernels
rs_status launch_raw_words(DevCtx &c, FillPlan &m, cudaStream_t st) {
    rs_status rc;
    if (rs::simd_engine(m.engine)) return launch_simd(c, m, FX_RAW, st);
    if (m.engine == RS_ENG_PHILOX) {
        const void *fn = philox_kernel(FX_RAW);
        for (int i = 0; i < 10; i++) {
            m.rk0[i] = m.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
            m.rk1[i] = m.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
        }
        m.vec_ok = (((uintptr_t)m.out) & 31) == 0;
        u64 nblk = (m.weng + 3) / 4;
        u64 g = (u64)c.sms * occupancy(fn);
        u64 need = (nblk + BLOCK - 1) / BLOCK;
        if (need < g) g = need;
        if (g < 1) g = 1;
        void *args[] = {&m};
        return launch(fn, dim3((unsigned)g), dim3(BLOCK), args, st);
    }
    const void *fn = fixed_kernel(m.engine, FX_RAW);
    if ((rc = plan_segments(c, m, m.weng, 64, occupancy(fn), st, true, 144))) return rc;
    void *args[] = {&m};
    return launch(fn, dim3(m.T / BLOCK), dim3(BLOCK), args, st);
}

// The device part of one fill. On return (sync=true) `E` holds the stream units
// consumed (64-bit words, or 32-bit halves incl. a used pending half when r.unit == 2)
// and `tal` the tallies.
rs_status run_fill(DevCtx &c, const rs_stream *s, const Resolved &r, u64 n, void *dout, cudaStream_t st, bool sync,
                   u64 &E, u64 *tal, int &rounds, u64 &chunks) {
    E = 0;
    rounds = 0;
    chunks = 0;
    for (int i = 0; i < 6; i++) tal[i] = 0;
    if (n == 0) return RS_OK;
    FillPlan p;
    memset(&p, 0, sizeof p);
    fill_plan_common(p, c, r, s->engine, s->full_mantissa);
    stream_prefix(s, p);
    p.out = dout;
    p.out0 = 0;
    memcpy(p.base, s->state, sizeof p.base);
    memcpy(p.lanes, s->state, sizeof p.lanes);
    const u64 u = (u64)r.unit;
    p.pending_used = (u == 2 && s->has_pending) ? 1 : 0;
    p.pending_val = (u32)s->pending;
    rs_status rc;

    if (is_serial(s->engine)) {  // sfc64 / sfc64simd single stream: no skip-ahead, serial
        p.n = n;
        if (s->engine == RS_ENG_SFC64_SIMD) memcpy(p.lanes, s->state, sizeof p.lanes);
        DevResult *res = c.res;
        void *args[] = {&p, &res};
        rc = launch(serial_kernel(s->engine, r.family, r.fixed_mode), dim3(1), dim3(32), args, st);
        if (rc) return rc;
        if (sync) {
            CK(cudaMemcpyAsync(c.res_host, c.res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            E = c.res_host->end_pos;
            for (int i = 0; i < 6; i++) tal[i] = c.res_host->tally[i];
        }
        chunks = 1;
        return RS_OK;
    }

    if (r.fixed_mode >= 0) {
        // fixed consumption: sample i <- logical unit i
        u64 words = u == 2 ? (n - p.pending_used + 1) / 2 : n;
        p.n = n;
        p.weng = words > (u64)p.P ? words - p.P : 0;
        if (s->engine == RS_ENG_PHILOX) {
            const void *fn = philox_kernel(r.fixed_mode);
            // round keys k + r*W (counter.py:95-96) live in the constant bank
            for (int i = 0; i < 10; i++) {
                p.rk0[i] = p.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
                p.rk1[i] = p.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
            }
            uintptr_t a = (uintptr_t)dout;
            if (u == 2)
                p.vec_ok = ((a + 4 * ((u64)p.pending_used + 2ULL * p.P)) & 31) == 0;
            else
                p.vec_ok = ((a + 8ULL * p.P) & 31) == 0;
            u64 nblk = (p.weng + 3) / 4;
            u64 g = (u64)c.sms * occupancy(fn);
            u64 need = (nblk + BLOCK - 1) / BLOCK;
            if (need < g) g = need;
            if (g < 1) g = 1;
            void *args[] = {&p};
            rc = launch(fn, dim3((unsigned)g), dim3(BLOCK), args, st);
            if (rc) return rc;
            E = n;
            chunks = 1;
            return RS_OK;
        }
        if (rs::simd_engine(s->engine)) {
            if ((rc = launch_simd(c, p, r.fixed_mode, st))) return rc;
            E = n;
            chunks = 1;
            return RS_OK;
        }
        const void *fn = fixed_kernel(s->engine, r.fixed_mode);
        rc = plan_segments(c, p, p.weng ? p.weng : 1, 64, occupancy(fn), st, true, 144);
        if (rc) return rc;
        void *args[] = {&p};
        rc = launch(fn, dim3(p.T / BLOCK), dim3(BLOCK), args, st);
        if (rc) return rc;
        E = n;
        chunks = 1;
        return RS_OK;
    }

    // variable consumption: chunks of provisioned words until n samples exist.
    // Chunk coordinates: chunk-local position lp in units; chunk 1 starts with the
    // pending half (u = 2) and the P buffered words, then the engine; a later chunk
    // has neither and lp counts engine units from its origin (thread 0 starts at lp0).
    VarKernels K = var_kernels(s->engine, r.family);
    const u64 P1 = (u64)p.P, pp1 = (u64)p.pending_used;
    u64 done = 0;    // samples produced so far
    u64 origin = 0;  // engine words from s->state to this chunk's origin (multiple of 36)
    u64 lp0 = 0;
    u64 Lmin = r.family == FAM_GAMMA ? (r.kind == GK_GAMMA ? 1024 : 2048) : 128;
    bool first = true;
    while (done < n) {
        u64 need = n - done;
        double ww = (double)need * r.words_per_sample;
        u64 words = (u64)(ww * 1.01 + 12.0 * std::sqrt(ww) + 2048.0);
        if (!first) {
            p.P = 0;
            p.pending_used = 0;
            u64 st32[32];
            memcpy(st32, s->state, sizeof st32);
            if (!rs::engine_advance_words(s->engine, st32, (u128)origin)) {
                rs::set_error("cannot position engine");
                return RS_ERR_INTERNAL;
            }
            memcpy(p.base, st32, sizeof p.base);
            memcpy(p.lanes, st32, sizeof p.lanes);
        }
        p.lp0 = lp0;
        p.n = need;
        p.out0 = done;
        int occ = std::min(occupancy(K.count), std::min(occupancy(K.fixup), occupancy(K.emit)));
        const bool mem = parse_from_memory(s->engine);
        rc = plan_segments(c, p, words + (lp0 + u - 1) / u, Lmin, occ, st, !mem);
        if (rc) return rc;
        if (mem) {
            // materialize the chunk's engine words (+ slack for the parses that run past the
            // last segment end) with the coalesced fixed-fill kernel
            u64 nw = (u64)p.T * p.L + std::max<u64>(1ULL << 16, (u64)p.T * p.L / 64);
            nw = (nw + 143) / 144 * 144;
            if (nw * 8 > c.words_bytes) {
                cudaFree(c.words);
                c.words = nullptr;
                CK(cudaMalloc(&c.words, nw * 8));
                c.words_bytes = nw * 8;
            }
            FillPlan m = p;
            m.P = 0;
            m.lp0 = 0;
            m.n = nw;
            m.weng = nw;
            m.out = c.words;
            m.out0 = 0;
            m.pending_used = 0;
            m.unit = 1;
            m.fmode = FX_RAW;
            if ((rc = launch_raw_words(c, m, st))) return rc;
            p.words = c.words;
            p.nwords = nw;
        }
        p.bm = r.family == FAM_GAMMA ? c.bm : nullptr;  // read now: the steps above may grow the scratch
        CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
        unsigned g = p.T / BLOCK;
        int round = 0;
        DevResult *res = c.res;
        {
            void *a1[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1};
            if ((rc = launch(K.count, dim3(g), dim3(BLOCK), a1, st))) return rc;
            const u32 *prev = c.ex0;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1, &prev, &c.entry, &c.cnt, &c.exA, &round, &res};
            if ((rc = launch(K.fixup, dim3(g), dim3(BLOCK), a2, st))) return rc;
        }
        u32 *ex_cur = c.exA, *ex_other = c.exB;
        for (;;) {
            size_t bytes = c.cub_bytes;
            CK(cub::DeviceScan::ExclusiveSum(c.cub_tmp, bytes, c.cnt, c.off, (int)p.T, st));
            void *a3[] = {&p, &c.entry, &c.cnt, &c.off, &ex_cur, &res};
            if ((rc = launch(K.emit, dim3(g), dim3(BLOCK), a3, st))) return rc;
            if (!sync) { chunks++; return RS_OK; }
            CK(cudaMemcpyAsync(c.res_host, c.res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (!c.res_host->flag) break;
            // entries not at a fixed point: iterate the resolution (SURVEY 7.2#1 fallback)
            // after round k threads 0..k have final exits, so p.T rounds always suffice
            if (++round > (int)p.T) { rs::set_error("segment entry resolution did not converge"); return RS_ERR_INTERNAL; }
            rounds++;
            CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
            const u32 *prev = ex_cur;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1, &prev, &c.entry, &c.cnt, &ex_other, &round, &res};
            if ((rc = launch(K.fixup, dim3(g), dim3(BLOCK), a2, st))) return rc;
            u32 *tmp = ex_cur; ex_cur = ex_other; ex_other = tmp;
        }
        chunks++;
        if (mem) {
            u32 over = 0, zero = 0;
            CK(cudaMemcpyFromSymbol(&over, g_mem_overrun, sizeof over));
            if (over) {
                CK(cudaMemcpyToSymbol(g_mem_overrun, &zero, sizeof zero));
                rs::set_error("parse ran past the materialized words (raise the slack)");
                return RS_ERR_INTERNAL;
            }
        }
        for (int i = 0; i < 6; i++) tal[i] += c.res_host->tally[i];
        u64 total = c.res_host->total;
        // chunk-local units -> engine units (from s->state) and whole-fill units
        u64 to_engine = first ? (u64)0 - (u * P1 + pp1) : u * origin;
        if (done + total >= n) {
            E = u * P1 + pp1 + (c.res_host->end_pos + to_engine);
            break;
        }
        done += total;
        u64 resume = c.res_host->next_start + to_engine;  // engine unit of the next boundary
        origin = resume / u / 72 * 72;  // whole Philox / ranlux / 8-word blocks
        lp0 = resume - u * origin;
        first = false;
    }
    return RS_OK;
}

// which reference tallies a fill touches (continuous.py:32-33: std_norm, std_exp, gamma)
void tally_seen(const Resolved &r, int32_t *seen) {
    seen[0] = seen[1] = seen[2] = 0;
    if (r.family == FAM_NORM) seen[0] = 1;
    if (r.family == FAM_EXP) seen[1] = 1;
    if (r.family == FAM_GAMMA) { seen[0] = 1; seen[2] = 1; }
}

rs_status check_stream(const rs_stream *s) {
    if (!s) { rs::set_error("null stream"); return RS_ERR_VALUE; }
    if (!rs::device_engine(s->engine)) { rs::set_error("engine not on the B200 fill path"); return RS_ERR_UNSUPPORTED; }
    if (s->fill < 0 || s->fill > CAP || s->cursor < 0 || s->cursor > s->fill) {
        rs::set_error("buffer cursor out of range");
        return RS_ERR_VALUE;
    }
    return RS_OK;
}

}  // namespace

// ============================================================================= C ABI
extern "C" {

rs_status rs_init_device(int32_t device) {
    std::lock_guard<std::mutex> g(g_mu);
    CK(cudaSetDevice(device));
    DevCtx *c;
    rs_status s = init_dev(device, &c);
    if (s == RS_OK) rs::clear_error();
    return s;
}

rs_status rs_fill(rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams, uint64_t n, void *out,
                  rs_fill_result *result, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    rs_status rc = check_stream(s);
    if (rc) return rc;
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (result) memset(result, 0, sizeof *result);
    if (n == 0) { rs::clear_error(); return RS_OK; }  // the reference consumes nothing for n == 0
    if (!out) { rs::set_error("null output"); return RS_ERR_VALUE; }
    int dev;
    if (is_device_ptr(out)) {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, out));
        dev = a.device;
        CK(cudaSetDevice(dev));
    } else {
        CK(cudaGetDevice(&dev));
    }
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t bytes = (size_t)n * elem_size(dist);
    Staging sg;
    if ((rc = get_out(*c, out, bytes, sg))) return rc;
    u64 Eu, tal[6];
    int rounds;
    u64 chunks;
    if ((rc = run_fill(*c, s, r, n, sg.dptr, st, true, Eu, tal, rounds, chunks))) return rc;
    if (sg.host) {
        CK(cudaMemcpyAsync(out, sg.dptr, bytes, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    // stream position after the fill (buffer.py:29-49)
    int P = s->fill - s->cursor;
    u64 pre_words[CAP];
    for (int i = 0; i < P; i++) pre_words[i] = s->buf[s->cursor + i];
    u64 E;            // 64-bit words taken from the buffer / engine
    bool odd = false; // a u32 consumer ended on a low half: the high half stays pending
    if (r.unit == 2) {
        u64 pp = s->has_pending ? 1 : 0;
        u64 rel = Eu > pp ? Eu - pp : 0;
        E = (rel + 1) / 2;
        odd = rel & 1;
    } else {
        E = Eu;
    }
    if ((rc = apply_consumption(s, E, is_serial(s->engine) ? c->res_host : nullptr))) return rc;
    if (odd) {
        u64 last = E - 1;
        u64 w = last < (u64)P ? pre_words[last] : s->buf[s->cursor - 1];
        s->has_pending = 1;
        s->pending = w >> 32;
    } else {
        s->has_pending = 0;
        s->pending = 0;
    }
    if (result) {
        result->words_consumed = E;
        for (int i = 0; i < 6; i++) result->tally[i] = tal[i];
        tally_seen(r, result->tally_seen);
        result->resync_rounds = rounds;
        result->chunks = chunks;
    }
    rs::clear_error();
    return RS_OK;
}

rs_status rs_fill_async(const rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams, uint64_t n,
                        void *out_device, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    rs_status rc = check_stream(s);
    if (rc) return rc;
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (n == 0) return RS_OK;
    int dev;
    CK(cudaGetDevice(&dev));
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    u64 E, tal[6];
    int rounds;
    u64 chunks;
    rc = run_fill(*c, s, r, n, out_device, (cudaStream_t)cuda_stream, false, E, tal, rounds, chunks);
    if (rc == RS_OK) rs::clear_error();
    return rc;
}

rs_status rs_fill_streams(int32_t engine, const uint64_t *seed, int32_t n_seed, const uint64_t *spawn_prefix,
                          int32_t n_prefix, uint64_t j0, uint64_t n_streams, int32_t dist, const double *fparams,
                          const uint64_t *iparams, uint64_t n_per_stream, void *out, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    if (engine != RS_ENG_SFC64 && engine != RS_ENG_PCG64 && engine != RS_ENG_PHILOX && engine != RS_ENG_X256SS &&
        engine != RS_ENG_X256PP && engine != RS_ENG_X128P && engine != RS_ENG_XORO && engine != RS_ENG_SQUARES &&
        engine != RS_ENG_CHACHA20 && engine != RS_ENG_CWG128) {
        rs::set_error("per-stream mode supports sfc64, pcg64, philox, x256**, x256++, x128+, xoro++, squares, chacha20, cwg128");
        return RS_ERR_UNSUPPORTED;
    }
    if (n_seed < 0 || n_seed > 16 || n_prefix < 0 || n_prefix > 7) {
        rs::set_error("seed / spawn key too long");
        return RS_ERR_VALUE;
    }
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rs_status rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (n_streams == 0 || n_per_stream == 0) { rs::clear_error(); return RS_OK; }
    int dev;
    if (is_device_ptr(out)) {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, out));
        dev = a.device;
        CK(cudaSetDevice(dev));
    } else {
        CK(cudaGetDevice(&dev));
    }
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t bytes = (size_t)n_streams * n_per_stream * elem_size(dist);
    Staging sg;
    if ((rc = get_out(*c, out, bytes, sg))) return rc;
    StreamArgs a;
    memset(&a, 0, sizeof a);
    a.engine = engine;
    a.nseed = n_seed;
    a.nprefix = n_prefix;
    for (int i = 0; i < n_seed; i++) a.seed[i] = seed[i];
    for (int i = 0; i < n_prefix; i++) a.prefix[i] = spawn_prefix[i];
    a.j0 = j0;
    a.nstreams = n_streams;
    a.nper = n_per_stream;
    a.dist = r.dist;
    a.fm = 0;
    memcpy(a.fp, r.fp, sizeof a.fp);
    memcpy(a.ip, r.ip, sizeof a.ip);
    a.ga = r.ga;
    a.gb = r.gb;
    a.kind = r.kind;
    a.zslow = (r.table == 0 || r.table == 1) ? c->zslow[r.table] : nullptr;
    a.zfast = (r.table == 0 || r.table == 1) ? c->zfast[r.table] : nullptr;
    a.zslowf = (r.table == 2 || r.table == 3) ? c->zslowf[r.table - 2] : nullptr;
    a.zfastf = (r.table == 2 || r.table == 3) ? c->zfastf[r.table - 2] : nullptr;
    a.rlx_A = c->rlxA;
    a.out = sg.dptr;
    int d = r.family;
    if (r.fixed_mode == FX_POW2) {  // b = 2^k: Lemire without a rejection zone
        d = FAM_LEMIRE;
        a.ip[0] = r.ip[0];
        a.ip[1] = 0;
        a.ip[2] = 0;
    } else if (r.fixed_mode == FX_HMAP && r.kind == HK_POW2) {
        d = FAM_U32;
        a.ip[0] = r.ip[0];
        a.ip[1] = 0;
        a.ip[2] = 0;
        a.ip[3] = r.ip[1];
    } else if (r.fixed_mode >= 0) {  // raw / u01 / u01f / unif / gumbel / masks / full spans
        d = FAM_FIXED;
        a.fmode = r.fixed_mode;
        memcpy(a.ip, r.ip, sizeof a.ip);
    }
    const void *fn = nullptr;
#define RS_STREAM_CASE(E)                                                     \
    switch (d) {                                                              \
    case FAM_NORM: fn = (const void *)k_streams<E, FAM_NORM>; break;          \
    case FAM_EXP: fn = (const void *)k_streams<E, FAM_EXP>; break;            \
    case FAM_GAMMA: fn = (const void *)k_streams<E, FAM_GAMMA>; break;        \
    case FAM_F32: fn = (const void *)k_streams<E, FAM_F32>; break;            \
    case FAM_U32: fn = (const void *)k_streams<E, FAM_U32>; break;            \
    case FAM_FIXED: fn = (const void *)k_streams<E, FAM_FIXED>; break;        \
    default: fn = (const void *)k_streams<E, FAM_LEMIRE>; break;              \
    }
    if (engine == RS_ENG_SFC64) { RS_STREAM_CASE(RS_ENG_SFC64) }
    else if (engine == RS_ENG_PCG64) { RS_STREAM_CASE(RS_ENG_PCG64) }
    else if (engine == RS_ENG_PHILOX) { RS_STREAM_CASE(RS_ENG_PHILOX) }
    else if (engine == RS_ENG_X256SS) { RS_STREAM_CASE(RS_ENG_X256SS) }
    else if (engine == RS_ENG_X128P) { RS_STREAM_CASE(RS_ENG_X128P) }
    else if (engine == RS_ENG_XORO) { RS_STREAM_CASE(RS_ENG_XORO) }
    else if (engine == RS_ENG_SQUARES) { RS_STREAM_CASE(RS_ENG_SQUARES) }
    else if (engine == RS_ENG_CHACHA20) { RS_STREAM_CASE(RS_ENG_CHACHA20) }
    else if (engine == RS_ENG_CWG128) { RS_STREAM_CASE(RS_ENG_CWG128) }
    else { RS_STREAM_CASE(RS_ENG_X256PP) }
#undef RS_STREAM_CASE
    void *args[] = {&a};
    unsigned g2 = (unsigned)((n_streams + BLOCK - 1) / BLOCK);
    if ((rc = launch(fn, dim3(g2), dim3(BLOCK), args, st))) return rc;
    if (sg.host) {
        CK(cudaMemcpyAsync(out, sg.dptr, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    CK(cudaGetLastError());
    rs::clear_error();
    return RS_OK;
}

rs_status rs_mvn(rs_stream *s, const double *L, const double *mean, int64_t d, uint64_t n, int32_t layout,
                 double *out, rs_fill_result *result, void *cuda_stream) {
    if (d < 1 || n < 1) { rs::set_error("mvn needs n >= 1"); return RS_ERR_VALUE; }
    if (layout != 0 && layout != 1) { rs::set_error("mvn layout must be 'n_d' or 'd_n'"); return RS_ERR_VALUE; }
    rs_status rc;
    int dev;
    {
        std::lock_guard<std::mutex> g(g_mu);
        if ((rc = check_stream(s))) return rc;
        if (is_device_ptr(out)) {
            cudaPointerAttributes a;
            CK(cudaPointerGetAttributes(&a, out));
            dev = a.device;
            CK(cudaSetDevice(dev));
        } else {
            CK(cudaGetDevice(&dev));
        }
    }
    DevCtx *c;
    {
        std::lock_guard<std::mutex> g(g_mu);
        if ((rc = init_dev(dev, &c))) return rc;
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t nz = (size_t)n * (size_t)d;
    // z and the factor / mean in device memory
    size_t need = nz * 8 + (size_t)d * d * 8 + (size_t)d * 8;
    {
        std::lock_guard<std::mutex> g(g_mu);
        if (need > c->mvn_bytes) {
            cudaFree(c->mvn_z);
            c->mvn_z = nullptr;
            CK(cudaMalloc(&c->mvn_z, need));
            c->mvn_bytes = need;
        }
        if (!c->blas) {
            if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) { rs::set_error("cublasCreate failed"); return RS_ERR_CUDA; }
        }
    }
    double *z = c->mvn_z, *Ld = z + nz, *md = Ld + (size_t)d * d;
    CK(cudaMemcpyAsync(Ld, L, (size_t)d * d * 8, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(md, mean, (size_t)d * 8, cudaMemcpyDefault, st));
    rs_fill_result fr;
    if ((rc = rs_fill(s, RS_DIST_STDNORM, nullptr, nullptr, nz, z, &fr, cuda_stream))) return rc;
    std::lock_guard<std::mutex> g(g_mu);
    bool host_out = !is_device_ptr(out);
    double *X;
    if (host_out) {
        if (nz * 8 > c->stage_bytes) {
            cudaFree(c->stage);
            c->stage = nullptr;
            CK(cudaMalloc(&c->stage, nz * 8));
            c->stage_bytes = nz * 8;
        }
        X = (double *)c->stage;
    } else {
        X = out;
    }
    k_mvn_init<<<(unsigned)std::min<u64>((nz + 255) / 256, 148 * 16), 256, 0, st>>>(X, md, d, n, layout);
    CK(cudaGetLastError());
    cublasSetStream(c->blas, st);
    double one = 1.0;
    cublasStatus_t bs;
    if (layout == 0) {
        // X (n x d row-major) = (d x n col-major) C = L * z^T : A = L buffer (row-major => col-major L^T), op T
        bs = cublasDgemm(c->blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)d, (int)n, (int)d, &one, Ld, (int)d, z, (int)d, &one,
                         X, (int)d);
    } else {
        // X^T (d x n row-major) = (n x d col-major) C = z * L^T : z buffer is (d x n) col-major -> op T
        bs = cublasDgemm(c->blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)d, (int)d, &one, z, (int)d, Ld, (int)d, &one,
                         X, (int)n);
    }
    if (bs != CUBLAS_STATUS_SUCCESS) { rs::set_error("cublasDgemm failed"); return RS_ERR_CUDA; }
    if (host_out) CK(cudaMemcpyAsync(out, X, nz * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (result) *result = fr;
    rs::clear_error();
    return RS_OK;
}

}  // extern "C"
