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
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "rs_device.cuh"
#include "rs_internal.h"

using rs::u128;

namespace {

constexpr int BLOCK = 256;
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
    int vec_ok;                   // counter-based fill: outputs 32-byte aligned per block
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int raw_norm;                 // std_norm without the epilogue (mvn z)
    const u64 *x256_states;
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
    u64 serial_state[9];
    u64 serial_buf[CAP];
    u64 serial_consumed;
};

// ----------------------------------------------------------------------------- device helpers
__device__ __forceinline__ u64 seg_start(const FillPlan &p, u32 t) { return t == 0 ? p.lp0 : (u64)p.P + (u64)t * p.L; }
__device__ __forceinline__ u64 seg_end(const FillPlan &p, u32 t) { return (u64)p.P + (u64)(t + 1) * p.L; }

template <int E>
struct EngOf;
template <> struct EngOf<RS_ENG_X256SS> { typedef EngX256<true> type; };
template <> struct EngOf<RS_ENG_X256PP> { typedef EngX256<false> type; };
template <> struct EngOf<RS_ENG_PCG64> { typedef EngPcg type; };
template <> struct EngOf<RS_ENG_PHILOX> { typedef EngPhilox type; };
template <> struct EngOf<RS_ENG_RANLUX> { typedef EngRanlux type; };
template <> struct EngOf<RS_ENG_SFC64> { typedef EngSfc type; };

// engine positioned at engine word t*L of the chunk (thread t's segment start)
template <int E>
__device__ __forceinline__ void make_engine(const FillPlan &p, u32 t, typename EngOf<E>::type &e) {
    if constexpr (E == RS_ENG_X256SS || E == RS_ENG_X256PP) {
        e.load(p.x256_states + 4 * (u64)t);
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

// word source positioned at logical position `pos` of segment t (pos >= seg_start)
template <int E>
__device__ __forceinline__ void make_src(const FillPlan &p, u32 t, u64 pos, Src<E> &s) {
    make_engine<E>(p, t, s.e);
    s.npre = 0;
    s.pre = p.prefix;
    s.pos = pos;
    u64 skip;
    if (t == 0) {
        if (pos < (u64)p.P) { s.pre = p.prefix + pos; s.npre = p.P - (int)pos; skip = 0; }
        else skip = pos - p.P;
    } else {
        skip = pos - seg_start(p, t);
    }
    for (u64 i = 0; i < skip; i++) s.e.next();
}

// ---- distributions from the plan
template <int D> struct DistOf;
template <> struct DistOf<RS_DIST_NORM> { typedef DistNorm type; };
template <> struct DistOf<RS_DIST_EXP> { typedef DistExp type; };
template <> struct DistOf<RS_DIST_GAMMA> { typedef DistGamma type; };
template <> struct DistOf<RS_DIST_BETA> { typedef DistBeta type; };
template <> struct DistOf<RS_DIST_UINT64> { typedef DistLemire type; };

template <int D>
__device__ __forceinline__ void make_dist_f(const double *fp, const u64 *ip, const GammaPrm &ga, const GammaPrm &gb,
                                            int raw, const RsZigSlow *zslow, int fm, const ZigFast *fast,
                                            typename DistOf<D>::type &d) {
    if constexpr (D == RS_DIST_UINT64) {
        d.b = ip[0];
        d.thr = ip[1];
    } else {
        d.z.fast = fast;
        d.z.slow = zslow;
        d.z.fm = fm;
        if constexpr (D == RS_DIST_NORM) {
            d.mu = fp[0];
            d.sd = fp[1];
            d.raw = raw;
        } else if constexpr (D == RS_DIST_EXP) {
            d.beta = fp[0];
        } else if constexpr (D == RS_DIST_GAMMA) {
            d.g = ga;
        } else {
            d.ga = ga;
            d.gb = gb;
        }
    }
}
template <int D>
__device__ __forceinline__ void make_dist(const FillPlan &p, const ZigFast *fast, typename DistOf<D>::type &d) {
    make_dist_f<D>(p.fp, p.ip, p.ga, p.gb, p.raw_norm, p.zslow, p.fm, fast, d);
}

__device__ __forceinline__ void stage_tables(const FillPlan &p, ZigFast *sm) {
    if (p.zfast) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = p.zfast[i];
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
    u64 v[4] = {p.base[0], p.base[1], p.base[2], p.base[3]};
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
    return E == RS_ENG_RANLUX ? 2 : (D == RS_DIST_GAMMA || D == RS_DIST_BETA) ? 2 : D == RS_DIST_UINT64 ? 4 : 3;
}

// ----------------------------------------------------------------------------- two-pass parse
// count: samples that START inside [seg_start, seg_end) and the exit (first sample
// boundary at or beyond seg_end), parsing from seg_start as if it were a boundary.
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_count(const __grid_constant__ FillPlan p, u64 *cnt0, u32 *ex0) {
    __shared__ ZigFast sm[256];
    stage_tables(p, sm);
    u32 t = blockIdx.x * BLOCK + threadIdx.x;
    if (t >= p.T) return;
    const u64 end = seg_end(p, t);
    Src<E> s;
    make_src<E>(p, t, seg_start(p, t), s);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl;
    u64 c = 0;
    if constexpr (D == RS_DIST_UINT64) {  // independent one-word tokens: word-level loop
        bool bnd = true;
        while (!(bnd && s.pos >= end)) {
            u64 o;
            bnd = d.accept(s.next(), o);
            c += bnd;
        }
    } else {
        while (s.pos < end) {
            d.sample(s, tl);
            c++;
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
__device__ void resolve_entry(const FillPlan &p, const ZigFast *sm, u32 t, u32 e, u64 c0, u32 x0, u64 &cnt,
                              u32 &ex) {
    const u64 start = seg_start(p, t), end = seg_end(p, t);
    Src<E> sa, sb;
    make_src<E>(p, t, start, sa);
    make_src<E>(p, t, start + e, sb);
    typename DistOf<D>::type d;
    make_dist<D>(p, sm, d);
    Tally tl;
    u64 na = 0, nb = 0;
    while (true) {
        if (sa.pos == sb.pos && sa.pos < end) {
            cnt = c0 - na + nb;
            ex = x0;
            return;
        }
        if (sb.pos >= end) {
            cnt = nb;
            ex = (u32)(sb.pos - end);
            return;
        }
        if (sa.pos < sb.pos && sa.pos < end) {
            d.sample(sa, tl);
            na++;
        } else {
            d.sample(sb, tl);
            nb++;
        }
    }
}

// round 0: prev_ex = ex0, every thread; round r>0: only threads whose entry changed.
template <int E, int D>
__global__ void __launch_bounds__(BLOCK, minb(E, D)) k_fixup(const __grid_constant__ FillPlan p, const u64 *cnt0, const u32 *ex0,
                                                 const u32 *prev_ex, u32 *entry, u64 *cnt, u32 *ex, int round,
                                                 DevResult *res) {
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
        resolve_entry<E, D>(p, sm, t, e, cnt0[t], ex0[t], c, x);
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
            Src<E> s;
            make_src<E>(p, t, seg_start(p, t) + entry[t], s);
            typename DistOf<D>::type d;
            make_dist<D>(p, sm, d);
            typedef typename DistOf<D>::type::out_t T;
            VecWriter8<T> wr;
            wr.init((T *)p.out, p.out0 + o);
            if constexpr (D == RS_DIST_UINT64) {
                for (u64 k = 0; k < kmax;) {
                    u64 o;
                    if (d.accept(s.next(), o)) { wr.put(o); k++; }
                }
            } else {
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
enum { FX_RAW = 0, FX_U01 = 1, FX_POW2 = 2, FX_U01F = 3 };

template <int MODE>
__device__ __forceinline__ u64 fx_map(const FillPlan &p, u64 w) {
    if constexpr (MODE == FX_RAW) return w;
    else if constexpr (MODE == FX_POW2) return __umul64hi(w, p.ip[0]);
    else if constexpr (MODE == FX_U01) return bits(u01_of(w, p.fm));
    else {  // two f32 halves, low half first, packed as one 8-byte element
        u32 lo = __float_as_uint(u01f_of((u32)w, p.fm)), hi = __float_as_uint(u01f_of((u32)(w >> 32), p.fm));
        return (u64)lo | ((u64)hi << 32);
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
    if constexpr (MODE != FX_U01F) {
        u64 *out = (u64 *)p.out;
        if (t == 0 && last > p.n) last = p.n;  // n < P: prefix only
        write_run<E, MODE>(p, s, out, first, last, tile, active);
    } else {
        float *out = (float *)p.out;
        u64 halves = p.n - p.pending_used;  // halves to emit
        if (t == 0 && p.pending_used) out[0] = u01f_of(p.pending_val, p.fm);
        u64 full_words = halves / 2;        // words whose both halves are emitted
        u64 lim = last < full_words ? last : full_words;
        float *o2 = out + p.pending_used;
        if ((((uintptr_t)o2) & 7) == 0) {  // warp-uniform: the whole grid shares o2
            write_run<E, MODE>(p, s, (u64 *)o2, first, lim > first ? lim : first, tile, active);
        } else if (active) {
            for (u64 i = first; i < lim; i++) {
                u64 w = s.next();
                o2[2 * i] = u01f_of((u32)w, p.fm);
                o2[2 * i + 1] = u01f_of((u32)(w >> 32), p.fm);
            }
        }
        if (active && (halves & 1) && full_words >= first && full_words < last) {  // trailing low half
            u64 w = 0;
            for (u64 i = lim; i <= full_words; i++) w = s.next();
            o2[2 * full_words] = u01f_of((u32)w, p.fm);
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
        if constexpr (MODE == FX_U01F) {
            float *out = (float *)p.out;
            if (p.pending_used) out[0] = u01f_of(p.pending_val, p.fm);
            for (int i = 0; i < p.P; i++) {
                u64 f = (u64)p.pending_used + 2ULL * i;
                if (f < p.n) out[f] = u01f_of((u32)p.prefix[i], p.fm);
                if (f + 1 < p.n) out[f + 1] = u01f_of((u32)(p.prefix[i] >> 32), p.fm);
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
            if constexpr (MODE == FX_U01F) {
                u64 f = (u64)p.pending_used + 2ULL * ((u64)p.P + 4 * bb);  // first f32 index of this block
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

// ----------------------------------------------------------------------------- serial (sfc64 single stream)
// sfc64 has no skip-ahead (rng.py:162-163): a single stream is parsed by one
// thread; per-stream mode (k_streams) is the parallel path for sfc64. The
// thread also rebuilds the reference's post-fill WordBuffer: it snapshots the
// engine at every 144-word refill boundary and replays the last refill.
struct SerialSrc {
    EngSfc e, snap;
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

template <int D>
__global__ void k_serial(const __grid_constant__ FillPlan p, DevResult *res) {
    __shared__ ZigFast sm[256];
    stage_tables(p, sm);
    if (threadIdx.x != 0) return;
    SerialSrc s;
    make_engine<RS_ENG_SFC64>(p, 0, s.e);
    s.snap = s.e;
    s.pre = p.prefix;
    s.npre = p.P;
    s.eng = 0;
    s.pos = 0;
    Tally tl = {0, 0, 0, 0, 0};
    if constexpr (D == 2) {  // u01f from halves, low half first
        float *out = (float *)p.out;
        u64 i = 0;
        if (p.pending_used) out[i++] = u01f_of(p.pending_val, p.fm);
        while (i < p.n) {
            u64 w = s.next();
            out[i++] = u01f_of((u32)w, p.fm);
            if (i < p.n) out[i++] = u01f_of((u32)(w >> 32), p.fm);
        }
    } else if constexpr (D == 0 || D == 1) {  // raw or power-of-two bound / u01
        u64 *out = (u64 *)p.out;
        for (u64 i = 0; i < p.n; i++) {
            u64 w = s.next();
            out[i] = D == 0 ? (p.ip[0] ? __umul64hi(w, p.ip[0]) : w) : bits(u01_of(w, p.fm));
        }
    } else {
        constexpr int DD = D - 10;
        typename DistOf<DD>::type d;
        make_dist<DD>(p, sm, d);
        typedef typename DistOf<DD>::type::out_t T;
        T *out = (T *)p.out;
        for (u64 i = 0; i < p.n; i++) out[i] = d.sample(s, tl);
    }
    res->end_pos = s.pos;
    res->tally[0] = tl.norm_att; res->tally[1] = tl.norm_pdf; res->tally[2] = tl.exp_att;
    res->tally[3] = tl.exp_pdf; res->tally[4] = tl.gamma_att; res->tally[5] = 0;
    res->serial_consumed = s.eng;
    EngSfc f = s.snap;
    if (s.eng > 0)
        for (int i = 0; i < CAP; i++) res->serial_buf[i] = f.next();
    res->serial_state[0] = f.a; res->serial_state[1] = f.b;
    res->serial_state[2] = f.c; res->serial_state[3] = f.w;
}

// ----------------------------------------------------------------------------- per-stream mode
// SeedSequenceFE128 on the device (seeding.py:48-116): stream j's state from
// entropy (ip words in `seedw`) + spawn key prefix + (j0 + j).
struct StreamArgs {
    int engine, nseed, nprefix, dist, fm;
    u64 seed[16];
    u64 prefix[8];
    u64 j0, nstreams, nper;
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    const RsZigSlow *zslow;
    const ZigFast *zfast;
    const u64 *rlx_A;
    void *out;
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
    } else {  // x256
        seed_fe128(a, a.j0 + j, w, 4);
        if (!(w[0] | w[1] | w[2] | w[3])) w[0] = 1;
        e.s0 = w[0]; e.s1 = w[1]; e.s2 = w[2]; e.s3 = w[3];
    }
    typedef typename DistOf<D>::type DT;
    DT d;
    make_dist_f<D>(a.fp, a.ip, a.ga, a.gb, 0, a.zslow, a.fm, sm, d);
    typedef typename DT::out_t T;
    VecWriter8<T> wr;
    wr.init((T *)a.out, j * a.nper);
    Tally tl;
    if constexpr (D == RS_DIST_UINT64) {
        for (u64 i = 0; i < a.nper;) {
            u64 o;
            if (d.accept(e.next(), o)) { wr.put(o); i++; }
        }
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
    u64 *rlxA = nullptr;
    // scratch
    size_t cap_T = 0;
    u64 *states = nullptr, *cnt0 = nullptr, *cnt = nullptr, *off = nullptr;
    u32 *ex0 = nullptr, *exA = nullptr, *exB = nullptr, *entry = nullptr;
    void *cub_tmp = nullptr;
    size_t cub_bytes = 0;
    DevResult *res = nullptr;
    DevResult *res_host = nullptr;
    std::map<std::pair<u64, int>, u64 *> x256_ml;  // (L, levels) -> matrices
    void *stage = nullptr;
    size_t stage_bytes = 0;
    cublasHandle_t blas = nullptr;
    double *mvn_z = nullptr;
    size_t mvn_bytes = 0;
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
    cudaFree(c.states); cudaFree(c.cnt0); cudaFree(c.cnt); cudaFree(c.off);
    cudaFree(c.ex0); cudaFree(c.exA); cudaFree(c.exB); cudaFree(c.entry); cudaFree(c.cub_tmp);
    CK(cudaMalloc(&c.states, nT * 32));
    CK(cudaMalloc(&c.cnt0, nT * 8));
    CK(cudaMalloc(&c.cnt, nT * 8));
    CK(cudaMalloc(&c.off, nT * 8));
    CK(cudaMalloc(&c.ex0, nT * 4));
    CK(cudaMalloc(&c.exA, nT * 4));
    CK(cudaMalloc(&c.exB, nT * 4));
    CK(cudaMalloc(&c.entry, nT * 4));
    c.cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c.cub_bytes, c.cnt, c.off, (int)nT);
    CK(cudaMalloc(&c.cub_tmp, c.cub_bytes));
    c.cap_T = nT;
    return RS_OK;
}

// x256: ML[0] = T^L, ML[1 + k] = T^(32 L 2^k) for k < levels; cached per (L, levels) on the device
rs_status x256_mats(DevCtx &c, u64 L, int levels, u64 **out) {
    auto key = std::make_pair(L, levels);
    auto it = c.x256_ml.find(key);
    if (it != c.x256_ml.end()) { *out = it->second; return RS_OK; }
    std::vector<rs::Mat256> m(1 + levels);
    bool init = false;
    for (int k = 0; k < 64; k++)
        if ((L >> k) & 1) {
            if (!init) { m[0] = rs::x256_pow2(k); init = true; }
            else rs::mat_mul(rs::x256_pow2(k), m[0], m[0]);
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

size_t elem_size(int dist) { return dist == RS_DIST_U01F ? 4 : 8; }

// ---- dispatch tables
typedef void (*KCount)(FillPlan, u64 *, u32 *);
typedef void (*KFixup)(FillPlan, const u64 *, const u32 *, const u32 *, u32 *, u64 *, u32 *, int, DevResult *);
typedef void (*KEmit)(FillPlan, const u32 *, const u64 *, const u64 *, const u32 *, DevResult *);
typedef void (*KFixed)(FillPlan);

struct VarKernels {
    const void *count, *fixup, *emit;
};

template <int E, int D>
VarKernels var_kernels_ed() {
    return VarKernels{(const void *)k_count<E, D>, (const void *)k_fixup<E, D>, (const void *)k_emit<E, D>};
}
template <int E>
VarKernels var_kernels_e(int d) {
    switch (d) {
    case RS_DIST_NORM: return var_kernels_ed<E, RS_DIST_NORM>();
    case RS_DIST_EXP: return var_kernels_ed<E, RS_DIST_EXP>();
    case RS_DIST_GAMMA: return var_kernels_ed<E, RS_DIST_GAMMA>();
    case RS_DIST_BETA: return var_kernels_ed<E, RS_DIST_BETA>();
    default: return var_kernels_ed<E, RS_DIST_UINT64>();
    }
}
VarKernels var_kernels(int e, int d) {
    switch (e) {
    case RS_ENG_X256SS: return var_kernels_e<RS_ENG_X256SS>(d);
    case RS_ENG_X256PP: return var_kernels_e<RS_ENG_X256PP>(d);
    case RS_ENG_PCG64: return var_kernels_e<RS_ENG_PCG64>(d);
    case RS_ENG_PHILOX: return var_kernels_e<RS_ENG_PHILOX>(d);
    default: return var_kernels_e<RS_ENG_RANLUX>(d);
    }
}
template <int E>
const void *fixed_kernel_e(int mode) {
    switch (mode) {
    case FX_RAW: return (const void *)k_fixed<E, FX_RAW>;
    case FX_U01: return (const void *)k_fixed<E, FX_U01>;
    case FX_POW2: return (const void *)k_fixed<E, FX_POW2>;
    default: return (const void *)k_fixed<E, FX_U01F>;
    }
}
const void *fixed_kernel(int e, int mode) {
    switch (e) {
    case RS_ENG_X256SS: return fixed_kernel_e<RS_ENG_X256SS>(mode);
    case RS_ENG_X256PP: return fixed_kernel_e<RS_ENG_X256PP>(mode);
    case RS_ENG_PCG64: return fixed_kernel_e<RS_ENG_PCG64>(mode);
    case RS_ENG_PHILOX: return fixed_kernel_e<RS_ENG_PHILOX>(mode);
    default: return fixed_kernel_e<RS_ENG_RANLUX>(mode);
    }
}
const void *philox_kernel(int mode) {
    static int variant = getenv("RS_PHILOX_VARIANT") ? atoi(getenv("RS_PHILOX_VARIANT")) : 0;
    if (variant == 1) {
        switch (mode) {
        case FX_RAW: return (const void *)k_philox_fixed<FX_RAW, 1>;
        case FX_U01: return (const void *)k_philox_fixed<FX_U01, 1>;
        case FX_POW2: return (const void *)k_philox_fixed<FX_POW2, 1>;
        default: return (const void *)k_philox_fixed<FX_U01F, 1>;
        }
    }
    switch (mode) {
    case FX_RAW: return (const void *)k_philox_fixed<FX_RAW>;
    case FX_U01: return (const void *)k_philox_fixed<FX_U01>;
    case FX_POW2: return (const void *)k_philox_fixed<FX_POW2>;
    default: return (const void *)k_philox_fixed<FX_U01F>;
    }
}
const void *serial_kernel(int d, int fixed_mode) {
    if (fixed_mode == FX_RAW || fixed_mode == FX_POW2) return (const void *)k_serial<0>;
    if (fixed_mode == FX_U01) return (const void *)k_serial<1>;
    if (fixed_mode == FX_U01F) return (const void *)k_serial<2>;
    switch (d) {
    case RS_DIST_NORM: return (const void *)k_serial<10 + RS_DIST_NORM>;
    case RS_DIST_EXP: return (const void *)k_serial<10 + RS_DIST_EXP>;
    case RS_DIST_GAMMA: return (const void *)k_serial<10 + RS_DIST_GAMMA>;
    case RS_DIST_BETA: return (const void *)k_serial<10 + RS_DIST_BETA>;
    default: return (const void *)k_serial<10 + RS_DIST_UINT64>;
    }
}

rs_status launch(const void *fn, dim3 g, dim3 b, void **args, cudaStream_t st) {
    CK(cudaLaunchKernel(fn, g, b, args, 0, st));
    return RS_OK;
}

// ---- parameter resolution (validated values)
struct Resolved {
    int dist;          // RS_DIST_*
    int fixed_mode;    // FX_* or -1 for variable
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int raw_norm;
    double words_per_sample;
    int table;         // 0 normal tables, 1 exp tables, -1 none
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

rs_status resolve(int dist, const double *fp, const u64 *ip, Resolved &r) {
    memset(&r, 0, sizeof r);
    r.dist = dist;
    r.fixed_mode = -1;
    r.table = -1;
    r.words_per_sample = 1.0;
    switch (dist) {
    case RS_DIST_UINT64: {
        u64 b = ip ? ip[0] : 0;
        bool b64 = ip && ip[1];
        if (b == 0 || b64) { r.fixed_mode = FX_RAW; }
        else if ((b & (b - 1)) == 0) { r.fixed_mode = FX_POW2; r.ip[0] = b; }
        else {
            r.ip[0] = b;
            r.ip[1] = (0 - b) % b;  // discrete.py:34
            r.words_per_sample = 1.0 / (1.0 - (double)r.ip[1] * 5.421010862427522e-20);
        }
        return RS_OK;
    }
    case RS_DIST_U01: r.fixed_mode = FX_U01; return RS_OK;
    case RS_DIST_U01F: r.fixed_mode = FX_U01F; return RS_OK;
    case RS_DIST_NORM: case RS_DIST_STDNORM:
        r.dist = RS_DIST_NORM;
        r.table = 0;
        r.words_per_sample = 1.03;
        if (dist == RS_DIST_STDNORM) { r.raw_norm = 1; return RS_OK; }
        if (!(fp[1] >= 0.0)) { rs::set_error("normal variance must be >= 0"); return RS_ERR_VALUE; }
        r.fp[0] = fp[0];
        r.fp[1] = std::sqrt(fp[1]);
        return RS_OK;
    case RS_DIST_EXP:
        if (!(fp[0] > 0.0)) { rs::set_error("exponential scale must be > 0"); return RS_ERR_VALUE; }
        r.table = 1;
        r.fp[0] = fp[0];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_GAMMA:
        if (!(fp[0] > 0.0)) { rs::set_error("gamma shape must be > 0"); return RS_ERR_VALUE; }
        if (!(fp[1] > 0.0)) { rs::set_error("gamma scale must be > 0"); return RS_ERR_VALUE; }
        r.table = 0;
        r.ga = gamma_prm(fp[0], fp[1]);
        r.words_per_sample = 2.2 + (r.ga.boost ? 1.0 : 0.0);
        return RS_OK;
    case RS_DIST_BETA:
        if (!(fp[0] > 0.0) || !(fp[1] > 0.0)) { rs::set_error("gamma shape must be > 0"); return RS_ERR_VALUE; }
        r.table = 0;
        r.ga = gamma_prm(fp[0], 1.0);
        r.gb = gamma_prm(fp[1], 1.0);
        r.words_per_sample = 4.4 + (r.ga.boost ? 1.0 : 0.0) + (r.gb.boost ? 1.0 : 0.0);
        return RS_OK;
    }
    rs::set_error("unknown distribution id");
    return RS_ERR_VALUE;
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
    p.zslow = r.table >= 0 ? c.zslow[r.table] : nullptr;
    p.zfast = r.table >= 0 ? c.zfast[r.table] : nullptr;
    p.rlx_A = c.rlxA;
}

// Segment geometry + per-engine jump tables for stride L (engine origin = p.base)
rs_status plan_segments(DevCtx &c, FillPlan &p, u64 words, u64 Lmin, int occ, cudaStream_t st) {
    // exactly one wave of resident threads: equal segments finish together
    u64 Tfull = (u64)c.sms * (u64)occ * BLOCK;
    u64 L = (words + Tfull - 1) / Tfull;
    if (L < Lmin) L = Lmin;
    L = (L + 35) / 36 * 36;  // a whole number of philox blocks and ranlux chunks
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
    } else if (p.engine == RS_ENG_X256SS || p.engine == RS_ENG_X256PP) {
        int lv = 0;  // bits of the warp index
        while ((1ULL << lv) < T / 32) lv++;
        u64 *ml;
        s = x256_mats(c, L, lv, &ml);
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
    if (s->engine == RS_ENG_SFC64) {  // rebuilt on the device by k_serial
        if (!sr || sr->serial_consumed != ep) {
            rs::set_error("serial fill bookkeeping mismatch");
            return RS_ERR_INTERNAL;
        }
        memcpy(s->state, sr->serial_state, 32);
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

// The device part of one fill. On return (sync=true) `E` holds the logical words
// consumed and `tal` the tallies.
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
    rs_status rc;

    if (s->engine == RS_ENG_SFC64) {  // single stream: serial
        p.n = n;
        p.pending_used = s->has_pending && r.dist == RS_DIST_U01F;
        p.pending_val = (u32)s->pending;
        if (r.fixed_mode == FX_POW2) p.ip[0] = r.ip[0];
        else if (r.fixed_mode == FX_RAW) p.ip[0] = 0;
        DevResult *res = c.res;
        void *args[] = {&p, &res};
        rc = launch(serial_kernel(r.dist, r.fixed_mode), dim3(1), dim3(32), args, st);
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
        // fixed consumption: sample i <- logical word i (u01f: half i)
        u64 words;
        if (r.fixed_mode == FX_U01F) {
            p.pending_used = s->has_pending ? 1 : 0;
            p.pending_val = (u32)s->pending;
            u64 halves = n - p.pending_used;
            words = (halves + 1) / 2;
        } else {
            words = n;
        }
        p.n = n;
        p.weng = words > (u64)p.P ? words - p.P : 0;
        if (r.fixed_mode == FX_POW2) p.ip[0] = r.ip[0];
        if (s->engine == RS_ENG_PHILOX) {
            const void *fn = philox_kernel(r.fixed_mode);
            // round keys k + r*W (counter.py:95-96) live in the constant bank
            for (int i = 0; i < 10; i++) {
                p.rk0[i] = p.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
                p.rk1[i] = p.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
            }
            uintptr_t a = (uintptr_t)dout;
            if (r.fixed_mode == FX_U01F)
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
            E = words;
            chunks = 1;
            return RS_OK;
        }
        const void *fn = fixed_kernel(s->engine, r.fixed_mode);
        rc = plan_segments(c, p, p.weng ? p.weng : 1, 64, occupancy(fn), st);
        if (rc) return rc;
        void *args[] = {&p};
        rc = launch(fn, dim3(p.T / BLOCK), dim3(BLOCK), args, st);
        if (rc) return rc;
        E = words;
        chunks = 1;
        return RS_OK;
    }

    // variable consumption: chunks of provisioned words until n samples exist.
    // Chunk coordinates: chunk-local logical position lp; chunk 1 starts with the
    // P buffered words (lp < P) then engine word lp - P; a later chunk has no
    // prefix and lp = engine word (origin + lp), with thread 0 starting at lp0.
    VarKernels K = var_kernels(s->engine, r.dist);
    const u64 P1 = (u64)p.P;
    u64 done = 0;    // samples produced so far
    u64 origin = 0;  // engine words from s->state to this chunk's origin (multiple of 36)
    u64 lp0 = 0;
    u64 Lmin = r.dist == RS_DIST_BETA ? 2048 : r.dist == RS_DIST_GAMMA ? 1024 : 128;
    bool first = true;
    while (done < n) {
        u64 need = n - done;
        double ww = (double)need * r.words_per_sample;
        u64 words = (u64)(ww * 1.01 + 12.0 * std::sqrt(ww) + 2048.0);
        if (!first) {
            p.P = 0;
            memcpy(p.base, s->state, sizeof p.base);
            if (!rs::engine_advance_words(s->engine, p.base, (u128)origin)) {
                rs::set_error("cannot position engine");
                return RS_ERR_INTERNAL;
            }
        }
        p.lp0 = lp0;
        p.n = need;
        p.out0 = done;
        int occ = std::min(occupancy(K.count), std::min(occupancy(K.fixup), occupancy(K.emit)));
        rc = plan_segments(c, p, words + lp0, Lmin, occ, st);
        if (rc) return rc;
        CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
        unsigned g = p.T / BLOCK;
        int round = 0;
        DevResult *res = c.res;
        {
            void *a1[] = {&p, &c.cnt0, &c.ex0};
            if ((rc = launch(K.count, dim3(g), dim3(BLOCK), a1, st))) return rc;
            const u32 *prev = c.ex0;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &prev, &c.entry, &c.cnt, &c.exA, &round, &res};
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
            if (++round > 64) { rs::set_error("segment entry resolution did not converge"); return RS_ERR_INTERNAL; }
            rounds++;
            CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
            const u32 *prev = ex_cur;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &prev, &c.entry, &c.cnt, &ex_other, &round, &res};
            if ((rc = launch(K.fixup, dim3(g), dim3(BLOCK), a2, st))) return rc;
            u32 *tmp = ex_cur; ex_cur = ex_other; ex_other = tmp;
        }
        chunks++;
        for (int i = 0; i < 6; i++) tal[i] += c.res_host->tally[i];
        u64 total = c.res_host->total;
        // chunk-local logical -> whole-fill logical / engine offset
        u64 to_engine = first ? (u64)0 - P1 : origin;  // engine word = lp + to_engine
        if (done + total >= n) {
            E = P1 + (c.res_host->end_pos + to_engine);
            break;
        }
        done += total;
        u64 resume = c.res_host->next_start + to_engine;  // engine word of the next boundary
        origin = resume / 36 * 36;
        lp0 = resume - origin;
        first = false;
    }
    return RS_OK;
}

void tally_seen(int dist, int32_t *seen) {
    seen[0] = seen[1] = seen[2] = 0;
    if (dist == RS_DIST_NORM || dist == RS_DIST_STDNORM) seen[0] = 1;
    if (dist == RS_DIST_EXP) seen[1] = 1;
    if (dist == RS_DIST_GAMMA || dist == RS_DIST_BETA) { seen[0] = 1; seen[2] = 1; }
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
    u64 E, tal[6];
    int rounds;
    u64 chunks;
    if ((rc = run_fill(*c, s, r, n, sg.dptr, st, true, E, tal, rounds, chunks))) return rc;
    if (sg.host) {
        CK(cudaMemcpyAsync(out, sg.dptr, bytes, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    // stream position after the fill (buffer.py:29-49)
    int P = s->fill - s->cursor;
    u64 pre_words[CAP];
    for (int i = 0; i < P; i++) pre_words[i] = s->buf[s->cursor + i];
    int had_pending = s->has_pending;
    if ((rc = apply_consumption(s, E, s->engine == RS_ENG_SFC64 ? c->res_host : nullptr))) return rc;
    if (dist == RS_DIST_U01F) {
        u64 halves = n - (had_pending ? 1 : 0);
        if (halves & 1) {
            u64 last = E - 1;
            u64 w = last < (u64)P ? pre_words[last] : s->buf[s->cursor - 1];
            s->has_pending = 1;
            s->pending = w >> 32;
        } else {
            s->has_pending = 0;
            s->pending = 0;
        }
    } else {
        s->has_pending = 0;
        s->pending = 0;
    }
    if (result) {
        result->words_consumed = E;
        for (int i = 0; i < 6; i++) result->tally[i] = tal[i];
        tally_seen(dist, result->tally_seen);
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
        engine != RS_ENG_X256PP) {
        rs::set_error("per-stream mode supports sfc64, pcg64, philox, x256**, x256++");
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
    if (dist == RS_DIST_U01F) { rs::set_error("u01f is not available in per-stream mode"); return RS_ERR_UNSUPPORTED; }
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
    size_t bytes = (size_t)n_streams * n_per_stream * 8;
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
    a.zslow = r.table >= 0 ? c->zslow[r.table] : nullptr;
    a.zfast = r.table >= 0 ? c->zfast[r.table] : nullptr;
    a.rlx_A = c->rlxA;
    a.out = sg.dptr;
    int d = r.dist;
    if (r.fixed_mode == FX_RAW || r.fixed_mode == FX_POW2) {  // Lemire with thr = 0
        d = RS_DIST_UINT64;
        a.ip[0] = r.fixed_mode == FX_RAW ? 0 : r.ip[0];
        a.ip[1] = 0;
    }
    if (r.fixed_mode == FX_U01 || (d == RS_DIST_UINT64 && a.ip[0] == 0)) {
        rs::set_error("per-stream mode covers bounded integers (b > 0) and the continuous samplers");
        return RS_ERR_UNSUPPORTED;
    }
    const void *fn = nullptr;
#define RS_STREAM_CASE(E)                                                     \
    switch (d) {                                                              \
    case RS_DIST_NORM: fn = (const void *)k_streams<E, RS_DIST_NORM>; break;  \
    case RS_DIST_EXP: fn = (const void *)k_streams<E, RS_DIST_EXP>; break;    \
    case RS_DIST_GAMMA: fn = (const void *)k_streams<E, RS_DIST_GAMMA>; break; \
    case RS_DIST_BETA: fn = (const void *)k_streams<E, RS_DIST_BETA>; break;  \
    default: fn = (const void *)k_streams<E, RS_DIST_UINT64>; break;          \
    }
    if (engine == RS_ENG_SFC64) { RS_STREAM_CASE(RS_ENG_SFC64) }
    else if (engine == RS_ENG_PCG64) { RS_STREAM_CASE(RS_ENG_PCG64) }
    else if (engine == RS_ENG_PHILOX) { RS_STREAM_CASE(RS_ENG_PHILOX) }
    else if (engine == RS_ENG_X256SS) { RS_STREAM_CASE(RS_ENG_X256SS) }
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
