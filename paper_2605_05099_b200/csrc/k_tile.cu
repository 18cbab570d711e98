// Warp-tile parse for the counter / affine engines (Philox-4x64-10, PCG64-DXSM) and the
// one-word-token laws (ziggurat normal and exponential with their word-level transforms,
// Lemire bounded integers): continuous.py:40-93, :157-169, :176-177, :252-274;
// discrete.py:20-39.
//
// These engines reach any word directly (counter + w/4; the LCG state A^w s0), so the
// stream is cut into warp-tiles of WT_WORDS = 512 consecutive words. Lane l of a warp owns
// the window of WT_W = 16 words at raw word 512 w + 16 l. Every warp-tile is processed
// independently -- no pass waits on another warp -- in four launches:
//
//  1. k_wt_count: each lane parses its window as if a token started at its first word and
//     records which words start tokens (S0) and which token starts emitted a sample (E0),
//     plus its exit (units past the window where its last token ends). Lane l's true entry
//     is lane l-1's exit; from an entry in S0 the parse coincides with the speculative one
//     (same exit, count = emits from the entry on). Only an entry inside a token (the second
//     word of a slow token, a tail pair: ~2 % of words for the normal) re-parses from the
//     entry, and meets the speculative parse within a token or two. Rounds
//     of shuffles repeat until no exit changes. The warp-tile's (exit, count) is tabulated
//     for entries 0..7 (WTTab); warp-tile 0 is a constant: the stream starts at `skip`.
//  2. k_wt_scan1: in blocks of 1024 warp-tiles, an inclusive scan of the tables (composition:
//     (a then b)(e) = b(a(e).exit), counts added) -> each warp-tile's exclusive in-block
//     prefix and each block's table.
//  3. k_wt_scan2: the block tables chained from the start -> each block's exact (entry,
//     sample offset).
//  4. k_wt_emit: each warp-tile, from its exact entry and offset, parses its windows once
//     with the samples' values going to per-lane rows in shared memory, resolves the lanes'
//     entries as in 1, copies the rows to the warp's run in shared memory and writes it with
//     one TMA bulk copy (cp.async.bulk global.shared::cta) plus at most two element stores
//     at unaligned ends. The lane holding sample n-1 reports the position after it; the
//     tallies (attempts, pdf evaluations) count the tokens that start before it, from the
//     masks, as the reference's counters do.
// An entry outside 0..7 where a table is needed (a tail token running 8+ words into the next
// warp-tile: ~1e-7 per boundary) sets a flag and the host redoes the fill on the two-pass
// path; so does a provisioning shortfall.
#include "rs_kernels.cuh"

namespace {

constexpr u32 FULL = 0xFFFFFFFFu;

// ---- engine word sources positioned at a lane window (raw word 0 = the rewound base)
template <int E, bool FOLD>
struct TSrc;

template <bool FOLD>
struct TSrc<RS_ENG_PCG64, FOLD> {
    EngPcg e;
    __device__ __forceinline__ void at(const WTPlan &p, const PhiloxFold &, u64 wt, u32 lane) {
        e.slo = __ldg(p.pcg_wt + 2 * wt);
        e.shi = __ldg(p.pcg_wt + 2 * wt + 1);
        e.ilo = p.base[2];
        e.ihi = p.base[3];
        const u64 *m = p.pcg_lane + 4 * lane;
        e.affine(__ldg(m), __ldg(m + 1), __ldg(m + 2), __ldg(m + 3));
    }
    __device__ __forceinline__ u64 next() { return e.next(); }
};

template <bool FOLD>
struct TSrc<RS_ENG_PHILOX, FOLD> {
    u64 blk;          // next block (from the rewound counter)
    u64 b1, b2, b3;   // rest of the current block
    int left;
    const WTPlan *pp;
    PhiloxFold f;
    __device__ __forceinline__ void at(const WTPlan &p, const PhiloxFold &fo, u64 wt, u32 lane) {
        pp = &p;
        f = fo;
        blk = (wt * WT_WORDS + (u64)WT_W * lane) / 4;
        left = 0;
    }
    __device__ __forceinline__ u64 next() {
        if (left == 0) {
            u64 o0;
            if constexpr (FOLD) {
                philox4x64_10_folded(pp->base[0] + blk, f, pp->rk0, pp->rk1, o0, b1, b2, b3);
            } else {
                u64 c0 = pp->base[0] + blk, c1 = pp->base[1], c2 = pp->base[2], c3 = pp->base[3];
                if (c0 < blk) { if (++c1 == 0) { if (++c2 == 0) ++c3; } }
                philox4x64_10_rk(c0, c1, c2, c3, pp->rk0, pp->rk1, o0, b1, b2, b3);
            }
            blk++;
            left = 3;
            return o0;
        }
        const u64 r = b1;
        b1 = b2;
        b2 = b3;
        left--;
        return r;
    }
};

__device__ __forceinline__ u32 above(u32 mask, u32 e) { return e >= 32 ? 0u : mask & ~((1u << e) - 1u); }

// One lane's window parsed from entry e (a token starts at window word e): the token-start,
// emit and density-evaluation masks and the exit; with VALUES, the samples (finished) go
// to `row`. `src` is positioned at window word e.
template <int D, bool VALUES, class DT, class S>
__device__ __forceinline__ void parse_window(const DT &d, S &src, u32 e, double *row, u32 &S0, u32 &E0, u32 &PD,
                                             u32 &x0) {
    S0 = E0 = PD = x0 = 0;
    u32 k = 0;
    if constexpr (D == FAM_LEMIRE) {
        for (u32 i = e; i < (u32)WT_W; i++) {
            u64 o;
            S0 |= 1u << i;
            if (d.accept(src.next(), o)) {
                E0 |= 1u << i;
                if constexpr (VALUES) ((u64 *)row)[k++] = o;
            }
        }
    } else {
        ZigWM m;
        m.st = 0;
        u32 ts = 0;
        for (u32 i = e; i < (u32)WT_W; i++) {
            const u64 w = src.next();
            if (m.st == 0) {
                S0 |= 1u << i;
                ts = i;
            }
            Tally t1 = {0, 0, 0, 0, 0};
            double z;
            const bool em = d.feed(m, w, d.strip(w), t1, z);
            if (t1.norm_pdf | t1.exp_pdf) PD |= 1u << ts;
            if (em) {
                E0 |= 1u << ts;
                if constexpr (VALUES) row[k++] = d.finish(z);
            }
        }
        while (m.st != 0) {  // the last token runs past the window
            Tally t1 = {0, 0, 0, 0, 0};
            double z;
            x0++;
            const bool em = d.feed(m, src.next(), t1, z);
            if (t1.norm_pdf | t1.exp_pdf) PD |= 1u << ts;
            if (em) {
                E0 |= 1u << ts;
                if constexpr (VALUES) row[k++] = d.finish(z);
            }
        }
    }
}

// The rare path (an entry inside a token of the speculative parse): the window re-parsed
// from entry e with regenerated words. Out of line, so the common path stays small.
template <int D, bool VALUES, class DT, class S>
__device__ __noinline__ void reparse_window(const DT &d, const S &src0, u32 e, double *row, u32 &S0, u32 &E0, u32 &PD,
                                            u32 &x0) {
    S s = src0;
    for (u32 i = 0; i < e; i++) s.next();
    parse_window<D, VALUES>(d, s, e, row, S0, E0, PD, x0);
}

// ---- tables: (exit, count) for entries 0..7
__device__ __forceinline__ u32 tx(const u32 (&x)[2], u32 e) { return (x[e >> 2] >> (8 * (e & 3))) & 0xFFu; }
__device__ __forceinline__ void set_tx(u32 (&x)[2], u32 e, u32 v) {
    x[e >> 2] = (x[e >> 2] & ~(0xFFu << (8 * (e & 3)))) | ((v > 0xFEu ? 0xFFu : v) << (8 * (e & 3)));
}
struct Tab {
    u32 x[2];
    u32 c[WT_D];
};
__device__ __forceinline__ Tab tab_identity() {
    Tab t;
    t.x[0] = 0x03020100u;
    t.x[1] = 0x07060504u;
#pragma unroll
    for (int e = 0; e < WT_D; e++) t.c[e] = 0;
    return t;
}
__device__ __forceinline__ Tab tab_then(const Tab &a, const Tab &b) {  // a, then b
    Tab r;
    r.x[0] = r.x[1] = 0;
#pragma unroll
    for (u32 e = 0; e < (u32)WT_D; e++) {
        const u32 xa = tx(a.x, e);
        u32 xr = 0xFFu, cr = 0;
        if (xa < (u32)WT_D) {
            xr = tx(b.x, xa);
            cr = a.c[e] + b.c[xa];
        }
        set_tx(r.x, e, xr);
        r.c[e] = cr;
    }
    return r;
}

template <class DT, int D>
__device__ __forceinline__ void make_tile_dist(const WTPlan &p, const ZigFast *sm, DT &d) {
    GammaPrm g{};
    DistArgs a{p.fp, p.ip, &g, &g, p.kind, p.fm, p.zslow, nullptr};
    make_dist_a<D>(a, sm, d);
}

// ----------------------------------------------------------------------------- 1. count
template <int E, int D, bool FOLD>
__global__ void __launch_bounds__(256, 2) k_wt_count(const __grid_constant__ WTPlan p) {
    typedef typename DistOf<D>::type DT;
    __shared__ ZigFast sm[256];
    if constexpr (D != FAM_LEMIRE) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = p.zfast[i];
    }
    __syncthreads();
    DT d;
    make_tile_dist<DT, D>(p, sm, d);
    PhiloxFold fold{};
    if constexpr (E == RS_ENG_PHILOX && FOLD) fold = philox_fold(p.base[1], p.base[2], p.base[3], p.rk0, p.rk1);
    const u32 lane = threadIdx.x & 31;
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 wt = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wt < p.nwt; wt += nw) {
        TSrc<E, FOLD> src0;
        src0.at(p, fold, wt, lane);
        u32 S0, E0, PD, x0;
        {
            TSrc<E, FOLD> s = src0;
            parse_window<D, false>(d, s, 0, nullptr, S0, E0, PD, x0);
        }
        // this lane's (count, exit) from entry e
        auto f = [&](u32 e, u32 &c, u32 &x) {
            if (e >= (u32)WT_W) { c = 0; x = e - WT_W; return; }
            if ((S0 >> e) & 1) { c = __popc(above(E0, e)); x = x0; return; }
            u32 a, b2, pd, xx;  // inside a token of the speculative parse: parse from e
            reparse_window<D, false>(d, src0, e, nullptr, a, b2, pd, xx);
            c = __popc(b2);
            x = xx;
        };
        // the warp-tile's (count, exit) with lane 0 entering at e0; also this lane's (c, x)
        u32 lc = 0, lx = 0;
        auto resolve = [&](u32 e0, u32 &C, u32 &X) {
            u32 e = __shfl_up_sync(FULL, x0, 1);
            if (lane == 0) e = e0;
            for (;;) {
                f(e, lc, lx);
                u32 ne = __shfl_up_sync(FULL, lx, 1);
                if (lane == 0) ne = e0;
                if (!__any_sync(FULL, ne != e)) break;
                e = ne;
            }
            u32 s = lc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            C = s;
            X = __shfl_sync(FULL, lx, 31);
        };
        u32 tx2[2] = {0, 0};
        u32 cp[4] = {0, 0, 0, 0};  // counts as u16 pairs (a warp-tile emits <= 512 samples)
        if (wt == 0) {  // the stream starts at raw word `skip`: a constant table
            u32 C, X;
            resolve((u32)p.skip, C, X);
#pragma unroll
            for (u32 e = 0; e < (u32)WT_D; e++) set_tx(tx2, e, X);
            cp[0] = cp[1] = cp[2] = cp[3] = C | (C << 16);
        } else {
            u32 C0, X0;
            resolve(0, C0, X0);
            const u32 c00 = __shfl_sync(FULL, lc, 0), x00 = __shfl_sync(FULL, lx, 0);
            set_tx(tx2, 0, X0);
            cp[0] = C0;
#pragma unroll 1
            for (u32 e = 1; e < (u32)WT_D; e++) {
                u32 ce = 0, xe = 0;
                if (lane == 0) f(e, ce, xe);
                ce = __shfl_sync(FULL, ce, 0);
                xe = __shfl_sync(FULL, xe, 0);
                u32 Ce, Xe;
                if (xe == x00) {  // lane 0 exits where it did from entry 0: the rest is unchanged
                    Ce = C0 - c00 + ce;
                    Xe = X0;
                } else {          // rare: lane 0's exit moved
                    resolve(e, Ce, Xe);
                }
                set_tx(tx2, e, Xe);
                const u32 sh = 16 * (e & 1);
                cp[e >> 1] = (cp[e >> 1] & ~(0xFFFFu << sh)) | (Ce << sh);
            }
        }
        if (lane == 0) {
            uint4 *t = (uint4 *)(p.tab + wt);
            t[0] = make_uint4(tx2[0], tx2[1], cp[0], cp[1]);
            t[1] = make_uint4(cp[2], cp[3], 0u, 0u);
        }
    }
}

// ----------------------------------------------------------------------------- 2. in-block scan
__device__ __forceinline__ Tab load_tab(const WTTab &w) {
    Tab t;
    t.x[0] = w.x[0];
    t.x[1] = w.x[1];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        t.c[2 * i] = w.c[i] & 0xFFFFu;
        t.c[2 * i + 1] = w.c[i] >> 16;
    }
    return t;
}
__device__ __forceinline__ void store_tab32(WTTab32 &w, const Tab &t) {
    w.x[0] = t.x[0];
    w.x[1] = t.x[1];
#pragma unroll
    for (int e = 0; e < WT_D; e++) w.c[e] = t.c[e];
}
__device__ __forceinline__ Tab load_tab32(const WTTab32 &w) {
    Tab t;
    t.x[0] = w.x[0];
    t.x[1] = w.x[1];
#pragma unroll
    for (int e = 0; e < WT_D; e++) t.c[e] = w.c[e];
    return t;
}

// block b of WT_BLK warp-tiles: pre[w] = tables of the block's warp-tiles before w (composed),
// blk[b] = all of them. Hillis-Steele in shared memory (dynamic: 2 x WT_BLK x sizeof(Tab)).
__global__ void __launch_bounds__(WT_BLK) k_wt_scan1(const __grid_constant__ WTPlan p) {
    extern __shared__ __align__(16) unsigned char sc_dyn[];
    Tab *A = (Tab *)sc_dyn, *B = A + WT_BLK;
    const u32 t = threadIdx.x;
    const u64 w = (u64)blockIdx.x * WT_BLK + t;
    A[t] = w < p.nwt ? load_tab(p.tab[w]) : tab_identity();
    __syncthreads();
    for (u32 s = 1; s < (u32)WT_BLK; s <<= 1) {
        Tab v = A[t];
        if (t >= s) v = tab_then(A[t - s], v);
        B[t] = v;
        __syncthreads();
        Tab *tmp = A; A = B; B = tmp;
    }
    // A[t]: inclusive prefix of warp-tiles 0..t of the block
    if (w < p.nwt) store_tab32(p.pre[w], t == 0 ? tab_identity() : A[t - 1]);
    if (t == WT_BLK - 1) store_tab32(p.blk[blockIdx.x], A[t]);
}

// the block tables chained from the start (the first block's table is constant in its
// entry): blk_in[b] = exact (entry, offset) entering block b; ctl[2..3] = total samples
__global__ void __launch_bounds__(WT_BLK) k_wt_scan2(const __grid_constant__ WTPlan p) {
    extern __shared__ __align__(16) unsigned char sc_dyn[];
    Tab *A = (Tab *)sc_dyn, *B = A + WT_BLK;
    __shared__ u32 s_e;
    __shared__ unsigned long long s_o;
    const u32 t = threadIdx.x;
    if (t == 0) { s_e = 0; s_o = 0; }
    __syncthreads();
    for (u32 c0 = 0; c0 < p.nblk; c0 += WT_BLK) {
        const u32 b = c0 + t;
        A[t] = b < p.nblk ? load_tab32(p.blk[b]) : tab_identity();
        __syncthreads();
        for (u32 s = 1; s < (u32)WT_BLK; s <<= 1) {
            Tab v = A[t];
            if (t >= s) v = tab_then(A[t - s], v);
            B[t] = v;
            __syncthreads();
            Tab *tmp = A; A = B; B = tmp;
        }
        const u32 e = s_e;
        const unsigned long long o = s_o;
        if (b < p.nblk) {
            u32 be = e;
            unsigned long long bo = o;
            if (t > 0) {
                const Tab &q = A[t - 1];
                if (e < (u32)WT_D && tx(q.x, e) != 0xFFu) {
                    be = tx(q.x, e);
                    bo = o + q.c[e];
                } else {
                    be = 0xFFFFFFFFu;
                    atomicOr(&p.ctl[0], 1u);
                }
            }
            p.blk_in[2 * b] = be;
            p.blk_in[2 * b + 1] = bo;
        }
        __syncthreads();
        if (t == WT_BLK - 1) {  // running entry / offset after this chunk
            const Tab &q = A[t];
            if (e < (u32)WT_D && tx(q.x, e) != 0xFFu) {
                s_e = tx(q.x, e);
                s_o = o + q.c[e];
            } else {
                s_e = 0xFFFFFFFFu;
                atomicOr(&p.ctl[0], 1u);
            }
        }
        __syncthreads();
    }
    if (t == 0) *(unsigned long long *)(p.ctl + 2) = s_o;
}

// ----------------------------------------------------------------------------- 4. emit
constexpr int WT_ROW = WT_W + 1;
constexpr size_t WT_WARP_SMEM = ((size_t)32 * WT_ROW + WT_WORDS + 2) * 8;  // rows + the warp's run

template <int E, int D, bool FOLD>
__global__ void __launch_bounds__(256, 2) k_wt_emit(const __grid_constant__ WTPlan p) {
    typedef typename DistOf<D>::type DT;
    extern __shared__ __align__(128) unsigned char wt_dyn[];
    __shared__ ZigFast sm[256];
    if constexpr (D != FAM_LEMIRE) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = p.zfast[i];
    }
    __syncthreads();
    DT d;
    make_tile_dist<DT, D>(p, sm, d);
    PhiloxFold fold{};
    if constexpr (E == RS_ENG_PHILOX && FOLD) fold = philox_fold(p.base[1], p.base[2], p.base[3], p.rk0, p.rk1);
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *const wbase = (double *)(wt_dyn + (size_t)warp * WT_WARP_SMEM);
    double *const sout = wbase;                                        // [WT_WORDS + 2] the run
    double *const row = wbase + WT_WORDS + 2 + (size_t)lane * WT_ROW;  // this lane's samples
    u64 att = 0, pdf = 0;
    bool bulk = false;  // lane 0: a bulk copy may still be reading sout
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 wt = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wt < p.nwt; wt += nw) {
        // exact entry and offset
        const u64 blk = wt / WT_BLK;
        const u32 eb = (u32)__ldg(p.blk_in + 2 * blk);
        const u64 ob = __ldg(p.blk_in + 2 * blk + 1);
        const WTTab32 &q = p.pre[wt];
        u32 qx[2] = {__ldg(&q.x[0]), __ldg(&q.x[1])};
        if (eb >= (u32)WT_D || tx(qx, eb) == 0xFFu) {
            if (lane == 0) atomicOr(&p.ctl[0], 1u);
            continue;
        }
        // warp-tile 0 starts the stream at `skip` (its table is the constant used by the others)
        const u32 E0in = wt == 0 ? (u32)p.skip : tx(qx, eb);
        const u64 O = wt == 0 ? 0 : ob + __ldg(&q.c[eb]);
        if (O >= p.n) continue;  // warp-uniform: the warp-tile is past the fill

        TSrc<E, FOLD> src0;
        src0.at(p, fold, wt, lane);
        u32 S0, E0, PD, x0;
        {
            TSrc<E, FOLD> s = src0;
            parse_window<D, true>(d, s, 0, row, S0, E0, PD, x0);
        }
        // lanes' entries: speculative first exits, rounds until no exit changes; an entry
        // inside a token re-parses the window from it (rewriting the row and the masks)
        u32 e = __shfl_up_sync(FULL, x0, 1), cnt = 0, rs = 0;
        if (lane == 0) e = E0in;
        for (;;) {
            u32 x;
            if (e >= (u32)WT_W) {
                cnt = 0;
                rs = 0;
                x = e - WT_W;
            } else {
                if (!((S0 >> e) & 1)) {
                    reparse_window<D, true>(d, src0, e, row, S0, E0, PD, x0);
                    rs = 0;
                } else {
                    rs = __popc(E0 & ((1u << e) - 1u));
                }
                cnt = __popc(above(E0, e));
                x = x0;
            }
            u32 ne = __shfl_up_sync(FULL, x, 1);
            if (lane == 0) ne = E0in;
            if (!__any_sync(FULL, ne != e)) break;
            e = ne;
        }
        // lane offsets in the warp-tile's run
        u32 lo = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(FULL, lo, o);
            if ((int)lane >= o) lo += y;
        }
        const u32 tot = __shfl_sync(FULL, lo, 31);
        lo -= cnt;
        // tallies and the end position, from the masks
        const u64 g0 = O + lo;  // global index of this lane's first sample
        if (e < (u32)WT_W && g0 < p.n) {
            u32 lim = WT_W;  // tokens counted: those starting before the end of sample n-1's token
            if (g0 + cnt >= p.n) {  // this lane holds sample n-1: its token starts at an emit bit
                u32 em = above(E0, e);
                for (u64 k = p.n - 1 - g0; k > 0; k--) em &= em - 1;
                const u32 ps = __ffs(em) - 1;
                const u32 nxt = above(S0, ps + 1);
                const u64 endw = nxt ? (u64)(__ffs(nxt) - 1) : (u64)WT_W + x0;
                p.res->end_pos = wt * WT_WORDS + (u64)WT_W * lane + endw;
                lim = ps + 1;
            }
            const u32 rng = above(lim >= 32 ? FULL : (1u << lim) - 1u, e);
            att += __popc(S0 & rng);
            pdf += __popc(PD & rng);
        }
        // the previous warp-tile's bulk copy must have finished reading sout
        if (lane == 0 && bulk) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bulk = false;
        }
        __syncwarp();
        const u32 b = (u32)(O & 1);  // sout[j] <-> out[O - b + j]: 16-byte alignment matches
        if (g0 < p.n) {
            const u32 c = g0 + cnt <= p.n ? cnt : (u32)(p.n - g0);
            u64 *dst = (u64 *)sout + b + lo;
            const u64 *srow = (const u64 *)row + rs;
            for (u32 k = 0; k < c; k++) dst[k] = srow[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const u64 cnt_t = O + tot <= p.n ? tot : p.n - O;
            u64 *gout = (u64 *)p.out + (O - b);
            const u64 *so = (const u64 *)sout;
            const u32 j0 = b, j1 = b + (u32)cnt_t;  // sout[j0, j1) holds the samples
            if (j1 > j0) {
                const u32 ja = (j0 + 1) & ~1u, jb = j1 & ~1u;  // the 16-byte-aligned middle [ja, jb)
                if (j0 & 1) gout[j0] = so[j0];
                if ((j1 & 1) && j1 - 1 >= ja) gout[j1 - 1] = so[j1 - 1];
                if (jb > ja) {
                    const unsigned saddr = (unsigned)__cvta_generic_to_shared(so + ja);
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gout + ja),
                                 "r"(saddr), "r"((jb - ja) * 8u) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    bulk = true;
                }
            }
        }
    }
    if (lane == 0 && bulk) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if constexpr (D != FAM_LEMIRE) {  // tallies: warp reduce, one atomic per warp
        const int ti = D == FAM_EXP ? 2 : 0;
        u64 tv[2] = {att, pdf};
#pragma unroll
        for (int i = 0; i < 2; i++) {
            u64 v = tv[i];
            for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULL, v, s);
            if (lane == 0 && v) atomicAdd((unsigned long long *)&p.res->tally[ti + i], (unsigned long long)v);
        }
    }
}

// the pcg64 state at raw word WT_WORDS w for w < nwt: A^(WT_WORDS w) s0, from the powers
// pw[j] = A^(WT_WORDS 2^j) (host, pcg.py:41-55 affine doubling)
__global__ void k_pcg_wt(const u64 *base, const u64 *pw, u64 *out, u64 nwt) {
    const u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwt) return;
    EngPcg e;
    e.slo = base[0];
    e.shi = base[1];
    e.ilo = base[2];
    e.ihi = base[3];
    for (int j = 0; j < 40 && (w >> j); j++)
        if ((w >> j) & 1) e.affine(pw[4 * j], pw[4 * j + 1], pw[4 * j + 2], pw[4 * j + 3]);
    out[2 * w] = e.slo;
    out[2 * w + 1] = e.shi;
}

template <int E, bool FOLD>
rsk::TileLaunch tile_e(int fam) {
    const size_t sm = 8 * WT_WARP_SMEM;
    switch (fam) {
    case FAM_NORM:
        return rsk::TileLaunch{(const void *)k_wt_count<E, FAM_NORM, FOLD>, (const void *)k_wt_emit<E, FAM_NORM, FOLD>, sm};
    case FAM_EXP:
        return rsk::TileLaunch{(const void *)k_wt_count<E, FAM_EXP, FOLD>, (const void *)k_wt_emit<E, FAM_EXP, FOLD>, sm};
    case FAM_LEMIRE:
        return rsk::TileLaunch{(const void *)k_wt_count<E, FAM_LEMIRE, FOLD>,
                               (const void *)k_wt_emit<E, FAM_LEMIRE, FOLD>, sm};
    default: return rsk::TileLaunch{nullptr, nullptr, 0};
    }
}

}  // namespace

rsk::TileLaunch rsk::tile_kernels(int engine, int fam, int fold) {
    if (engine == RS_ENG_PCG64) return tile_e<RS_ENG_PCG64, false>(fam);
    if (engine == RS_ENG_PHILOX) return fold ? tile_e<RS_ENG_PHILOX, true>(fam) : tile_e<RS_ENG_PHILOX, false>(fam);
    return rsk::TileLaunch{nullptr, nullptr, 0};
}
const void *rsk::pcg_wt_kernel() { return (const void *)k_pcg_wt; }
const void *rsk::wt_scan1_kernel() { return (const void *)k_wt_scan1; }
const void *rsk::wt_scan2_kernel() { return (const void *)k_wt_scan2; }
