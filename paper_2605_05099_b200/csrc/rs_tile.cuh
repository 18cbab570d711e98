// Single-pass tile parse for the ziggurat normal / exponential families over engines that
// reach any word directly (PCG64-DXSM by an affine power, Philox by its counter).
//
// The two-pass path (k_count -> k_fixup -> k_emit) runs the engine and the ziggurat
// machine twice per word. Here every word is generated and parsed once:
//
//  * The chunk's engine words are cut into tiles of TL_T threads x TL_W words. A persistent
//    grid of G co-resident CTAs takes tiles c, c + G, c + 2G, ... (static, so a thread moves
//    to its next tile with one fixed affine step / counter add).
//  * A thread parses its TL_W words as if a sample boundary sat on its first word and leaves
//    its samples in a shared-memory row. Its exit (words its last token runs past its end) is
//    its neighbour's entry. An entry of 1 on a one-word first token just drops that sample;
//    any other non-zero entry re-parses the thread's words with the exact machine, and the
//    tile repeats the exchange until no exit changes (a fixed point, as in k_fixup).
//  * What a tile needs from the stream before it is one bit: whether its predecessor's last
//    word started a wedge. A tile's exit does not depend on its entry once the two parses of
//    thread 0 meet inside thread 0's words (checked, never assumed), so each tile publishes
//    ONE record right after its parse: its sample count for entry 0, for entry 1, and its
//    exit. No tile waits for another tile's resolution: there is no chain.
//  * The CTA then parses its NEXT tile (double-buffered rows) and only afterwards finishes
//    the previous one: it sums the exact counts of the G - 1 tiles between its own last two
//    (one record load per thread; they were published a whole tile time ago), which gives
//    the tile's output offset, and copies the rows out as contiguous runs.
//  * Anything outside this model -- a tile exit of 2 or more words (a tail token across a
//    tile edge), thread 0's two parses not meeting, a record that never arrives -- raises a
//    flag and the host runs the chunk through the two-pass path instead. Results are the
//    reference's in every case.
#pragma once
#include "rs_kernels.cuh"

namespace {

constexpr int TL_ROW = TL_W + 1;  // odd row stride: conflict-free 8-byte rows

// ---- per-thread engines: 8-word batches, single words on the rare paths, seek inside a tile
template <int E> struct TileEng;
template <> struct TileEng<RS_ENG_PCG64> {
    EngPcg e;
    u64 tlo, thi;  // state at the thread's first word of the current tile
    u64 plo, phi;  // ... of the tile awaiting its finish
    __device__ __forceinline__ void init(const FillPlan &p, u32 t) {
        make_engine<RS_ENG_PCG64>(p, t, e);  // plan stride L = TL_W
        tlo = e.slo; thi = e.shi;
        plo = tlo; phi = thi;
    }
    __device__ __forceinline__ void next_tile(const FillPlan &p) {
        plo = tlo; phi = thi;
        e.slo = tlo; e.shi = thi;
        e.affine(p.tile_m[0], p.tile_m[1], p.tile_a[0], p.tile_a[1]);
        tlo = e.slo; thi = e.shi;
    }
    __device__ __forceinline__ void gen8(const FillPlan &, u64 *w) {
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = e.next();
    }
    __device__ __forceinline__ u64 next(const FillPlan &) { return e.next(); }
    __device__ __forceinline__ void seek(const FillPlan &, bool prev, u32 off) {
        e.slo = prev ? plo : tlo; e.shi = prev ? phi : thi;
        for (u32 k = 0; k < off; k++) e.next();
    }
};
template <> struct TileEng<RS_ENG_PHILOX> {
    u64 blk, tblk, pblk;  // next block / first block of the current tile / of the tile awaiting its finish
    u64 b0, b1, b2, b3;
    int left;
    u64 stride;
    __device__ __forceinline__ void init(const FillPlan &p, u32 t) {
        tblk = pblk = blk = (u64)t * (TL_W / 4);
        left = 0;
        stride = (u64)gridDim.x * (TL_T * TL_W / 4);
    }
    __device__ __forceinline__ void next_tile(const FillPlan &) {
        pblk = tblk;
        tblk += stride;
        blk = tblk;
        left = 0;
    }
    __device__ __forceinline__ void block(const FillPlan &p, u64 bi, u64 &o0, u64 &o1, u64 &o2, u64 &o3) {
        u64 c0 = p.base[0] + bi, c1 = p.base[1], c2 = p.base[2], c3 = p.base[3];
        if (c0 < bi) { c1 += 1; if (c1 == 0) { c2 += 1; if (c2 == 0) c3 += 1; } }
        philox4x64_10_rk<0>(c0, c1, c2, c3, p.rk0, p.rk1, o0, o1, o2, o3);
    }
    __device__ __forceinline__ void gen8(const FillPlan &p, u64 *w) {  // block-aligned (left == 0)
        block(p, blk, w[0], w[1], w[2], w[3]);
        block(p, blk + 1, w[4], w[5], w[6], w[7]);
        blk += 2;
    }
    __device__ __forceinline__ u64 next(const FillPlan &p) {
        if (left == 0) { block(p, blk, b0, b1, b2, b3); blk++; left = 4; }
        u64 r = b0;
        b0 = b1; b1 = b2; b2 = b3;
        left--;
        return r;
    }
    __device__ __forceinline__ void seek(const FillPlan &p, bool prev, u32 off) {
        blk = (prev ? pblk : tblk) + off / 4;
        left = 0;
        for (u32 k = 0; k < (off & 3); k++) next(p);
    }
};

// ---- tile records: one 64-bit word per tile, written once, polled by later tiles
//   [63:32] epoch of the launch  [31:30] exit (0, 1; 3 = outside the model)
//   [29:15] samples for entry 1  [14:0] samples for entry 0
__device__ __forceinline__ u64 rec_pack(u32 epoch, u32 cntA, u32 cntB, u32 ex) {
    return ((u64)epoch << 32) | ((u64)(ex > 1 ? 3u : ex) << 30) | ((u64)cntB << 15) | (u64)cntA;
}
__device__ __forceinline__ u32 rec_a(u64 r) { return (u32)r & 0x7FFFu; }
__device__ __forceinline__ u32 rec_b(u64 r) { return (u32)(r >> 15) & 0x7FFFu; }
__device__ __forceinline__ u32 rec_exit(u64 r) { return (u32)(r >> 30) & 3u; }
__device__ __forceinline__ void rec_store(u64 *p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 rec_load(const u64 *p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// exact re-parse of a thread's words from word offset `ent` of its tile slot (the engine is
// already positioned there): samples that START in the slot, written from dst[0]. Returns the
// count; ex = words consumed past the slot's end; stops after `upto` samples when upto > 0
// (then `used` = words consumed from the slot's first word up to and including the word that
// completed that sample).
template <int E, class DI>
__device__ __noinline__ u32 tile_reparse(const FillPlan &p, const DI &d, TileEng<E> &eng, u32 ent, double *dst,
                                        Tally &tl, u32 &ex, u32 upto, u32 &used) {
    ZigWM m;
    m.st = 0;
    u32 pos = ent, c = 0;
    used = 0;
    if (ent >= (u32)TL_W) { ex = ent - TL_W; return 0; }
    while (pos < (u32)TL_W || m.st != 0) {
        double z;
        u64 w = eng.next(p);
        pos++;
        if (d.feed(m, w, tl, z)) {
            dst[c++] = d.finish(z);
            if (upto && c == upto) { used = pos; break; }
        }
    }
    ex = pos > (u32)TL_W ? pos - TL_W : 0;
    return c;
}

template <class DI> __device__ __forceinline__ u32 tl_att(const Tally &t) {
    return std::is_same<DI, DistNorm>::value ? t.norm_att : t.exp_att;
}
template <class DI> __device__ __forceinline__ u32 tl_pdf(const Tally &t) {
    return std::is_same<DI, DistNorm>::value ? t.norm_pdf : t.exp_pdf;
}

struct TileInfo {  // per buffer, written after the tile's resolution (CTA-uniform data)
    u32 cntA;      // tile samples for entry 0
    u32 tal;       // att | pdf << 16, summed over the tile, entry 0
    u32 d_cnt;     // thread 0: samples(entry 0) - samples(entry 1)
    u32 tal0A, tal0B;  // thread 0's own tallies (att | pdf << 16) for entry 0 / entry 1
    u32 cntB0;     // thread 0's samples for entry 1
    u32 startB;    // first slot of thread 0's run for entry 1 (in its row, or in rowB)
    u32 use_rowB;
    u32 exit;      // tile exit (words past the tile's end)
    u32 bad;       // entry 1 cannot be served (thread 0's parses did not meet)
};

template <int E, int D>
__global__ void __launch_bounds__(TL_T, 1) k_tile(const __grid_constant__ FillPlan p, DevResult *res) {
    typedef typename DistOf<D>::type DI;
    extern __shared__ __align__(16) unsigned char tl_dyn[];
    double *rows = (double *)tl_dyn;                      // [2][TL_T][TL_ROW]
    double *rowB = rows + 2 * TL_T * TL_ROW;              // [2][TL_ROW]
    __shared__ ZigFast sm[256];
    __shared__ u32 s_exit[TL_T];
    __shared__ u64 s_rec[TL_T];
    __shared__ u32 s_wc[TL_T / 32];
    __shared__ u32 s_tal, s_tal2[2], s_e0, s_abort;
    __shared__ TileInfo s_ti[2];
    stage_tables(p, sm);
    DI d;
    make_dist<D>(p, sm, d);
    const u32 j = threadIdx.x, lane = j & 31, wid = j >> 5;
    const u32 c = blockIdx.x, G = gridDim.x, NT = p.tile_nt, epoch = p.tile_epoch;
    u64 *rec = p.tile_rec;
    double *out = (double *)p.out + p.out0;
    constexpr int TI = D == FAM_NORM ? 0 : 2;  // tally slots (norm_att, norm_pdf | exp_att, exp_pdf)

    TileEng<E> eng;
    eng.init(p, c * TL_T + j);
    if (j == 0) { s_tal = 0; s_e0 = 0; s_abort = 0; }

    // ---- the stream ahead of engine word 0: the buffered prefix (first chunk) or lp0 engine
    // words to skip (later chunks). CTA 0 parses the prefix exactly, straight to the output
    // (the host takes this path only for fills far larger than the prefix).
    if (c == 0 && j == 0) {
        u32 e0 = 0, cpre = 0;
        Tally tp = {0, 0, 0, 0, 0};
        if (p.P > 0) {
            ZigWM m;
            m.st = 0;
            for (u32 q = (u32)p.lp0; q < (u32)p.P; q++) {
                double z;
                if (d.feed(m, p.prefix[q], tp, z)) out[cpre++] = d.finish(z);
            }
            while (m.st != 0) {  // the last buffered token runs into the engine words
                double z;
                u64 w = eng.next(p);
                e0++;
                if (d.feed(m, w, tp, z)) out[cpre++] = d.finish(z);
            }
            eng.seek(p, false, 0);
        } else {
            e0 = (u32)p.lp0;
        }
        s_e0 = e0;
        if (tl_att<DI>(tp)) atomicAdd((unsigned long long *)&res->tally[TI], (unsigned long long)tl_att<DI>(tp));
        if (tl_pdf<DI>(tp)) atomicAdd((unsigned long long *)&res->tally[TI + 1], (unsigned long long)tl_pdf<DI>(tp));
        rec_store(rec, rec_pack(epoch, cpre, cpre, 0));
    }
    __syncthreads();

    // per-thread state of the tile awaiting its finish
    u32 pv_i = 0, pv_off = 0, pv_cnt = 0, pv_start = 0, pv_ent = 0, pv_tal = 0;
    bool have_prev = false;
    u64 own_pref = 0;  // output offset just past this CTA's last finished tile

    for (u32 k = 0, i = c;; k++, i += G) {
        const bool has = i < NT;
        const u32 buf = k & 1;
        double *row = rows + ((size_t)buf * TL_T + j) * TL_ROW;
        u32 cnt = 0, start = 0, ent = 0, ex = 0, off = 0, att = 0, pdf = 0;
        if (has) {
            if (k > 0) eng.next_tile(p);
            // ---- speculative parse: a boundary on my first word
            ZigWM m;
            m.st = 0;
            Tally tl = {0, 0, 0, 0, 0};
            u32 f0 = 0;
#pragma unroll 1
            for (int h = 0; h < TL_W / ZB; h++) {
                u64 w[ZB];
                eng.gen8(p, w);
                u32 F = 0, Z = 0;
                double x[ZB];
#pragma unroll
                for (int g = 0; g < ZB; g += 4) {
                    ZigFast f[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) f[q] = d.strip(w[g + q]);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        F |= (d.zfast(w[g + q], f[q]) ? 1u : 0u) << (g + q);
                        Z |= (((u32)w[g + q] & 0xFFu) == 0 ? 1u : 0u) << (g + q);
                        x[g + q] = d.zval(w[g + q], f[q]);
                    }
                }
                if (h == 0) f0 = F & 1u;
                u32 O = 0xFFu;
                if (F != 0xFFu || m.st != 0) {
                    // stage the words in the row's free slots (cnt <= 8h, the row holds 17): the
                    // batch's samples overwrite them in order after the words have been read
                    u64 *wst = (u64 *)(row + cnt);
#pragma unroll
                    for (int q = 0; q < ZB; q++) wst[q] = w[q];
                    auto ws = [wst](int q) -> u64 { return wst[q]; };
                    u32 a;
                    bool bnd;
                    double xc = 0.0;
                    const u32 cin = m.st;
                    if (zb_tokens(d, m, ws, F, Z, O, a, bnd, xc, tl)) {
                        d.zatt(tl, a);
                        if (cin) x[0] = xc;
                    } else {  // exact machine over the batch (a tail token)
                        O = 0;
                        for (int q = 0; q < ZB; q++) {
                            double z;
                            if (d.feed(m, ws(q), tl, z)) row[cnt++] = d.finish(z);
                        }
                    }
                } else {
                    d.zatt(tl, ZB);
                }
                {
                    u32 cc = 0;
#pragma unroll
                    for (int q = 0; q < ZB; q++) {
                        row[cnt + cc] = d.finish(x[q]);
                        cc += (O >> q) & 1;
                    }
                    cnt += cc;
                }
            }
            while (m.st != 0) {  // my last token runs past my words: its sample is mine
                double z;
                u64 w = eng.next(p);
                ex++;
                if (d.feed(m, w, tl, z)) row[cnt++] = d.finish(z);
            }
            att = tl_att<DI>(tl);
            pdf = tl_pdf<DI>(tl);

            // ---- entries: my entry is my neighbour's exit; repeat to a fixed point
            s_exit[j] = ex;
            __syncthreads();
            for (;;) {
                const u32 e = j == 0 ? (i == 0 ? s_e0 : 0u) : s_exit[j - 1];
                bool ch = false;
                if (e != ent) {
                    if (ent == 0 && start == 0 && e == 1 && f0) {  // drop my one-word first token
                        start = 1; cnt -= 1; att -= 1; ent = 1;
                    } else {
                        Tally t2 = {0, 0, 0, 0, 0};
                        u32 x2, used;
                        eng.seek(p, false, e < (u32)TL_W ? e : 0u);
                        cnt = tile_reparse<E>(p, d, eng, e, row, t2, x2, 0u, used);
                        att = tl_att<DI>(t2);
                        pdf = tl_pdf<DI>(t2);
                        start = 0;
                        ent = e;
                        f0 = 0;
                        if (x2 != ex) { ex = x2; ch = true; }
                    }
                }
                const int any = __syncthreads_or(ch ? 1 : 0);
                if (!any) break;
                if (ch) s_exit[j] = ex;
                __syncthreads();
            }

            // ---- thread 0 of a later tile also serves entry 1 (its predecessor's last word
            // started a wedge); which one applies is known when the tile is finished
            if (j == 0) {
                TileInfo &ti = s_ti[buf];
                ti.d_cnt = 0;
                ti.tal0A = ti.tal0B = att | (pdf << 16);
                ti.cntB0 = cnt; ti.startB = start; ti.use_rowB = 0; ti.bad = 0;
                if (i > 0) {
                    if (f0 && start == 0) {
                        ti.d_cnt = 1;
                        ti.tal0B = (att - 1) | (pdf << 16);
                        ti.cntB0 = cnt - 1; ti.startB = 1;
                    } else {
                        Tally t2 = {0, 0, 0, 0, 0};
                        u32 x2, used;
                        eng.seek(p, false, 1);
                        u32 cb = tile_reparse<E>(p, d, eng, 1, rowB + buf * TL_ROW, t2, x2, 0u, used);
                        ti.cntB0 = cb; ti.startB = 0; ti.use_rowB = 1;
                        ti.d_cnt = cnt - cb;  // (mod 2^32: the sum below wraps back)
                        ti.tal0B = tl_att<DI>(t2) | (tl_pdf<DI>(t2) << 16);
                        if (x2 != ex) ti.bad = 1;
                    }
                }
            }

            // ---- offsets inside the tile (entry 0) and the tile's tallies
            u32 inc = cnt;
#pragma unroll
            for (int sh = 1; sh < 32; sh <<= 1) {
                u32 v = __shfl_up_sync(0xFFFFFFFFu, inc, sh);
                if (lane >= (u32)sh) inc += v;
            }
            if (lane == 31) s_wc[wid] = inc;
            const u32 tv = __reduce_add_sync(0xFFFFFFFFu, att | (pdf << 16));
            if (lane == 0) atomicAdd(&s_tal, tv);
            __syncthreads();
            u32 wb = 0, tot = 0;
#pragma unroll
            for (int w2 = 0; w2 < TL_T / 32; w2++) {
                const u32 v = s_wc[w2];
                if ((u32)w2 < wid) wb += v;
                tot += v;
            }
            off = wb + inc - cnt;
            if (j == 0) {
                TileInfo &ti = s_ti[buf];
                ti.cntA = tot;
                ti.tal = s_tal;
                ti.exit = s_exit[TL_T - 1];
                s_tal = 0;
                u32 xr = ti.exit;
                if (xr > 1) { xr = 3; atomicExch(&res->pad, 1u); }
                const u32 cb = tot - ti.d_cnt;
                if (ti.bad) {
                    // entry 1 cannot be served: only legal if the predecessor's exit is 0;
                    // publishing cntB = 0x7FFF marks it (checked when summed)
                    rec_store(rec + 1 + i, rec_pack(epoch, tot, 0x7FFFu, xr));
                } else {
                    rec_store(rec + 1 + i, rec_pack(epoch, tot, i == 0 ? tot : cb, xr));
                }
            }
        }
        __syncthreads();

        // ---- finish the previous tile: its output offset, then its rows
        if (have_prev) {
            const u32 ip = pv_i, pb = buf ^ 1;
            const u32 nrec = ip + 1 < G ? ip + 1 : G;   // records rec[lo .. lo + nrec): tiles ip - nrec .. ip - 1 (+1)
            const u32 lo = ip + 1 - nrec;
            u64 v = 0;
            if (j < nrec) {
                u32 polls = 0;
                for (;;) {
                    v = rec_load(rec + lo + j);
                    if ((u32)(v >> 32) == epoch) break;
                    if ((++polls & 0x3FFu) == 0) {
                        if (polls > (1u << 24) || *(volatile u32 *)&res->pad) { atomicExch(&res->pad, 1u); s_abort = 1; break; }
                    }
                    __nanosleep(64);
                }
            }
            s_rec[j] = v;
            __syncthreads();
            u32 cv = 0;
            if (j < nrec) {
                if (j == 0) {
                    cv = ip < G ? rec_a(v) : 0u;  // the pre-record counts; my own previous tile is in own_pref
                } else {
                    const u32 pe = rec_exit(s_rec[j - 1]);
                    cv = pe ? rec_b(v) : rec_a(v);
                    if (pe == 3 || (pe && rec_b(v) == 0x7FFFu)) atomicExch(&res->pad, 1u);
                }
            }
            cv = __reduce_add_sync(0xFFFFFFFFu, cv);
            if (lane == 0) s_wc[wid] = cv;
            __syncthreads();
            u32 between = 0;
#pragma unroll
            for (int w2 = 0; w2 < TL_T / 32; w2++) between += s_wc[w2];
            const u32 entT = ip == 0 ? 0u : rec_exit(s_rec[nrec - 1]);
            const TileInfo ti = s_ti[pb];
            const bool B = entT != 0;
            if (B && (entT == 3 || ti.bad) && j == 0) atomicExch(&res->pad, 1u);
            const u64 base = own_pref + between;
            const u32 cntT = B ? ti.cntA - ti.d_cnt : ti.cntA;
            own_pref = base + cntT;
            const bool aborted = s_abort != 0;
            double *prow0 = rows + (size_t)pb * TL_T * TL_ROW;
            if (B && j == 0) {
                if (ti.use_rowB) {
                    for (u32 q = 0; q < ti.cntB0; q++) prow0[q] = rowB[pb * TL_ROW + q];
                }
                pv_cnt = ti.cntB0; pv_start = ti.startB; pv_ent = 1;
                pv_tal = ti.tal0B;
            }
            if (B && j > 0) pv_off -= ti.d_cnt;
            __syncthreads();
            if (!aborted && base < p.n) {
                // rows out as contiguous runs: a half-warp per row, two adjacent rows per step
                const u32 meta = pv_off | (pv_cnt << 14) | (pv_start << 19);
                const u32 l16 = lane & 15, hh = lane >> 4;
#pragma unroll 4
                for (int it = 0; it < 16; it++) {
                    const u32 r = (u32)it * 2 + hh;
                    const u32 mr = __shfl_sync(0xFFFFFFFFu, meta, r);
                    const u32 ro = mr & 0x3FFFu, rc = (mr >> 14) & 31u, rs = (mr >> 19) & 1u;
                    const u64 g = base + ro + l16;
                    if (l16 < rc && g < p.n) out[g] = prow0[(size_t)(wid * 32 + r) * TL_ROW + rs + l16];
                }
                // tallies and, in the tile that holds sample n - 1, the position after it
                if (base + cntT <= p.n) {
                    if (j == 0) {
                        const u32 t = B ? ti.tal - ti.tal0A + ti.tal0B : ti.tal;  // (no borrow: tal includes tal0A)
                        atomicAdd((unsigned long long *)&res->tally[TI], (unsigned long long)(t & 0xFFFFu));
                        atomicAdd((unsigned long long *)&res->tally[TI + 1], (unsigned long long)(t >> 16));
                    }
                } else {
                    const u32 q = (u32)(p.n - 1 - base);  // the tile's sample index of sample n - 1
                    if (j == 0) { s_tal2[0] = 0; s_tal2[1] = 0; }
                    __syncthreads();
                    u32 a2 = 0, p2 = 0;
                    if (pv_off + pv_cnt <= q) {
                        a2 = pv_tal & 0xFFFFu; p2 = pv_tal >> 16;
                    } else if (pv_off <= q) {
                        Tally t2 = {0, 0, 0, 0, 0};
                        u32 x2, used;
                        double *scratch = prow0 + (size_t)j * TL_ROW;  // (already copied out)
                        eng.seek(p, has, pv_ent < (u32)TL_W ? pv_ent : 0u);  // (no next_tile() ran when !has)
                        tile_reparse<E>(p, d, eng, pv_ent, scratch, t2, x2, q - pv_off + 1, used);
                        a2 = tl_att<DI>(t2); p2 = tl_pdf<DI>(t2);
                        res->end_pos = (u64)p.P + (u64)ip * (TL_T * TL_W) + (u64)j * TL_W + used;
                        eng.seek(p, false, 0);
                    }
                    if (a2) atomicAdd(&s_tal2[0], a2);
                    if (p2) atomicAdd(&s_tal2[1], p2);
                    __syncthreads();
                    if (j == 0) {
                        atomicAdd((unsigned long long *)&res->tally[TI], (unsigned long long)s_tal2[0]);
                        atomicAdd((unsigned long long *)&res->tally[TI + 1], (unsigned long long)s_tal2[1]);
                    }
                }
            }
            if (ip == NT - 1 && j == 0) {
                res->total = base + cntT;
                res->next_start = (u64)p.P + (u64)NT * (TL_T * TL_W) + ti.exit;
            }
            if (aborted) break;
        }
        if (!has) break;
        pv_i = i; pv_off = off; pv_cnt = cnt; pv_start = start; pv_ent = ent; pv_tal = att | (pdf << 16);
        have_prev = true;
        __syncthreads();
    }
}

}  // namespace
