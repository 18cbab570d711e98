"""Multi-GPU partitioning of one logical stream.

Rank g of N fills a contiguous slice of the engine's word stream. Its generator is
positioned by exact skip-ahead: GF(2) jump (x256), LCG advance (pcg64), counter
offset (philox), A^(W/9) (ranlux++). sfc64 has no skip-ahead and shards by spawned
streams instead. No collective touches the data path; the concatenation over
ranks equals the single-stream fill, and every rank ends with the generator
position the single-stream fill leaves (buffer.py:29-49 semantics).

* Fixed-consumption laws (raw, u01, u01f, ...): sample i comes from stream unit i,
  so rank g takes the words [g*W, (g+1)*W) (W a multiple of 144).
* Variable-consumption laws (ziggurat normal / exponential, gamma family, Lemire):
  rank g takes the samples that START in its slice [g*R, (g+1)*R) of a provisioned
  word range. It does not know where its first sample starts (that is decided by
  everything before it), so it
    1. guesses its entry by parsing a warm-up window just before its slice (the
       parses of these grammars converge within a few words),
    2. counts its samples from that entry and records its exit, the first sample
       boundary at or past its slice end (rs_range_count),
    3. exchanges (entry, exit, count) with the other ranks -- 3 integers per rank,
       the path's one real exchange step -- and re-counts if rank g-1's exit is not
       its guessed entry (iterated to a fixed point: at most N rounds),
    4. writes its first min(count, n - offset) samples, offset = the exclusive prefix
       of the counts (rs_range_emit).
  If the provisioned range holds fewer than n samples, the last rank continues the
  stream from its exit with an ordinary fill.
"""

import ctypes
import math

import torch

from . import _lib, engines, rng as _rng, state_io

CAP = 144


def shard_rng(engine, seed, rank, words_per_rank, spawn_key=(), full_mantissa=False):
    """A fresh Rng (empty buffer) positioned at engine word rank * words_per_rank."""
    r = state_io.create(engine, seed=seed, spawn_key=spawn_key)
    r.set_full_mantissa(full_mantissa)
    _advance_engine(r, int(rank) * int(words_per_rank))
    return r


def shard_streams(n_streams, rank, world):
    """Per-stream mode: rank's block [j0, j0 + count) of the spawned stream indices."""
    per = (int(n_streams) + world - 1) // world
    j0 = min(rank * per, n_streams)
    return j0, max(0, min(per, n_streams - j0))


def supported_skip_ahead(engine):
    return engines.normalize(engine) in ("x256**", "x256++", "pcg64", "philox", "ranlux++")


# ----------------------------------------------------------------------------- positioning
def _advance_engine(r, words):
    if words:
        st = _lib.u64_array(r.engine.s, 32)
        _lib.check(_lib.lib.rs_engine_advance_words(r.engine.native, st, words & (2 ** 64 - 1), words >> 64))
        r.engine.s = [int(st[i]) for i in range(r.engine.STATE_WORDS)]


def positioned(base, word):
    """A copy of `base` (at a fresh stream position) moved `word` engine words on, empty buffer."""
    r = base.duplicate()
    r.buffer.reset()
    _advance_engine(r, int(word))
    return r


def consume_units(r, units, unit):
    """Move a fresh-position `r` past `units` stream units exactly as the reference's buffer
    would after consuming them (buffer.py:29-49): ceil(W/144) refills, the buffer holds the
    last refill, and an odd number of 32-bit halves leaves the high half pending."""
    units = int(units)
    if unit == 2:
        words, odd = (units + 1) // 2, units & 1
    else:
        words, odd = units, 0
    if words == 0:
        return r
    refills = (words + CAP - 1) // CAP
    _advance_engine(r, (refills - 1) * CAP)
    r.buffer.words = r.engine.generate(CAP)
    r.buffer.cursor = words - (refills - 1) * CAP
    r.buffer.pending = (r.buffer.words[r.buffer.cursor - 1] >> 32) if odd else None
    return r


# ----------------------------------------------------------------------------- device slices
class DeviceRanges:
    """The product's range primitive: rs_range_geometry / rs_range_count / rs_range_emit on
    the current CUDA device. One counted slice per device at a time: emit() re-counts if
    another slice (or any fill) ran on the device after this one was counted."""

    _slot = {}  # device index -> token of the counted slice

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise _lib.LibraryError("no CUDA device: the fill path runs only on the GPU")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    def geometry(self, rng, dist_id, fp, ip, words):
        L = ctypes.c_uint64(0)
        T = ctypes.c_uint32(0)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.rs_range_geometry(rng.engine.native, dist_id, _fp(fp), _ip(ip), int(words),
                                                  _byref(L), _byref(T)))
        return int(L.value), int(T.value)

    def window(self, info):
        return int(info.min_seg_len), 256

    def count(self, rng, dist_id, fp, ip, entry, seg_len, n_seg):
        self._args = (rng, dist_id, fp, ip, entry, seg_len, n_seg)
        res = _lib.RsRangeInfo()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.rs_range_count(_byref(rng.to_stream()), dist_id, _fp(fp), _ip(ip), int(entry),
                                               int(seg_len), int(n_seg), _byref(res), self._stream()))
        self._token = object()
        DeviceRanges._slot[self.device.index] = self._token
        return int(res.count), int(res.exit), int(res.resync_rounds)

    def count_warm(self, wrng, dist_id, fp, ip, n_warm, seg_len, n_seg):
        """rs_range_count_warm: the slice counted behind n_warm warm-up segments in the same
        launches (the entry guess without a separate warm-up count). -> (count, exit, entry, rounds)"""
        res = _lib.RsRangeInfo()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.rs_range_count_warm(_byref(wrng.to_stream()), dist_id, _fp(fp), _ip(ip), int(n_warm),
                                                    int(seg_len), int(n_seg), _byref(res), self._stream()))
        # a re-count (emit after another slice ran on the device) goes through rs_range_count
        self._args = (positioned(wrng, int(n_warm) * int(seg_len)), dist_id, fp, ip, int(res.end_pos), seg_len, n_seg)
        self._token = object()
        DeviceRanges._slot[self.device.index] = self._token
        return int(res.count), int(res.exit), int(res.end_pos), int(res.resync_rounds)

    def emit(self, keep, out_dtype):
        if DeviceRanges._slot.get(self.device.index) is not self._token:
            self.count(*self._args)
        out = torch.empty(int(keep), dtype=out_dtype, device=self.device)
        res = _lib.RsRangeInfo()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.rs_range_emit(int(keep), _vp(out.data_ptr() if keep else 0), _byref(res),
                                              self._stream()))
        return out, int(res.end_pos), [int(res.tally[i]) for i in range(6)]

    def tail(self, t, dist, params, m):
        """An ordinary fill of m samples from the positioned generator `t` (the stream
        past the provisioned range); returns (samples, tallies)."""
        before = {k: dict(v) for k, v in t.counters.items()}
        out = t.fill(dist, params, m)
        tal = [0] * 6
        for i, name in enumerate(_rng._TALLY_NAMES):
            c, b = t.counters.get(name, {}), before.get(name, {})
            tal[2 * i] = c.get("attempts", 0) - b.get("attempts", 0)
            tal[2 * i + 1] = c.get("pdf_evals", 0) - b.get("pdf_evals", 0)
        return out, tal

    def _stream(self):
        return _vp(torch.cuda.current_stream(self.device).cuda_stream)


def _byref(x):
    return ctypes.byref(x)


def _vp(p):
    return ctypes.c_void_p(p)


def _fp(fp):
    return (ctypes.c_double * 4)(*(list(fp) + [0.0] * (4 - len(fp))))


def _ip(ip):
    return _lib.u64_array(list(ip), 4)


def dist_info(dist_id, fp, ip):
    info = _lib.RsDistInfo()
    _lib.check(_lib.lib.rs_dist_info(dist_id, _fp(fp), _ip(ip), _byref(info)))
    return info


def _validated(r, dist, params, n):
    """The reference's validation (rng.Rng.fill) -> (native dist id, fparams, iparams)."""
    params = dict(params or {})
    if dist in ("perm", "sample"):
        raise NotImplementedError("%s draws are sequences, not bulk fills" % dist)
    if n < 0:
        raise ValueError("draw count must be >= 0")
    if dist in _rng.SCALAR_NAMES:
        return _lib.DIST_IDS[dist], r._continuous_params(dist, params, n), []
    if dist in _rng.DISCRETE_NAMES:
        return _lib.DIST_IDS[dist], [], r._discrete_params(dist, params, n)
    raise ValueError("unknown discrete distribution %r" % dist)


def provision_words(n, words_per_sample):
    """Engine words provisioned for n samples (run_fill's rule: +1 % + 12 sigma + 2048)."""
    ww = n * words_per_sample
    return int(ww * 1.01 + 12.0 * math.sqrt(ww) + 2048.0)


# ----------------------------------------------------------------------------- the protocol
class ShardedFill:
    """One rank's state through the protocol; `fill_sharded` drives it with an allgather.
    Tests drive several instances in one process to simulate a world on one device."""

    def __init__(self, rng, dist, params, n, rank, world, ranges=None, words_per_rank=None, window=None):
        self.rng, self.dist, self.params, self.n = rng, dist, dict(params or {}), int(n)
        self.rank, self.world = int(rank), int(world)
        if rng.buffer.cursor < len(rng.buffer.words) or rng.buffer.pending is not None:
            raise ValueError("a sharded fill starts at a fresh stream position (no buffered words)")
        self.dist_id, self.fp, self.ip = _validated(rng, dist, self.params, self.n)
        self.info = dist_info(self.dist_id, self.fp, self.ip)
        self.unit = int(self.info.unit)
        self.variable = bool(self.info.variable)
        self.ranges = ranges
        self.out_dtype = _rng._out_dtype(dist)
        self.rounds = 0
        if self.variable:
            if self.ranges is None:
                self.ranges = DeviceRanges()
            words = provision_words(self.n, float(self.info.words_per_sample))
            wr = words_per_rank or (words + self.world - 1) // self.world
            self.L, self.T = self.ranges.geometry(rng, self.dist_id, self.fp, self.ip, wr)
            self.R = self.L * self.T  # engine words per slice, a multiple of 144
            self.window = window or self.ranges.window(self.info)
        else:
            words = (self.n + self.unit - 1) // self.unit
            per = words_per_rank or (words + self.world - 1) // self.world
            self.R = (per + CAP - 1) // CAP * CAP

    # -- variable consumption ------------------------------------------------
    def count(self):
        """Steps 1-2: entry guess from the warm-up window, then count + exit of the slice."""
        g = self.rank
        self.slice_rng = positioned(self.rng, g * self.R)
        if g > 0 and self.n and self.window[0] * self.window[1] and hasattr(self.ranges, "count_warm"):
            # the warm-up window as leading segments of the slice's own plan (one count)
            nw = -(-self.window[0] * self.window[1] // self.L)
            nw = (nw + 255) // 256 * 256
            if nw * self.L <= g * self.R:
                wr = positioned(self.rng, g * self.R - nw * self.L)
                self.cnt, self.exit, self.entry, rr = self.ranges.count_warm(wr, self.dist_id, self.fp, self.ip, nw,
                                                                             self.L, self.T)
                self.rounds += rr
                return
        if g == 0 or self.n == 0 or self.window[0] * self.window[1] == 0:  # (0, 0): no warm-up, guess 0
            self.entry = 0
        else:
            Lw, Tw = self.window
            wr = positioned(self.rng, g * self.R - Lw * Tw)
            _, self.entry, _ = self.ranges.count(wr, self.dist_id, self.fp, self.ip, 0, Lw, Tw)
        self._count()

    def _count(self):
        if self.n == 0:
            self.cnt, self.exit = 0, 0
            return
        self.cnt, self.exit, rr = self.ranges.count(self.slice_rng, self.dist_id, self.fp, self.ip, self.entry,
                                                    self.L, self.T)
        self.rounds += rr

    def record(self):
        return [self.entry, self.exit, self.cnt]

    def resolve(self, table):
        """Step 3: True if this or any rank's guessed entry was wrong (then re-counted here)."""
        bad = [h for h in range(1, self.world) if table[h - 1][1] != table[h][0]]
        if self.rank in bad:
            self.entry = table[self.rank - 1][1]
            self._count()
        return bool(bad)

    def emit(self, table):
        """Step 4: this rank's samples (device tensor) and its global offset."""
        counts = [int(t[2]) for t in table]
        self.off = sum(counts[:self.rank])
        self.total = sum(counts)
        self.keep = max(0, min(self.cnt, self.n - self.off))
        self.out, self.end_pos, self.tally = self.ranges.emit(self.keep, self.out_dtype) if self.keep else (
            torch.empty(0, dtype=self.out_dtype, device=self._dev()), self.entry, [0] * 6)
        self.last_exit = int(table[-1][1])
        return self.out, self.off

    def _dev(self):
        return getattr(self.ranges, "device", "cpu")

    def final_record(self):
        """What the others need to finish: this rank's end position (if it holds sample
        n-1) and its tallies; the last rank also runs the tail when the range fell short."""
        ends_here = self.keep > 0 and self.off + self.keep == self.n
        rec = [1 if ends_here else 0, self.end_pos] + list(self.tally)
        self.tail_units = 0
        if self.total < self.n and self.rank == self.world - 1:
            # continue the stream from the last exit with an ordinary fill
            t = positioned(self.rng, self.world * self.R)
            for _ in range(self.last_exit):
                t.next_u32() if self.unit == 2 else t.next_u64()
            tail, tal = self.ranges.tail(t, self.dist, self.params, self.n - self.total)
            self.out = torch.cat([self.out, tail.to(self.out.device)])
            self.keep += int(tail.numel())
            rec = [2, 0] + [a + b for a, b in zip(self.tally, tal)]
            rec += list(t.engine.s) + [len(t.buffer.words), t.buffer.cursor, 0 if t.buffer.pending is None else 1,
                                       t.buffer.pending or 0] + list(t.buffer.words)
        return rec

    def finish(self, table):
        """Every rank: the generator's post-fill position and the summed tallies."""
        r = self.rng
        if self.n == 0:  # nothing consumed, no tally touched (continuous.py:422-427 runs zero times)
            return
        tal = [sum(int(t[2 + i]) for t in table) for i in range(6)]
        for i, name in enumerate(_rng._TALLY_NAMES):
            if self.info.tally_seen[i]:
                c = r.counters.setdefault(name, {"attempts": 0, "pdf_evals": 0})
                c["attempts"] += tal[2 * i]
                c["pdf_evals"] += tal[2 * i + 1]
        tails = [t for t in table if t[0] == 2]
        if tails:
            t = tails[0][8:]
            sw = r.engine.STATE_WORDS
            r.engine.s = [int(v) for v in t[:sw]]
            nbuf, cur, has, pend = int(t[sw]), int(t[sw + 1]), int(t[sw + 2]), int(t[sw + 3])
            r.buffer.words = [int(v) for v in t[sw + 4:sw + 4 + nbuf]]
            r.buffer.cursor = cur
            r.buffer.pending = pend if has else None
            return
        ends = [(h, t[1]) for h, t in enumerate(table) if t[0] == 1]
        if not ends:  # n == 0: nothing consumed
            return
        h, end_pos = ends[0]
        units = h * self.R * self.unit + int(end_pos)
        fresh = positioned(r, 0)
        consume_units(fresh, units, self.unit)
        r.engine.s, r.buffer = fresh.engine.s, fresh.buffer
        r.buffer.engine = r.engine

    # -- fixed consumption ---------------------------------------------------
    def fixed(self):
        g = self.rank
        first = min(self.n, g * self.R * self.unit)
        last = min(self.n, (g + 1) * self.R * self.unit)
        self.off, self.keep = first, last - first
        part = positioned(self.rng, g * self.R)
        if self.keep:
            self.out = part.fill(self.dist, self.params, self.keep)
        else:
            dev = part._device() if torch.cuda.is_available() else "cpu"
            self.out = torch.empty(0, dtype=self.out_dtype, device=dev)
        return self.out, self.off

    def finish_fixed(self):
        if self.n:
            fresh = positioned(self.rng, 0)
            consume_units(fresh, self.n, self.unit)
            self.rng.engine.s, self.rng.buffer = fresh.engine.s, fresh.buffer
            self.rng.buffer.engine = self.rng.engine


def fill_sharded(rng, dist, params, n, rank, world, allgather, ranges=None, words_per_rank=None, window=None):
    """Rank-local part of `rng.fill(dist, params, n)` split over `world` ranks.

    Every rank passes an identical `rng` at a fresh stream position. Returns
    (samples, offset): this rank's piece of the single-stream result and where it
    starts in it. On return `rng` holds the single-stream post-fill position on every
    rank. `allgather(list_of_ints) -> list over ranks` is the exchange (see
    `torch_allgather`)."""
    sf = ShardedFill(rng, dist, params, n, rank, world, ranges, words_per_rank, window)
    if not sf.variable:
        out, off = sf.fixed()
        sf.finish_fixed()
        return out, off
    sf.count()
    for _ in range(world + 1):
        table = allgather(sf.record())
        if not sf.resolve(table):
            break
    else:
        raise _lib.LibraryError("slice entries did not reach a fixed point")
    out, off = sf.emit(table)
    sf.finish(allgather(sf.final_record()))
    return sf.out, off


def torch_allgather(group=None, width=256):
    """allgather over torch.distributed (NCCL or gloo): each rank's record is a few
    integers (at most `width`, u64 values as their int64 bit patterns), sent as one
    fixed-size int64 tensor on the rank's device (NCCL) or host (gloo)."""
    import torch.distributed as dist

    def gather(rec):
        rec = [int(v) for v in rec]
        if len(rec) + 1 > width:
            raise ValueError("allgather record longer than %d words" % width)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        row = [len(rec)] + [v - (1 << 64) if v >= (1 << 63) else v for v in rec]
        t = torch.zeros(width, dtype=torch.int64, device=dev)
        t[:len(row)] = torch.tensor(row, dtype=torch.int64)
        world = dist.get_world_size(group)
        parts = [torch.empty(width, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        rows = torch.stack(parts).cpu().tolist()
        return [[v & 0xFFFFFFFFFFFFFFFF if v < 0 else v for v in r[1:1 + r[0]]] for r in rows]

    return gather
