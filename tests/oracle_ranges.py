"""Test infrastructure: the range primitive of paper_2605_05099_b200.shard restated on the
oracle (a sequential parse), so the sharding protocol's host logic can run on CPU ranks.
It is the checker's stand-in for rs_range_count / rs_range_emit, never the product."""
import math

import numpy as np
import torch

from oracle import oracle as O

CAP = 144


class _Tracker:
    """Unit position of an oracle generator from its slice start (fresh buffer)."""

    def __init__(self, engine, state, unit, full_mantissa):
        self.engine, self.unit = engine, unit
        self.o = O.OracleRng(engine, seed=[1], full_mantissa=full_mantissa)
        self.o.set_state(state)
        self.states = [list(state)]
        self.k = 0

    def pos(self):
        if self.o.r.fill == 0:
            return 0
        st = self.o.get_state()
        k = max(self.k, 1)
        while True:
            while k >= len(self.states):
                _, nxt = O.engine_generate(self.engine, self.states[-1], CAP)
                self.states.append(nxt)
            if self.states[k] == st:
                break
            k += 1
            assert k < self.k + 100000, "oracle position lost"
        self.k = k
        words = CAP * k - (self.o.r.fill - self.o.r.cursor)
        if self.unit == 2:
            return 2 * words - (1 if self.o.r.has_pending else 0)
        return words

    def skip(self, units):
        for _ in range(int(units)):
            self.o.next_u32() if self.unit == 2 else self.o.next_u64()


class OracleRanges:
    device = "cpu"

    def __init__(self, engine, dist, params, full_mantissa=False, window=(72, 2), seg_len=72):
        self.engine, self.dist, self.params = engine, dist, dict(params or {})
        self.fm = full_mantissa
        self._window = window
        self.seg_len = seg_len
        self.unit = 2 if dist in ("u01f", "uniff", "normf", "expf", "uint8", "uint16", "uint32", "int") else 1

    def geometry(self, rng, dist_id, fp, ip, words):
        return self.seg_len, max(1, math.ceil(words / self.seg_len))

    def window(self, info):
        return self._window

    def _tracker(self, rng):
        return _Tracker(self.engine, list(rng.engine.s), self.unit, self.fm)

    def count(self, rng, dist_id, fp, ip, entry, seg_len, n_seg):
        self._rng, self._entry = rng, entry
        t = self._tracker(rng)
        t.skip(entry)
        end = self.unit * seg_len * n_seg
        pos, c = entry, 0
        while pos < end:
            t.o.fill(self.dist, self.params, 1)
            pos = t.pos()
            c += 1
        return c, pos - end, 0

    def emit(self, keep, out_dtype):
        t = self._tracker(self._rng)
        t.skip(self._entry)
        vals = t.o.fill(self.dist, self.params, keep)
        return _tensor(vals), t.pos(), _tallies(t.o)

    def tail(self, t, dist, params, m):
        """The oracle continues from the product generator's exact position (state + buffer)."""
        o = O.OracleRng(self.engine, seed=[1], full_mantissa=self.fm)
        o.set_state(t.engine.s)
        for i, w in enumerate(t.buffer.words):
            o.r.buf[i] = w
        o.r.fill, o.r.cursor = len(t.buffer.words), t.buffer.cursor
        o.r.has_pending = 0 if t.buffer.pending is None else 1
        o.r.pending = t.buffer.pending or 0
        vals = o.fill(dist, params, m)
        t.engine.s = o.get_state()
        t.buffer.words, t.buffer.cursor, t.buffer.pending = o.buffer()
        return _tensor(vals), _tallies(o)


def _tallies(o):
    tal = o.tallies()
    v = [0] * 6
    for i, name in enumerate(("norm", "exp", "gamma")):
        if name in tal:
            v[2 * i], v[2 * i + 1] = tal[name]["attempts"], tal[name]["pdf_evals"]
    return v


def _tensor(vals):
    if vals.dtype == np.uint64:
        return torch.from_numpy(vals.view(np.int64).copy()).view(torch.uint64)
    return torch.from_numpy(vals.copy())


def simulate(make_rng, dist, params, n, world, make_ranges, **kw):
    """Drive `world` ShardedFill ranks in one process (the allgathers become lists):
    returns (concatenated samples as numpy, rank-0 generator, per-rank instances)."""
    from paper_2605_05099_b200 import shard

    sfs = [shard.ShardedFill(make_rng(), dist, params, n, g, world, make_ranges(), **kw) for g in range(world)]
    if not sfs[0].variable:
        outs = [sf.fixed()[0] for sf in sfs]
        for sf in sfs:
            sf.finish_fixed()
    else:
        for sf in sfs:
            sf.count()
        for _ in range(world + 1):
            table = [sf.record() for sf in sfs]
            flags = [sf.resolve(table) for sf in sfs]
            if not any(flags):
                break
        for sf in sfs:
            sf.emit(table)
        fin = [sf.final_record() for sf in sfs]
        for sf in sfs:
            sf.finish(fin)
        outs = [sf.out for sf in sfs]
    got = torch.cat([o.cpu() for o in outs])
    return got, sfs[0].rng, sfs
