"""Multi-GPU partitioning of one logical stream.

Rank g of N fills the contiguous slice [g*W, (g+1)*W) of the engine's word stream:
its generator is positioned by exact skip-ahead -- GF(2) jump (x256), LCG advance
(pcg64), counter offset (philox), A^(W/9) (ranlux++). sfc64 has no skip-ahead and
shards by spawned streams instead. No collective touches the data path; the
concatenation over ranks equals the single-stream fill.
"""

from . import _lib, engines, state_io


def shard_rng(engine, seed, rank, words_per_rank, spawn_key=(), full_mantissa=False):
    """A fresh Rng (empty buffer) positioned at engine word rank * words_per_rank."""
    r = state_io.create(engine, seed=seed, spawn_key=spawn_key)
    r.set_full_mantissa(full_mantissa)
    off = int(rank) * int(words_per_rank)
    if off:
        st = _lib.u64_array(r.engine.s, 32)
        _lib.check(_lib.lib.rs_engine_advance_words(r.engine.native, st, off & (2 ** 64 - 1), off >> 64))
        r.engine.s = [int(st[i]) for i in range(r.engine.STATE_WORDS)]
    return r


def shard_streams(n_streams, rank, world):
    """Per-stream mode: rank's block [j0, j0 + count) of the spawned stream indices."""
    per = (int(n_streams) + world - 1) // world
    j0 = min(rank * per, n_streams)
    return j0, max(0, min(per, n_streams - j0))


def supported_skip_ahead(engine):
    return engines.normalize(engine) in ("x256**", "x256++", "pcg64", "philox", "ranlux++")
