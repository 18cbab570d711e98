"""Seed conditioning: SeedSequenceFE128 (numpy SeedSequence, pool_size=4).

Same mixing as the reference (pkg/src/randstream/seeding.py:21-116); the 32-bit
lane arithmetic runs in the native library (rs_seed_words). Spawn keys append
words after the (zero-padded) entropy so children never collide with parents.
"""

import os
import time

from . import _lib

MASK64 = 0xFFFFFFFFFFFFFFFF


def words32_from_words64(words64):
    out = []
    for w in words64:
        w = int(w) & MASK64
        out += [w & 0xFFFFFFFF, w >> 32]
    return out


def derive_seed_words(n_words, entropy_words, spawn_key=()):
    ent = [int(w) & MASK64 for w in (entropy_words or [])]
    key = [int(w) & MASK64 for w in spawn_key]
    out = _lib.u64_array([], n_words)
    _lib.check(_lib.lib.rs_seed_words(_lib.u64_array(ent), len(ent), _lib.u64_array(key), len(key), out, n_words))
    return [int(out[i]) for i in range(n_words)]


class SeedSequenceFE128:
    def __init__(self, entropy_words=None, spawn_key=()):
        self.entropy_words = [int(w) & MASK64 for w in (entropy_words or [])]
        self.spawn_key = tuple(int(w) & MASK64 for w in spawn_key)

    def generate_words64(self, n):
        return derive_seed_words(n, self.entropy_words, self.spawn_key)

    def generate_words32(self, n):
        w64 = self.generate_words64((n + 1) // 2)
        return words32_from_words64(w64)[:n]

    def child(self, index):
        return SeedSequenceFE128(self.entropy_words, self.spawn_key + (int(index) & MASK64,))


def seed_engine(engine, entropy_words, spawn_key=()):
    engine.seed_from(derive_seed_words(engine.SEED_WORDS, entropy_words, spawn_key))


def random_entropy(n_words=4):
    """OS entropy with the reference's degradation chain (seeding.py:119-152):
    os.urandom -> /dev/urandom -> clock (flagged degraded)."""
    try:
        raw = os.urandom(8 * n_words)
        return [int.from_bytes(raw[8 * i:8 * i + 8], "little") for i in range(n_words)], "os.urandom", False
    except (NotImplementedError, OSError):
        pass
    try:
        with open("/dev/urandom", "rb") as fh:
            raw = fh.read(8 * n_words)
        if len(raw) == 8 * n_words:
            return [int.from_bytes(raw[8 * i:8 * i + 8], "little") for i in range(n_words)], "/dev/urandom", False
    except OSError:
        pass
    mixer = SeedSequenceFE128([time.time_ns() & MASK64, os.getpid() & MASK64, id(object()) & MASK64])
    return mixer.generate_words64(n_words), "clock", True
