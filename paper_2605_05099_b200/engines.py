"""Engine registry and the engine protocol (host side).

Mirrors the reference registry (pkg/src/randstream/engines/__init__.py:11-78):
14 engine ids in registry order, case-insensitive selectors, "" / "0" / None ->
the default id. Each engine object keeps its state words on the host and
implements the reference engine protocol -- ID, NAME, AUTHORS, YEAR,
STATE_WORDS, SEED_WORDS, CHUNK, PERIOD, FAMILY, generate(n), get_state(),
set_state(words) (validating), seed_from(words) (repairing) -- by calling the
native library (the per-word arithmetic lives in C++, the bulk fills on the GPU).

Engines outside the B200 fill path (north star: xoshiro256**, PCG64, Philox,
sfc64, ranlux++; x256++ shares the xoshiro256 machinery) are listed by
catalogue() but cannot be constructed.
"""

from . import _lib

MASK64 = 0xFFFFFFFFFFFFFFFF

# (id, name, authors, year, state_words, seed_words, chunk, period, family, native id)
_REGISTRY = [
    ("x256++", "xoshiro256++", "Vigna and Blackman", 2019, 4, 4, 1, "2^256-1", "x256", 1),
    ("x256**", "xoshiro256**", "Vigna and Blackman", 2018, 4, 4, 1, "2^256-1", "x256", 2),
    ("x128+", "xorshift128+", "Vigna", 2014, 2, 2, 1, "2^128-1", "x128+", 3),
    ("xoro++", "xoroshiro128++", "Vigna and Blackman", 2019, 2, 2, 1, "2^128-1", "xoro", 4),
    ("pcg64", "PCG64 DXSM", "O'Neill", 2019, 4, 4, 1, "2^128 per increment", None, 5),
    ("philox", "Philox-4x64", "Salmon and Moraes", 2011, 6, 2, 4, "2^256 per key", None, 6),
    ("squares", "squares64", "Widynski", 2021, 2, 1, 1, "2^64 per key", None, 7),
    ("sfc64", "sfc64", "Chris Doty-Humphrey", 2010, 4, 3, 1, ">=2^64", None, 8),
    ("cwg128", "cwg128", "Dziala", 2022, 8, 8, 1, "2^128 per increment", None, 9),
    ("ranlux++", "ranlux++", "Sibidanov", 2017, 9, 9, 9, "~2^570", None, 10),
    ("chacha20", "ChaCha20", "Bernstein", 2008, 6, 6, 8, "2^35 bytes per nonce", None, 11),
    ("x256++simd", "xoshiro256++ x8", "Blackman, Vigna", 2019, 32, 4, 8, "2^256 - 1 per lane", "x256", 12),
    ("x256**simd", "xoshiro256** x8", "Blackman, Vigna", 2019, 32, 4, 8, "2^256 - 1 per lane", "x256", 13),
    ("sfc64simd", "sfc64 x8", "Doty-Humphrey", 2010, 32, 3, 8, ">= 2^64 per lane", None, 14),
]

ENGINE_IDS = [r[0] for r in _REGISTRY]
NATIVE_ID = {r[0]: r[9] for r in _REGISTRY}
_LOWER = {r[0].lower(): r[0] for r in _REGISTRY}

DEFAULT_ID = "x256++simd"


class UnknownEngineError(ValueError):
    pass


def normalize(selector):
    """engines/__init__.py:38-60: case-insensitive; None / "" / "0" -> default."""
    if selector is None:
        return DEFAULT_ID
    sel = str(selector).strip()
    if sel == "" or sel == "0":
        return DEFAULT_ID
    canon = _LOWER.get(sel.lower())
    if canon is None:
        raise UnknownEngineError(
            "unknown engine %r; known engines: %s" % (selector, ", ".join(sorted(ENGINE_IDS))))
    return canon


class Engine:
    """Host-side engine state + protocol, backed by the native library."""

    def __init__(self, eid, name, authors, year, state_words, seed_words, chunk, period, family, native):
        self.ID, self.NAME, self.AUTHORS, self.YEAR = eid, name, authors, year
        self.STATE_WORDS, self.SEED_WORDS, self.CHUNK = state_words, seed_words, chunk
        self.PERIOD, self.FAMILY, self.native = period, family, native
        self.s = [0] * state_words
        # reference constructors' initial states (xorfam.py:52-54, pcg.py:21-23, counter.py:80-82,
        # sfc.py:19-23, ranlux.py:75-76)
        if eid in ("x256++", "x256**"):
            self.s[0] = 1
        elif eid == "pcg64":
            self.s = [0, 0, 1, 0]
        elif eid == "sfc64":
            self.s = [0, 0, 0, 1]
        elif eid == "ranlux++":
            self.s[0] = 1
        elif eid in ("x128+", "xoro++"):  # xorfam.py:52-54
            self.s[0] = 1
        elif eid == "squares":  # counter.py:23-25: counter 0, key 1
            self.s = [0, 1]
        elif eid == "cwg128":  # cwg.py:22-26: x = weyl = extra = 0, inc = 1
            self.s = [0, 0, 0, 0, 0, 0, 1, 0]
        elif eid in ("x256++simd", "x256**simd"):  # lane k = [4k+1, 4k+2, 4k+3, 4k+4]
            self.s = [4 * k + w + 1 for k in range(8) for w in range(4)]
        elif eid == "sfc64simd":  # lanes from a default sfc64 (a=b=c=0, w=1), counters + k*2^61
            self.s = [v for k in range(8) for v in (0, 0, 0, (1 + k * (1 << 61)) & MASK64)]

    def get_state(self):
        return list(self.s)

    def set_state(self, words):
        words = [int(w) & MASK64 for w in words]
        if len(words) != self.STATE_WORDS:
            raise ValueError("%s expects %d state words, got %d" % (self.ID, self.STATE_WORDS, len(words)))
        _lib.check(_lib.lib.rs_engine_check_state(self.native, _lib.u64_array(words)))
        self.s = words

    def seed_from(self, words):
        w = _lib.u64_array(list(words)[:16], 16)
        out = _lib.u64_array([], 32)
        _lib.check(_lib.lib.rs_engine_seed_from(self.native, w, out))
        self.s = [int(out[i]) for i in range(self.STATE_WORDS)]

    def generate(self, n):
        n = int(n)
        st = _lib.u64_array(self.s, 32)
        out = (_lib.ctypes.c_uint64 * max(1, n))()
        _lib.check(_lib.lib.rs_engine_generate(self.native, st, out, n))
        self.s = [int(st[i]) for i in range(self.STATE_WORDS)]
        return [int(out[i]) for i in range(n)]

    # stream-control hooks used by Rng.set_stream (rng.py:27-35)
    def set_inc(self, words):  # pcg.py:57-61
        if len(words) != 2:
            raise ValueError("pcg64 increment is 2 words")
        self.s[2] = int(words[0]) & MASK64 | 1
        self.s[3] = int(words[1]) & MASK64

    def set_key(self, words):  # philox counter.py:123-127; squares counter.py:50-54
        if self.ID == "squares":
            if len(words) != 1:
                raise ValueError("squares key is 1 word")
            self.s = [0, int(words[0]) & MASK64]
            return
        if len(words) != 2:
            raise ValueError("philox key is 2 words")
        self.s = [0, 0, 0, 0, int(words[0]) & MASK64, int(words[1]) & MASK64]

    def set_weyl(self, words):  # cwg.py:40-45: odd increment, then a 96-word warm-up
        if len(words) != 2:
            raise ValueError("cwg128 Weyl increment is 2 words")
        self.s[6] = (int(words[0]) & MASK64) | 1
        self.s[7] = int(words[1]) & MASK64
        self.generate(96)

    def set_nonce(self, words):  # counter.py:218-224: 96-bit nonce, counter 0
        if len(words) != 2:
            raise ValueError("chacha20 nonce is 96 bits passed as 2 words")
        self.s[4] = int(words[0]) & MASK64
        self.s[5] = int(words[1]) & 0xFFFFFFFF

    def set_abc(self, words):  # sfc.py:38-43: (a, b, c), w = 0, 18-step warmup
        if len(words) != 3:
            raise ValueError("sfc64 stream selector is 3 words (a, b, c)")
        base = [int(w) & MASK64 for w in words] + [0]
        st = _lib.u64_array(base, 32)
        out = (_lib.ctypes.c_uint64 * 18)()
        _lib.check(_lib.lib.rs_engine_generate(NATIVE_ID["sfc64"], st, out, 18))
        a, b, c, w = (int(st[i]) for i in range(4))
        if self.ID == "sfc64simd":  # interleave.py:217-228: lanes offset the counter by k*2^61
            self.s = [v for k in range(8) for v in (a, b, c, (w + k * (1 << 61)) & MASK64)]
        else:
            self.s = [a, b, c, w]


def engine_class_info():
    return list(_REGISTRY)


def make(selector=None):
    eid = normalize(selector)
    row = next(r for r in _REGISTRY if r[0] == eid)
    if not _lib.lib.rs_engine_supported(row[9]):
        raise NotImplementedError(
            "engine %r is not on the B200 fill path"
            % eid)
    return Engine(*row)


def supported(selector):
    try:
        eid = normalize(selector)
    except UnknownEngineError:
        return False
    return bool(_lib.lib.rs_engine_supported(NATIVE_ID[eid]))


def catalogue():
    """engines/__init__.py:67-78: static description of every engine, registry order."""
    return [
        {"id": r[0], "name": r[1], "authors": r[2], "year": r[3], "state_words": r[4], "seed_words": r[5],
         "period": r[7]}
        for r in _REGISTRY
    ]
