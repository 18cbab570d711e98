"""ctypes front of the C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker. The product package never
imports this module.

The interface mirrors the reference `randstream` surface that the parity
tests need: create(engine, seed, spawn_key) (src/state_io.py:13-19),
fill(dist, params, n) (src/rng.py:223-241), get_state/set_state,
buffer capture (src/buffer.py:51-60), tallies (src/continuous.py:32-33),
and the jump math (src/jumps.py, src/engines/pcg.py:41-55,
src/engines/ranlux.py:90-93).
"""

import ctypes
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

ENGINE_IDS = {"x256++": 1, "x256**": 2, "x128+": 3, "xoro++": 4, "pcg64": 5, "philox": 6, "squares": 7,
              "sfc64": 8, "cwg128": 9, "ranlux++": 10, "chacha20": 11, "x256++simd": 12, "x256**simd": 13,
              "sfc64simd": 14}
STATE_WORDS = {1: 4, 2: 4, 3: 2, 4: 2, 5: 4, 6: 6, 7: 2, 8: 4, 9: 8, 10: 9, 11: 6, 12: 32, 13: 32, 14: 32}
DIST_IDS = {"uint64": 1, "u01": 2, "u01f": 3, "norm": 4, "exp": 5, "gamma": 6, "beta": 7, "stdnorm": 8,
            "unif": 9, "uniff": 10, "normf": 11, "expf": 12, "lognormal": 13, "chi2": 14, "t": 15, "f": 16,
            "gumbel": 17, "pareto": 18, "gpd": 19, "weibull": 20, "skew_normal": 21,
            "uint8": 22, "uint16": 22, "uint32": 22, "int": 23, "long_long": 24}
F32_DISTS = ("u01f", "uniff", "normf", "expf")
TALLY_NAMES = ("norm", "exp", "gamma")
CAP = 144

U64P = ctypes.POINTER(ctypes.c_uint64)


class _Rng(ctypes.Structure):
    _fields_ = [
        ("eid", ctypes.c_int),
        ("full_mantissa", ctypes.c_int),
        ("st", ctypes.c_uint64 * 32),
        ("buf", ctypes.c_uint64 * CAP),
        ("fill", ctypes.c_int),
        ("cursor", ctypes.c_int),
        ("has_pending", ctypes.c_int),
        ("pending", ctypes.c_uint64),
        ("tally", ctypes.c_uint64 * 6),
        ("tally_seen", ctypes.c_int * 3),
    ]


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        assert L.orc_sizeof_rng() == ctypes.sizeof(_Rng), "oracle struct layout mismatch"
        L.orc_create.argtypes = [ctypes.POINTER(_Rng), ctypes.c_int, U64P, ctypes.c_int, U64P, ctypes.c_int]
        L.orc_set_state.argtypes = [ctypes.POINTER(_Rng), ctypes.c_int, U64P]
        L.orc_fill.argtypes = [ctypes.POINTER(_Rng), ctypes.c_int, ctypes.POINTER(ctypes.c_double), U64P,
                               ctypes.c_uint64, ctypes.c_void_p]
        L.orc_fill_threads.argtypes = [ctypes.POINTER(_Rng), ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_double), U64P, ctypes.c_uint64,
                                       ctypes.POINTER(ctypes.c_void_p)]
        L.orc_next_u64.argtypes = [ctypes.POINTER(_Rng)]
        L.orc_next_u64.restype = ctypes.c_uint64
        L.orc_next_u32.argtypes = [ctypes.POINTER(_Rng)]
        L.orc_next_u32.restype = ctypes.c_uint32
        L.orc_det_exp.argtypes = [ctypes.c_double]
        L.orc_det_exp.restype = ctypes.c_double
        L.orc_det_log.argtypes = [ctypes.c_double]
        L.orc_det_log.restype = ctypes.c_double
        L.orc_seed_words.argtypes = [U64P, ctypes.c_int, U64P, ctypes.c_int, U64P, ctypes.c_int]
        L.orc_x_pow_mod.argtypes = [ctypes.c_uint64, ctypes.c_uint64, U64P, U64P]
        L.orc_x256_charpoly.argtypes = [U64P]
        L.orc_x_pow2k_mod.argtypes = [ctypes.c_int, U64P, U64P]
        L.orc_x256_apply_poly.argtypes = [U64P, U64P]
        L.orc_pcg_advance.argtypes = [U64P, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_ranlux_advance_chunks.argtypes = [U64P, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_ranlux_jump_pow2k.argtypes = [U64P, ctypes.c_int]
        L.orc_x128_jump_pow2k.argtypes = [ctypes.c_int, U64P, ctypes.c_int]
        L.orc_engine_generate.argtypes = [ctypes.c_int, U64P, U64P, ctypes.c_int]
        _LIB = L
    return _LIB


def _u64arr(vals):
    vals = [int(v) & 0xFFFFFFFFFFFFFFFF for v in vals]
    return (ctypes.c_uint64 * max(1, len(vals)))(*vals), len(vals)


def fparams_for(dist, params):
    """Resolve the reference's defaults (src/continuous.py:157-218)."""
    p = dict(params or {})
    if dist == "norm":
        return [float(p.get("mu", 0.0)), float(p.get("var", 1.0)), 0.0, 0.0]
    if dist == "exp":
        return [float(p.get("beta", 1.0)), 0.0, 0.0, 0.0]
    if dist == "gamma":
        return [float(p["alpha"]), float(p.get("theta", 1.0)), 0.0, 0.0]
    if dist == "beta":
        return [float(p["a"]), float(p["b"]), 0.0, 0.0]
    if dist in ("unif", "uniff"):
        return [float(p.get("a", 0.0)), float(p.get("b", 1.0)), 0.0, 0.0]
    if dist in ("normf", "lognormal"):
        return [float(p.get("mu", 0.0)), float(p.get("var", 1.0)), 0.0, 0.0]
    if dist == "expf":
        return [float(p.get("beta", 1.0)), 0.0, 0.0, 0.0]
    if dist in ("chi2", "t"):
        return [float(p["nu"]), 0.0, 0.0, 0.0]
    if dist == "f":
        return [float(p["nu1"]), float(p["nu2"]), 0.0, 0.0]
    if dist == "gumbel":
        return [float(p.get("mu", 0.0)), float(p.get("beta", 1.0)), 0.0, 0.0]
    if dist == "pareto":
        return [float(p["alpha"]), float(p.get("xm", 1.0)), 0.0, 0.0]
    if dist == "gpd":
        return [float(p["xi"]), float(p.get("mu", 0.0)), float(p.get("sigma", 1.0)), 0.0]
    if dist == "weibull":
        return [float(p["k"]), float(p.get("lam", 1.0)), 0.0, 0.0]
    if dist == "skew_normal":
        return [float(p.get("alpha", 0.0)), float(p.get("mu", 0.0)), float(p.get("sigma", 1.0)), 0.0]
    return [0.0, 0.0, 0.0, 0.0]


WIDTH = {"uint8": 8, "uint16": 16, "uint32": 32}


def iparams_for(dist, params):
    p = dict(params or {})
    if dist == "uint64":
        b = int(p.get("b", 0))
        if b == 1 << 64:
            return [0, 1, 0, 0]
        return [b, 0, 0, 0]
    if dist in WIDTH:
        return [int(p.get("b", 0)), WIDTH[dist], 0, 0]
    if dist in ("int", "long_long"):
        w = 32 if dist == "int" else 64
        half = 1 << (w - 1)
        m, hi = int(p.get("m", -half)), int(p.get("n", half - 1))
        span = hi - m + 1
        full = 1 if span == 1 << w else 0
        return [0 if full else span, w, m & 0xFFFFFFFFFFFFFFFF, full]
    return [0, 0, 0, 0]


def out_dtype(dist):
    if dist == "uint64":
        return np.uint64
    if dist in F32_DISTS:
        return np.float32
    if dist in WIDTH:
        return np.uint32
    if dist == "int":
        return np.int32
    if dist == "long_long":
        return np.int64
    return np.float64


class OracleRng:
    def __init__(self, engine, seed=None, spawn_key=(), full_mantissa=False):
        self.L = lib()
        self.eid = ENGINE_IDS[engine]
        self.engine = engine
        self.r = _Rng()
        s, ns = _u64arr(seed or [])
        k, nk = _u64arr(spawn_key)
        self.L.orc_create(ctypes.byref(self.r), self.eid, s, ns if seed else 0, k, nk if spawn_key else 0)
        self.r.full_mantissa = int(bool(full_mantissa))

    def set_full_mantissa(self, flag):
        self.r.full_mantissa = int(bool(flag))

    def set_state(self, words):
        a, _ = _u64arr(words)
        self.L.orc_set_state(ctypes.byref(self.r), self.eid, a)

    def get_state(self):
        return [int(self.r.st[i]) for i in range(STATE_WORDS[self.eid])]

    def buffer(self):
        """(words, cursor, pending) as in WordBuffer.capture (src/buffer.py:51-60)."""
        words = [int(self.r.buf[i]) for i in range(self.r.fill)]
        pending = int(self.r.pending) if self.r.has_pending else None
        return words, int(self.r.cursor), pending

    def tallies(self):
        out = {}
        for i, name in enumerate(TALLY_NAMES):
            if self.r.tally_seen[i]:
                out[name] = {"attempts": int(self.r.tally[2 * i]), "pdf_evals": int(self.r.tally[2 * i + 1])}
        return out

    def next_u64(self):
        return int(self.L.orc_next_u64(ctypes.byref(self.r)))

    def next_u32(self):
        return int(self.L.orc_next_u32(ctypes.byref(self.r)))

    def fill(self, dist, params=None, n=1):
        out = np.empty(int(n), dtype=out_dtype(dist))
        fp = (ctypes.c_double * 4)(*fparams_for(dist, params))
        ip, _ = _u64arr(iparams_for(dist, params))
        rc = self.L.orc_fill(ctypes.byref(self.r), DIST_IDS[dist], fp, ip, int(n),
                             out.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            raise ValueError("oracle: unsupported dist %s" % dist)
        return out

    def clone(self):
        o = OracleRng.__new__(OracleRng)
        o.L, o.eid, o.engine = self.L, self.eid, self.engine
        o.r = _Rng()
        ctypes.memmove(ctypes.byref(o.r), ctypes.byref(self.r), ctypes.sizeof(_Rng))
        return o


def det_exp(x):
    return lib().orc_det_exp(float(x))


def det_log(x):
    return lib().orc_det_log(float(x))


def seed_words(entropy, spawn_key, n):
    e, ne = _u64arr(entropy)
    k, nk = _u64arr(spawn_key)
    out = (ctypes.c_uint64 * n)()
    lib().orc_seed_words(e, ne if entropy else 0, k, nk if spawn_key else 0, out, n)
    return [int(v) for v in out]


def x256_charpoly():
    out = (ctypes.c_uint64 * 5)()
    lib().orc_x256_charpoly(out)
    return sum(int(out[i]) << (64 * i) for i in range(5))


def x_pow_mod(n, c):
    cw, _ = _u64arr([(c >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(5)])
    out = (ctypes.c_uint64 * 5)()
    lib().orc_x_pow_mod(n & 0xFFFFFFFFFFFFFFFF, n >> 64, cw, out)
    return sum(int(out[i]) << (64 * i) for i in range(5))


def x_pow2k_mod(k, c):
    cw, _ = _u64arr([(c >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(5)])
    out = (ctypes.c_uint64 * 5)()
    lib().orc_x_pow2k_mod(int(k), cw, out)
    return sum(int(out[i]) << (64 * i) for i in range(5))


def x256_apply_poly(state, poly):
    s, _ = _u64arr(state)
    pw, _ = _u64arr([(poly >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(5)])
    lib().orc_x256_apply_poly(s, pw)
    return [int(s[i]) for i in range(4)]


def pcg_advance(state, delta):
    s, _ = _u64arr(state)
    lib().orc_pcg_advance(s, delta & 0xFFFFFFFFFFFFFFFF, (delta >> 64) & 0xFFFFFFFFFFFFFFFF)
    return [int(s[i]) for i in range(4)]


def ranlux_advance_chunks(state, nchunks):
    s, _ = _u64arr(state)
    lib().orc_ranlux_advance_chunks(s, nchunks & 0xFFFFFFFFFFFFFFFF, nchunks >> 64)
    return [int(s[i]) for i in range(9)]


def x128_jump(engine, state, k):
    """2^k steps of x128+ / xoro++ (jumps.py FAMILY_JUMPS)."""
    s, _ = _u64arr(state)
    lib().orc_x128_jump_pow2k(ENGINE_IDS[engine], s, int(k))
    return [int(s[i]) for i in range(2)]


def ranlux_jump(state, k):
    s, _ = _u64arr(state)
    lib().orc_ranlux_jump_pow2k(s, int(k))
    return [int(s[i]) for i in range(9)]


def engine_generate(engine, state, n):
    eid = ENGINE_IDS[engine]
    s, _ = _u64arr(list(state) + [0] * (32 - len(state)))
    out = (ctypes.c_uint64 * n)()
    lib().orc_engine_generate(eid, s, out, n)
    return [int(v) for v in out], [int(s[i]) for i in range(STATE_WORDS[eid])]


def threaded_fill(rngs, dist, params, n_per_thread, outs=None):
    """Run len(rngs) oracle streams on host threads (the CPU baseline leg). `outs`: optional
    preallocated per-thread output arrays (each >= n_per_thread elements of the law's dtype)."""
    L = lib()
    k = len(rngs)
    arr = (_Rng * k)()
    for i, r in enumerate(rngs):
        ctypes.memmove(ctypes.byref(arr[i]), ctypes.byref(r.r), ctypes.sizeof(_Rng))
    if outs is None:
        outs = [np.empty(int(n_per_thread), dtype=out_dtype(dist)) for _ in range(k)]
    assert len(outs) == k and all(o.size >= n_per_thread and o.dtype == out_dtype(dist) for o in outs)
    ptrs = (ctypes.c_void_p * k)(*[o.ctypes.data for o in outs])
    fp = (ctypes.c_double * 4)(*fparams_for(dist, params))
    ip, _ = _u64arr(iparams_for(dist, params))
    L.orc_fill_threads(arr, k, DIST_IDS[dist], fp, ip, int(n_per_thread), ptrs)
    for i, r in enumerate(rngs):
        ctypes.memmove(ctypes.byref(r.r), ctypes.byref(arr[i]), ctypes.sizeof(_Rng))
    return outs


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
