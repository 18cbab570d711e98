"""The generator facade: drop-in for the reference's `Rng` (pkg/src/randstream/rng.py).

Same surface and semantics -- word primitives, uniforms, seed / randomize /
jump / advance / set_stream, state, modes, duplicate, fill, mvn, the
per-instance error slot -- with one difference in *where* work runs:
`fill` and `mvn` (the bulk hot path, rng.py:223-241 / 273-275) always run on
the GPU through the C ABI (`rs_fill`, `rs_mvn`) and return device tensors.
Scalar word primitives (next_u64 / next_u32 / u01 / u01f / raw) consume the
host-side 144-word buffer exactly as the reference does; the scalar sampler
conveniences (norm, expo, gamma, unif, bounded_uint) are one-element device
fills. After any fill the engine state and buffer equal the reference's
(SURVEY 8(b)), so scalar draws, duplicate() and to_blob() continue bit-exactly.
"""

import ctypes
import math
import warnings
from functools import wraps
from struct import pack, unpack

import numpy as np
import torch

from . import _lib, engines, seeding
from .buffer import CAPACITY, WordBuffer

MASK64 = 0xFFFFFFFFFFFFFFFF

_POLY_JUMP = {"x256++", "x256**", "x256++simd", "x256**simd"}
STANDARD_JUMPS = (32, 64, 96, 128, 192)  # jumps.py:24
_NARROW_JUMP = {"x128+": "x128+", "xoro++": "xoro"}  # rng.py:20-25 -> jumps.py:25-29 families
_NARROW_JUMPS = (32, 64, 96)
_STREAM_METHODS = {  # rng.py:27-35
    "pcg64": ("set_inc", 2),
    "squares": ("set_key", 1),
    "philox": ("set_key", 2),
    "sfc64": ("set_abc", 3),
    "sfc64simd": ("set_abc", 3),
    "cwg128": ("set_weyl", 2),
    "chacha20": ("set_nonce", 2),
}

# the reference's continuous + discrete names (continuous.py:339-359, discrete.py:95-100)
RAW_DEVICE_WORDS = 4096  # raw(nbytes) from this many words on goes through the device uint64 fill

SCALAR_NAMES = ("u01", "u01f", "unif", "uniff", "norm", "normf", "exp", "expf", "lognormal", "gamma", "beta",
                "chi2", "t", "f", "gumbel", "pareto", "gpd", "weibull", "skew_normal")
DISCRETE_NAMES = ("uint8", "uint16", "uint32", "uint64", "int", "long_long")
_TRANSFORMED = ("lognormal", "gumbel", "pareto", "weibull", "gpd")  # continuous.py:361
_WIDTH = {"uint8": 8, "uint16": 16, "uint32": 32, "uint64": 64}

# keyword signatures of the reference samplers: (allowed, required) -- continuous.py:136-290
_SIGNATURES = {
    "u01": ((), ()),
    "u01f": ((), ()),
    "unif": (("a", "b"), ()),
    "uniff": (("a", "b"), ()),
    "norm": (("mu", "var"), ()),
    "normf": (("mu", "var"), ()),
    "exp": (("beta",), ()),
    "expf": (("beta",), ()),
    "lognormal": (("mu", "var"), ()),
    "gamma": (("alpha", "theta"), ("alpha",)),
    "beta": (("a", "b"), ("a", "b")),
    "chi2": (("nu",), ("nu",)),
    "t": (("nu",), ("nu",)),
    "f": (("nu1", "nu2"), ("nu1", "nu2")),
    "gumbel": (("mu", "beta"), ()),
    "pareto": (("alpha", "xm"), ("alpha",)),
    "gpd": (("xi", "mu", "sigma"), ("xi",)),
    "weibull": (("k", "lam"), ("k",)),
    "skew_normal": (("alpha", "mu", "sigma"), ()),
}
_TALLY_NAMES = ("norm", "exp", "gamma")

# Engines without skip-ahead (sfc.py / rng.py:162-163: "jump unsupported"): one stream cannot
# be split over GPU threads, so a single-stream fill replays it on ONE device thread
# (~10 Msamples/s). Their parallel form is per-stream mode (fill_streams: one spawned stream
# per thread, C5b). Warn once per engine when such a fill is large enough to matter.
_SERIAL_ENGINES = ("sfc64", "sfc64simd", "cwg128")
_SERIAL_WARN_N = 1 << 16
_serial_warned = set()


def _warn_serial(eid):
    if eid not in _serial_warned:
        _serial_warned.add(eid)
        warnings.warn("%s has no skip-ahead: a single-stream device fill runs on one GPU thread (~10 Msamples/s); "
                      "use fill_streams (one spawned stream per thread) for bulk draws" % eid, RuntimeWarning,
                      stacklevel=4)


def _op(fn):
    """Per-instance error slot (rng.py:38-52): success clears, failure records."""

    @wraps(fn)
    def guarded(self, *args, **kwargs):
        try:
            result = fn(self, *args, **kwargs)
        except Exception as exc:
            self.last_error = str(exc) or type(exc).__name__
            raise
        self.last_error = None
        return result

    return guarded


def _cuda_stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _out_dtype(dist):
    if dist == "uint64":
        return torch.uint64
    if dist in ("u01f", "uniff", "normf", "expf"):
        return torch.float32
    if dist in ("uint8", "uint16", "uint32"):
        return torch.uint32
    if dist == "int":
        return torch.int32
    if dist == "long_long":
        return torch.int64
    return torch.float64


_NP_OUT = {torch.uint64: np.dtype(np.uint64), torch.float32: np.dtype(np.float32), torch.uint32: np.dtype(np.uint32),
           torch.int32: np.dtype(np.int32), torch.int64: np.dtype(np.int64), torch.float64: np.dtype(np.float64)}


class Rng:
    def __init__(self, engine):
        self.engine = engine
        self.buffer = WordBuffer(engine)
        self.bitexact = False
        self.full_mantissa = False
        self.counters = {}
        self.last_error = None
        self.entropy_source = None
        self.entropy_degraded = False
        self.device = None  # torch device for fills (default: current CUDA device)

    @property
    def engine_id(self):
        return self.engine.ID

    # ---------------------------------------------------------------- word primitives (host)
    @_op
    def next_u64(self):
        return self.buffer.take_u64()

    @_op
    def next_u32(self):
        return self.buffer.take_u32()

    @_op
    def raw(self, nbytes):
        """rng.py:80-94: little-endian bytes; a trailing partial word is truncated.

        The byte pipe is ceil(nbytes / 8) u64 takes, i.e. a raw uint64 fill: from
        RAW_DEVICE_WORDS words on it runs on the device (same words, same position)."""
        nbytes = int(nbytes)
        if nbytes < 0:
            raise ValueError("byte count must be >= 0")
        words = (nbytes + 7) // 8
        if words >= RAW_DEVICE_WORDS:
            host = np.empty(words, dtype="<u8")
            self.device_fill("uint64", [], [0, 0], words, out=host)
            return host.view(np.uint8)[:nbytes].tobytes()
        full, rest = divmod(nbytes, 8)
        out = bytearray()
        for _ in range(full):
            out += pack("<Q", self.buffer.take_u64())
        if rest:
            out += pack("<Q", self.buffer.take_u64())[:rest]
        return bytes(out)

    @_op
    def u01(self):
        w = self.buffer.take_u64()
        if self.full_mantissa:
            return (w >> 11) * 1.1102230246251565e-16
        return unpack("<d", pack("<Q", (w >> 12) | 0x3FF0000000000000))[0] - 1.0

    @_op
    def u01f(self):
        w = self.buffer.take_u32()
        if self.full_mantissa:
            return (w >> 8) * 5.9604644775390625e-08
        return float(unpack("<f", pack("<I", (w >> 9) | 0x3F800000))[0]) - 1.0

    # ---------------------------------------------------------------- seeding / streams
    @_op
    def seed(self, entropy_words, spawn_key=()):
        seeding.seed_engine(self.engine, entropy_words, spawn_key)
        self.buffer.reset()
        self.entropy_source = "seed"
        self.entropy_degraded = False

    @_op
    def randomize(self):
        words, source, degraded = seeding.random_entropy()
        seeding.seed_engine(self.engine, words)
        self.buffer.reset()
        self.entropy_source = source
        self.entropy_degraded = degraded
        return source, degraded

    @_op
    def jump(self, k):
        """rng.py:135-164: x256 / x128+ / xoro families 2^k steps (k in the committed
        table), pcg64 advance(2^k), ranlux++ x*A^(2^k); others raise."""
        k = int(k)
        eid = self.engine_id
        if eid in _POLY_JUMP:
            if k not in STANDARD_JUMPS + (253,):
                raise ValueError("no jump polynomial for family 'x256' at 2^%d" % k)
        elif eid in _NARROW_JUMP:  # jumps.py:179-188
            if k not in _NARROW_JUMPS:
                raise ValueError("no jump polynomial for family %r at 2^%d" % (_NARROW_JUMP[eid], k))
        elif eid in ("pcg64", "ranlux++"):
            if k not in STANDARD_JUMPS:
                raise ValueError("%s jump exponent must be one of %s" % (eid, STANDARD_JUMPS))
        else:
            raise ValueError("jump unsupported for engine %s" % eid)
        st = _lib.u64_array(self.engine.s, 32)
        _lib.check(_lib.lib.rs_engine_jump(self.engine.native, st, k))
        self.engine.s = [int(st[i]) for i in range(self.engine.STATE_WORDS)]
        self.buffer.reset()

    @_op
    def advance(self, delta):
        if self.engine_id != "pcg64":
            raise ValueError("advance unsupported for engine %s" % self.engine_id)
        d = int(delta) & ((1 << 128) - 1)
        st = _lib.u64_array(self.engine.s, 32)
        _lib.check(_lib.lib.rs_pcg_advance(st, d & MASK64, d >> 64))
        self.engine.s = [int(st[i]) for i in range(4)]
        self.buffer.reset()

    @_op
    def set_stream(self, words):
        eid = self.engine_id
        if eid not in _STREAM_METHODS:
            raise ValueError("stream selection unsupported for engine %s; use jumps or spawn keys" % eid)
        method, nwords = _STREAM_METHODS[eid]
        if len(words) != nwords:
            raise ValueError("%s stream selector takes %d words, got %d" % (eid, nwords, len(words)))
        getattr(self.engine, method)([int(w) & MASK64 for w in words])
        self.buffer.reset()

    # ---------------------------------------------------------------- state / modes
    @_op
    def get_state(self):
        return self.engine.get_state()

    @_op
    def set_state(self, words):
        self.engine.set_state(words)
        self.buffer.reset()

    @_op
    def set_bitexact(self, flag):
        self.bitexact = bool(flag)

    @_op
    def set_full_mantissa(self, flag):
        self.full_mantissa = bool(flag)

    @_op
    def duplicate(self):
        other = Rng(engines.make(self.engine_id))
        other.engine.s = list(self.engine.s)
        other.buffer.restore(self.buffer.capture())
        other.bitexact = self.bitexact
        other.full_mantissa = self.full_mantissa
        other.counters = {k: dict(v) for k, v in self.counters.items()}
        other.device = self.device
        return other

    # ---------------------------------------------------------------- device boundary
    def to_stream(self):
        """The generator's logical position as an rs_stream (C ABI struct)."""
        s = _lib.RsStream()
        s.engine = self.engine.native
        s.full_mantissa = int(self.full_mantissa)
        s.bitexact = int(self.bitexact)
        s.has_pending = 0 if self.buffer.pending is None else 1
        s.pending = self.buffer.pending or 0
        for i, w in enumerate(self.engine.s):
            s.state[i] = w
        words = self.buffer.words
        for i, w in enumerate(words):
            s.buf[i] = w
        s.fill = len(words)
        s.cursor = self.buffer.cursor
        return s

    def from_stream(self, s):
        self.engine.s = [int(s.state[i]) for i in range(self.engine.STATE_WORDS)]
        self.buffer.words = [int(s.buf[i]) for i in range(s.fill)]
        self.buffer.cursor = int(s.cursor)
        self.buffer.pending = int(s.pending) if s.has_pending else None

    def _device(self):
        if self.device is not None:
            return torch.device(self.device)
        if not torch.cuda.is_available():
            raise _lib.LibraryError("no CUDA device: the fill path runs only on the GPU")
        return torch.device("cuda", torch.cuda.current_device())

    def _add_tallies(self, res):
        for i, name in enumerate(_TALLY_NAMES):
            if res.tally_seen[i]:
                c = self.counters.setdefault(name, {"attempts": 0, "pdf_evals": 0})
                c["attempts"] += int(res.tally[2 * i])
                c["pdf_evals"] += int(res.tally[2 * i + 1])

    def device_fill(self, dist, fparams, iparams, n, out=None):
        """Run rs_fill for `n` samples of a validated device distribution."""
        n = int(n)
        if n == 0 and out is None:  # nothing is consumed (continuous.py:422-427 runs zero times)
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
            return torch.empty(0, dtype=_out_dtype(dist), device=dev)
        if out is None:
            dev = self._device()
            out = torch.empty(n, dtype=_out_dtype(dist), device=dev)
        # rs_fill writes n * (the law's element size) bytes: the caller's buffer must hold
        # exactly that element type, or the fill would run past its end
        want = _out_dtype(dist)
        if isinstance(out, torch.Tensor):
            if out.dtype != want:
                raise ValueError("out must have dtype %s for %s (got %s)" % (want, dist, out.dtype))
            if out.numel() < n or not out.is_contiguous():
                raise ValueError("out must be a contiguous tensor with at least n elements")
            ptr = out.data_ptr()
            stream = _cuda_stream_ptr(out.device) if out.is_cuda else ctypes.c_void_p(0)
        else:  # numpy host array (the e2e path: the library stages through device memory)
            arr = out
            want_np = _NP_OUT[want]
            if not isinstance(arr, np.ndarray) or arr.dtype.newbyteorder("=") != want_np:
                raise ValueError("out must be a numpy array of dtype %s for %s" % (np.dtype(want_np), dist))
            if arr.size < n or not arr.flags["C_CONTIGUOUS"]:
                raise ValueError("out must be a contiguous array with at least n elements")
            ptr = arr.ctypes.data
            stream = _cuda_stream_ptr(self._device())
        st = self.to_stream()
        res = _lib.RsFillResult()
        fp = (ctypes.c_double * 4)(*(list(fparams) + [0.0] * (4 - len(fparams))))
        ip = _lib.u64_array(list(iparams), 4)
        _lib.check(_lib.lib.rs_fill(ctypes.byref(st), _lib.DIST_IDS[dist], fp, ip, n, ctypes.c_void_p(ptr),
                                    ctypes.byref(res), stream))
        self.from_stream(st)
        self._add_tallies(res)
        self.last_fill = res
        return out

    # ---------------------------------------------------------------- fill (the hot path)
    @_op
    def fill(self, dist, params=None, n=1, out=None):
        """n draws of a named distribution on the GPU (rng.py:223-241).

        Returns a 1-D device tensor (uint64 / float64; float32 for the 32-bit-half
        laws u01f/uniff/normf/expf; uint32 for uint8/16/32; int32 / int64 for
        int / long_long); `.tolist()` gives the reference's list. `out` may be a
        device tensor or a host numpy array (staged through device memory)."""
        params = dict(params or {})
        if dist in ("perm", "sample"):
            raise NotImplementedError("%s draws are sequences, not bulk fills; not on the B200 fill path" % dist)
        n = int(n)
        if n < 0:
            raise ValueError("draw count must be >= 0")
        if n >= _SERIAL_WARN_N and self.engine_id in _SERIAL_ENGINES:
            _warn_serial(self.engine_id)
        if dist in SCALAR_NAMES:
            fp = self._continuous_params(dist, params, n)
            return self.device_fill(dist, fp, [], n, out)
        if dist in DISCRETE_NAMES:
            ip = self._discrete_params(dist, params, n)
            return self.device_fill(dist, [], ip, n, out)
        raise ValueError("unknown discrete distribution %r" % dist)

    def _discrete_params(self, dist, params, n):
        """discrete.py:103-118 + bounded_uint/bounded_int checks (per call, so n >= 1 only)."""
        if dist in _WIDTH:
            width = _WIDTH[dist]
            b = int(params.get("b", 0))
            if n > 0 and (b < 0 or b > (1 << width)):
                raise ValueError("bound must be in [0, 2^%d]" % width)
            if width == 64:
                return [0, 1, 0, 0] if b == 1 << 64 else [b, 0, 0, 0]
            return [b, width, 0, 0]
        width = 32 if dist == "int" else 64
        half = 1 << (width - 1)
        m, hi = int(params.get("m", -half)), int(params.get("n", half - 1))
        if n > 0 and not (-half <= m <= hi <= half - 1):
            raise ValueError("range [%d, %d] does not fit a signed %d-bit span" % (m, hi, width))
        span = hi - m + 1
        full = 1 if span == 1 << width else 0
        return [0 if full else span, width, m & MASK64, full]

    def _continuous_params(self, dist, params, n):
        """Reference validation order (continuous.py:413-431 + sampler bodies): the
        numpy-vectorised transform path (default mode) validates its parameters even
        for n == 0 (continuous.py:364-410); every other sampler validates per call, i.e.
        nothing for n == 0, then bad keywords -> 'bad parameters', then its own value
        checks -- always before any word is consumed."""
        vec = dist in _TRANSFORMED and not self.bitexact
        if vec:
            return self._vectorized_params(dist, params)
        if n == 0:
            return [0.0] * 4
        allowed, required = _SIGNATURES[dist]
        if any(k not in allowed for k in params) or any(k not in params for k in required):
            raise ValueError("bad parameters for %s: %r" % (dist, sorted(params)))
        g = params.get
        if dist in ("u01", "u01f"):
            return [0.0] * 4
        if dist in ("unif", "uniff"):
            a, b = float(g("a", 0.0)), float(g("b", 1.0))
            if not b > a:
                raise ValueError("%s needs b > a" % dist)
            return [a, b, 0.0, 0.0]
        if dist in ("norm", "normf", "lognormal"):
            mu, var = float(g("mu", 0.0)), float(g("var", 1.0))
            if not var >= 0.0:  # lognormal = det_exp(norm(...)) checks as "normal"
                raise ValueError("%s variance must be >= 0" % ("normf" if dist == "normf" else "normal"))
            return [mu, var, 0.0, 0.0]
        if dist in ("exp", "expf"):
            beta = float(g("beta", 1.0))
            if not beta > 0.0:
                raise ValueError("exponential scale must be > 0" if dist == "exp" else "expf scale must be > 0")
            return [beta, 0.0, 0.0, 0.0]
        if dist == "gamma":
            alpha, theta = float(params["alpha"]), float(g("theta", 1.0))
            if not alpha > 0.0:
                raise ValueError("gamma shape must be > 0")
            if not theta > 0.0:
                raise ValueError("gamma scale must be > 0")
            return [alpha, theta, 0.0, 0.0]
        if dist == "beta":
            a, b = float(params["a"]), float(params["b"])
            if not a > 0.0:
                raise ValueError("gamma shape must be > 0")
            if not b > 0.0:
                # beta draws gamma(a) before gamma(b) raises (continuous.py:215-218):
                # consume exactly that one gamma(a) sample, then fail.
                self.device_fill("gamma", [a, 1.0], [], 1)
                raise ValueError("gamma shape must be > 0")
            return [a, b, 0.0, 0.0]
        if dist in ("chi2", "t"):
            nu = float(params["nu"])
            if not nu > 0.0:
                raise ValueError("%s degrees of freedom must be > 0" % dist)
            return [nu, 0.0, 0.0, 0.0]
        if dist == "f":
            nu1, nu2 = float(params["nu1"]), float(params["nu2"])
            if not (nu1 > 0.0 and nu2 > 0.0):
                raise ValueError("f degrees of freedom must be > 0")
            return [nu1, nu2, 0.0, 0.0]
        if dist == "skew_normal":
            alpha, mu, sigma = float(g("alpha", 0.0)), float(g("mu", 0.0)), float(g("sigma", 1.0))
            if not sigma > 0.0:
                raise ValueError("skew_normal scale must be > 0")
            return [alpha, mu, sigma, 0.0]
        return self._vectorized_params(dist, params)  # bitexact transforms: same checks

    @staticmethod
    def _vectorized_params(dist, params):
        """_fill_vectorized's parameter reading (continuous.py:364-410): unknown keys are
        ignored, a missing required key raises KeyError, checks run even for n == 0."""
        g = params.get
        if dist == "lognormal":
            mu, var = float(g("mu", 0.0)), float(g("var", 1.0))
            if not var >= 0.0:
                raise ValueError("lognormal variance must be >= 0")
            return [mu, var, 0.0, 0.0]
        if dist == "gumbel":
            mu, b = float(g("mu", 0.0)), float(g("beta", 1.0))
            if not b > 0.0:
                raise ValueError("gumbel scale must be > 0")
            return [mu, b, 0.0, 0.0]
        if dist == "pareto":
            alpha, xm = float(params["alpha"]), float(g("xm", 1.0))
            if not (alpha > 0.0 and xm > 0.0):
                raise ValueError("pareto needs alpha > 0 and xm > 0")
            return [alpha, xm, 0.0, 0.0]
        if dist == "weibull":
            k, lam = float(params["k"]), float(g("lam", 1.0))
            if not (k > 0.0 and lam > 0.0):
                raise ValueError("weibull needs k > 0 and lambda > 0")
            return [k, lam, 0.0, 0.0]
        xi, mu, sigma = float(params["xi"]), float(g("mu", 0.0)), float(g("sigma", 1.0))  # gpd
        if not sigma > 0.0:
            raise ValueError("gpd scale must be > 0")
        return [xi, mu, sigma, 0.0]

    # ---------------------------------------------------------------- scalar conveniences
    @_op
    def unif(self, a=0.0, b=1.0):
        a, b = float(a), float(b)
        if not b > a:
            raise ValueError("unif needs b > a")
        return a + self.u01() * (b - a)

    @_op
    def norm(self, mu=0.0, var=1.0):
        return float(self.fill("norm", {"mu": mu, "var": var}, 1)[0].item())

    @_op
    def expo(self, beta=1.0):
        return float(self.fill("exp", {"beta": beta}, 1)[0].item())

    @_op
    def gamma(self, alpha, theta=1.0):
        return float(self.fill("gamma", {"alpha": alpha, "theta": theta}, 1)[0].item())

    @_op
    def bounded_uint(self, b, width=64):
        if width != 64:
            raise NotImplementedError("only 64-bit bounded draws are on the B200 fill path")
        return int(self.fill("uint64", {"b": b}, 1).tolist()[0])

    @_op
    def mvn(self, mean, cov, n=1, layout="n_d"):
        """continuous.py:312-336: X = mean + z @ L^T, z = n*d std_norm draws (row-major),
        L = Cholesky factor (pivoted LAPACK fallback for semidefinite S).

        The host checks symmetry and factorises S on a worker thread while the device draws z
        (numpy and LAPACK release the GIL, and so does the ctypes fill); the contraction
        (rs_mvn_apply_rows) is queued on the current stream once the factor is ready."""
        mean = np.asarray(mean, dtype=np.float64)
        cov = np.asarray(cov, dtype=np.float64)
        if mean.ndim != 1 or cov.shape != (mean.size, mean.size):
            raise ValueError("mvn needs a length-d mean and a d x d covariance")

        def symmetric():
            if not np.allclose(cov, cov.T, rtol=1e-9, atol=1e-12):
                raise ValueError("mvn covariance must be symmetric")

        # the reference's error order: symmetry, layout, n (an earlier error wins)
        if layout not in ("n_d", "d_n"):
            symmetric()
            raise ValueError("mvn layout must be 'n_d' or 'd_n'")
        try:
            n = int(n)
        except Exception:
            symmetric()
            raise
        if n < 1:
            symmetric()
            raise ValueError("mvn needs n >= 1")
        d = mean.size
        dev = self._device()

        def factorise():
            f = np.ascontiguousarray(semidefinite_factor(cov))
            return f, not np.triu(f, 1).any()

        out = torch.empty((n, d) if layout == "n_d" else (d, n), dtype=torch.float64, device=dev)
        z = torch.empty(n * d, dtype=torch.float64, device=dev)
        # The reference factorises before drawing (continuous.py:331), so a failed
        # factorisation puts the generator back where it was: nothing observable is consumed.
        before = (list(self.engine.s), self.buffer.capture(), {k: dict(v) for k, v in self.counters.items()})
        # (two host workers: the symmetry check and the factorisation each take about as long
        # as half the z fill at d = 512; its error is the earlier one in the reference's order)
        fsym = _host_pool().submit(symmetric)
        fut = _host_pool().submit(factorise)
        try:
            self.device_fill("stdnorm", [], [], n * d, out=z)
        finally:
            try:
                sym_err = fsym.exception()
                if sym_err is not None:
                    fut.cancel()
                    try:
                        fut.result()  # (let a running factorisation finish before the state is restored)
                    except Exception:
                        pass
                    raise sym_err
                factor, lower = fut.result()
            except Exception:
                self.engine.s, self.counters = before[0], before[2]
                self.buffer.restore(before[1])
                raise
        Ld = torch.from_numpy(factor).to(dev)
        md = torch.from_numpy(np.ascontiguousarray(mean)).to(dev)
        _lib.check(_lib.lib.rs_mvn_apply_rows(
            ctypes.c_void_p(Ld.data_ptr()), ctypes.c_void_p(md.data_ptr()), d, 1 if lower else 0, n,
            ctypes.c_void_p(z.data_ptr()), 0 if layout == "n_d" else 1, ctypes.c_void_p(out.data_ptr()), n,
            _cuda_stream_ptr(dev)))
        return out


_POOL = None


def _host_pool():
    """Two worker threads for host work that overlaps a device fill (mvn's symmetry check and factorisation)."""
    global _POOL
    if _POOL is None:
        import concurrent.futures

        _POOL = concurrent.futures.ThreadPoolExecutor(2, thread_name_prefix="randstream-host")
    return _POOL


def semidefinite_factor(cov):
    """continuous.py:293-309: numpy Cholesky, else pivoted dpstrf + reconstruction check."""
    try:
        return np.linalg.cholesky(cov)
    except np.linalg.LinAlgError:
        from scipy.linalg.lapack import dpstrf

        c, piv, rank, info = dpstrf(cov, lower=1)
        if info < 0:
            raise ValueError("covariance factorization failed")
        low = np.tril(c)
        low[:, rank:] = 0.0
        m = np.zeros_like(low)
        m[piv - 1, :] = low
        scale = max(1.0, float(np.abs(cov).max()))
        if not np.allclose(m @ m.T, cov, rtol=0.0, atol=1e-8 * scale):
            raise ValueError("mvn covariance must be positive semidefinite")
        return m


def fill_streams(engine, seed, spawn_prefix, j0, n_streams, dist, params, n_per_stream, device=None, out=None):
    """Per-stream mode: row s = create(engine, seed, spawn_key=prefix + (j0 + s,)).fill(dist, params, n)
    for s < n_streams, computed by one GPU thread per stream (sfc64's parallel form).
    `out`: an optional contiguous CUDA tensor of shape (n_streams, n_per_stream) and the
    law's dtype to fill in place (returned)."""
    eid = engines.normalize(engine)
    params = dict(params or {})
    n_streams, n_per_stream = int(n_streams), int(n_per_stream)
    probe = Rng(engines.make(eid))
    if dist in DISCRETE_NAMES:
        fp, ip = [0.0] * 4, probe._discrete_params(dist, params, 1)
    else:
        fp, ip = probe._continuous_params(dist, params, 1), [0, 0, 0, 0]
    if out is not None:
        if (not out.is_cuda or not out.is_contiguous() or tuple(out.shape) != (n_streams, n_per_stream)
                or out.dtype != _out_dtype(dist)):
            raise ValueError("out must be a contiguous CUDA tensor of shape (n_streams, n_per_stream) and dtype %s"
                             % _out_dtype(dist))
        dev = out.device
    else:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        out = torch.empty((n_streams, n_per_stream), dtype=_out_dtype(dist), device=dev)
    seedw = [int(w) & MASK64 for w in seed]
    pre = [int(w) & MASK64 for w in spawn_prefix]
    _lib.check(_lib.lib.rs_fill_streams(engines.NATIVE_ID[eid], _lib.u64_array(seedw), len(seedw),
                                        _lib.u64_array(pre), len(pre), int(j0), n_streams, _lib.DIST_IDS[dist],
                                        (ctypes.c_double * 4)(*fp[:4]), _lib.u64_array(ip, 4), n_per_stream,
                                        ctypes.c_void_p(out.data_ptr()), _cuda_stream_ptr(dev)))
    return out
