"""ctypes binding of librandstream_b200.so (the C ABI in include/randstream_b200.h).

The product has no CPU fallback: if the shared library is missing or cannot be
loaded, importing the package raises. Build it with `make -C paper_2605_05099_b200`
(or `python -c "import __graft_entry__ as g; g.build()"`).
"""

import ctypes
import os
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ.get("RANDSTREAM_B200_LIB", HERE / "librandstream_b200.so"))  # override: A/B builds

CAP = 144

RS_OK, RS_ERR_VALUE, RS_ERR_UNSUPPORTED, RS_ERR_CUDA, RS_ERR_INTERNAL = range(5)

DIST_IDS = {"uint64": 1, "u01": 2, "u01f": 3, "norm": 4, "exp": 5, "gamma": 6, "beta": 7, "stdnorm": 8,
            "unif": 9, "uniff": 10, "normf": 11, "expf": 12, "lognormal": 13, "chi2": 14, "t": 15, "f": 16,
            "gumbel": 17, "pareto": 18, "gpd": 19, "weibull": 20, "skew_normal": 21,
            "uint8": 22, "uint16": 22, "uint32": 22, "int": 23, "long_long": 24}

U64P = ctypes.POINTER(ctypes.c_uint64)
DBLP = ctypes.POINTER(ctypes.c_double)


class RsStream(ctypes.Structure):
    _fields_ = [
        ("engine", ctypes.c_int32),
        ("full_mantissa", ctypes.c_int32),
        ("bitexact", ctypes.c_int32),
        ("has_pending", ctypes.c_int32),
        ("pending", ctypes.c_uint64),
        ("state", ctypes.c_uint64 * 32),
        ("buf", ctypes.c_uint64 * CAP),
        ("fill", ctypes.c_int32),
        ("cursor", ctypes.c_int32),
    ]


class RsFillResult(ctypes.Structure):
    _fields_ = [
        ("words_consumed", ctypes.c_uint64),
        ("tally", ctypes.c_uint64 * 6),
        ("tally_seen", ctypes.c_int32 * 3),
        ("resync_rounds", ctypes.c_int32),
        ("chunks", ctypes.c_uint64),
    ]


class RsDistInfo(ctypes.Structure):
    _fields_ = [
        ("unit", ctypes.c_int32),
        ("variable", ctypes.c_int32),
        ("words_per_sample", ctypes.c_double),
        ("min_seg_len", ctypes.c_uint64),
        ("tally_seen", ctypes.c_int32 * 3),
        ("pad", ctypes.c_int32),
    ]


class RsRangeInfo(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_uint64),
        ("exit", ctypes.c_uint64),
        ("end_pos", ctypes.c_uint64),
        ("tally", ctypes.c_uint64 * 6),
        ("unit", ctypes.c_int32),
        ("resync_rounds", ctypes.c_int32),
    ]


RANGE_ALIGN = 72  # RS_RANGE_ALIGN


class LibraryError(RuntimeError):
    pass


def _load():
    if not LIB_PATH.exists():
        raise LibraryError(
            "librandstream_b200.so is not built (%s); run `make -C %s`. "
            "There is no CPU fallback for the fill path." % (LIB_PATH, HERE))
    L = ctypes.CDLL(str(LIB_PATH))
    L.rs_abi_version.restype = ctypes.c_int32
    L.rs_last_error.restype = ctypes.c_char_p
    L.rs_init_device.argtypes = [ctypes.c_int32]
    L.rs_engine_supported.argtypes = [ctypes.c_int32]
    L.rs_engine_state_words.argtypes = [ctypes.c_int32]
    L.rs_engine_seed_words.argtypes = [ctypes.c_int32]
    L.rs_engine_chunk.argtypes = [ctypes.c_int32]
    L.rs_seed_words.argtypes = [U64P, ctypes.c_int32, U64P, ctypes.c_int32, U64P, ctypes.c_int32]
    L.rs_engine_seed.argtypes = [ctypes.c_int32, U64P, ctypes.c_int32, U64P, ctypes.c_int32, U64P]
    L.rs_engine_seed_from.argtypes = [ctypes.c_int32, U64P, U64P]
    L.rs_engine_check_state.argtypes = [ctypes.c_int32, U64P]
    L.rs_engine_generate.argtypes = [ctypes.c_int32, U64P, U64P, ctypes.c_int32]
    L.rs_engine_jump.argtypes = [ctypes.c_int32, U64P, ctypes.c_int32]
    L.rs_engine_advance_words.argtypes = [ctypes.c_int32, U64P, ctypes.c_uint64, ctypes.c_uint64]
    L.rs_pcg_advance.argtypes = [U64P, ctypes.c_uint64, ctypes.c_uint64]
    L.rs_fill.argtypes = [ctypes.POINTER(RsStream), ctypes.c_int32, DBLP, U64P, ctypes.c_uint64, ctypes.c_void_p,
                          ctypes.POINTER(RsFillResult), ctypes.c_void_p]
    L.rs_fill_async.argtypes = [ctypes.POINTER(RsStream), ctypes.c_int32, DBLP, U64P, ctypes.c_uint64,
                                ctypes.c_void_p, ctypes.c_void_p]
    L.rs_fill_streams.argtypes = [ctypes.c_int32, U64P, ctypes.c_int32, U64P, ctypes.c_int32, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_int32, DBLP, U64P, ctypes.c_uint64, ctypes.c_void_p,
                                  ctypes.c_void_p]
    L.rs_mvn.argtypes = [ctypes.POINTER(RsStream), ctypes.c_void_p, DBLP, ctypes.c_int64, ctypes.c_uint64,
                         ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(RsFillResult), ctypes.c_void_p]
    L.rs_mvn_apply.argtypes = [ctypes.c_void_p, DBLP, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.rs_mvn_apply.restype = ctypes.c_int
    if hasattr(L, "rs_mvn_apply_rows"):  # (absent from older builds used in A/B timing)
        L.rs_mvn_apply_rows.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_void_p]
        L.rs_mvn_apply_rows.restype = ctypes.c_int
    L.rs_dist_info.argtypes = [ctypes.c_int32, DBLP, U64P, ctypes.POINTER(RsDistInfo)]
    L.rs_range_geometry.argtypes = [ctypes.c_int32, ctypes.c_int32, DBLP, U64P, ctypes.c_uint64, U64P,
                                    ctypes.POINTER(ctypes.c_uint32)]
    L.rs_range_count.argtypes = [ctypes.POINTER(RsStream), ctypes.c_int32, DBLP, U64P, ctypes.c_uint64,
                                 ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(RsRangeInfo), ctypes.c_void_p]
    L.rs_range_count_warm.argtypes = [ctypes.POINTER(RsStream), ctypes.c_int32, DBLP, U64P, ctypes.c_uint32,
                                      ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(RsRangeInfo), ctypes.c_void_p]
    L.rs_range_emit.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(RsRangeInfo), ctypes.c_void_p]
    for name in ("rs_dist_info", "rs_range_geometry", "rs_range_count", "rs_range_count_warm", "rs_range_emit"):
        getattr(L, name).restype = ctypes.c_int
    for name in ("rs_init_device", "rs_seed_words", "rs_engine_seed", "rs_engine_seed_from", "rs_engine_check_state",
                 "rs_engine_generate", "rs_engine_jump", "rs_engine_advance_words", "rs_pcg_advance", "rs_fill",
                 "rs_fill_async", "rs_fill_streams", "rs_mvn"):
        getattr(L, name).restype = ctypes.c_int
    for name in ("rs_engine_supported", "rs_engine_state_words", "rs_engine_seed_words", "rs_engine_chunk"):
        getattr(L, name).restype = ctypes.c_int32
    return L


lib = _load()

EXPORTED = (
    "rs_abi_version", "rs_last_error", "rs_init_device", "rs_engine_supported", "rs_engine_state_words",
    "rs_engine_seed_words", "rs_engine_chunk", "rs_seed_words", "rs_engine_seed", "rs_engine_seed_from",
    "rs_engine_check_state", "rs_engine_generate", "rs_engine_jump", "rs_engine_advance_words", "rs_pcg_advance",
    "rs_fill", "rs_fill_async", "rs_fill_streams", "rs_mvn", "rs_mvn_apply", "rs_mvn_apply_rows",
    "rs_dist_info", "rs_range_geometry", "rs_range_count", "rs_range_count_warm", "rs_range_emit",
)


def last_error():
    return (lib.rs_last_error() or b"").decode()


def check(status):
    """Map an rs_status to the reference's exception types (ValueError for bad input)."""
    if status == RS_OK:
        return
    msg = last_error() or "status %d" % status
    if status == RS_ERR_VALUE:
        if "stream exhausted" in msg:  # chacha20's 32-bit block counter, counter.py:212-213
            raise OverflowError("stream exhausted")
        raise ValueError(msg)
    if status == RS_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise LibraryError(msg)


def u64_array(vals, n=None):
    vals = [int(v) & 0xFFFFFFFFFFFFFFFF for v in vals]
    size = max(1, n if n is not None else len(vals))
    arr = (ctypes.c_uint64 * size)()
    for i, v in enumerate(vals):
        arr[i] = v
    return arr
