"""Pin the C oracle (oracle/oracle.c) against vectors produced by the
reference itself (tests/golden/make_golden.py). CPU only."""
import hashlib
import struct

import numpy as np
import pytest

from oracle import oracle as O
from conftest import golden_params, is_vectorized, vec_close


def _h(words):
    return [int(w, 16) for w in words]


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _run_pre(o, pre):
    for op in pre:
        for _ in range(op[1]):
            (o.next_u64 if op[0] == "u64" else o.next_u32)()


def test_engine_kats(golden):
    assert {k["engine"] for k in golden["kats"]} >= {"x256**", "pcg64", "philox", "sfc64", "ranlux++"}
    for k in golden["kats"]:
        if k["how"] == "set_state":
            words, st = O.engine_generate(k["engine"], _h(k["words"]), len(k["expect"]))
        else:
            o = O.OracleRng(k["engine"], seed=[1])
            # seed_from path: ranlux++ residue reduction (src/engines/ranlux.py:106-110)
            x = sum(w << (64 * i) for i, w in enumerate(_h(k["words"]))) % ((1 << 576) - (1 << 240) + 1) or 1
            st0 = [(x >> (64 * i)) & (2 ** 64 - 1) for i in range(9)]
            words, st = O.engine_generate(k["engine"], st0, len(k["expect"]))
        assert words == _h(k["expect"]), k["engine"]


@pytest.mark.parametrize("which", ["det_exp", "det_log"])
def test_detmath_bits(golden, which):
    fn = O.det_exp if which == "det_exp" else O.det_log
    bad = [(x, w) for x, w in golden[which] if _bits(fn(float.fromhex(x))) != int(w, 16)]
    assert not bad, bad[:5]


def test_seeding(golden):
    for s in golden["seeding"]:
        got = O.seed_words(_h(s["entropy"]), _h(s["spawn"]), 9)
        assert got == _h(s["words"])


def test_jump_polynomials(golden):
    p = O.x256_charpoly()
    assert p == int(golden["x256_charpoly"], 16)
    for k, poly in golden["x256_jump_polys"].items():
        assert O.x_pow2k_mod(int(k), p) == int(poly, 16)
    for n, poly in golden["x256_x_pow_mod"].items():
        assert O.x_pow_mod(int(n), p) == int(poly, 16)


def test_jumped_states(golden):
    p = O.x256_charpoly()
    for j in golden["jumps"]:
        o = O.OracleRng(j["engine"], seed=[77])
        o.next_u64()
        st = o.get_state()
        if "advance" in j:
            st = O.pcg_advance(O.OracleRng("pcg64", seed=[77]).get_state(), int(j["advance"]))
        elif j["engine"] in ("x256**", "x256++"):
            st = O.x256_apply_poly(st, O.x_pow2k_mod(j["k"], p))
        elif j["engine"] == "pcg64":
            st = O.pcg_advance(st, 1 << j["k"])
        elif j["engine"] in ("x128+", "xoro++"):
            st = O.x128_jump(j["engine"], st, j["k"])
        else:
            st = O.ranlux_jump(st, j["k"])
        assert st == _h(j["state"]), j
        o.set_state(st)
        assert [o.next_u64() for _ in range(5)] == _h(j["next"])


def _fill_cases(golden, large):
    for rec in golden["fills"]:
        if (rec["n"] > 70000) == large:
            yield rec


def _check_fill(rec, golden_arrays):
    o = O.OracleRng(rec["engine"] or "x256++simd", seed=rec["seed"], spawn_key=tuple(rec["spawn"]),
                    full_mantissa=rec["full_mantissa"])
    assert o.get_state() == _h(rec["start_state"])
    _run_pre(o, rec["pre"])
    out = o.fill(rec["dist"], golden_params(rec), rec["n"])
    if is_vectorized(rec):  # reference default mode uses numpy exp/log: 4-ulp bar
        assert vec_close(out, golden_arrays[rec["name"]]), rec["name"]
    else:
        assert hashlib.sha256(out.tobytes()).hexdigest() == rec["sha256"], rec["name"]
    if rec["name"] in golden_arrays and not is_vectorized(rec):
        assert np.array_equal(out.view(np.uint8), golden_arrays[rec["name"]].view(np.uint8))
    words, cursor, pending = o.buffer()
    assert o.get_state() == _h(rec["final_state"])
    assert hashlib.sha256(np.asarray(words, dtype=np.uint64).tobytes()).hexdigest() == rec["buffer_sha256"]
    assert cursor == rec["cursor"]
    assert (None if pending is None else "%08x" % pending) == rec["pending"]
    assert o.tallies() == rec["tallies"]


def test_fills_small(golden, golden_arrays):
    n = 0
    for rec in _fill_cases(golden, large=False):
        _check_fill(rec, golden_arrays)
        n += 1
    assert n > 100


def test_fills_large(golden, golden_arrays):
    for rec in _fill_cases(golden, large=True):
        _check_fill(rec, golden_arrays)


def test_mvn_z_and_x(golden, golden_arrays):
    m = golden["mvn"]
    d, n = m["d"], m["n"]
    o = O.OracleRng("philox", seed=m["seed"])
    A = o.fill("norm", {}, d * d).reshape(d, d)
    S = A @ A.T / d + np.eye(d)
    assert np.array_equal(S, golden_arrays["mvn_S"])
    L = np.linalg.cholesky(S)
    z = o.fill("stdnorm", {}, n * d).reshape(n, d)
    X = z @ L.T
    ref = golden_arrays["mvn_X"]
    scale = np.abs(z) @ np.abs(L).T
    assert np.max(np.abs(X - ref) / scale) <= 1e-12
    assert o.get_state() == _h(m["final_state"])
