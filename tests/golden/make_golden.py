"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Imports the reference `randstream` package read-only from
/root/reference/pkg/src (pure Python; only importable in the build
container, never on the GPU box) and records, for every case below, what
the reference itself produces:

* fills: output (full array for small n, sha256 + head otherwise), final
  engine state, final 144-word buffer (sha256), cursor, pending half and the
  diagnostic tallies -- the state contract of src/buffer.py:29-60;
* engine known-answer vectors, restated from the reference's
  pkg/tests/golden/engines_kat.json (external oracles: rand_xoshiro, numpy);
* det_exp/det_log bit patterns (src/detmath.py) on a grid plus the frozen
  canaries of pkg/tests/test_detmath.py:131-152;
* SeedSequenceFE128 words (src/seeding.py) and the GF(2) jump polynomials
  (src/_tables/jump_polynomials.txt via src/jumps.py);
* jumped states (src/rng.py:135-171);
* one small multivariate-normal draw (src/continuous.py:312-336).

Run:  python tests/golden/make_golden.py      (takes about a minute)
"""

import hashlib
import json
import math
import pathlib
import random
import struct
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from randstream import continuous, detmath, jumps, seeding, state_io  # noqa: E402

HERE = pathlib.Path(__file__).resolve().parent
M64 = (1 << 64) - 1


def f64bits(vals):
    return np.asarray(vals, dtype=np.float64).view(np.uint64)


def out_array(dist, vals):
    if dist == "uint64":
        return np.asarray(vals, dtype=np.uint64)
    if dist in ("uint8", "uint16", "uint32"):
        return np.asarray(vals, dtype=np.uint32)
    if dist == "int":
        return np.asarray(vals, dtype=np.int32)
    if dist == "long_long":
        return np.asarray(vals, dtype=np.int64)
    if dist in ("u01f", "uniff", "normf", "expf"):
        return np.asarray(vals, dtype=np.float32)
    return np.asarray(vals, dtype=np.float64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def buf_sha(words):
    return hashlib.sha256(np.asarray(words, dtype=np.uint64).tobytes()).hexdigest()


# (name, engine, seed, spawn_key, full_mantissa, pre_ops, dist, params, n, keep_full)
# pre_ops: list of ("u64", k) | ("u32", k) | ("fill", dist, params, k) applied before the fill,
# so the fill starts mid-buffer (the hand-off of SURVEY 8(b)).
CASES = []


def case(name, engine, seed, dist, params, n, spawn=(), fm=False, pre=(), keep=None, bitexact=False):
    if keep is None:
        keep = n <= 20000
    CASES.append(dict(name=name, engine=engine, seed=list(seed), spawn=list(spawn), full_mantissa=fm,
                      pre=[list(p) for p in pre], dist=dist, params=params, n=n, keep=keep, bitexact=bitexact))


# BASELINE configs (prefix sizes the reference finishes in seconds)
case("c1_x256ss_raw_2p20", "x256**", [12345], "uint64", {}, 1 << 20, keep=False)
case("c1_x256ss_raw_4096", "x256**", [12345], "uint64", {}, 4096)
case("c2_philox_u01_fm", "philox", [7], "u01", {}, 1 << 16, fm=True, keep=False)
case("c2_philox_u01f_fm", "philox", [7], "u01f", {}, 1 << 16, fm=True, keep=False)
case("c2_philox_u01_fm_small", "philox", [7], "u01", {}, 4099, fm=True)
case("c2_philox_u01f_fm_small", "philox", [7], "u01f", {}, 4099, fm=True)
case("c3_x256ss_norm", "x256**", [2024], "norm", {}, 1 << 16, keep=False)
case("c3_pcg64_norm", "pcg64", [2024], "norm", {}, 1 << 16, keep=False)
case("c3_x256ss_norm_small", "x256**", [2024], "norm", {}, 5000)
case("c3_pcg64_norm_small", "pcg64", [2024], "norm", {}, 5000)
case("c4_pcg64_exp", "pcg64", [99], "exp", {}, 1 << 15, keep=False)
case("c4_pcg64_exp_small", "pcg64", [99], "exp", {}, 3000)
for k in (0.3, 1.0, 2.5, 10.0):
    case("c4_pcg64_gamma_%g" % k, "pcg64", [99], "gamma", {"alpha": k}, 1 << 14, keep=False)
    case("c4_pcg64_gamma_%g_small" % k, "pcg64", [99], "gamma", {"alpha": k}, 2000)
case("c4_pcg64_beta_2_5", "pcg64", [99], "beta", {"a": 2.0, "b": 5.0}, 1 << 14, keep=False)
case("c4_pcg64_beta_2_5_small", "pcg64", [99], "beta", {"a": 2.0, "b": 5.0}, 2000)
for m in (6, 1000003, (1 << 63) + 1):
    for j in (0, 1, 7, 65535):
        case("c5b_sfc64_b%d_j%d" % (m, j), "sfc64", [31], "uint64", {"b": m}, 4096, spawn=[j])
case("extra_ranlux_raw", "ranlux++", [12345], "uint64", {}, 1 << 14, keep=False)
case("extra_ranlux_raw_small", "ranlux++", [12345], "uint64", {}, 999)
# the library default engine (create() with no name): x256++simd
case("default_engine_raw", None, [2024], "uint64", {}, 1 << 16, keep=False)
case("default_engine_norm", None, [2024], "norm", {}, 1 << 16, keep=False)

# edge cases: empty / single / parameters / modes / mid-buffer starts
ENG = ("x256**", "x256++", "pcg64", "philox", "sfc64", "ranlux++", "x256++simd", "x256**simd", "sfc64simd",
       "x128+", "xoro++", "squares", "cwg128", "chacha20")
for e in ENG:
    tag = e.replace("+", "p").replace("*", "s")
    case("edge_%s_n0" % tag, e, [5], "norm", {}, 0)
    case("edge_%s_n1" % tag, e, [5], "norm", {}, 1)
    case("edge_%s_raw_mid" % tag, e, [6], "uint64", {}, 1000, pre=[("u64", 37)])
    case("edge_%s_raw_pending" % tag, e, [6], "uint64", {}, 301, pre=[("u32", 3)])
    case("edge_%s_u01f_pending" % tag, e, [6], "u01f", {}, 777, pre=[("u32", 1)])
    case("edge_%s_u01f_odd" % tag, e, [6], "u01f", {}, 289, pre=[("u64", 143)])
    case("edge_%s_u01_default" % tag, e, [8], "u01", {}, 500)
    case("edge_%s_u01f_default" % tag, e, [8], "u01f", {}, 501)
    case("edge_%s_norm_mid" % tag, e, [9], "norm", {"mu": 1.5, "var": 4.0}, 3000, pre=[("u64", 100)])
    case("edge_%s_norm_fm" % tag, e, [10], "norm", {}, 3000, fm=True)
    case("edge_%s_exp_beta" % tag, e, [11], "exp", {"beta": 2.5}, 3000, pre=[("u32", 1)])
    case("edge_%s_gamma_small_theta" % tag, e, [12], "gamma", {"alpha": 0.5, "theta": 3.0}, 1500, fm=True)
    case("edge_%s_gamma_3" % tag, e, [13], "gamma", {"alpha": 3.0}, 1500, pre=[("u64", 143)])
    case("edge_%s_beta" % tag, e, [14], "beta", {"a": 0.7, "b": 1.3}, 800)
    for b in (1, 2, 3, 1 << 32, (1 << 64) - 1, 1 << 64, 12345678901234567):
        case("edge_%s_bounded_%d" % (tag, b), e, [15], "uint64", {"b": b}, 400)
    case("edge_%s_stdnorm_tail" % tag, e, [16], "norm", {}, 40000, keep=False)
    case("edge_%s_exp_tail" % tag, e, [17], "exp", {}, 40000, keep=False)
# derived laws, transforms and narrower / signed integers
DERIVED = [("unif", {"a": -2.0, "b": 3.0}), ("unif", {}), ("uniff", {"a": -2.0, "b": 3.0}),
           ("normf", {"mu": 1.0, "var": 4.0}), ("normf", {}), ("expf", {"beta": 2.5}), ("expf", {}),
           ("lognormal", {"mu": 0.5, "var": 0.25}), ("chi2", {"nu": 3.0}), ("chi2", {"nu": 0.8}),
           ("t", {"nu": 5.0}), ("f", {"nu1": 3.0, "nu2": 7.0}), ("gumbel", {"mu": 1.0, "beta": 2.0}),
           ("pareto", {"alpha": 2.5}), ("gpd", {"xi": 0.3}), ("gpd", {"xi": -0.2, "sigma": 2.0}),
           ("gpd", {"xi": 0.0, "mu": 1.0}), ("weibull", {"k": 1.7}), ("skew_normal", {"alpha": 3.0, "mu": 1.0, "sigma": 2.0}),
           ("skew_normal", {}), ("uint8", {"b": 200}), ("uint8", {}), ("uint16", {"b": 1000}), ("uint16", {"b": 1024}),
           ("uint32", {"b": 3000000001}), ("uint32", {}), ("uint32", {"b": 1 << 32}), ("int", {"m": -5, "n": 17}),
           ("int", {}), ("int", {"m": -(1 << 31), "n": 0}), ("long_long", {"m": -10 ** 15, "n": 10 ** 18}),
           ("long_long", {}), ("long_long", {"m": 7, "n": 7 + (1 << 40) - 1})]
TRANSFORMED = ("lognormal", "gumbel", "pareto", "weibull", "gpd")
for e in ("x256**", "pcg64", "philox", "sfc64", "ranlux++", "x256++simd", "xoro++", "chacha20", "cwg128"):
    tag = e.replace("+", "p").replace("*", "s")
    for i, (dist, params) in enumerate(DERIVED):
        case("derived_%s_%s_%d" % (tag, dist, i), e, [100 + i], dist, params, 1500, pre=[("u32", 1)],
             fm=(i % 2 == 1), bitexact=True)
        if dist in TRANSFORMED:
            case("derived_%s_%s_%d_vec" % (tag, dist, i), e, [100 + i], dist, params, 1500, pre=[("u32", 1)])

# long runs for the diagnostic tallies (gate 04 reads them)
case("tally_sfc64_norm", "sfc64", [40401], "norm", {}, 1 << 18, keep=False)
case("tally_sfc64_exp", "sfc64", [40402], "exp", {}, 1 << 18, keep=False)


def run_pre(rng, pre):
    for op in pre:
        if op[0] == "u64":
            for _ in range(op[1]):
                rng.next_u64()
        elif op[0] == "u32":
            for _ in range(op[1]):
                rng.next_u32()


def run_case(c):
    rng = state_io.create(c["engine"], seed=c["seed"], spawn_key=tuple(c["spawn"]))
    rng.set_full_mantissa(c["full_mantissa"])
    rng.set_bitexact(c.get("bitexact", False))
    start_state = rng.get_state()
    run_pre(rng, c["pre"])
    vals = rng.fill(c["dist"], dict(c["params"]), c["n"])
    arr = out_array(c["dist"], vals)
    cap = rng.buffer.capture()
    rec = dict(c)
    rec["params"] = {k: (str(v) if isinstance(v, int) else v) for k, v in c["params"].items()}
    rec["start_state"] = ["%016x" % w for w in start_state]
    rec["sha256"] = sha(arr)
    rec["head"] = [("%016x" % int(v)) if arr.dtype == np.uint64 else float(v).hex() for v in arr[:16]]
    rec["final_state"] = ["%016x" % w for w in rng.get_state()]
    rec["buffer_sha256"] = buf_sha(cap["words"])
    rec["buffer_fill"] = cap["fill"]
    rec["cursor"] = cap["cursor"]
    rec["pending"] = None if cap["pending"] is None else "%08x" % cap["pending"]
    rec["tallies"] = rng.counters
    return rec, arr


def main():
    out = {"generated_by": "tests/golden/make_golden.py", "reference": REF}
    arrays = {}
    recs = []
    for c in CASES:
        rec, arr = run_case(c)
        if c["keep"]:
            arrays[c["name"]] = arr
        recs.append(rec)
        print("case", c["name"], rec["sha256"][:12])
    out["fills"] = recs

    # engine KATs restated from the reference's external-oracle vectors
    kat_src = json.loads(pathlib.Path("/root/reference/pkg/tests/golden/engines_kat.json").read_text())
    kats = []
    for e in kat_src:
        if e["engine"] in ENG:
            kats.append({"engine": e["engine"], "origin": e["source"],
                         "how": "seed_from" if "seed_words" in e else "set_state",
                         "words": e.get("seed_words", e.get("set_state")), "expect": e["expect"]})
    out["kats"] = kats

    # detmath: canaries (pkg/tests/test_detmath.py:131-152) + a random grid
    rnd = random.Random(20240615)
    xs_exp = [1.0, -0.5, 42.0, 1e-09, -700.25, 709.0, 0.0, -0.0, 1e-320, 700.0, -745.0, -744.4, 0.34657359027997264,
              0.34657359027997265, 1.0397207708399179, -1.0397207708399179, 7.09782712893383973096e+02]
    xs_exp += [rnd.uniform(-745, 709.7) for _ in range(3000)] + [rnd.uniform(-1, 1) for _ in range(2000)]
    xs_exp += [-0.5 * x * x for x in (rnd.uniform(0, 3.7) for _ in range(2000))]
    xs_log = [0.5, 1.0000009536743164, 3.141592653589793, 1e-300, 6.02e23, 2.0, 1.0, 5e-324, 2.2250738585072014e-308,
              1.7976931348623157e308, 0.9999999999999999, 1.0000000000000002]
    xs_log += [10 ** rnd.uniform(-320, 308) for _ in range(3000)] + [rnd.uniform(0, 2) for _ in range(3000)]
    xs_log += [1.0 - k * 2.0 ** -53 for k in range(1, 200)]
    out["det_exp"] = [[float(x).hex(), "%016x" % struct.unpack("<Q", struct.pack("<d", detmath.det_exp(x)))[0]]
                      for x in xs_exp]
    out["det_log"] = [[float(x).hex(), "%016x" % struct.unpack("<Q", struct.pack("<d", detmath.det_log(x)))[0]]
                      for x in xs_log]

    # seeding
    seeds = []
    for ent, key in (([42], ()), ([1, 2, 3], ()), ([7], (0, 4)), ([], (1,)), ([12345], ()), ([31], (65535,)),
                     ([2 ** 64 - 1, 0, 5, 6, 7], (3, 2, 1)), ([0], ())):
        seeds.append({"entropy": ["%016x" % w for w in ent], "spawn": ["%016x" % w for w in key],
                      "words": ["%016x" % w for w in seeding.derive_seed_words(9, list(ent), tuple(key))]})
    out["seeding"] = seeds

    # jumps
    p = jumps.characteristic_polynomial("x256")
    out["x256_charpoly"] = "%x" % p
    out["x256_jump_polys"] = {str(k): "%x" % jumps.jump_polynomial("x256", k) for k in (32, 64, 96, 128, 192, 253)}
    out["x256_x_pow_mod"] = {str(n): "%x" % jumps.x_pow_mod(n, p) for n in (1, 1000, 10 ** 6, 144 * 7919, 2 ** 40 + 3)}
    jstates = []
    for e in ("x256**", "x256++", "pcg64", "ranlux++"):
        for k in (32, 64, 96, 128, 192):
            r = state_io.create(e, seed=[77])
            r.next_u64()
            r.jump(k)
            jstates.append({"engine": e, "k": k, "state": ["%016x" % w for w in r.get_state()],
                            "next": ["%016x" % r.next_u64() for _ in range(5)]})
    for e in ("x128+", "xoro++"):  # jumps.py FAMILY_JUMPS for the 128-bit families
        for k in (32, 64, 96):
            r = state_io.create(e, seed=[77])
            r.next_u64()
            r.jump(k)
            jstates.append({"engine": e, "k": k, "state": ["%016x" % w for w in r.get_state()],
                            "next": ["%016x" % r.next_u64() for _ in range(5)]})
    r = state_io.create("pcg64", seed=[77])
    r.advance(123456789012345)
    jstates.append({"engine": "pcg64", "advance": "123456789012345", "state": ["%016x" % w for w in r.get_state()],
                    "next": ["%016x" % r.next_u64() for _ in range(5)]})
    out["jumps"] = jstates

    # stream selection (rng.py:27-35, 173-188) for every engine that has one
    streams = []
    for e, words in (("pcg64", [5, 6]), ("squares", [123]), ("philox", [9, 10]), ("sfc64", [1, 2, 3]),
                     ("sfc64simd", [1, 2, 3]), ("cwg128", [5, 6]), ("chacha20", [9, 10])):
        r = state_io.create(e, seed=[88])
        r.next_u32()
        r.set_stream(words)
        streams.append({"engine": e, "words": ["%016x" % w for w in words],
                        "state": ["%016x" % w for w in r.get_state()],
                        "next": ["%016x" % r.next_u64() for _ in range(20)]})
    out["streams"] = streams

    # multivariate normal (config 5a, scaled down): S from the same philox stream
    d, n = 16, 64
    r = state_io.create("philox", seed=[31])
    A = np.array(r.fill("norm", {}, d * d)).reshape(d, d)
    S = A @ A.T / d + np.eye(d)
    X = r.mvn(np.zeros(d), S, n=n)
    arrays["mvn_S"] = S
    arrays["mvn_X"] = np.asarray(X)
    out["mvn"] = {"engine": "philox", "seed": [31], "d": d, "n": n,
                  "final_state": ["%016x" % w for w in r.get_state()], "cursor": r.buffer.capture()["cursor"],
                  "tallies": r.counters}

    (HERE / "reference_vectors.json").write_text(json.dumps(out, indent=0, sort_keys=True))
    np.savez_compressed(HERE / "reference_arrays.npz", **arrays)
    print("wrote", len(recs), "fill cases")


if __name__ == "__main__":
    main()
