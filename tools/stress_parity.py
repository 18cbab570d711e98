"""Randomised parity stress on the GPU box: random engine / law / size / start position
(buffered words, pending half, chained fills) against the oracle, for SECONDS seconds.

    python tools/stress_parity.py [SECONDS] [SEED]
"""
import os, sys, time, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2605_05099_b200 import state_io, fill_streams

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ENG = ["x256**", "x256++", "pcg64", "philox", "ranlux++", "x256++simd", "x256**simd", "xoro++", "squares", "chacha20"]
LAWS = [("uint64", {}), ("u01", {}), ("u01f", {}), ("norm", {}), ("exp", {}), ("gamma", {"alpha": 2.5}),
        ("gamma", {"alpha": 0.4}), ("beta", {"a": 2.0, "b": 5.0}), ("uint64", {"b": 6}), ("uint64", {"b": (1 << 44) + 1}),
        ("uint64", {"b": (1 << 63) + 1}), ("normf", {}), ("uint32", {"b": 1000}), ("chi2", {"nu": 3.0}),
        ("norm", {"mu": 1.0, "var": 4.0}), ("exp", {"beta": 2.0})]


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)


t0, n_ok = time.time(), 0
while time.time() - t0 < secs:
    eng = rnd.choice(ENG)
    seed = [rnd.getrandbits(40)]
    r = state_io.create(eng, seed=seed)
    o = O.OracleRng(eng, seed=seed)
    for _ in range(rnd.choice([0, 0, 1, 3, 7, 143, 144, 200])):
        if rnd.random() < 0.5:
            assert r.next_u64() == o.next_u64()
        else:
            assert r.next_u32() == o.next_u32()
    for _ in range(rnd.choice([1, 2, 3])):
        dist, params = rnd.choice(LAWS)
        n = rnd.choice([1, 33, 4097, 65535, 65536, 70001, (1 << 18) + rnd.randrange(100), (1 << 20) + rnd.randrange(5000),
                        (1 << 22) + rnd.randrange(1 << 16)])
        if dist in ("gamma", "beta", "chi2") and n > (1 << 21):
            n >>= 2
        got = r.fill(dist, params, n).cpu().numpy()
        ref = o.fill(dist, params, n)
        if not (np.array_equal(bits(got), bits(ref)) and r.get_state() == o.get_state()
                and r.buffer.capture()["cursor"] == o.buffer()[1] and r.counters == o.tallies()):
            d = np.nonzero(bits(got) != bits(ref))[0]
            print("MISMATCH", eng, seed, dist, params, n, "first diff", d[:3], "ndiff", d.size)
            sys.exit(1)
        n_ok += 1
    if rnd.random() < 0.15:  # per-stream rows
        e2 = rnd.choice(["sfc64", "pcg64", "x256**", "philox"])
        dist, params = rnd.choice([("uint64", {"b": 6}), ("uint64", {"b": (1 << 44) + 1}), ("uint64", {"b": (1 << 63) + 1}),
                                   ("uint64", {}), ("norm", {}), ("u01", {})])
        S, n = rnd.choice([1, 33, 64, 97]), rnd.choice([1, 31, 32, 64, 1000, 4096, 4097])
        out = fill_streams(e2, seed, [3], 5, S, dist, params, n).cpu().numpy()
        for j in (0, S - 1):
            oo = O.OracleRng(e2, seed=seed, spawn_key=(3, 5 + j))
            if not np.array_equal(bits(out[j]), bits(oo.fill(dist, params, n))):
                print("MISMATCH streams", e2, seed, dist, params, S, n, j)
                sys.exit(1)
        n_ok += 1
print("stress ok: %d fills in %.0f s" % (n_ok, time.time() - t0))
