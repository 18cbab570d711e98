"""Quick parity check of the single-pass tile parse against the oracle (GPU box)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2605_05099_b200 import state_io

cases = [("pcg64", "norm", {}, 1 << 16), ("pcg64", "norm", {}, (1 << 20) + 77), ("philox", "norm", {}, 1 << 20),
         ("pcg64", "exp", {}, 1 << 20), ("philox", "exp", {}, (1 << 21) + 5), ("pcg64", "norm", {"mu": 1.5, "var": 2.0}, 1 << 22),
         ("philox", "exp", {}, (1 << 21) + 6), ("philox", "exp", {}, 1 << 17), ("pcg64", "exp", {}, (1 << 21) + 5)]
bad = 0
for eng, dist, params, n in cases:
    for pre in (0, 5):
        r = state_io.create(eng, seed=[99])
        o = O.OracleRng(eng, seed=[99])
        for _ in range(pre):
            r.next_u64(); o.next_u64()
        t0 = time.time()
        got = r.fill(dist, params, n).cpu().numpy()
        t1 = time.time()
        ref = o.fill(dist, params, n)
        ok = np.array_equal(got.view(np.uint64), ref.view(np.uint64)) and r.get_state() == o.get_state() and r.counters == o.tallies()
        if not ok:
            bad += 1
            d = np.nonzero(got.view(np.uint64) != ref.view(np.uint64))[0]
            print("MISMATCH", eng, dist, n, pre, "first diff", d[:5], "ndiff", d.size, "state", r.get_state() == o.get_state(), r.counters, o.tallies())
        else:
            print("ok", eng, dist, n, pre, "%.1f ms" % ((t1 - t0) * 1e3))
        # chained second fill continues from the exact position
        got2 = r.fill(dist, params, 70000).cpu().numpy()
        ref2 = o.fill(dist, params, 70000)
        if not (np.array_equal(got2.view(np.uint64), ref2.view(np.uint64)) and r.get_state() == o.get_state()):
            bad += 1
            d = np.nonzero(got2.view(np.uint64) != ref2.view(np.uint64))[0]
            print("MISMATCH chained", eng, dist, n, pre, "first diff", d[:5], "ndiff", d.size, "state", r.get_state() == o.get_state(), r.counters, o.tallies(), "cursor", r.buffer.cursor if hasattr(r, "buffer") else None)
print("bad", bad)
sys.exit(1 if bad else 0)
