"""Fills beyond 2^32 samples: one call equals two chained calls (chunk / grid / offset arithmetic
at sizes no other test reaches), compared on the device; the split point is mid-buffer.

    python tools/big_fill_check.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_05099_b200 import state_io

CASES = [("x256**", "uint64", {}, (1 << 32) + 12345), ("philox", "u01", {}, (1 << 32) + 7),
         ("pcg64", "u01f", {}, (1 << 33) + 3), ("pcg64", "norm", {}, (1 << 31) + 1001),
         ("x256++simd", "uint64", {}, (1 << 32) + 8 * 1000 + 5), ("philox", "exp", {}, (1 << 30) + 77)]
bad = 0
for eng, dist, params, n in CASES:
    n1 = n // 3 + 11
    a = state_io.create(eng, seed=[5]); b = state_io.create(eng, seed=[5])
    t0 = time.time()
    whole = a.fill(dist, params, n)
    torch.cuda.synchronize(); t1 = time.time()
    p1 = b.fill(dist, params, n1)
    p2 = b.fill(dist, params, n - n1)
    ok = torch.equal(whole[:n1], p1) and torch.equal(whole[n1:], p2) and a.get_state() == b.get_state() \
        and a.buffer.capture() == b.buffer.capture() and a.counters == b.counters
    print("%s %s n=%d: %s (%.1f ms)" % (eng, dist, n, "ok" if ok else "MISMATCH", (t1 - t0) * 1e3))
    bad += 0 if ok else 1
    del whole, p1, p2
    torch.cuda.empty_cache()
sys.exit(1 if bad else 0)
