import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import oracle as O
from paper_2605_05099_b200 import state_io
for eng, dist, n1 in (("philox","exp",2097157),):
    r = state_io.create(eng, seed=[99]); o = O.OracleRng(eng, seed=[99])
    a = r.fill(dist, {}, n1).cpu().numpy(); b = o.fill(dist, {}, n1)
    a = r.fill(dist, {}, 70000).cpu().numpy(); b = o.fill(dist, {}, 70000 + 8)
    n = 70000
    off = np.full(n, 99)
    for k in range(-3, 4):
        idx = np.arange(n) + k
        ok = (idx >= 0) & (idx < b.size)
        m = np.zeros(n, bool); m[ok] = a[ok] == b[idx[ok]]
        off[m & (off == 99)] = k
    ch = np.nonzero(np.diff(off))[0]
    print("offset runs:", [(int(i + 1), int(off[i + 1])) for i in ch][:20], "start", off[0], "end", off[-1])
    print(a[:3], b[:4]); print(a[60:70]); print(b[60:71])
