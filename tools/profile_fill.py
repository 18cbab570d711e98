"""Run one BASELINE fill config a few times through rs_fill, the product call (for ncu /
timing; each rep restarts from the same stream position).

    python tools/profile_fill.py ENGINE DIST LOG2N [key=value ...] [--reps R] [--fm]
e.g. python tools/profile_fill.py philox u01 30 --fm
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_05099_b200 import _lib, state_io  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("engine")
ap.add_argument("dist")
ap.add_argument("log2n", type=int)
ap.add_argument("params", nargs="*")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fm", action="store_true")
ap.add_argument("--seed", type=int, default=2024)
a = ap.parse_args()
params = {}
for kv in a.params:
    k, v = kv.split("=")
    params[k] = int(v) if (k == "b" and a.dist == "uint64") else float(v)
n = 1 << a.log2n
r = state_io.create(a.engine, seed=[a.seed])
r.set_full_mantissa(a.fm)
s = r.to_stream()
fp = r._continuous_params(a.dist, params, n) if a.dist != "uint64" else []
fpa = (ctypes.c_double * 4)(*(list(fp) + [0.0] * (4 - len(fp))))
b = int(params.get("b", 0))
ipa = _lib.u64_array([b, 0], 4)
el = 4 if a.dist in ("u01f", "uniff", "normf", "expf") else 8
out = torch.empty(n * el, dtype=torch.uint8, device="cuda")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
res = _lib.RsFillResult()
for i in range(a.reps):
    s2 = _lib.RsStream()
    ctypes.memmove(ctypes.byref(s2), ctypes.byref(s), ctypes.sizeof(s))
    ev[i].record()
    _lib.check(_lib.lib.rs_fill(ctypes.byref(s2), _lib.DIST_IDS[a.dist], fpa, ipa, n,
                                ctypes.c_void_p(out.data_ptr()), ctypes.byref(res), sp))
ev[a.reps].record()
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.reps)]
best = min(ms[1:] if len(ms) > 1 else ms)
print("%s %s n=2^%d: %s ms; best %.4f ms = %.1f Gsamples/s, %.1f GB/s" % (
    a.engine, a.dist, a.log2n, ["%.3f" % x for x in ms], best, n / best / 1e6, n * el / best / 1e6))
