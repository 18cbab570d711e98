"""Where the time of one C5a Rng.mvn call goes (d = 512, n = 2^20, the BASELINE recipe):
the whole public call, the z fill alone, the host factorisation alone, the contraction
(rs_mvn_apply) alone. Wall clock around synchronised calls, best of 3."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import _lib, state_io  # noqa: E402
from paper_2605_05099_b200.rng import semidefinite_factor  # noqa: E402


def best(fn, reps=3):
    out = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out = min(out, time.perf_counter() - t0)
    return out * 1e3


d = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = 1 << 20
r = state_io.create("philox", seed=[31])
A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
S = A @ A.T / d + np.eye(d)
print("whole r.mvn        %.3f ms" % best(lambda: r.mvn(np.zeros(d), S, n=n)))
print("sym check (host)   %.3f ms" % best(lambda: np.allclose(S, S.T, rtol=1e-9, atol=1e-12)))
Ld = torch.from_numpy(np.ascontiguousarray(np.linalg.cholesky(S))).cuda()
stC = r.to_stream()
Xc = torch.empty((n, d), dtype=torch.float64, device="cuda")
mz = np.zeros(d)
print("rs_mvn (C ABI)      %.3f ms" % best(lambda: _lib.check(_lib.lib.rs_mvn(
    ctypes.byref(stC), ctypes.c_void_p(Ld.data_ptr()), mz.ctypes.data_as(_lib.DBLP), d, n, 0,
    ctypes.c_void_p(Xc.data_ptr()), None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))))
del Xc
z = torch.empty(n * d, dtype=torch.float64, device="cuda")
print("z fill (stdnorm)   %.3f ms" % best(lambda: r.device_fill("stdnorm", [], [], n * d, out=z)))
print("cholesky (host)    %.3f ms" % best(lambda: semidefinite_factor(S)))
L = np.ascontiguousarray(semidefinite_factor(S))
X = torch.empty(n * d, dtype=torch.float64, device="cuda")
mean = np.zeros(d)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
print("rs_mvn_apply       %.3f ms" % best(lambda: _lib.check(_lib.lib.rs_mvn_apply(
    ctypes.c_void_p(L.ctypes.data), mean.ctypes.data_as(_lib.DBLP), d, n, 0, ctypes.c_void_p(z.data_ptr()),
    ctypes.c_void_p(X.data_ptr()), st))))
print("torch.empty x2     %.3f ms" % best(lambda: (torch.empty((n, d), dtype=torch.float64, device="cuda"),
                                                   torch.empty(n * d, dtype=torch.float64, device="cuda"))))
