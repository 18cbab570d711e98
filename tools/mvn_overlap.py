"""Does a z fill overlap a running contraction? Times (1) the contraction alone, (2) the
z fill alone, (3) both issued together on two streams (fill high priority, contraction low),
(4) the same with the priorities swapped. d = 512, n = 2^20 (C5a). CUDA events on the
default stream bracketing both side streams; best of 3."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import _lib, state_io  # noqa: E402

d, n = 512, 1 << 20
r = state_io.create("philox", seed=[31])
A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
L = torch.from_numpy(np.ascontiguousarray(np.linalg.cholesky(A @ A.T / d + np.eye(d)))).cuda()
mean = torch.zeros(d, dtype=torch.float64, device="cuda")
z = torch.empty(n * d, dtype=torch.float64, device="cuda")
z2 = torch.empty(n * d, dtype=torch.float64, device="cuda")
X = torch.empty(n * d, dtype=torch.float64, device="cuda")
r.device_fill("stdnorm", [], [], n * d, out=z)
hi = torch.cuda.Stream(priority=-1)
lo = torch.cuda.Stream(priority=0)


def contract(st):
    _lib.check(_lib.lib.rs_mvn_apply_rows(ctypes.c_void_p(L.data_ptr()), ctypes.c_void_p(mean.data_ptr()), d, 1, n,
                                          ctypes.c_void_p(z.data_ptr()), 0, ctypes.c_void_p(X.data_ptr()), n,
                                          ctypes.c_void_p(st.cuda_stream)))


def fill(st):
    with torch.cuda.stream(st):
        r.device_fill("stdnorm", [], [], n * d, out=z2)


def timed(fn):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        hi.wait_stream(torch.cuda.current_stream())
        lo.wait_stream(torch.cuda.current_stream())
        fn()
        torch.cuda.current_stream().wait_stream(hi)
        torch.cuda.current_stream().wait_stream(lo)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


print("contraction alone        %.3f ms" % timed(lambda: contract(lo)))
print("z fill alone             %.3f ms" % timed(lambda: fill(hi)))
print("contraction(lo) + fill(hi) %.3f ms" % timed(lambda: (contract(lo), fill(hi))))
print("contraction(hi) + fill(lo) %.3f ms" % timed(lambda: (contract(hi), fill(lo))))
print("fill(hi) then contraction(lo) queued after %.3f ms" % timed(lambda: (fill(hi), contract(lo))))
