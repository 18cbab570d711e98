"""Time the MVN contraction (k_mvn_dmma through rs_mvn_apply) on the device: C5a shapes,
d in {64, 256, 512}, n = 2^20, lower-triangular Cholesky factor and a dense factor.
CUDA events around rs_mvn_apply (which synchronises; the host-side triangularity scan of
L is included). Checks X against torch's fp64 matmul (normwise 1e-12)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import _lib  # noqa: E402


def run(d, n, dense=False, layout=0, reps=5):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(d)
    z = torch.randn(n * d, dtype=torch.float64, device=dev, generator=g)
    A = np.random.default_rng(d).standard_normal((d, d))
    S = A @ A.T / d + np.eye(d)
    L = np.linalg.cholesky(S)
    if dense:
        L = L + np.triu(np.full((d, d), 1e-3), 1)
    L = np.ascontiguousarray(L)
    mean = np.zeros(d)
    X = torch.empty(n * d, dtype=torch.float64, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def go():
        _lib.check(_lib.lib.rs_mvn_apply(ctypes.c_void_p(L.ctypes.data), mean.ctypes.data_as(_lib.DBLP), d, n, layout,
                                         ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(X.data_ptr()), st))
    go()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        go()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    Lt = torch.from_numpy(L).to(dev)
    zz = z.view(n, d)
    ref = zz @ Lt.T
    got = X.view(n, d) if layout == 0 else X.view(d, n).T
    scale = zz.abs() @ Lt.abs().T
    err = float(((got - ref).abs() / scale).max())
    tri = n * d * (d + 1) / (best / 1e3) / 1e12
    dense_tf = 2.0 * n * d * d / (best / 1e3) / 1e12
    # cuBLAS DGEMM through torch on the same shape (for comparison only)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    zz @ Lt.T
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        zz @ Lt.T
    b.record()
    torch.cuda.synchronize()
    cub = a.elapsed_time(b) / 3
    print("d=%4d n=2^%d %s layout=%s: %.3f ms  %.1f TF/s triangular (%.1f dense-equiv)  err %.2e | torch DGEMM %.3f ms"
          % (d, int(np.log2(n)), "dense" if dense else "chol ", "n_d" if layout == 0 else "d_n", best, tri, dense_tf,
             err, cub), flush=True)
    assert err <= 1e-12


if __name__ == "__main__":
    if len(sys.argv) > 1:  # e.g. `512`: one C5a shape (for ncu)
        run(int(sys.argv[1]), 1 << 20, reps=1)
        sys.exit(0)
    for d in (64, 256, 512):
        run(d, 1 << 20)
    run(512, 1 << 20, layout=1)
    run(512, 1 << 20, dense=True)
    run(24, 1000, dense=True)
    run(33, 1001)
    run(7, 4099, layout=1)
