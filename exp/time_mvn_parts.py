"""MVN C5a d=512 breakdown: host Cholesky, z fill (std_norm philox), the whole rs_mvn."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2605_05099_b200 import state_io
from paper_2605_05099_b200.rng import semidefinite_factor
for d in (64, 256, 512):
    r = state_io.create("philox", seed=[31])
    A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
    S = A @ A.T / d + np.eye(d)
    n = 1 << 20
    t = time.perf_counter(); L = semidefinite_factor(S); tc = time.perf_counter() - t
    q = r.duplicate()
    q.device_fill("stdnorm", [], [], n * d); torch.cuda.synchronize()
    q = r.duplicate()
    torch.cuda.synchronize(); t = time.perf_counter(); q.device_fill("stdnorm", [], [], n * d); torch.cuda.synchronize(); tz = time.perf_counter() - t
    q = r.duplicate(); q.mvn(np.zeros(d), S, n=n); torch.cuda.synchronize()
    q = r.duplicate()
    torch.cuda.synchronize(); t = time.perf_counter(); q.mvn(np.zeros(d), S, n=n); torch.cuda.synchronize(); tm = time.perf_counter() - t
    print("d=%d chol %.2f ms, z fill %.2f ms, mvn total %.2f ms -> rest (GEMM + copies) %.2f ms" % (d, tc * 1e3, tz * 1e3, tm * 1e3, (tm - tc - tz) * 1e3), flush=True)
