import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2605_05099_b200 import state_io
for d in (64, 256, 512):
    r = state_io.create("philox", seed=[31])
    A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
    S = A @ A.T / d + np.eye(d)
    r.mvn(np.zeros(d), S, n=1 << 20); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter(); r.mvn(np.zeros(d), S, n=1 << 20); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    z = torch.empty((1 << 20) * d, dtype=torch.float64, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r.fill("stdnorm", {}, (1 << 20) * d, out=z) if False else None
    print("mvn d=%d n=2^20: %.2f ms (wall, incl. host Cholesky)" % (d, best * 1e3))
