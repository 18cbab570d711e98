import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_05099_b200 import fill_streams
for m in (6, 1000003, (1 << 63) + 1):
    rows = fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096)
    torch.cuda.synchronize()
    best = 1e9
    for r in range(5):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        try:
            fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096, out=rows)
        except TypeError:
            fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096)
        z.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(z))
    print("sfc64 streams lemire m=%d: %.3f ms = %.1f Gsamples/s, %.0f GB/s" % (m, best, 2**28 / best / 1e6, 2**31 / best / 1e6))
