"""C5b per-stream fill for ncu / timing: sfc64 seed 31, 2^16 streams x 4096, Lemire bound m.

    python tools/streams_fill.py M [--time]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import fill_streams  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rows = torch.empty((1 << 16, 4096), dtype=torch.uint64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for i in range(4):
    ev[i].record()
    fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096, out=rows)
ev[4].record()
torch.cuda.synchronize()
if "--time" in sys.argv:
    ms = min(ev[i].elapsed_time(ev[i + 1]) for i in range(1, 4))
    print("c5b sfc64 m=%d 2^28: best %.4f ms = %.1f Gsamples/s, %.1f GB/s" % (m, ms, (1 << 28) / ms / 1e6,
                                                                            (1 << 31) / ms / 1e6))
else:
    print("ok")
