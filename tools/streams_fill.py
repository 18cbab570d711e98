"""C5b per-stream fill for ncu / timing: sfc64 seed 31, 2^16 streams x 4096, Lemire bound m."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_05099_b200 import fill_streams  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rows = torch.empty((1 << 16, 4096), dtype=torch.uint64, device="cuda")
for _ in range(3):
    fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096, out=rows)
torch.cuda.synchronize()
print("ok")
