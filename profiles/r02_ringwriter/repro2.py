import sys
import torch
sys.path.insert(0, ".")
from paper_2605_05099_b200 import fill_streams
for ns, nper in ((8, 4096), (64, 777), (64, 4096), (256, 4096), (64, 4097)):
    out = fill_streams("x256**", [5], [2], 10, ns, "norm", {}, nper)
    torch.cuda.synchronize()
    print("x256** norm", ns, nper, "ok", flush=True)
print("all ok")
