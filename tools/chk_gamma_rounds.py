"""Chained product fills (bench.py's per-config pattern): time, resolution rounds and chunks per call."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_05099_b200 import _lib, state_io
eng, dist, log2n = sys.argv[1], sys.argv[2], int(sys.argv[3])
params = {k: float(v) for k, v in (a.split("=") for a in sys.argv[4:])}
n = 1 << log2n
r = state_io.create(eng, seed=[99])
s = r.to_stream()
fp = r._continuous_params(dist, params, n)
fpa = (ctypes.c_double * 4)(*(list(fp) + [0.0] * (4 - len(fp))))
ipa = _lib.u64_array([0, 0], 4)
out = torch.empty(n, dtype=torch.float64, device="cuda")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = _lib.RsFillResult()
for i in range(6):
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(_lib.lib.rs_fill(ctypes.byref(s), _lib.DIST_IDS[dist], fpa, ipa, n, ctypes.c_void_p(out.data_ptr()), ctypes.byref(res), sp))
    z.record(); torch.cuda.synchronize()
    print("call %d: %.3f ms rounds=%d chunks=%d words=%d" % (i, a.elapsed_time(z), res.resync_rounds, res.chunks, res.words_consumed))
