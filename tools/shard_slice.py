"""One rank's slice of an N-rank fill, repeated (for ncu launch lists): tools/shard_slice.py ENGINE DIST N WORLD [k=v]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import shard, state_io  # noqa: E402

engine, dist, log2n, world = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
params = {k: float(v) for k, v in (a.split("=") for a in sys.argv[5:])}
for rep in range(3):
    r = state_io.create(engine, seed=[2024])
    sf = shard.ShardedFill(r, dist, params, 1 << log2n, world - 1, world, shard.DeviceRanges())
    torch.cuda.nvtx.range_push("rep%d" % rep)
    sf.count()
    table = [[0, 0, 0] for _ in range(world)]
    table[world - 1] = sf.record()
    sf.emit(table)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
print("ok", sf.rounds)
