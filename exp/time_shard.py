"""Per-rank device time of a sharded variable fill (one slice = what one GPU of N does)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2605_05099_b200 import shard, state_io

def t_single(engine, dist, params, n, reps=3):
    best = 1e9
    for _ in range(reps):
        r = state_io.create(engine, seed=[2024])
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r.fill(dist, params, n); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3

def t_rank(engine, dist, params, n, world, g, reps=3):
    best = 1e9
    for _ in range(reps):
        r = state_io.create(engine, seed=[2024])
        sf = shard.ShardedFill(r, dist, params, n, g, world, shard.DeviceRanges())
        global L_
        L_ = sf.L
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sf.count()
        table = [[0, 0, sf.cnt]] * world
        table[g] = sf.record()
        sf.emit([[0, 0, sf.cnt if h == g else 0] for h in range(world)] if g == 0 else [[0,0,0]]*g + [sf.record()] + [[0,0,0]]*(world-g-1))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    global ROUNDS
    ROUNDS = sf.rounds
    return best * 1e3

ROUNDS = 0
for engine, dist, params, n in [("x256**", "norm", {}, 1 << 28), ("pcg64", "gamma", {"alpha": 2.5}, 1 << 26),
                                ("pcg64", "beta", {"a": 2.0, "b": 5.0}, 1 << 26), ("pcg64", "exp", {}, 1 << 26)]:
    s = t_single(engine, dist, params, n)
    line = "%s %s n=%d single %.3f ms" % (engine, dist, n, s)
    for world in (2, 4, 8):
        ts = [t_rank(engine, dist, params, n, world, g) for g in (0, world - 1)]
        line += " | N=%d rank0 %.3f last %.3f (x%.2f, L=%d rounds=%d)" % (world, ts[0], ts[1], s / max(ts), L_, ROUNDS)
    print(line, flush=True)
