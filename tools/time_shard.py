"""Per-rank cost of a sharded variable-consumption fill: one GPU timing one
rank's slice of an N-rank fill (warm-up entry guess, count, emit; the exchange is left out:
it is a few integers over the process group). Wall time per phase, best of 3, against the
single-GPU fill; `overhead` = slice time - single / N, the fixed cost that caps scaling."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_05099_b200 import shard, state_io  # noqa: E402


def _sync_time(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


def t_single(engine, dist, params, n, reps=3):
    return min(_sync_time(lambda: state_io.create(engine, seed=[2024]).fill(dist, params, n)) for _ in range(reps))


def t_rank(engine, dist, params, n, world, g, reps=3):
    best = None
    for _ in range(reps):
        r = state_io.create(engine, seed=[2024])
        sf = shard.ShardedFill(r, dist, params, n, g, world, shard.DeviceRanges())
        tc = _sync_time(sf.count)
        table = [[0, 0, 0] for _ in range(world)]
        table[g] = sf.record()
        te = _sync_time(lambda: sf.emit(table))
        if best is None or tc + te < best[0] + best[1]:
            best = (tc, te, sf.rounds, sf.L, sf.T)
    return best


if __name__ == "__main__":
    cases = [("x256**", "norm", {}, 1 << 28), ("pcg64", "exp", {}, 1 << 26), ("pcg64", "gamma", {"alpha": 2.5}, 1 << 26),
             ("pcg64", "beta", {"a": 2.0, "b": 5.0}, 1 << 26)]
    for engine, dist, params, n in cases:
        s = t_single(engine, dist, params, n)
        print("%s %s n=2^%d single %.3f ms" % (engine, dist, n.bit_length() - 1, s), flush=True)
        for world in (2, 4, 8):
            g = world - 1
            tc, te, rr, L, T = t_rank(engine, dist, params, n, world, g)
            print("   N=%d rank %d: count %.3f + emit %.3f = %.3f ms (single/N %.3f, overhead %.3f, speed-up x%.2f)"
                  " L=%d T=%d rounds=%d" % (world, g, tc, te, tc + te, s / world, tc + te - s / world,
                                              s / (tc + te), L, T, rr), flush=True)
