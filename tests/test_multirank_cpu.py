"""N>1 path on CPU: two gloo ranks each position their slice of one logical stream
with the product's skip-ahead (paper_2605_05099_b200.shard) and the oracle checks that
the gathered concatenation equals the single-stream reference sequence."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, engine, dist_name, words_per_rank, n_per_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import oracle as O
        from paper_2605_05099_b200 import shard

        r = shard.shard_rng(engine, [2024], rank, words_per_rank, full_mantissa=True)
        o = O.OracleRng(engine, seed=[1], full_mantissa=True)
        o.set_state(r.get_state())            # the oracle checks what this rank would fill
        part = o.fill(dist_name, {}, n_per_rank)
        t = torch.from_numpy(part.view(np.int64).copy() if part.dtype.itemsize == 8
                             else part.view(np.int32).astype(np.int64))
        out = [torch.empty_like(t) for _ in range(WORLD)]
        dist.all_gather(out, t)
        if rank == 0:
            q.put(torch.cat(out).numpy())
        j0, cnt = shard.shard_streams(65536, rank, WORLD)
        js = torch.tensor([j0, cnt])
        allj = [torch.empty_like(js) for _ in range(WORLD)]
        dist.all_gather(allj, js)
        if rank == 0:
            q.put([tuple(int(v) for v in a) for a in allj])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("engine,dist_name,wpr,npr", [
    ("philox", "u01", 4096, 4096),
    ("x256**", "uint64", 1000, 1000),
    ("pcg64", "u01", 777, 777),
    ("ranlux++", "uint64", 9 * 144, 9 * 144),
    ("philox", "u01f", 2048, 4096),
])
def test_two_rank_slices_concatenate(engine, dist_name, wpr, npr):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, engine, dist_name, wpr, npr, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    js = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = O.OracleRng(engine, seed=[2024], full_mantissa=True).fill(dist_name, {}, WORLD * npr)
    ref = ref.view(np.int64) if ref.dtype.itemsize == 8 else ref.view(np.int32).astype(np.int64)
    assert np.array_equal(got, ref)
    assert js == [(0, 32768), (32768, 32768)]


# ----------------------------------------------------------------------------- variable-consumption sharding
# The rank protocol of shard.ShardedFill (warm-up entry guess, count, exchange, re-count,
# prefix offsets, emit, final position) with the range primitive restated on the oracle.

def _ref(engine, dist_name, params, n):
    from oracle import oracle as O

    o = O.OracleRng(engine, seed=[2024])
    vals = o.fill(dist_name, params, n)
    return vals, o.get_state(), o.buffer(), o.tallies()


def _as_int(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)


def _check(got, r, engine, dist_name, params, n):
    vals, st, buf, tal = _ref(engine, dist_name, params, n)
    g = got.numpy() if got.dtype != torch.uint64 else got.view(torch.int64).numpy()
    assert np.array_equal(_as_int(g), _as_int(vals))
    assert r.get_state() == st
    assert (r.buffer.words, r.buffer.cursor, r.buffer.pending) == buf
    assert {k: v for k, v in r.counters.items()} == tal


SIM_CASES = [
    # engine, dist, params, n, world, ShardedFill kwargs, OracleRanges kwargs
    ("x256**", "norm", {}, 3000, 2, {}, {}),
    ("x256**", "norm", {}, 3000, 3, {}, {}),
    ("pcg64", "exp", {}, 2500, 4, {}, {}),
    ("pcg64", "gamma", {"alpha": 2.5}, 1200, 3, {}, {}),
    ("philox", "beta", {"a": 2.0, "b": 5.0}, 500, 2, {}, {}),
    ("pcg64", "uint64", {"b": (1 << 63) + 1}, 2000, 3, {}, {}),
    ("x256**", "normf", {}, 3001, 2, {}, {}),
    # a one-word warm-up window: guesses are often wrong, so the re-count path runs
    ("pcg64", "gamma", {"alpha": 0.3}, 1000, 4, {"window": (1, 1)}, {}),
    ("x256**", "norm", {}, 2000, 3, {"window": (1, 1)}, {}),
    # provisioned range too small: the last rank continues with an ordinary fill
    ("x256**", "norm", {}, 2000, 2, {"words_per_rank": 500}, {}),
    ("pcg64", "gamma", {"alpha": 2.5}, 700, 2, {"words_per_rank": 300}, {}),
    # n = 0 consumes nothing
    ("x256**", "norm", {}, 0, 2, {}, {}),
]


@pytest.mark.parametrize("engine,dist_name,params,n,world,kw,okw", SIM_CASES)
def test_sharded_variable_fill_simulated(engine, dist_name, params, n, world, kw, okw):
    from oracle_ranges import OracleRanges, simulate
    from paper_2605_05099_b200 import state_io

    got, r, sfs = simulate(lambda: state_io.create(engine, seed=[2024]), dist_name, params, n, world,
                           lambda: OracleRanges(engine, dist_name, params, **okw), **kw)
    _check(got, r, engine, dist_name, params, n)
    for sf in sfs[1:]:  # every rank ends at the same position
        assert sf.rng.get_state() == r.get_state() and sf.rng.buffer.cursor == r.buffer.cursor


def _sharded_worker(rank, port, engine, dist_name, params, n, kw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle_ranges import OracleRanges
        from paper_2605_05099_b200 import shard, state_io

        r = state_io.create(engine, seed=[2024])
        out, off = shard.fill_sharded(r, dist_name, params, n, rank, WORLD, shard.torch_allgather(),
                                      ranges=OracleRanges(engine, dist_name, params), **kw)
        a = out.view(torch.int64) if out.dtype == torch.uint64 else out
        parts = [None] * WORLD
        dist.all_gather_object(parts, (off, a.numpy().tobytes(), str(a.dtype), r.get_state(),
                                       (r.buffer.words, r.buffer.cursor, r.buffer.pending), r.counters))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("engine,dist_name,params,n,kw", [
    ("x256**", "norm", {}, 3000, {}),
    ("pcg64", "gamma", {"alpha": 2.5}, 1000, {"window": (1, 1)}),
    ("x256**", "exp", {}, 1500, {"words_per_rank": 400}),
])
def test_two_rank_sharded_variable_fill(engine, dist_name, params, n, kw):
    import sys

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    sys.path.insert(0, os.path.dirname(__file__))
    procs = [ctx.Process(target=_sharded_worker, args=(r, port, engine, dist_name, params, n, kw, q))
             for r in range(WORLD)]
    for p in procs:
        p.start()
    parts = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    vals, st, buf, tal = _ref(engine, dist_name, params, n)
    offs = [p[0] for p in parts]
    assert offs[0] == 0
    got = np.concatenate([np.frombuffer(p[1], dtype=np.float64 if "float64" in p[2] else np.int64) for p in parts])
    assert np.array_equal(_as_int(got), _as_int(vals))
    assert len(np.frombuffer(parts[0][1], dtype=np.int64)) == min(offs[1], n)
    for p in parts:
        assert p[3] == st and p[4] == buf and p[5] == tal
