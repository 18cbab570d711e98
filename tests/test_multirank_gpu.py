"""Two processes sharing one GPU, each a rank of one logical stream through the product's
device range primitive (shard.DeviceRanges: rs_range_count / rs_range_emit) with the
(entry, exit, count) exchange over a real gloo process group -- the multi-process form of
SURVEY 8(e) that the simulated-world tests run in one process. The gathered samples, the
final generator position on every rank and the tallies equal the single-stream device
fill and the oracle. (No kernel waits on another process: the exchange is host-side.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, engine, dist_name, params, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        from paper_2605_05099_b200 import shard, state_io
        r = state_io.create(engine, seed=[2024])
        out, off = shard.fill_sharded(r, dist_name, params, n, rank, WORLD, shard.torch_allgather())
        host = out.cpu().numpy()
        q.put((rank, int(off), host.view(np.uint64 if host.dtype.itemsize == 8 else np.uint32).copy(),
               r.get_state(), r.buffer.capture(), {k: dict(v) for k, v in r.counters.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("engine,dist_name,params,n", [
    ("x256**", "norm", {}, 1 << 20),
    ("pcg64", "gamma", {"alpha": 2.5}, 1 << 18),
    ("philox", "exp", {}, 300001),
    ("pcg64", "uint64", {"b": 6}, 1 << 19),
])
def test_two_process_device_ranges(engine, dist_name, params, n):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, engine, dist_name, params, n, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(WORLD)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    parts = [(off, arr) for _, off, arr, _, _, _ in res]
    assert parts[0][0] == 0 and parts[1][0] == len(parts[0][1])
    got = np.concatenate([a for _, a in parts])
    o = O.OracleRng(engine, seed=[2024])
    ref = o.fill(dist_name, params, n)
    assert np.array_equal(got, ref.view(got.dtype))
    for _, _, _, st, cap, counters in res:  # every rank ends where the single-stream fill does
        words, cursor, pending = o.buffer()
        assert st == o.get_state() and cap["words"] == words and cap["cursor"] == cursor
        assert cap["pending"] == pending
        assert counters == o.tallies()


@pytest.mark.slow
def test_bench_two_ranks_plumbing():
    """bench.py's N > 1 path (the driver's torchrun launch line: barriers, max-over-ranks
    time, one JSON line from rank 0, the sharded C3 line) with two ranks sharing this GPU
    over gloo (RS_BENCH_BACKEND=gloo). A plumbing check only: the numbers mean nothing."""
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    env = dict(os.environ, RS_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--no-e2e"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, "rank 0 prints exactly one JSON line"
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["scaling"] == "weak"
    assert line["value"] > 0 and line["sharded_c3"]["gsamples_s"] > 0
    assert line["gpu_launches"] == 4
