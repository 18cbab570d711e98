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
