#!/usr/bin/env python
"""Benchmark of the B200 bulk stream-fill path (one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], "config 2"): Philox-4x64-10
(the reference `philox`), seed 7, full-mantissa uniforms:
u01 float64 n=2^30 plus u01f float32 n=2^30 per GPU. A step = both fills.
With N GPUs each rank fills its own contiguous counter-offset slice of the one
logical stream (rank g starts 2^30 words / 2^29 words in), so per-GPU work is
fixed ("weak") and there is no collective on the data path.

  value     device-timed whole-job Gsamples/s (outputs resident in HBM; CUDA
            events on the launch stream, max over ranks)
  e2e       the same fills through the public API with pinned HOST output
            buffers (library stages through HBM; D2H inside the timed region)
  roofline  the dominant kernel (u01 f64 fill): algorithmic bytes 8 B/sample x
            2^30 per launch / its average CUDA-event duration, against the
            measured HBM figure in MEASURED_PEAKS.json
  cpu_baseline  the C restatement of the reference (oracle/, "port") on all
            host threads, each on a disjoint counter-offset substream
  per_config    device-time Gsamples/s of the other BASELINE configs (N=1 only)

--impl reference runs the reference's CPU path (the oracle port; the Python
reference itself is not on the GPU box) on the same metric and prints
"impl": "reference".
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gsamples/s per engine×distribution at 1/2/4/8 B200; % of HBM write roofline"
UNIT = "Gsamples/s"
N_HEAD = 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ CPU reference / baseline
def cpu_reference(seconds, dist_pairs=(("u01", 8), ("u01f", 4))):
    """Oracle port on all host threads: thread t fills from the counter-offset slice t of
    the philox seed-7 stream (full mantissa), repeated 2^22-sample fills (bench.py of the
    reference fills fixed-size buffers the same way, src/bench.py:50-67)."""
    from oracle import oracle as O

    P = O.cpu_count()
    m = 1 << 22
    rngs = {}
    for dist, _ in dist_pairs:
        rs = []
        for t in range(P):
            o = O.OracleRng("philox", seed=[7], full_mantissa=True)
            st = o.get_state()
            words_per_thread = 1 << 34
            if dist == "u01f":
                words_per_thread //= 2
            st[0] = (st[0] + t * (words_per_thread // 4)) & (2 ** 64 - 1)
            o.set_state(st)
            rs.append(o)
        rngs[dist] = rs
    done = 0
    t0 = time.perf_counter()
    while True:
        for dist, _ in dist_pairs:
            O.threaded_fill(rngs[dist], dist, {}, m)
            done += P * m
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el / 1e9, P, "%d host threads x repeated 2^22-sample philox fills (u01 f64 + u01f f32), %.1f s" % (
        P, el)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = float(parts[1])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2605_05099_b200 import _lib, fill_streams, state_io

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.check(_lib.lib.rs_init_device(local_rank))
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    peak, peak_src = measured_peaks()

    from paper_2605_05099_b200 import shard

    # rank g fills words [g*W, (g+1)*W) of the one logical stream (counter offset, no collective)
    r64 = shard.shard_rng("philox", [7], rank, N_HEAD, full_mantissa=True)
    r32 = shard.shard_rng("philox", [7], rank, N_HEAD // 2, full_mantissa=True)
    s64, s32 = r64.to_stream(), r32.to_stream()
    out64 = torch.empty(N_HEAD, dtype=torch.float64, device=dev)
    out32 = torch.empty(N_HEAD, dtype=torch.float32, device=dev)
    zero_f = (ctypes.c_double * 4)()
    zero_i = _lib.u64_array([], 4)

    def fill_async(s, dist_id, n, out):
        _lib.check(_lib.lib.rs_fill_async(ctypes.byref(s), dist_id, zero_f, zero_i, n, ctypes.c_void_p(out.data_ptr()),
                                          sptr))

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        fill_async(s64, _lib.DIST_IDS["u01"], N_HEAD, out64)
        if ev is not None:
            ev[1].record(stream)
        fill_async(s32, _lib.DIST_IDS["u01f"], N_HEAD, out32)
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clock = ClockSampler(local_rank)
    clock.start()
    time.sleep(0.3)  # let the sampler attach before the timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t_stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clock.stop()
    total_ms = t_start.elapsed_time(t_stop)
    k64 = [e[0].elapsed_time(e[1]) for e in evs]
    k32 = [e[1].elapsed_time(e[2]) for e in evs]
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    samples = 2 * N_HEAD * world * args.steps
    value = samples / (total_ms / 1e3) / 1e9
    avg64 = float(np.mean(k64))
    avg32 = float(np.mean(k32))
    bytes64 = 8.0 * N_HEAD
    achieved = bytes64 / (avg64 / 1e3) / 1e9

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        h64 = torch.empty(N_HEAD, dtype=torch.float64, pin_memory=True).numpy()
        h32 = torch.empty(N_HEAD, dtype=torch.float32, pin_memory=True).numpy()
        e2e_steps = max(1, min(args.steps, 3))
        r64.fill("u01", {}, N_HEAD, out=h64)  # warm-up (also allocates the staging buffer)
        r32.fill("u01f", {}, N_HEAD, out=h32)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r64.fill("u01", {}, N_HEAD, out=h64)
            r32.fill("u01f", {}, N_HEAD, out=h32)
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": 2 * N_HEAD * world * e2e_steps / el / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * ctypes.sizeof(_lib.RsStream),
               "d2h_bytes_per_step": N_HEAD * 8 + N_HEAD * 4, "steps": e2e_steps,
               "path": "Rng.fill(..., out=pinned numpy) -> rs_fill(host ptr): kernels into HBM staging + "
                       "cudaMemcpyAsync D2H, synchronous"}
        del h64, h32

    per_config = None
    if world == 1 and not args.no_per_config:
        per_config = run_per_config(dev, stream, sptr, out64, peak)
    sharded = None
    if world > 1 and not args.no_per_config:
        sharded = run_sharded(rank, world, dev)

    traffic, limiter = None, None
    prof = os.path.join(ROOT, "profiles", "r01_ncu_philox_u01_f64.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        traffic = pj.get("traffic_bytes_per_launch")
        heavy = pj["metrics"].get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", {}).get("value")
        if heavy:
            limiter = ("integer multiply: Philox-4x64-10 needs 72 IMAD.WIDE.U32 per 4-word block (18 products after the "
                       "round fold, DESIGN 4.1); ncu: fmaheavy "
                       "pipe %.1f%% busy, DRAM %.1f%% (profiles/r01_ncu_philox_u01_f64.json)" % (
                           heavy, pj["metrics"]["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]["value"]))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic: seeded stream fills (no dataset is involved)",
        "config": {"workload": "BASELINE config 2: philox (Philox-4x64-10) seed=7 full_mantissa; u01 f64 n=2^30 "
                               "+ u01f f32 n=2^30 per GPU; rank g = counter-offset slice g",
                   "l2": "outputs 12 GiB per step >> 126 MB L2 (inputs larger than L2, no flush)",
                   "parallelism": "dp%d (independent counter slices, no collective)" % world},
        "roofline": {"bound": "hbm", "kernel": "k_philox_fixed<FX_U01> (u01 f64 fill)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu --set full, same kernel)", "limiter": limiter,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes64,
                     "avg_launch_ms": avg64, "u01f_f32_launch_ms": avg32,
                     "u01f_f32_achieved_gbs": 4.0 * N_HEAD / (avg32 / 1e3) / 1e9},
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if per_config:
        line["per_config"] = per_config
    if sharded:
        line["sharded_c3"] = sharded
    return line


def run_sharded(rank, world, dev, reps=3):
    """C3 over N GPUs as ONE logical stream: x256** seed 2024 normals,
    2^28 per GPU (weak), split by shard.fill_sharded -- warm-up entry guess, count, an
    allgather of (entry, exit, count) per rank over NCCL, emit. Wall time per rank around
    the whole protocol (it synchronises with the host), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2605_05099_b200 import shard, state_io

    n = (1 << 28) * world
    gather = shard.torch_allgather()
    best = None
    for it in range(reps + 1):
        r = state_io.create("x256**", seed=[2024])
        dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        out, off = shard.fill_sharded(r, "norm", {}, n, rank, world, gather)
        torch.cuda.synchronize(dev)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        del out
        if it > 0:  # the first pass warms the plan caches
            best = el.item() if best is None else min(best, el.item())
    return {"workload": "x256** seed 2024 norm, 2^28 per GPU, one logical stream over %d ranks" % world,
            "gsamples_s": n / best / 1e9, "ms": best * 1e3, "reps": reps,
            "timing": "wall clock per rank around fill_sharded (host-synchronising protocol), max over ranks"}


def run_per_config(dev, stream, sptr, buf, peak):
    """Device-time Gsamples/s for the other BASELINE configs (3 timed reps each)."""
    import torch

    from paper_2605_05099_b200 import _lib, fill_streams, state_io

    res = {}
    # store-only HBM figure of this box: torch's fill_ over the 8 GiB buffer
    wbest = 1e9
    for _ in range(6):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        buf.fill_(0.0)
        z.record(stream)
        torch.cuda.synchronize()
        wbest = min(wbest, a.elapsed_time(z))
    wpeak = buf.numel() * 8 / (wbest / 1e3) / 1e9
    res["hbm_write_peak"] = {"gbs": wpeak, "how": "torch fill_ of an 8 GiB tensor, best of 6, CUDA events"}

    def time_fill(label, engine, seed, dist, params, n, fm=False, reps=3, bytes_per=8):
        r = state_io.create(engine, seed=seed)
        r.set_full_mantissa(fm)
        s = r.to_stream()
        fp = r._continuous_params(dist, params, n) if dist not in ("uint64",) else []
        fpa = (ctypes.c_double * 4)(*(list(fp) + [0.0] * (4 - len(fp))))
        b = int(params.get("b", 0)) if dist == "uint64" else 0
        ipa = _lib.u64_array([b, 0] if b != 1 << 64 else [0, 1], 4)
        out = buf.view(torch.uint8)[: n * bytes_per]
        did = _lib.DIST_IDS[dist]

        def go():
            _lib.check(_lib.lib.rs_fill_async(ctypes.byref(s), did, fpa, ipa, n, ctypes.c_void_p(out.data_ptr()),
                                              sptr))
        go()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            go()
        z.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(z) / reps
        gbs = n * bytes_per / (ms / 1e3) / 1e9
        res[label] = {"gsamples_s": n / (ms / 1e3) / 1e9, "ms": ms, "n": n, "hbm_frac": gbs / peak,
                      "write_frac": gbs / wpeak}

    time_fill("c1_x256ss_raw_u64_2p30", "x256**", [12345], "uint64", {}, 1 << 30)
    time_fill("c2_philox_u01_f64_2p30", "philox", [7], "u01", {}, 1 << 30, fm=True)
    time_fill("c2_philox_u01f_f32_2p30", "philox", [7], "u01f", {}, 1 << 30, fm=True, bytes_per=4)
    time_fill("c3_x256ss_norm_2p28", "x256**", [2024], "norm", {}, 1 << 28)
    time_fill("c3_pcg64_norm_2p28", "pcg64", [2024], "norm", {}, 1 << 28)
    time_fill("c4_pcg64_exp_2p26", "pcg64", [99], "exp", {}, 1 << 26)
    for k in (0.3, 1.0, 2.5, 10.0):
        time_fill("c4_pcg64_gamma_%g_2p26" % k, "pcg64", [99], "gamma", {"alpha": k}, 1 << 26)
    time_fill("c4_pcg64_beta_2_5_2p26", "pcg64", [99], "beta", {"a": 2.0, "b": 5.0}, 1 << 26)
    time_fill("extra_ranlux_raw_2p28", "ranlux++", [12345], "uint64", {}, 1 << 28, reps=2)
    # C5b: sfc64 per-stream Lemire, 2^16 streams x 4096
    for m in (6, 1000003, (1 << 63) + 1):
        rows = fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096)
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            fill_streams("sfc64", [31], [], 0, 1 << 16, "uint64", {"b": m}, 4096, out=rows)
        z.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(z) / 3
        n = 1 << 28
        res["c5b_sfc64_streams_lemire_%d_2p28" % m] = {"gsamples_s": n / (ms / 1e3) / 1e9, "ms": ms, "n": n,
                                                       "hbm_frac": n * 8 / (ms / 1e3) / 1e9 / peak,
                                                       "write_frac": n * 8 / (ms / 1e3) / 1e9 / wpeak,
                                                       "note": "fill_streams(..., out=) into a resident 2 GiB tensor"}
    # C5a: mvn (z fill + cuBLAS DGEMM), d in {64, 256, 512}, n = 2^20
    for d in (64, 256, 512):
        r = state_io.create("philox", seed=[31])
        A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
        S = A @ A.T / d + np.eye(d)
        r.mvn(np.zeros(d), S, n=1 << 20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r.mvn(np.zeros(d), S, n=1 << 20)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        res["c5a_mvn_d%d_2p20" % d] = {"vectors_per_s": (1 << 20) / el, "ms": el * 1e3,
                                        "gflops_dense": 2.0 * (1 << 20) * d * d / el / 1e9,
                                        "gflops_triangular": 1.0 * (1 << 20) * d * (d + 1) / el / 1e9,
                                        "note": "wall clock incl. host Cholesky and sync (rs_mvn is synchronous)"}
    # FP64 peak for the MVN contraction: cuBLAS DGEMM 8192^3 through torch
    m = 8192
    a64 = torch.randn(m, m, dtype=torch.float64, device=dev)
    b64 = torch.randn(m, m, dtype=torch.float64, device=dev)
    c64 = torch.matmul(a64, b64)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.matmul(a64, b64, out=c64)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    tf = 2.0 * m ** 3 / (best / 1e3) / 1e12
    res["fp64_dgemm_peak"] = {"tflops": tf, "how": "torch.matmul f64 8192^3 (cuBLAS DGEMM), best of 3, CUDA events"}
    for d in (64, 256, 512):
        row = res["c5a_mvn_d%d_2p20" % d]
        row["dense_frac_of_dgemm"] = row["gflops_dense"] / 1e3 / tf
    del a64, b64, c64
    return res


# ------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        for _ in range(max(0, min(args.warmup, 1))):
            cpu_reference(0.2)
        vals = []
        for _ in range(max(1, min(args.steps, 3))):
            v, P, sample = cpu_reference(args.cpu_seconds)
            vals.append(v)
        v = float(np.median(vals))
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                "steps": len(vals), "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic: seeded stream fills",
                "config": {"workload": "BASELINE config 2 (philox seed=7 full_mantissa, u01 f64 + u01f f32), "
                                       "bounded CPU sample"},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": P, "kind": "port", "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1:
            v, P, sample = cpu_reference(args.cpu_seconds)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": P, "kind": "port", "sample": sample}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
