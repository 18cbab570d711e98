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
  roofline  the dominant kernel (k_philox_fixed, u01 f64): it is bound by the
            integer-multiply (fmaheavy) pipe, not HBM -- `frac` is its 64x64->128
            products per second against that pipe's capacity; the HBM fraction of
            the same launch is reported beside it
  cpu_baseline  the C restatement of the reference (oracle/, "port") on all
            host threads, each on a disjoint counter-offset substream
  per_config    every other BASELINE row (N=1 only), each timed through the product
            call (Rng.fill / fill_streams / Rng.mvn, CUDA events on the stream),
            with its roofline fraction and the same-run CPU rate of the port at
            P = all host threads and P = 1 (same partition scheme as the GPU)

--impl reference runs the reference's CPU path (the oracle port: the reference is
pure Python and is not on the GPU box) on the headline's full config -- 2^30 u01 +
2^30 u01f per GPU per step, all host threads -- and prints "impl": "reference".
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
    ap.add_argument("--cpu-seconds", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ CPU reference / baseline
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class C2Reference:
    """The headline config on the host: the oracle port (C restatement of the reference),
    P threads, thread t filling counter-offset slice t of the philox seed-7 stream (full
    mantissa) -- the GPU's partition (counter.py:108-112). One step = u01 f64 2^30 plus
    u01f f32 2^30 per GPU of the run, into preallocated host arrays."""

    def __init__(self, world=1):
        from oracle import oracle as O
        self.O = O
        self.P = O.cpu_count()
        self.world = world
        self.per = {d: (N_HEAD // self.P + 7) // 8 * 8 for d in ("u01", "u01f")}
        self.outs = {d: [np.empty(self.per[d], dtype=np.float64 if d == "u01" else np.float32)
                         for _ in range(self.P)] for d in ("u01", "u01f")}

    def rngs(self, dist, g):
        O = self.O
        out = []
        for t in range(self.P):
            o = O.OracleRng("philox", seed=[7], full_mantissa=True)
            st = o.get_state()
            w0 = g * N_HEAD + t * self.per[dist]  # first sample of the slice
            words = w0 if dist == "u01" else w0 // 2
            st[0] = (st[0] + words // 4) & (2 ** 64 - 1)
            o.set_state(st)
            out.append(o)
        return out

    def step(self):
        t0 = time.perf_counter()
        for g in range(self.world):
            for dist in ("u01", "u01f"):
                self.O.threaded_fill(self.rngs(dist, g), dist, {}, self.per[dist], self.outs[dist])
        return time.perf_counter() - t0

    def sample(self):
        return ("%d host threads (%s): the full config, %d x (2^30 u01 f64 + 2^30 u01f f32) per step, thread t = "
                "counter-offset slice t" % (self.P, cpu_model(), self.world))


def cpu_rate(engine, seed, dist, params, P, seconds, fm=False, spawn_streams=False):
    """Samples/s of the oracle port on P host threads, each on a disjoint substream of the
    engine (offset t * 2^50 words) or, for per-stream mode, its own spawned stream."""
    from oracle import oracle as O

    rngs = []
    for t in range(P):
        if spawn_streams:
            o = O.OracleRng(engine, seed=seed, spawn_key=(t,))
        else:
            o = O.OracleRng(engine, seed=seed)
            st = o.get_state()
            off = t << 50
            if engine == "philox":
                st[0] = (st[0] + off // 4) & (2 ** 64 - 1)
            elif engine == "x256**":
                st = O.x256_apply_poly(st, O.x_pow_mod(off, O.x256_charpoly()))
            elif engine == "pcg64":
                st = O.pcg_advance(st, off)
            elif engine == "ranlux++":
                st = O.ranlux_advance_chunks(st, off // 9)
            o.set_state(st)
        o.set_full_mantissa(fm)
        rngs.append(o)
    m = 1 << 12
    outs = None
    while True:  # size one call at ~50 ms
        t0 = time.perf_counter()
        O.threaded_fill(rngs, dist, params, m)
        if time.perf_counter() - t0 > 0.05 or m >= 1 << 26:
            break
        m *= 4
    outs = [np.empty(m, dtype=O.out_dtype(dist)) for _ in range(P)]
    done, t0 = 0, time.perf_counter()
    while True:
        O.threaded_fill(rngs, dist, params, m, outs)
        done += P * m
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"gsamples_s": done / el / 1e9, "cores": P, "seconds": round(el, 3), "per_call": m}


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
        per_config = run_per_config(dev, stream, sptr, out64, peak, args.cpu_seconds, not args.no_cpu,
                                    clocks.get("sm_max_mhz") or 1965.0)
    sharded = None
    if world > 1 and not args.no_per_config:
        sharded = run_sharded(rank, world, dev)

    # Roofline of the dominant kernel. k_philox_fixed is bound by the integer multiplies,
    # not by HBM (DESIGN 4.1): Philox-4x64-10 needs 20 64x64->128 products per 4-word
    # block, 18 after the round fold. A 64x64 product is four IMAD.WIDE.U32, and one
    # IMAD.WIDE warp instruction holds an SMSP's fmaheavy pipe 4 cycles, so the pipe
    # completes 2 products per cycle per SMSP: 148 SMs x 4 SMSPs x 2 x f_max.
    mhz = clocks.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    int_peak = sms * 4 * 2 * mhz * 1e6 / 1e9  # G products/s
    prods = 18.0 * (N_HEAD / 4)               # products per u01 launch (folded rounds)
    int_achieved = prods / (avg64 / 1e3) / 1e9
    traffic, pipe = None, None
    prof = os.path.join(ROOT, "profiles", "r01_ncu_philox_u01_f64.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        traffic = pj.get("traffic_bytes_per_launch")
        pipe = {"fmaheavy_busy_pct": pj["metrics"].get(
                    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", {}).get("value"),
                "dram_busy_pct": pj["metrics"]["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]["value"],
                "source": "profiles/r01_ncu_philox_u01_f64.json (ncu --set full, same kernel)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic: seeded stream fills (no dataset is involved)",
        "config": {"workload": "BASELINE config 2: philox (Philox-4x64-10) seed=7 full_mantissa; u01 f64 n=2^30 "
                               "+ u01f f32 n=2^30 per GPU; rank g = counter-offset slice g",
                   "l2": "outputs 12 GiB per step >> 126 MB L2 (inputs larger than L2, no flush)",
                   "parallelism": "dp%d (independent counter slices, no collective)" % world},
        "roofline": {"bound": "int", "pipe": "fmaheavy (IMAD.WIDE, integer multiply)",
                     "kernel": "k_philox_fixed<FX_U01> (u01 f64 fill)",
                     "achieved": int_achieved, "peak": int_peak, "unit": "G 64x64->128-bit products/s",
                     "frac": int_achieved / int_peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu --set full, same kernel)",
                     "peak_source": "fmaheavy pipe capacity: %d SMs x 4 SMSPs x 2 products/cycle x %.0f MHz "
                                    "(IMAD.WIDE.U32 = 4 pipe cycles, 4 per product)" % (sms, mhz),
                     "algorithmic_products_per_launch": prods, "avg_launch_ms": avg64, "ncu": pipe,
                     "hbm": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                             "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes64},
                     "u01f_f32_launch_ms": avg32, "u01f_f32_achieved_gbs": 4.0 * N_HEAD / (avg32 / 1e3) / 1e9},
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


def run_per_config(dev, stream, sptr, buf, peak, cpu_seconds, cpu=True, issue_mhz=1965.0):
    """Every BASELINE row at its stated size, timed through the product call (Rng.fill with
    a device `out`, fill_streams, Rng.mvn): CUDA events on the stream around the
    synchronous call, best of 5 after two warm-up calls. Beside each: the fraction of the store-only
    HBM figure (the ceiling of a fill) and of the copy figure, and the same-run
    CPU rate of the port (P = all host threads, and P = 1)."""
    import torch

    from oracle import oracle as O
    from paper_2605_05099_b200 import _lib, fill_streams, state_io
    from paper_2605_05099_b200.rng import _out_dtype

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
    P = O.cpu_count()
    res["cpu"] = {"model": cpu_model(), "threads": P,
                  "how": "oracle port (C restatement of the reference), P threads on disjoint substreams "
                         "(philox counter offsets, x256 GF(2) jumps, pcg64 advance, ranlux A^k, sfc64 spawned "
                         "streams), repeated fills of ~50 ms per call for %.1f s; and P = 1" % cpu_seconds}

    def timed(go, reps=5):
        # two warm-up calls (plan caches, scratch growth, and the SM clock back up after the
        # host-bound legs before this row), then the best of `reps`
        go()
        go()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            go()
            z.record(stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(z))
        return best

    def cpu_pair(engine, seed, dist, params, fm=False, spawn=False):
        if not cpu:
            return None
        return {"p_all": cpu_rate(engine, seed, dist, params, P, cpu_seconds, fm, spawn),
                "p_1": cpu_rate(engine, seed, dist, params, 1, cpu_seconds, fm, spawn)}

    def row(label, engine, seed, dist, params, n, fm=False):
        r = state_io.create(engine, seed=seed)
        r.set_full_mantissa(fm)
        out = buf.view(_out_dtype(dist))[:n]
        ms = timed(lambda: r.fill(dist, params, n, out=out))
        bpe = out.element_size()
        gbs = n * bpe / (ms / 1e3) / 1e9
        res[label] = {"gsamples_s": n / (ms / 1e3) / 1e9, "ms": ms, "n": n, "bytes_per_sample": bpe,
                      "write_frac": gbs / wpeak, "hbm_frac": gbs / peak,
                      "timed": "Rng.fill(dist, params, n, out=device tensor) -> rs_fill (synchronous)",
                      "cpu": cpu_pair(engine, seed, dist, params, fm)}

    row("c1_x256ss_raw_u64_2p30", "x256**", [12345], "uint64", {}, 1 << 30)
    row("c2_philox_u01_f64_2p30", "philox", [7], "u01", {}, 1 << 30, fm=True)
    row("c2_philox_u01f_f32_2p30", "philox", [7], "u01f", {}, 1 << 30, fm=True)
    row("c3_x256ss_norm_2p28", "x256**", [2024], "norm", {}, 1 << 28)
    row("c3_pcg64_norm_2p28", "pcg64", [2024], "norm", {}, 1 << 28)
    row("c4_pcg64_exp_2p26", "pcg64", [99], "exp", {}, 1 << 26)
    for k in (0.3, 1.0, 2.5, 10.0):
        row("c4_pcg64_gamma_%g_2p26" % k, "pcg64", [99], "gamma", {"alpha": k}, 1 << 26)
    row("c4_pcg64_beta_2_5_2p26", "pcg64", [99], "beta", {"a": 2.0, "b": 5.0}, 1 << 26)
    row("extra_ranlux_raw_2p30", "ranlux++", [12345], "uint64", {}, 1 << 30)
    # C5b: sfc64 per-stream Lemire, 2^16 streams x 4096
    S, per = 1 << 16, 4096
    for m in (6, 1000003, (1 << 63) + 1):
        rows = torch.empty((S, per), dtype=torch.uint64, device=dev)
        ms = timed(lambda: fill_streams("sfc64", [31], [], 0, S, "uint64", {"b": m}, per, out=rows))
        n = S * per
        gbs = n * 8 / (ms / 1e3) / 1e9
        res["c5b_sfc64_streams_lemire_%d_2p28" % m] = {
            "gsamples_s": n / (ms / 1e3) / 1e9, "ms": ms, "n": n, "write_frac": gbs / wpeak, "hbm_frac": gbs / peak,
            "timed": "fill_streams(..., out=) into a resident 2 GiB tensor -> rs_fill_streams",
            "cpu": cpu_pair("sfc64", [31], "uint64", {"b": m}, spawn=True)}
        del rows
    # FP64 peak for the MVN contraction: cuBLAS DGEMM 8192^3 through torch
    mm = 8192
    a64 = torch.randn(mm, mm, dtype=torch.float64, device=dev)
    b64 = torch.randn(mm, mm, dtype=torch.float64, device=dev)
    c64 = torch.matmul(a64, b64)
    ms = timed(lambda: torch.matmul(a64, b64, out=c64))
    tf = 2.0 * mm ** 3 / (ms / 1e3) / 1e12
    res["fp64_dgemm_peak"] = {"tflops": tf, "how": "torch.matmul f64 8192^3 (cuBLAS DGEMM), best of 3, CUDA events"}
    del a64, b64, c64
    # C5a: mvn, d in {64, 256, 512}, n = 2^20 (the BASELINE recipe: philox seed 31, S from the
    # same r, mvn on the same r). Whole call (z draw overlapping the host Cholesky, then the
    # contraction) and the contraction alone (rs_mvn_apply: k_mvn_dmma, FP64 tensor cores)
    # (all three GPU timings first: the CPU leg's OpenBLAS threads keep spinning for a while
    # after a call and slowed the next row's host-side symmetry check and Cholesky by 2-4 ms)
    mvn_rows = {}
    for d in (64, 256, 512):
        n = 1 << 20
        r = state_io.create("philox", seed=[31])
        A = r.fill("norm", {}, d * d).cpu().numpy().reshape(d, d)
        S_ = A @ A.T / d + np.eye(d)
        ms_all = timed(lambda: r.mvn(np.zeros(d), S_, n=n), reps=3)
        Lf = np.ascontiguousarray(np.linalg.cholesky(S_))
        mean = np.zeros(d)
        z = r.device_fill("stdnorm", [], [], n * d)
        X = torch.empty(n * d, dtype=torch.float64, device=dev)
        ms_k = timed(lambda: _lib.check(_lib.lib.rs_mvn_apply(
            ctypes.c_void_p(Lf.ctypes.data), mean.ctypes.data_as(_lib.DBLP), d, n, 0, ctypes.c_void_p(z.data_ptr()),
            ctypes.c_void_p(X.data_ptr()), sptr)))
        zt = torch.empty(n * d, dtype=torch.float64, device=dev)
        ms_z = timed(lambda: r.device_fill("stdnorm", [], [], n * d, out=zt))
        del z, X, zt
        mvn_rows[d] = (ms_all, ms_k, ms_z, Lf)
    for d in (64, 256, 512):
        n = 1 << 20
        ms_all, ms_k, ms_z, Lf = mvn_rows[d]
        tri = n * d * (d + 1)
        cpu_r = None
        if cpu:  # the reference's CPU path: z by the port (P threads), X = z @ L^T by numpy
            nn = 1 << 14
            o = O.OracleRng("philox", seed=[31])
            t0 = time.perf_counter()
            reps = 0
            while True:
                zs = O.threaded_fill([o.clone() for _ in range(P)], "stdnorm", {}, nn * d // P)
                zz = np.concatenate(zs).reshape(-1, d)
                _ = zz @ Lf.T
                reps += 1
                el = time.perf_counter() - t0
                if el >= cpu_seconds:
                    break
            cpu_r = {"vectors_per_s": reps * nn / el, "cores": P,
                     "how": "z by the port on P threads + numpy z @ L^T (OpenBLAS), 2^14 vectors per call"}
        res["c5a_mvn_d%d_2p20" % d] = {
            "vectors_per_s": n / (ms_all / 1e3), "ms": ms_all,
            "timed": "Rng.mvn(0, S, 2^20): z fill + host symmetry check and Cholesky (overlapped) + contraction",
            "z_fill_ms": ms_z, "z_fill_gsamples_s": n * d / (ms_z / 1e3) / 1e9,
            "contraction_ms": ms_k, "contraction_tflops_triangular": tri / (ms_k / 1e3) / 1e12,
            "contraction_tflops_dense_equiv": 2.0 * n * d * d / (ms_k / 1e3) / 1e12,
            "contraction_frac_of_dgemm_peak": tri / (ms_k / 1e3) / 1e12 / tf,
            "contraction_kernel": "k_mvn_dmma (mma.sync f64 / DMMA.8x8x4; triangular skip)",
            "cpu": cpu_r}
    # Issue roofline of every row whose ceiling is instruction issue, not HBM (parse kernels,
    # per-stream Lemire, the integer-bound engines): warp instructions of one fill (ncu
    # smsp__inst_executed.sum over the fill's kernels, profiles/r02_issue_counts.json) / the
    # row's time measured above, against one warp instruction per SMSP per cycle.
    prof = os.path.join(ROOT, "profiles", "r02_issue_counts.json")
    if os.path.exists(prof):
        with open(prof) as f:
            counts = json.load(f)["configs"]
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ipeak = sms * 4 * issue_mhz * 1e6 / 1e9  # G warp instructions / s
        for label, c in counts.items():
            if label in res and "ms" in res[label] and c.get("warp_instr"):
                ach = c["warp_instr"] / (res[label]["ms"] / 1e3) / 1e9
                res[label]["issue_roofline"] = {
                    "bound": "issue", "warp_instr_per_sample": c["warp_instr"] / res[label]["n"],
                    "lanes_per_warp_instr": c["thread_instr"] / c["warp_instr"],
                    "achieved": ach, "peak": ipeak, "unit": "G warp instructions/s", "frac": ach / ipeak,
                    "peak_source": "%d SMs x 4 SMSPs x 1 warp instruction/cycle x %.0f MHz" % (sms, issue_mhz),
                    "source": "profiles/r02_issue_counts.json (ncu --metrics smsp__inst_executed.sum, same fill)"}
        z = counts.get("c5a_z_philox_norm_2p29")
        row512 = res.get("c5a_mvn_d512_2p20")
        if z and row512 and row512.get("z_fill_ms"):
            ach = z["warp_instr"] / (row512["z_fill_ms"] / 1e3) / 1e9
            row512["z_fill_issue_roofline"] = {
                "bound": "issue", "warp_instr_per_sample": z["warp_instr"] / float(1 << 29),
                "lanes_per_warp_instr": z["thread_instr"] / z["warp_instr"],
                "achieved": ach, "peak": ipeak, "unit": "G warp instructions/s", "frac": ach / ipeak,
                "note": "2^29 Philox normals: materialise (integer-bound) + count + emit over the words",
                "source": "profiles/r02_issue_counts.json"}
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
        ref = C2Reference(world)
        for _ in range(args.warmup):
            ref.step()
        times = [ref.step() for _ in range(args.steps)]
        el = float(np.sum(times))
        v = 2 * N_HEAD * world * args.steps / el / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
                "data": "synthetic: seeded stream fills (no dataset is involved)",
                "config": {"workload": "BASELINE config 2: philox (Philox-4x64-10) seed=7 full_mantissa; u01 f64 "
                                       "n=2^30 + u01f f32 n=2^30 per GPU; rank g = counter-offset slice g",
                           "same_config": True, "parallelism": "%d host threads" % ref.P},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": ref.P, "kind": "port", "sample": ref.sample()},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist

    if world > 1:
        # RS_BENCH_BACKEND=gloo: plumbing test of the N > 1 path on a box with fewer GPUs than
        # ranks (ranks share devices; no kernel waits on another rank). Never a bench number.
        backend = os.environ.get("RS_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    line = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            ref = C2Reference(1)
            ref.step()  # first touch of the host arrays
            el = ref.step()
            v = 2 * N_HEAD / el / 1e9
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": ref.P, "kind": "port",
                                    "sample": ref.sample() + "; one timed step after one warm-up"}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
