"""Condense an `ncu --page raw --csv` export into the JSON summary kept under profiles/.

    python tools/ncu_summary.py RAW.csv OUT.json --capture "<the ncu command>" [--algorithmic-bytes B]

Keeps the metrics the roofline and the DESIGN.md tables cite: duration, DRAM bytes and
throughput, pipe utilisation, issue activity, warp stalls, occupancy, divergence.
"""
import argparse
import csv
import json

KEEP_PREFIX = (
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__warps_active.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("out")
    ap.add_argument("--capture", required=True)
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--row", type=int, default=0, help="which captured launch (0 = first)")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units, vals = rows[0], rows[1], rows[2 + a.row]
    metrics = {}
    kernel = None
    for k, u, v in zip(hdr, units, vals):
        if k == "Kernel Name":
            kernel = v
        stall = k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
        if not (k in KEEP_PREFIX or stall):
            continue
        try:
            f = float(v.replace(",", ""))
        except ValueError:
            continue
        if stall and f < 0.05:
            continue
        metrics[k] = {"value": f, "unit": u}
    out = {"kernel": kernel, "capture": a.capture, "metrics": metrics}
    rd, wr = metrics.get("dram__bytes_read.sum"), metrics.get("dram__bytes_write.sum")
    if rd and wr:
        out["traffic_bytes_per_launch"] = rd["value"] * SCALE.get(rd["unit"], 1) + wr["value"] * SCALE.get(wr["unit"], 1)
    if a.algorithmic_bytes:
        out["algorithmic_bytes_per_launch"] = a.algorithmic_bytes
    json.dump(out, open(a.out, "w"), indent=1)
    print("wrote", a.out, "traffic", out.get("traffic_bytes_per_launch"))


if __name__ == "__main__":
    main()
