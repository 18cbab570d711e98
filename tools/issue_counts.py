"""Sum the ncu --metrics launch lists written by tools/issue_counts.sh per config:
warp instructions, thread instructions and kernel time of one fill -> profiles JSON.

    python tools/issue_counts.py DIR OUT.json
"""
import csv
import glob
import json
import os
import sys

d, out = sys.argv[1], sys.argv[2]
res = {}
for path in sorted(glob.glob(os.path.join(d, "*.csv"))):
    label = os.path.basename(path)[:-4]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    per = {}
    for r in rows:
        kid, kname, metric, val = r[0], r[4], r[-3], float(r[-1].replace(",", ""))
        unit = r[-2]
        k = per.setdefault(kid, {"kernel": kname.split("(")[0].replace("void <unnamed>::", "")})
        if metric == "gpu__time_duration.sum":
            val *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(unit, 1.0)
        k[metric] = val
    ks = list(per.values())
    # streams_fill.py launches the fill 4 times: keep one launch of each kernel name
    if label.startswith("c5b"):
        ks = ks[-1:]
    res[label] = {
        "warp_instr": sum(k.get("smsp__inst_executed.sum", 0) for k in ks),
        "thread_instr": sum(k.get("smsp__thread_inst_executed.sum", 0) for k in ks),
        "kernel_us_under_ncu": sum(k.get("gpu__time_duration.sum", 0) for k in ks),
        "kernels": [{"kernel": k["kernel"][:60], "warp_instr": k.get("smsp__inst_executed.sum"),
                     "us": k.get("gpu__time_duration.sum"),
                     "issue_active_pct": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active")} for k in ks],
    }
json.dump({"how": "bash tools/issue_counts.sh: ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,"
                  "gpu__time_duration.sum,smsp__issue_active... --clock-control none over one fill per config "
                  "(tools/profile_fill.py / tools/streams_fill.py, bench.py's seeds); summed over the fill's kernels",
           "configs": res}, open(out, "w"), indent=1)
print("wrote", out, len(res), "configs")
