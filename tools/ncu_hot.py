"""Hot basic blocks of an `ncu --page source --csv --print-source sass` export.

    python tools/ncu_hot.py SRC.csv [N]
Groups consecutive SASS lines with equal execution counts and prints the N blocks with
the most executed warp instructions (count x length), per kernel.
"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    kern, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            kern.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and len(r) > 5:
            cur["rows"].append(r)
    seen = set()
    for k in kern:
        if k["name"] in seen:
            continue
        seen.add(k["name"])
        h = k["hdr"]
        iE, iS, iT = h.index("Instructions Executed"), h.index("Source"), h.index("Avg. Threads Executed")
        iW = h.index("Warp Stall Sampling (All Samples)")
        d = k["rows"]
        tot = sum(num(r[iE]) for r in d)
        ws = sum(num(r[iW]) for r in d)
        print("%s  warp-instr %.0f  stall samples %.0f" % (k["name"][:70], tot, ws))
        blocks = []
        for i, r in enumerate(d):
            e = num(r[iE])
            if blocks and blocks[-1]["e"] == e and blocks[-1]["end"] == i - 1:
                blocks[-1]["end"] = i
                blocks[-1]["w"] += num(r[iW])
            else:
                blocks.append({"e": e, "start": i, "end": i, "w": num(r[iW]), "t": r[iT]})
        blocks.sort(key=lambda b: -b["e"] * (b["end"] - b["start"] + 1))
        for b in blocks[:top]:
            n = b["end"] - b["start"] + 1
            print("  rows %5d-%5d n=%3d exec=%9d %5.1f%% thr=%s stall=%5.1f%%  %s" % (
                b["start"], b["end"], n, b["e"], 100 * b["e"] * n / tot, b["t"], 100 * b["w"] / max(ws, 1),
                d[b["start"]][iS].strip()[:60]))


if __name__ == "__main__":
    main()
