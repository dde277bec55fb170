"""Instruction / stall-sample share per (file, line range) region of an ncu report.

    python tools/ncu_regions.py report.ncu-rep
Regions are the named line ranges below (warp_seg.cuh / batch.cu of round 1).
"""
import csv
import io
import subprocess
import sys

REGIONS = {
    "warp_seg.cuh": [(0, "init"), (80, "new-component"), (101, "row+guess"), (127, "movers"),
                     (161, "ext-scan"), (173, "pre-split"), (200, "split-scan"), (251, "split-loops"),
                     (293, "append"), (306, "tail")],
    "batch.cu": [(0, "batch-setup"), (66, "write-order"), (69, "peo"), (131, "witness")],
}


def _i(x):
    try:
        return int(float(x))
    except (TypeError, ValueError):
        return 0


def region(f, ln):
    best = f
    for start, name in REGIONS.get(f, []):
        if ln >= start:
            best = f"{f}:{name}"
    return best


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, fname, agg = None, None, {}
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr, r))
        a = agg.setdefault(region(fname, ln), [0, 0])
        a[0] += _i(d.get("Instructions Executed"))
        a[1] += _i(d.get("Warp Stall Sampling (All Samples)"))
    T = sum(a[0] for a in agg.values()) or 1
    S = sum(a[1] for a in agg.values()) or 1
    print(f"instructions {T}, stall samples {S}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} inst {100 * v[0] / T:5.1f}%  samples {100 * v[1] / S:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
