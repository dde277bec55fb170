"""Summarise an ncu report per CUDA source line: instructions executed and stall samples.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = []
    cur = None
    for r in rows:
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            d = dict(zip(hdr, r))
            try:
                cur = [int(r[0]), r[1].strip()[:90], int(d["Warp Stall Sampling (All Samples)"] or 0),
                       int(float(d["Instructions Executed"] or 0))]
            except ValueError:
                continue
            lines.append(cur)
    tot_s = sum(x[2] for x in lines) or 1
    tot_i = sum(x[3] for x in lines) or 1
    print(f"total stall samples {tot_s}, instructions {tot_i}")
    for ln in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln[0]:5d} samp {100 * ln[2] / tot_s:5.1f}%  inst {100 * ln[3] / tot_i:5.1f}%  {ln[1]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
