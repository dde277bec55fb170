"""Summarise an ncu report per CUDA source line: stall samples, instructions,
dominant stall reasons and the memory spaces the line's SASS touches.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_lg", "stall_mio", "stall_branch_resolving",
           "stall_barrier", "stall_membar", "stall_math", "stall_no_inst", "stall_dispatch", "stall_selected",
           "stall_not_selected", "stall_drain", "stall_misc", "stall_tex", "stall_sleep"]


def _i(x):
    try:
        return int(float(x))
    except (TypeError, ValueError):
        return 0


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = {}
    cur = None
    for r in rows:
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        d = dict(zip(hdr, r))
        if r[0]:
            try:
                ln = int(r[0])
            except ValueError:
                continue
            cur = lines.setdefault(ln, {"src": r[1].strip()[:80], "samp": 0, "inst": 0, "why": {}, "space": set()})
            cur["samp"] += _i(d.get("Warp Stall Sampling (All Samples)"))
            cur["inst"] += _i(d.get("Instructions Executed"))
            for k in REASONS:
                cur["why"][k] = cur["why"].get(k, 0) + _i(d.get(k))
        elif cur is not None:
            # SASS rows under the current source line (the second "Source"/"Address Space" columns)
            sp = r[13] if len(r) > 13 else "-"
            if sp and sp != "-":
                cur["space"].add(sp)
    tot_s = sum(x["samp"] for x in lines.values()) or 1
    tot_i = sum(x["inst"] for x in lines.values()) or 1
    print(f"total stall samples {tot_s}, instructions {tot_i}")
    for ln, x in sorted(lines.items(), key=lambda kv: -kv[1]["samp"])[:top]:
        why = sorted(x["why"].items(), key=lambda kv: -kv[1])[:2]
        ws = " ".join(f"{k[6:]}={100 * v / max(x['samp'], 1):.0f}%" for k, v in why if v)
        print(f"{ln:5d} samp {100 * x['samp'] / tot_s:5.1f}% inst {100 * x['inst'] / tot_i:5.1f}% "
              f"[{ws}] {','.join(sorted(x['space']))[:20]:20s} {x['src']}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
