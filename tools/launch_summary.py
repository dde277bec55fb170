"""Per-kernel totals of an ncu launch list (the --metrics gpu__time_duration.sum
--csv pass of bench.py), largest first.

    python tools/launch_summary.py launches.csv "bench.py --steps 2 --warmup 3 --no-cpu"
"""
import collections
import csv
import sys


def main(path, command):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        a = agg[r[ki]]
        a[0] += 1
        a[1] += v * scale.get(r[ui], 1e-6)
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none -c 400 (cold, serialised): {command}")
    print("count total_ms avg_us kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:4d} {t:10.3f} {t * 1e3 / c:10.2f} {k[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
