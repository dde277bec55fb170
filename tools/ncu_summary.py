"""Key counters of every kernel in an ncu report (raw page).

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active%"),
    ("sm__maximum_warps_per_active_cycle_pct", "occ_limit%"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "?")[:90])
        for k, name in KEYS:
            if k in d:
                print(f"  {name:14s} {d[k]:>16s} {units[hdr.index(k)]}")
        st = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  stalls/issue  " + "  ".join(f"{n}={v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
