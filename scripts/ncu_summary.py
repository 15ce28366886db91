"""Summarise an ncu report (raw page) into the metrics we track; usage: python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("---", r[h.index("Kernel Name")][:70])
        for w in WANT:
            if w in h:
                print(f"  {w:58s} {r[h.index(w)]:>16s} {units[h.index(w)]}")
        stalls = []
        for i, w in enumerate(h):
            if w.startswith("smsp__pcsamp_warps_issue_stalled") and not w.endswith("not_issued"):
                try:
                    v = float(r[i] or 0)
                except ValueError:
                    continue
                if v > 0:
                    stalls.append((v, w.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in stalls) or 1
        print("  stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
