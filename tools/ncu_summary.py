"""Compact summary of an ncu report (raw page) for profiles/.
usage: python tools/ncu_summary.py report.ncu-rep [label]"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    print(f"# ncu --set full summary: {label}")
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        print(f"kernel: {name[:160]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w} = {row[i]} {u[i]}")
        rd = row[h.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h else None
        print()


if __name__ == "__main__":
    main()
