"""Compact summary of an ncu report (raw page) for profiles/.
usage: python tools/ncu_summary.py report.ncu-rep [label] [--json out.json]

--json also writes the per-launch DRAM traffic (dram__bytes_read.sum +
dram__bytes_write.sum) and duration of every captured launch, the source of
bench.py's roofline "traffic" (profiles/traffic.json)."""
import csv
import io
import json
import subprocess
import sys

_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
]


def _val(row, h, u, name):
    i = h.index(name)
    return float(row[i].replace(",", "")) * _SCALE.get(u[i], 1.0)


def main():
    argv = list(sys.argv[1:])
    jout = None
    if "--json" in argv:
        k = argv.index("--json")
        jout = argv[k + 1]
        del argv[k:k + 2]
    rep = argv[0]
    label = argv[1] if len(argv) > 1 else rep
    launches = []
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
        if "dram__bytes_read.sum" in h and "gpu__time_duration.sum" in h:
            launches.append({"kernel": name[:160], "us": _val(row, h, u, "gpu__time_duration.sum"),
                             "dram_bytes": _val(row, h, u, "dram__bytes_read.sum") +
                             _val(row, h, u, "dram__bytes_write.sum")})
        print()
    if jout:
        with open(jout, "w") as fh:
            json.dump({"label": label, "launches": launches}, fh, indent=1)


if __name__ == "__main__":
    main()
