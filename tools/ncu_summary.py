"""Print the key sections of an ncu report (details page) — for profiles/ summaries."""
import csv
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
            "Scheduler Statistics", "Warp State Statistics", "Compute Workload Analysis")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = set(sys.argv[2:]) if len(sys.argv) > 2 else None
for row in r[1:]:
    sec, name, unit, val = (row[h.index(c)] for c in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    if sec in SECTIONS and (want is None or any(w in name for w in want)):
        print(f"{sec[:26]:26s} {name:48s} {val:>14s} {unit}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active",
        "smsp__inst_executed_pipe_tensor", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak"]
hdr, units, vals = rr[0], rr[1], rr[2]
for i, k in enumerate(hdr):
    if any(k.startswith(x) for x in keys):
        print(f"raw {k:70s} {vals[i]:>16s} {units[i]}")
