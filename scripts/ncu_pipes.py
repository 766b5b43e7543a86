"""Pipe utilisation and issue metrics of an ncu report (run where the report is).

python scripts/ncu_pipes.py <rep.ncu-rep>   -> prints metric, value for pipe / issue / stall keys
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, unit, val = rows[0], rows[1], rows[2]
keys = ("pipe_", "issue_active", "inst_executed.avg.per_cycle", "warps_active", "throughput",
        "smsp__average_warp", "inst_executed_pipe")
for h, u, v in zip(hdr, unit, val):
    if any(k in h for k in keys) and ("pct" in h or "per_cycle" in h or "ratio" in h):
        try:
            if float(v) == 0:
                continue
        except ValueError:
            continue
        print(f"{h:90s} {v:>14s} {u}")
