"""Top warp-stall-sampled SASS lines of an ncu report (with their neighbours)."""
import csv, subprocess, sys

rep, ntop = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr, data = rows[0], rows[1:]
i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
tot = sum(float(r[i_s] or 0) for r in data)
print("total samples", tot)
order = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:ntop]
for k in order:
    prev = data[k - 1][i_src].strip()[:50] if k else ""
    print(f"{float(data[k][i_s]) / tot * 100:5.1f}%  [{k:5d}] {data[k][i_src].strip()[:60]:60s} | prev: {prev}")
