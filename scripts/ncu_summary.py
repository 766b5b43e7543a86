"""Summarise ncu artefacts from gpurun_out/ into committed text under profiles/.

python scripts/ncu_summary.py gpurun_out/prof_X.ncu-rep profiles/rNN_X.md [workload-key]
python scripts/ncu_summary.py --launches gpurun_out/launches.csv profiles/rNN_launches.md

The .ncu-rep files themselves stay in gpurun_out/ (scratch); the summary holds the numbers
the roofline claims rest on: duration, DRAM bytes (traffic), DRAM % of peak, per-instruction
shared-memory wavefronts (ideal vs. actual), stall reasons, registers, launch shape.
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def summarize_rep(rep, out_md, key=None):
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", "",
             f"Kernel: `{kname}`", "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in m:
            lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    lines += ["", f"DRAM traffic per launch (read + write): {(rd + wr) / 1e6:.1f} MB "
              "(cold L2: ncu flushes caches before the launch, so the tail of the output is "
              "still dirty in L2 when the kernel ends and is written back afterwards)."]
    # per-instruction shared-memory wavefronts and stalls
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    h = src[1]
    idx = {x: i for i, x in enumerate(h)}
    lines += ["", "## Shared-memory instructions (address-pattern conflicts)", "",
              "| SASS | executed | wavefronts | ideal | excessive |", "|---|---|---|---|---|"]
    for r in src[2:]:
        s = r[idx["Source"]].strip()
        if re.search(r"\b(LDS|STS)", s):
            lines.append(f"| `{s}` | {r[idx['Instructions Executed']]} | "
                         f"{r[idx['L1 Wavefronts Shared']]} | {r[idx['L1 Wavefronts Shared Ideal']]} | "
                         f"{r[idx['L1 Wavefronts Shared Excessive']]} |")
    tma = collections.Counter()
    for r in src[2:]:
        s = r[idx["Source"]].strip()
        mm = re.search(r"\b(UTMALDG|UTMASTG|UBLKCP)\S*", s)
        if mm:
            tma[mm.group(0)] += int(float(r[idx["Instructions Executed"]] or 0))
    lines += ["", "TMA instructions executed: " + ", ".join(f"`{k}` x{v}" for k, v in tma.items())]
    stall_cols = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    agg = collections.Counter()
    for r in src[2:]:
        for c in stall_cols:
            try:
                agg[c] += float(r[idx[c]] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    lines += ["", "## Warp stall sampling (all samples)", "", "| reason | share |", "|---|---|"]
    for c, v in agg.most_common(8):
        lines.append(f"| {c} | {100 * v / tot:.1f}% |")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if key:
        tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(tj)) if os.path.exists(tj) else {}
        d[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                  "duration_us": float(m["gpu__time_duration.sum"][0].replace(",", "")),
                  "source": os.path.basename(out_md), "kernel": kname,
                  "note": "ncu --set full, single launch, cold L2 (caches flushed by ncu)"}
        json.dump(d, open(tj, "w"), indent=1)
    print(open(out_md).read())


def summarize_launches(path, out_md):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    idx = {x: i for i, x in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[idx["Metric Value"]].replace(",", "")) * scale[r[idx["Metric Unit"]]]
        agg[r[idx["Kernel Name"]]][0] += 1
        agg[r[idx["Kernel Name"]]][1] += v
    # bench.py's untimed device spin (torch.cuda._sleep, queued before the timed region so the
    # region times the GPU, not the host's launches) is not part of a step: listed apart
    gate = {k: v for k, v in agg.items() if "spin_kernel" in k}
    agg = {k: v for k, v in agg.items() if "spin_kernel" not in k}
    tot = sum(t for _, t in agg.values())
    lines = [f"# Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`): "
             f"`{os.path.basename(path)}`", "",
             "Serialised, cold-cache per-launch device times: compare shares, not absolutes.", "",
             "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:90]}` | {n} | {t:.1f} | {100 * t / tot:.1f}% | {t / n:.2f} |")
    for k, (n, t) in gate.items():
        lines += ["", f"Not in a step: `{k[:60]}` x{n} ({t:.0f} us) -- bench.py's untimed device "
                      "spin before the timed region (its length follows the host's launch time, "
                      "which ncu inflates)."]
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(open(out_md).read())


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarize_launches(sys.argv[2], sys.argv[3])
    else:
        summarize_rep(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
