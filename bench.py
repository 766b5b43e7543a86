#!/usr/bin/env python
"""bench.py -- effective transpose GB/s (read+write) and % of HBM peak on 1..8 B200.

Contract (task ③/④, BASELINE.json "metric"):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]
A "step" is one pass of the whole hot path over one batch of synthetic input: one
C-ABI call (one kernel launch) transposing the workload's matrices.  Rank 0 prints ONE
JSON line.  Under torchrun (N > 1) every rank transposes its own matrices (independent
problems, no data-path collective: "scaling": "weak"); the time is the max over ranks.

Default workload: 8192 x 8192 f32 (BASELINE.json configs[2], the headline target).
Other workloads (--workload): 2048f64 (configs[1], L2-flushed), 3000x5000f64 (configs[2]),
batched (configs[3], 256 x 1024^2 f32 sharded over ranks), dist65536 (configs[4]).

--impl reference times the CPU oracle (oracle/, naive single-thread C loop) on the same
workload -- the one other place bench.py executes oracle/ besides the cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded input generators only; no method arithmetic)

METRIC = "transpose effective GB/s (read+write) and % of HBM peak at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024
KERNEL_FN = {"tma_st": "desc::transpose_tma2_kernel (TMA load + TMA store)",
             "tma": "desc::transpose_tma_kernel (TMA load + st.global)",
             "smem": "desc::transpose_smem_kernel (32x33 smem tile)",
             "tiled": "desc::transpose_tiled_kernel (64x64-cell tiles for 4-byte cells, 32x32 for 8-byte; padded smem tile, 16 / 8 loads in flight per thread)",
             "tma_tile": "desc::transpose_tma_tile_kernel (one 16 KB tile per CTA: TMA load, "
                         "register micro-transpose, TMA store)",
             "vtiled": "desc::transpose_vtiled_kernel (one tile per CTA: 16-byte cp.async staging "
                       "into a 16-byte-swizzled tile, register micro-transposes, 16-byte stores)"}

WORKLOADS = {
    "8192f32": dict(batch=1, rows=8192, cols=8192, dtype="f32", es=4,
                    name="8192x8192 f32 transpose (BASELINE.json configs[2], headline target)"),
    "2048f64": dict(batch=1, rows=2048, cols=2048, dtype="f64", es=8,
                    name="2048x2048 f64 transpose (BASELINE.json configs[1], the paper's listing shape)"),
    "3000x5000f64": dict(batch=1, rows=3000, cols=5000, dtype="f64", es=8,
                         name="3000x5000 f64 non-tile-multiple transpose (BASELINE.json configs[2])"),
    "4096f64": dict(batch=1, rows=4096, cols=4096, dtype="f64", es=8,
                    name="4096x4096 f64 transpose (paper-size extra: 256 MB in+out, P:1051)"),
    "8192i32": dict(batch=1, rows=8192, cols=8192, dtype="i32", es=4,
                    name="8192x8192 i32 transpose (configs[2] shape, int32: dtype independence)"),
    "8192f64": dict(batch=1, rows=8192, cols=8192, dtype="f64", es=8,
                    name="8192x8192 f64 transpose (paper-size extra: 1 GiB in+out, P:1051)"),
    "3000x5000f64_ld5001": dict(batch=1, rows=3000, cols=5000, dtype="f64", es=8, ld_in=5001,
                                name="3000x5000 f64 with ld_in = 5001 (TMA-ineligible: 40008-byte pitch; "
                                     "BASELINE.json configs[2] fallback variant)"),
    "8192f32_ld8193": dict(batch=1, rows=8192, cols=8192, dtype="f32", es=4, ld_in=8193,
                           name="8192x8192 f32 with ld_in = 8193 (TMA-ineligible pitch)"),
    "batched": dict(batch=256, rows=1024, cols=1024, dtype="f32", es=4, shard=True,
                    name="batched 256x(1024x1024) f32, batch sharded over ranks (BASELINE.json configs[3])"),
    "dist65536": dict(batch=1, rows=65536, cols=65536, dtype="f32", es=4, dist=True,
                      name="65536x65536 f32 distributed transpose, row slabs + exchange (BASELINE.json configs[4])"),
}
GBT = [("group", 64, 0), ("group", 64, 2), ("transpose", 0, 1)]   # group_by_tile<64,64>
VIEW_WORKLOADS = {
    "view_tiles8192f32": ("8192x8192 f32 view copy: group_by_tile<64,64> (tile-major layout)", GBT),
    "view_transpose8192f32": ("8192x8192 f32 view copy: transpose", [("transpose", 0, 0)]),
    "view_rot90_8192f32": ("8192x8192 f32 view copy: transpose.map(reverse) (rot90)",
                           [("transpose", 0, 0), ("reverse", 0, 1)]),
    "view_flip8192f32": ("8192x8192 f32 view copy: reverse.map(reverse) (rot180)",
                         [("reverse", 0, 0), ("reverse", 0, 1)]),
}
for _k, (_n, _ops) in VIEW_WORKLOADS.items():
    WORKLOADS[_k] = dict(batch=1, rows=8192, cols=8192, dtype="f32", es=4, view=_ops,
                         name=_n + " (SURVEY 8(f) NEXT #2)")
WORKLOADS["reduce64M_f32"] = dict(batch=1, rows=1, cols=1 << 26, dtype="f32", es=4, op="reduce",
                                  block=1024, name="block-wide reduction, n = 2^26 f32 (256 MB), "
                                  "block 1024 (SURVEY 8(f) NEXT #3, P:1047)")
WORKLOADS["scan64M_f32"] = dict(batch=1, rows=1, cols=1 << 26, dtype="f32", es=4, op="scan",
                                name="inclusive scan, n = 2^26 f32 (256 MB) (SURVEY 8(f) NEXT #4, P:1047)")
WORKLOADS["scan64M_i32"] = dict(batch=1, rows=1, cols=1 << 26, dtype="i32", es=4, op="scan",
                                name="inclusive scan, n = 2^26 i32 (256 MB) (SURVEY 8(f) NEXT #4, P:1047)")
WORKLOADS["scan32M_f64"] = dict(batch=1, rows=1, cols=1 << 25, dtype="f64", es=8, op="scan",
                                name="inclusive scan, n = 2^25 f64 (256 MB) (SURVEY 8(f) NEXT #4, P:1047)")
NOMINAL_HBM_GBS = 8000.0  # BASELINE.json north star / SURVEY 8(d): the nominal B200 HBM3e figure
NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction per GPU


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload: str, kernel: str = "auto"):
    """dram bytes (read+write) per launch of the dominant kernel from the committed
    `ncu --set full` summary, if one exists for this workload (and, for an explicit
    --kernel, for that kernel: key "<workload>:<kernel>")."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(workload if kernel in ("auto", None) else f"{workload}:{kernel}")
        return None if v is None else float(v["dram_bytes_per_launch"])
    except Exception:
        return None


_SAMPLER_CHILD = r"""
import sys, time, json, select
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print(json.dumps({"max": pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)}), flush=True)
out = []
while True:
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    out.append((time.perf_counter(), mhz, r))
    if select.select([sys.stdin], [], [], 0)[0]:
        break
    time.sleep(1e-4)
print(json.dumps(out), flush=True)
"""


class ClockSampler:
    """Samples the SM clock and the throttle reasons with NVML, as fast as NVML answers, with
    host timestamps (CLOCK_MONOTONIC, shared by all processes), in a CHILD PROCESS: a sampler
    thread here would wait for the GIL while the launching thread runs, and missed the
    1.7 ms timed region of the default line entirely.  ``region(t0, t1)`` marks the host-time
    window of the timed region (from just before its first event is recorded to the return
    of the synchronize after it); the summary reports the samples taken inside it."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []            # (host time, sm MHz, reason bits)
        self.ok = False
        self.max_mhz = None
        self.t0 = self.t1 = None
        self.extended = 0
        self.proc = None
        try:
            import pynvml  # noqa: F401  (the child needs it)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def __enter__(self):
        if self.ok:
            import subprocess
            # NVML numbers devices physically: map the CUDA index through CUDA_VISIBLE_DEVICES
            idx = self.index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.index])
                except (ValueError, IndexError):
                    pass
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_CHILD, str(idx)],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            try:
                self.max_mhz = json.loads(self.proc.stdout.readline())["max"]
            except Exception:
                self.ok = False
            time.sleep(0.002)        # the first samples land before the region starts
        return self

    def __exit__(self, *exc):
        if self.ok and self.proc is not None:
            out, _ = self.proc.communicate(input="stop\n", timeout=120)
            try:
                self.samples += [tuple(x) for x in json.loads(out.strip().splitlines()[-1])]
            except Exception:
                pass
            self.proc = None

    def region(self, t0: float, t1: float):
        self.t0, self.t1 = t0, t1

    def _in_region(self):
        if self.t0 is None:
            return list(self.samples)
        return [x for x in self.samples if self.t0 <= x[0] <= self.t1]

    def extend(self, work, torch, dev, seconds: float = 0.3, min_samples: int = 10):
        """A timed region too short for min_samples NVML answers: keep sampling over `seconds`
        of untimed repeats of the same work right after it (reported separately)."""
        if not self.ok or len(self._in_region()) >= min_samples:
            return
        n0 = len(self.samples)
        self.__enter__()
        t_end = time.time() + seconds
        while True:
            for _ in range(20 if seconds > 0 else 1):
                work()
            torch.cuda.synchronize(dev)
            if time.time() >= t_end:
                break
        self.__exit__()
        self.extended = len(self.samples) - n0

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        inr = self._in_region()
        use = inr if inr else self.samples
        reasons = set()
        for _, _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        out = {"sm_mhz": statistics.median(m for _, m, _ in use) if use else None,
               "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
               "samples": len(self.samples), "samples_in_timed_region": len(inr),
               "sm_mhz_from": "samples in the timed region" if inr else "all samples",
               "sampler": "NVML polled in a child process, host CLOCK_MONOTONIC timestamps"}
        if self.extended:
            ext = [m for _, m, _ in self.samples[-self.extended:]]
            out["extension"] = {"samples": self.extended,
                                "sm_mhz": statistics.median(ext),
                                "what": "timed region gave < 10 NVML samples: untimed "
                                        "repeats of the same step right after it"}
        return out


def host_gate(torch, stream, seconds: float):
    """Queue a device-side spin (torch.cuda._sleep) of about `seconds` on `stream` before the
    timed region, so that the host enqueues all K steps while the GPU is still busy: the
    region then measures the device executing K queued steps back to back, not the host's
    launch rate (a 2048^2 f64 step takes ~12 us on B200, about one Python + C-ABI call).
    The spin runs BEFORE the region's first event and is not timed."""
    torch.cuda._sleep(int(max(seconds, 1e-3) * 2.0e9))     # SM clock <= 1.965 GHz


def gate_seconds(host_s_per_step: float, steps: int) -> float:
    """Spin long enough to cover the host's enqueue of `steps` steps twice over (capped)."""
    return min(5.0, 1e-3 + 2.0 * host_s_per_step * steps)


def bench_backend():
    """Process-group backend: NCCL (one GPU per rank, the driver's launch).  DESC_BENCH_BACKEND=
    gloo lets several ranks share one GPU to exercise the N > 1 code path on a 1-GPU box
    (host-side collectives only; the data path never uses a collective here)."""
    return os.environ.get("DESC_BENCH_BACKEND", "nccl")


def init_pg(dev):
    import torch.distributed as dist
    if bench_backend() == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(bench_backend())


def reduce_scalar(x: float, op: str, dev) -> float:
    """max/min of a host scalar over ranks (device tensor for NCCL, host tensor for gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64,
                     device=dev if bench_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return float(t.item())


def local_device(local: int):
    import torch
    n = torch.cuda.device_count()
    return local % n if bench_backend() != "nccl" else local


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info():
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    cpu = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu": cpu, "cpu_count": os.cpu_count(), "affinity": aff}


# ------------------------------------------------------------------------- oracle arm
def run_oracle(wl, budget_s: float, steps: int | None = None, warmup: int = 0,
               band_rows: int | None = None, full_pass: bool = True):
    """Time the oracle (naive single-thread C loop) on a bounded sample of the workload.

    The sample is a sequence of row bands of the workload's matrices, each transposed by
    the oracle into the FULL-size output buffer (same ld_out, so the access pattern is that
    of the whole transpose).  With full_pass the bands cover every matrix of the sample once
    (the output then is the complete oracle result, used for the parity check).
    Returns dict(gbs, reps, sample, times, out, in)."""
    import oracle
    es, rows, cols, batch = wl["es"], wl["rows"], wl["cols"], wl["batch"]
    sample_batch = min(batch, 4)
    if wl.get("dist"):     # bounded sample of the 16 GiB matrix: a 4096-row slab of it
        rows, wl = 4096, dict(wl, name=wl["name"] + " (4096-row slab sample)")
    a = synth.random_bits((sample_batch, rows, cols), es, synth.BASE_SEED + 2)
    out = np.empty((sample_batch, cols, rows), dtype=a.dtype)

    def band(k, br):
        nb = -(-rows // br)
        m, b = divmod(k % (nb * sample_batch), nb)
        r0 = b * br
        r1 = min(rows, r0 + br)
        t0 = time.perf_counter()
        oracle.transpose_raw(a, out, 1, r1 - r0, cols, cols, rows, 0, 0, es,
                             in_offset=m * rows * cols + r0 * cols,
                             out_offset=m * cols * rows + r0)
        return time.perf_counter() - t0, 2 * (r1 - r0) * cols * es

    if band_rows is None:  # calibrate: seconds per row
        dt, _ = band(0, 64)
        per_row = max(dt / 64, 1e-7)
        if steps:
            band_rows = int(budget_s / (steps + warmup) / per_row)
        else:
            band_rows = rows
        band_rows = max(8, min(rows, band_rows))
    nbands = -(-rows // band_rows) * sample_batch
    for k in range(warmup):
        band(k, band_rows)
    times, nbytes = [], 0
    t_end = time.perf_counter() + budget_s
    k = warmup
    while True:
        dt, b = band(k, band_rows)
        times.append(dt)
        nbytes += b
        k += 1
        if steps and len(times) >= steps:
            break
        if not steps and time.perf_counter() >= t_end and (not full_pass or k >= nbands):
            break
    gbs = nbytes / sum(times) / 1e9
    desc = (f"{len(times)} row bands of {band_rows} x {cols} {wl['dtype']} "
            f"(out of {sample_batch} of {batch} {rows}x{cols} matrices), each transposed into the "
            f"full-size output (ld_out={rows}); GB/s = 2*bytes/sum(time)")
    return dict(gbs=gbs, reps=len(times), sample=desc, times=times, out=out, inp=a,
                complete=(k >= nbands and full_pass), band_rows=band_rows,
                sample_batch=sample_batch)


def reference_arm(args, wl, world, rank):
    if rank != 0:
        return 0
    r = run_oracle(wl, budget_s=args.reference_seconds, steps=args.steps, warmup=args.warmup,
                   full_pass=False)
    hi = host_info()
    ms = sum(r["times"]) / len(r["times"]) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": round(r["gbs"], 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": r["reps"], "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": wl["dtype"], "data": "synthetic (seeded random bit patterns)",
        "config": {"workload": wl["name"], "rows": wl["rows"], "cols": wl["cols"],
                   "batch": wl["batch"], "parallelism": "single host thread (CPU oracle)"},
        "cpu_baseline": {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": 1,
                         "kind": "oracle", "sample": r["sample"], "host": hi},
        "e2e": {"value": round(r["gbs"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------- our arm
def small_problem_context(desc, torch, dev, stream, wl, kernel, step, l2_flush, step_bytes,
                          reps: int = 100):
    """Context for small workloads (working set < 2 x L2), outside the timed region: (1) the
    launch floor -- the same kernel on a one-tile problem of the same dtype, timed with a
    flush and events around the launch, i.e. launch + prologue + one load/store round trip;
    (2) the workload itself timed that way (flush + events around each launch); (3) the same
    launches back to back on ONE buffer pair (L2-resident, not the metric)."""
    tdt = {"f32": torch.float32, "f64": torch.float64, "i32": torch.int32}[wl["dtype"]]
    tr = 64 if wl["es"] == 8 else 128
    xt = torch.zeros((tr, 128 // wl["es"]), dtype=tdt, device=dev)
    yt = torch.empty((128 // wl["es"], tr), dtype=tdt, device=dev)
    sptr = stream.cuda_stream

    def tiny():
        desc.desc_transpose_ex(xt.data_ptr(), yt.data_ptr(), 1, xt.shape[0], xt.shape[1],
                               xt.shape[1], xt.shape[0], 0, 0, wl["dtype"], kernel, sptr)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for k in range(reps):
        l2_flush()
        ev[2 * k].record(stream)
        tiny()
        ev[2 * k + 1].record(stream)
    torch.cuda.synchronize(dev)
    floor = statistics.median(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(reps))
    for k in range(reps):
        l2_flush()
        ev[2 * k].record(stream)
        step(0)
        ev[2 * k + 1].record(stream)
    torch.cuda.synchronize(dev)
    med = statistics.median(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(reps))
    warm0, warm1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        step(0)
    warm0.record(stream)
    for _ in range(reps):
        step(0)
    warm1.record(stream)
    torch.cuda.synchronize(dev)
    warm_ms = warm0.elapsed_time(warm1) / reps
    return {"launch_floor_ms": round(floor, 5),
            "launch_floor_what": f"same kernel, one {tuple(xt.shape)} tile, flushed L2, "
                                 "events around the launch (median of 100); an empty torch "
                                 "kernel timed this way takes ~6.2 us on B200 "
                                 "(profiles/r01_exp_floor.txt)",
            "flushed_launch_median_ms": round(med, 5),
            "flushed_gbs": round(step_bytes / (med / 1e3) / 1e9, 1),
            "flushed_what": "the workload with a 252 MiB read flush before each launch and "
                            "events around it (median of 100; includes the event floor)",
            "l2_resident_gbs": round(step_bytes / (warm_ms / 1e3) / 1e9, 1),
            "l2_resident_what": "the same launches back to back, no flush (working set in "
                                "the 126 MB L2; context, not the metric)"}


def live_ceiling_context(desc, torch, dev, stream, wl, xs, ys, R, batch, rows, cols, ld_in,
                         step_bytes, kernel, graph: bool, reps: int = 20):
    """Outside the timed region, on the same buffers and in the same launch pattern as the
    metric (K launches back to back over the R rotating pairs): (1) the SAME BYTES moved by a
    plain copy, no transpose -- this library's 16-byte row copy (desc_copy_batched, PDL) and
    torch's copy_ -- the practical ceiling SURVEY 8(d) M3 asks to report beside the
    transpose; (2) for small working sets, the transpose captured in a CUDA graph (2R
    launches per graph) and replayed with events around each replay: the graph-captured
    back-to-back median SURVEY 8(d) M2 asks for."""
    import statistics as _st
    sptr = stream.cuda_stream
    tdt = xs[0].dtype

    def region(fn, k=reps):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / k

    def own_copy(i):
        xi, yi = xs[i % R], ys[i % R]
        desc.desc_copy_batched(xi.data_ptr(), yi.data_ptr(), batch, rows, cols, ld_in, cols,
                               rows * ld_in, rows * cols, wl["dtype"], sptr)

    def torch_copy(i):
        xi, yi = xs[i % R], ys[i % R]
        yi.view(batch, rows, cols).copy_(xi[..., :cols] if ld_in != cols else xi.view(batch, rows, cols))

    out = {}
    for name, fn in (("desc_copy_batched", own_copy), ("torch_copy", torch_copy)):
        try:
            ms = region(fn)
            out[name + "_gbs"] = round(step_bytes / (ms / 1e3) / 1e9, 1)
        except Exception as e:  # noqa: BLE001
            out[name + "_error"] = f"{type(e).__name__}: {e}"[:200]
    out["what"] = ("the same bytes (read + write) moved without transposing, same buffers, K "
                   "launches back to back: the practical ceiling of this workload's layout")
    if graph:
        try:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(stream)
            n_in = 2 * R
            with torch.cuda.stream(cs):
                for i in range(n_in):        # warm the capture stream once
                    xi, yi = xs[i % R], ys[i % R]
                    desc.desc_transpose_ex(xi.data_ptr(), yi.data_ptr(), batch, rows, cols, ld_in,
                                           rows, rows * ld_in if batch > 1 else 0,
                                           rows * cols if batch > 1 else 0, wl["dtype"], kernel,
                                           cs.cuda_stream)
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(g, stream=cs):
                    for i in range(n_in):
                        xi, yi = xs[i % R], ys[i % R]
                        desc.desc_transpose_ex(xi.data_ptr(), yi.data_ptr(), batch, rows, cols,
                                               ld_in, rows, rows * ld_in if batch > 1 else 0,
                                               rows * cols if batch > 1 else 0, wl["dtype"],
                                               kernel, torch.cuda.current_stream(dev).cuda_stream)
            stream.wait_stream(cs)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize(dev)
            per = []
            for _ in range(100):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                per.append(e0.elapsed_time(e1) / n_in)
            med = _st.median(per)
            out["graph_replay_ms_per_launch_median"] = round(med, 5)
            out["graph_replay_gbs"] = round(step_bytes / (med / 1e3) / 1e9, 1)
            out["graph_what"] = (f"{n_in} transposes over the {R} rotating pairs captured in one "
                                 "CUDA graph (PDL edges kept), 100 replays with events around "
                                 "each, median per launch")
        except Exception as e:  # noqa: BLE001
            out["graph_error"] = f"{type(e).__name__}: {e}"[:200]
    return out


def ours_arm(args, wl, world, rank, local):
    import torch
    import torch.distributed as dist
    import paper_2305_03448_b200 as desc

    local = local_device(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    desc.load()
    if world > 1:
        init_pg(dev)

    es, rows, cols = wl["es"], wl["rows"], wl["cols"]
    batch = wl["batch"]
    if wl.get("shard"):
        if batch % world:
            raise SystemExit(f"batch {batch} not divisible by world {world}")
        batch = batch // world
    elem = {4: torch.int32, 8: torch.int64}[es]
    tdt = {"f32": torch.float32, "f64": torch.float64, "i32": torch.int32}[wl["dtype"]]

    # seeded synthetic input, generated on the host (so the oracle sees the same bits)
    src = synth.random_bits((batch, rows, cols), es, synth.BASE_SEED + 2 + 1000 * rank)
    src_t = torch.from_numpy(src.view(np.int32 if es == 4 else np.int64))
    ld_in = wl.get("ld_in", cols)
    if ld_in == cols:
        x = src_t.to(dev).view(tdt)
    else:          # padded input pitch (TMA-ineligible workloads): logical rows x cols view
        xp = torch.zeros((batch, rows, ld_in), dtype=src_t.dtype, device=dev)
        xp[:, :, :cols] = src_t.to(dev)
        x = xp.view(tdt)
    y = torch.empty((batch, cols, rows), dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    kernel = args.kernel
    mat_bytes = rows * cols * es
    step_bytes = 2 * batch * mat_bytes                     # algorithmic: read + write
    small_ws = (batch * mat_bytes) < 2 * L2_BYTES
    # A working set that fits the 126 MB L2 is kept out of it one of two ways:
    #  * "rotate" (default): R copies of the (input, output) pair, R * 2 * bytes >= 4 x L2,
    #    launched round robin back to back -- each launch finds its pair evicted by the R - 1
    #    launches since its last use, and the region is timed without per-launch events
    #    (which add ~6 us of event overhead per launch on B200, profiles/r01_exp_floor.txt);
    #  * "flush": a read of a 2 x L2 buffer before every launch, events around each launch.
    flush = small_ws and args.l2 == "flush"
    R = max(2, -(-4 * L2_BYTES // (2 * batch * mat_bytes))) if small_ws and not flush else 1
    xs, ys = [x], [y]
    for _ in range(R - 1):
        xs.append(x.clone())
        ys.append(torch.empty_like(y))
    # L2 flush by READING a 2 x L2 buffer: leaves L2 full of clean, unrelated lines (a write
    # flush would leave 126 MB of dirty lines that the timed kernel would have to write back)
    scratch = torch.ones(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if small_ws else None
    sink = torch.empty((), dtype=torch.int64, device=dev) if small_ws else None

    def l2_flush():
        torch.sum(scratch, dim=0, dtype=torch.int64, out=sink)

    turn = [0]

    def step(pair=None):
        if pair is None:
            pair = turn[0] % R
            turn[0] += 1
        xi, yi = xs[pair], ys[pair]
        if batch == 1:
            desc.desc_transpose_ex(xi.data_ptr(), yi.data_ptr(), 1, rows, cols, ld_in, rows, 0,
                                   0, wl["dtype"], kernel, sptr)
        else:
            desc.desc_transpose_ex(xi.data_ptr(), yi.data_ptr(), batch, rows, cols, ld_in, rows,
                                   rows * ld_in, rows * cols, wl["dtype"], kernel, sptr)
        return desc.desc_last_launch_count()

    selected = desc.desc_select_kernel(x.data_ptr(), y.data_ptr(), batch, rows, cols, ld_in, rows,
                                       rows * ld_in if batch > 1 else 0,
                                       rows * cols if batch > 1 else 0, wl["dtype"])
    if kernel != "auto":
        selected = kernel

    h0 = time.perf_counter()
    for _ in range(args.warmup):
        if flush:
            l2_flush()
        step()
    host_step = (time.perf_counter() - h0) / args.warmup     # host enqueue time per step
    torch.cuda.synchronize(dev)

    # Timed region.  Without an L2 flush the K launches run back to back and only the two
    # region events are recorded (events between launches would add ~5 us gaps and block
    # the PDL overlap); the kernel's average launch duration is then region / launches
    # (nothing else runs on the stream).  With a flush, each launch is bracketed by its own
    # events and only the launches are summed.
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if flush else []
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if flush else []
    region0 = torch.cuda.Event(enable_timing=True)
    region1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        if not flush:
            host_gate(torch, stream, gate_seconds(host_step, args.steps))
        region0.record(stream)
        for k in range(args.steps):
            if flush:
                l2_flush()             # evict the working set from the 126 MB L2 (clean)
                starts[k].record(stream)
            launches += step()
            if flush:
                ends[k].record(stream)
        region1.record(stream)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        clk.region(t1 - region0.elapsed_time(region1) / 1e3 - 1e-4, t1)
    clk.extend(step, torch, dev)
    if world > 1:
        dist.barrier()
    region_ms = region0.elapsed_time(region1)
    if flush:
        per_launch = [s.elapsed_time(e) for s, e in zip(starts, ends)]   # ms, device time
        timed_ms = sum(per_launch)
    else:
        timed_ms = region_ms
    timed_ms_max = reduce_scalar(timed_ms, "max", dev)

    total_bytes = step_bytes * world * args.steps
    value = total_bytes / (timed_ms_max / 1e3) / 1e9
    avg_launch_ms = timed_ms / launches            # this rank's average launch duration
    achieved = step_bytes / (avg_launch_ms / 1e3) / 1e9
    if not flush:  # untimed diagnostic pass: per-launch spread (events between launches),
        # >= 100 launches whatever K is -- the median the paper reports
        n_diag = max(100, min(args.steps, 200))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n_diag)]
        for k in range(n_diag):
            ev[2 * k].record(stream)
            step()
            ev[2 * k + 1].record(stream)
        torch.cuda.synchronize(dev)
        per_launch = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(n_diag)]
    peak, peak_src = load_peak()
    small = small_problem_context(desc, torch, dev, stream, wl, kernel, step, l2_flush,
                                  step_bytes) if small_ws else None

    # ---- parity of the timed output (rank-local) ------------------------------------
    parity = None
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_oracle:
        r = run_oracle(wl, budget_s=args.oracle_seconds)
        cpu_baseline = {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": 1,
                        "kind": "oracle", "sample": r["sample"], "host": host_info()}
        nb = r["sample_batch"]
        got = y[:nb].view(elem).cpu().numpy().view(r["out"].dtype)
        same_in = np.array_equal(r["inp"], src[:nb])
        if not (same_in and r["complete"]):
            parity = "not checked (oracle sample incomplete)"
        else:
            parity = ("bit-exact vs oracle" if got.tobytes() == r["out"].tobytes()
                      else "MISMATCH vs oracle")

    # ---- context: the same bytes copied, graph replay (overwrites the output buffers, so
    # it runs after the parity check above) -------------------------------------------
    ceiling = None if args.no_context else live_ceiling_context(
        desc, torch, dev, stream, wl, xs, ys, R, batch, rows, cols, ld_in, step_bytes, kernel,
        graph=small_ws and not flush)

    # ---- end to end through the public API with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, desc, torch, dev, stream, src_t, tdt, batch, rows, cols, wl,
                          kernel, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(timed_ms_max / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic (seeded random bit patterns, host-generated)",
            "config": {"workload": wl["name"], "rows": rows, "cols": cols, "ld_in": ld_in,
                       "batch_per_gpu": batch, "kernel": selected,
                       "queued": "the K steps are enqueued behind an untimed device spin, so the "
                                 "region times the GPU running them back to back",
                       "parallelism": f"{world} independent replica(s), no collective",
                       "l2": ("flushed before every step (read of a 252 MiB buffer, untimed)" if flush else
                              f"{R} (input, output) pairs of {batch * mat_bytes / 1e6:.0f} MB each "
                              f"used round robin ({2 * R * batch * mat_bytes / 1e6:.0f} MB >= 4 x the "
                              "126 MB L2): every launch starts with its pair evicted, no flush"
                              if R > 1 else
                              f"inputs larger than L2 ({batch * mat_bytes / 1e6:.0f} MB > 126 MB), no flush"),
                       "timing": ("CUDA events on the launch stream around the K launches "
                                  "(per launch when flushing), max over ranks")},
            "pct_of_hbm_peak": round(100.0 * value / world / peak, 2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "nominal_peak": NOMINAL_HBM_GBS,
                         "frac_of_nominal": round(achieved / NOMINAL_HBM_GBS, 4),
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": load_traffic(args.workload, args.kernel), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": step_bytes,
                         "kernel": KERNEL_FN[selected],
                         "launch_ms_mean_in_region": round(avg_launch_ms, 5),
                         "launch_spread_from": ("the timed launches" if flush else
                                                f"an untimed pass of {len(per_launch)} launches "
                                                "with events around each launch"),
                         "launch_ms_median": round(statistics.median(per_launch), 5),
                         "launch_ms_median_of": len(per_launch),
                         "median_frac": round(step_bytes / (statistics.median(per_launch) / 1e3)
                                              / 1e9 / peak, 4),
                         "launch_ms_p10": round(float(np.percentile(per_launch, 10)), 5),
                         "launch_ms_p90": round(float(np.percentile(per_launch, 90)), 5),
                         "launch_ms_min": round(min(per_launch), 5)},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "parity": parity,
            "gpu_launches": launches,
            **({"small_problem": small} if small else {}),
            "same_bytes_copy": ceiling,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------- configs[4]
class _Done:
    def wait(self):
        return True


def staged_all_to_all(out, inp, group=None, async_op=False):
    """DESC_BENCH_BACKEND=gloo only (several ranks sharing ONE GPU to exercise the N > 1 code
    path on a 1-GPU box): the all-to-all through host memory -- gloo has no CUDA all-to-all
    and NCCL refuses two ranks on one GPU.  Never used with the NCCL backend."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    o = torch.empty(out.shape, dtype=out.dtype)
    dist.all_to_all_single(o, inp.cpu(), group=group)
    out.copy_(o)
    return _Done()


def slab_roofline(lay, es, step_s):
    """T* = max(2S / HBM, S(P-1)/P / NVLink) per rank; frac = T* / t_step."""
    peak, peak_src = load_peak()
    S = lay.Rm * lay.N * es
    t_hbm = 2 * S / (peak * 1e9)
    t_nvl = lay.nvlink_bytes(es) / (NVLINK_PEER_GBS * 1e9)
    t_star = max(t_hbm, t_nvl)
    hbm_bound = t_hbm >= t_nvl
    return {"bound": "hbm" if hbm_bound else "nvlink",
            "achieved": round((2 * S if hbm_bound else lay.nvlink_bytes(es)) / step_s / 1e9, 2),
            "peak": peak if hbm_bound else NVLINK_PEER_GBS,
            "unit": "GB/s", "frac": round(t_star / step_s, 4), "traffic": None,
            "t_star_ms": round(t_star * 1e3, 4), "t_hbm_ms": round(t_hbm * 1e3, 4),
            "t_nvlink_ms": round(t_nvl * 1e3, 4),
            "peak_source": peak_src + "; NVLink: B200_PROFILING.md measured peer copy 770 GB/s "
                                      "per direction",
            "note": "frac = T*/t_step, T* = max(2S/HBM, S(P-1)/P / 770 GB/s), S = slab bytes"}


def slab_buffers(world, rank, dev, n, es=4, ws=True):
    """Rank's input slab (hash-filled in HBM: in[i][j] = H(seed, i*n + j)), its output slab and
    the NCCL path's (send, recv) workspace."""
    import torch
    from paper_2305_03448_b200 import dist as ddist
    lay = ddist.SlabLayout(n, n, world, rank)
    it = {4: torch.int32, 8: torch.int64}[es]
    x = torch.empty((lay.Rm, lay.N), dtype=it, device=dev)
    synth.hash_fill_torch(x, lay.in_rows()[0], 0, lay.N, SLAB_SEED, chunk_rows=1024)
    out = torch.empty((lay.Rn, lay.M), dtype=it, device=dev)
    w = None
    if ws:
        w = (torch.empty(lay.Rm * lay.N, dtype=it, device=dev),
             torch.empty(lay.Rm * lay.N, dtype=it, device=dev))
    return lay, x, out, w


SLAB_SEED = synth.BASE_SEED + 5


def slab_verify(lay, out, dev, blocks: int = 4):
    """EVERY element of this rank's output slab against the closed form of the hash input
    (tests/fullcheck.py), plus `blocks` 64 x 64 blocks against the oracle itself; the verdict
    is the min over ranks."""
    import torch
    import oracle
    from tests.fullcheck import hash_transpose_mismatches
    r0, _ = lay.out_rows()
    bad, first = hash_transpose_mismatches(out, r0, lay.N, SLAB_SEED, chunk_rows=512)
    rng = np.random.default_rng(SLAB_SEED + lay.r)
    es = out.element_size()
    picks = [(0, 0), (lay.Rn - 64, lay.M - 64)] + [
        (int(rng.integers(0, lay.Rn - 63)), int(rng.integers(0, lay.M - 63)))
        for _ in range(blocks)]
    ok_blocks = True
    for j0, i0 in picks:           # out_r[j0:j0+64, i0:i0+64] = A[i0:i0+64, r0+j0:r0+j0+64]^T
        j0, i0 = max(0, j0), max(0, i0)
        h = min(64, lay.Rn - j0)
        w = min(64, lay.M - i0)
        ii, jj = np.meshgrid(np.arange(i0, i0 + w), np.arange(r0 + j0, r0 + j0 + h), indexing="ij")
        exp = oracle.transpose(synth.hash_expected_np(ii, jj, lay.N, SLAB_SEED, es))
        got = out[j0:j0 + h, i0:i0 + w].cpu().numpy().view(exp.dtype)
        ok_blocks &= got.tobytes() == exp.tobytes()
    total_bad = reduce_scalar(float(bad), "max", dev)
    all_ok = reduce_scalar(1.0 if (bad == 0 and ok_blocks) else 0.0, "min", dev) > 0.5
    if all_ok:
        return (f"bit-exact: every element of every rank's slab ({lay.M * lay.N} in total) vs the "
                "closed form of the hash input, plus 64x64 blocks vs the oracle")
    return f"MISMATCH (max over ranks {int(total_bad)} elements; rank {lay.r} first at {first})"


def slab_step_fn(impl, lay, x, out, ws, chunks, group=None):
    """One distributed transpose step; returns (step(), chunks) -- step() returns the number of
    our kernel launches it made."""
    from paper_2305_03448_b200 import dist as ddist
    if impl == "p2p":
        xp = ddist.PeerSlabTranspose(out, lay.M, group=group,
                                     force_remote=bench_backend() != "nccl")
        # back to back without the per-call group barriers: inside the loop no rank reads its
        # slab and the ranks write disjoint column blocks of each slab in stream order, so
        # the result only needs the barrier after the last step (taken by the caller)
        return (lambda: xp(x, barrier=False)[1]), None, xp
    if impl == "local":
        def step_local():
            ddist.slab_transpose(x, out)
            return 1
        return step_local, 1, None
    a2a = staged_all_to_all if bench_backend() != "nccl" else None
    C = ddist.default_chunks(lay.Rm, lay.P) if chunks is None else chunks

    def step():
        ddist.slab_transpose(x, out, workspace=ws, chunks=C, all_to_all=a2a, group=group)
        return 2 * C
    return step, C, None


def timed_region(step, steps, warmup, dev, world):
    """W untimed steps, then EXACTLY K steps between a barrier + synchronize on both sides,
    CUDA events on the launch stream, NVML clocks sampled in the region; max over ranks."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream(dev)
    h0 = time.perf_counter()
    for _ in range(warmup):
        step()
    host_step = (time.perf_counter() - h0) / max(warmup, 1)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        host_gate(torch, stream, gate_seconds(host_step, steps))
        e0.record(stream)
        for _ in range(steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        clk.region(t1 - e0.elapsed_time(e1) / 1e3 - 1e-4, t1)
    if world > 1:
        dist.barrier()
    ms_max = reduce_scalar(e0.elapsed_time(e1), "max", dev)
    # too few NVML samples in the region: every rank repeats the step the SAME number of
    # times (the steps may contain collectives), decided from values equal on all ranks
    short = reduce_scalar(1.0 if clk.ok and len(clk._in_region()) < 10 else 0.0, "max", dev)
    if short > 0.5:
        reps = max(1, min(2000, int(0.3 / max(ms_max / steps / 1e3, 1e-6))))
        clk.extend(lambda: [step() for _ in range(reps)], torch, dev, seconds=0.0, min_samples=10**9)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    return ms_max, launches, clk


def slab_phases(lay, x, out, ws, dev, world, reps: int = 3):
    """The NCCL path's three phases timed separately (unchunked: pack = local transpose into
    the send buffer, the all-to-all, unpack), median of `reps`, each the max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2305_03448_b200 as desc
    stream = torch.cuda.current_stream(dev)
    send, recv = (w.view(-1) for w in ws)
    a2a = dist.all_to_all_single if bench_backend() == "nccl" else staged_all_to_all
    N, Rm, Rn, M, P = lay.N, lay.Rm, lay.Rn, lay.M, lay.P
    ts = []
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        desc.transpose(x, send[:N * Rm].view(N, Rm))
        ev[1].record(stream)
        a2a(recv[:N * Rm], send[:N * Rm])
        ev[2].record(stream)
        desc.desc_copy_batched(recv.data_ptr(), out.data_ptr(), P, Rn, Rm, Rm, M, Rn * Rm, Rm,
                               out.dtype, stream.cuda_stream)
        ev[3].record(stream)
        torch.cuda.synchronize(dev)
        ts.append([ev[k].elapsed_time(ev[k + 1]) for k in range(3)])
    med = [statistics.median(t[k] for t in ts) for k in range(3)]
    med = [reduce_scalar(v, "max", dev) for v in med]
    S = Rm * N * out.element_size()
    peak, _ = load_peak()
    return {"pack_ms": round(med[0], 4), "all_to_all_ms": round(med[1], 4),
            "unpack_ms": round(med[2], 4), "sum_ms": round(sum(med), 4),
            "pack_hbm_frac": round(2 * S / (med[0] / 1e3) / 1e9 / peak, 4),
            "unpack_hbm_frac": round(2 * S / (med[2] / 1e3) / 1e9 / peak, 4),
            "all_to_all_gbs_per_direction": round(lay.nvlink_bytes(out.element_size())
                                                  / (med[1] / 1e3) / 1e9, 2),
            "what": "unchunked step, phases timed by CUDA events on the compute stream (the "
                    "all-to-all synchronous), median of 3, max over ranks"
                    + ("" if bench_backend() == "nccl" else
                       "; all-to-all staged through the host (gloo 1-GPU test mode)")}


def replicas_object(world, rank, dev, steps: int = 50, warmup: int = 5):
    """Weak-scaling context at N > 1: one 8192^2 f32 transpose per rank (configs[2] replicas,
    no collective), K launches back to back, max over ranks."""
    import torch
    import paper_2305_03448_b200 as desc
    x = torch.from_numpy(synth.random_bits((8192, 8192), 4, synth.BASE_SEED + 2 + 1000 * rank)
                         .view(np.int32)).to(dev)
    y = torch.empty_like(x)
    ms, launches, clk = timed_region(lambda: (desc.transpose(x, y), 1)[1], steps, warmup, dev, world)
    peak, _ = load_peak()
    step_bytes = 2 * 8192 * 8192 * 4
    value = step_bytes * world * steps / (ms / 1e3) / 1e9
    ok = bool(torch.equal(y[:64, :64], x[:64, :64].t()))
    del x, y
    return {"workload": "8192x8192 f32 per rank (configs[2] replicas, no collective)",
            "value": round(value, 2), "unit": "GB/s", "scaling": "weak",
            "ms_per_step": round(ms / steps, 5), "frac_per_gpu": round(value / world / peak, 4),
            "gpu_launches": launches, "spot_check": "ok" if ok else "MISMATCH"}


def dist_e2e(world, rank, dev, n, steps: int = 5):
    """configs[4]'s e2e through the public API at a bounded size (n x n, host memory per rank
    2 * n^2 * 4 / P bytes): every step copies this rank's input slab from pinned host memory,
    runs the distributed transpose, and copies its output slab back to pinned host memory."""
    import torch
    from paper_2305_03448_b200 import dist as ddist
    lay, x, out, ws = slab_buffers(world, rank, dev, n, ws=world > 1)
    h_in = x.cpu().pin_memory()
    h_out = torch.empty((lay.Rn, lay.M), dtype=x.dtype, pin_memory=True)
    a2a = staged_all_to_all if bench_backend() != "nccl" else None

    import paper_2305_03448_b200 as desc
    hws = None
    if world == 1:   # one rank holds the whole matrix: the public host-buffer entry point
        nws = desc.desc_transpose_host_workspace(lay.M, lay.N, "f32")
        hws = torch.empty(nws, dtype=torch.uint8, device=dev)

    def step():
        if hws is not None:
            desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), 1, lay.M, lay.N, lay.N,
                                     lay.M, 0, 0, "f32", hws.data_ptr(), hws.numel(),
                                     torch.cuda.current_stream(dev).cuda_stream)
            return desc.desc_last_launch_count()
        # the host-buffer pipeline: H2D chunks, the chunked exchange, 2-D D2H stripes
        ddist.slab_transpose_host(h_in, h_out, x, out, workspace=ws, all_to_all=a2a)
        return 2 * ddist.default_host_chunks(lay.Rn, 4)
    ms, launches, _ = timed_region(step, steps, 3, dev, world)
    out.copy_(h_out)                   # what reached the host, verified on the device
    parity = slab_verify(lay, out, dev, blocks=1)
    es = 4
    value = 2 * n * n * es * steps / (ms / 1e3) / 1e9
    bi = lay.Rm * lay.N * es
    del x, out, ws
    return {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": bi * world,
            "d2h_bytes_per_step": bi * world, "bytes_per_rank_each_way": bi,
            "workload": f"{n}x{n} f32 (configs[4] layout at a host-memory-bounded size)",
            "steps": steps, "gpu_launches": launches, "parity": parity,
            "path": ("pinned host matrix -> desc_transpose_host (banded H2D | transpose | "
                     "D2H) -> pinned host, every step" if world == 1 else
                     "pinned host slab -> dist.slab_transpose_host (H2D of row chunks | "
                     "chunked transpose + all-to-all + unpack | 2-D D2H of the output column "
                     "stripes) -> pinned host slab, every step")}


def dist_arm(args, wl, world, rank, local):
    """configs[4]: the global n x n matrix lives as row slabs, one per rank; a step is one
    full distributed transpose.  Headline: the NCCL all-to-all path (pipelined over row
    chunks) with strong scaling; beside it the fused peer-to-peer path
    (exchange_p2p), the phases of the NCCL path, the 8192^2 replicas (weak), e2e; every
    element of every rank's slab verified after each path."""
    import torch
    import torch.distributed as dist
    import paper_2305_03448_b200 as desc

    local = local_device(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    desc.load()
    if world > 1:
        init_pg(dev)
    n, es = args.dist_n, wl["es"]
    impl = args.dist_impl if world > 1 else "local"
    lay, x, out, ws = slab_buffers(world, rank, dev, n, es, ws=world > 1)

    def run(impl_, chunks=None):
        out.fill_(0x5A5A5A5A)
        step, C, xp = slab_step_fn(impl_, lay, x, out, ws, chunks)
        ms, launches, clk = timed_region(step, args.steps, args.warmup, dev, world)
        if xp is not None:
            xp.close()
        parity = slab_verify(lay, out, dev)
        step_s = ms / args.steps / 1e3
        return {"ms": ms, "launches": launches, "clk": clk, "chunks": C, "parity": parity,
                "value": 2 * lay.M * lay.N * es * args.steps / (ms / 1e3) / 1e9,
                "roofline": slab_roofline(lay, es, step_s)}

    head = run(impl, args.dist_chunks)
    extra = {}
    if world > 1:
        other = "p2p" if impl == "nccl" else "nccl"
        try:
            r = run(other)
            extra["exchange_p2p" if other == "p2p" else "exchange_nccl"] = {
                "impl": other, "value": round(r["value"], 2), "unit": "GB/s",
                "ms_per_step": round(r["ms"] / args.steps, 4), "roofline": r["roofline"],
                "parity": r["parity"], "gpu_launches": r["launches"], "chunks": r["chunks"],
                "what": ("fused transpose + exchange: ONE kernel per step "
                         "(desc_slab_transpose_peer) writes block (r,s)^T straight into every "
                         "rank s's slab through CUDA IPC (2S HBM per rank, no NCCL kernels)"
                         if other == "p2p" else "NCCL all-to-all path")}
        except Exception as e:  # noqa: BLE001  (reported, the headline stays)
            extra["exchange_" + other] = {"error": f"{type(e).__name__}: {e}"[:300]}
        if impl == "nccl" and head["chunks"] > 1:
            r1 = run("nccl", 1)
            extra["unchunked"] = {"ms_per_step": round(r1["ms"] / args.steps, 4),
                                  "frac": r1["roofline"]["frac"], "parity": r1["parity"]}
        try:
            extra["phases"] = slab_phases(lay, x, out, ws, dev, world)
        except Exception as e:  # noqa: BLE001
            extra["phases"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    del x, out, ws
    torch.cuda.empty_cache()
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_oracle:
        r = run_oracle(wl, budget_s=args.oracle_seconds)
        cpu_baseline = {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                        "sample": r["sample"], "host": host_info()}
    e2e = None
    if not args.no_e2e:
        e2e = dist_e2e(world, rank, dev, min(n, args.dist_e2e_n))
    if world > 1:
        extra["replicas"] = replicas_object(world, rank, dev)
    if rank == 0:
        rf = dict(head["roofline"])
        line = {
            "metric": METRIC, "value": round(head["value"], 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(head["ms"] / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"],
            "data": "synthetic (counter-based hash, generated in HBM)",
            "config": {"workload": wl["name"], "rows": lay.M, "cols": lay.N, "ranks": world,
                       "slab_rows": lay.Rm, "impl": impl, "chunks": head["chunks"],
                       "parallelism": (f"row slabs over {world} ranks, "
                                       + ("NCCL all-to-all" if impl == "nccl" else
                                          "fused peer-to-peer stores") if world > 1 else
                                       "one rank: a single local transpose"),
                       "backend": bench_backend() if world > 1 else None,
                       "l2": "inputs larger than L2 (slab >= 2 GiB), no flush",
                       "timing": "CUDA events around exactly K steps after barrier + "
                                 "synchronize, max over ranks"},
            "roofline": rf,
            "parity": head["parity"],
            "gpu_launches": head["launches"], "cpu_baseline": cpu_baseline, "e2e": e2e,
            **extra,
            "clocks": head["clk"].summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def view_arm(args, wl, world, rank, local):
    """materialise a view chain of Listing 3 over an 8192^2 f32 root;
    one step = one desc_view_copy launch; parity vs oracle/views.py materialize."""
    import torch
    import paper_2305_03448_b200 as desc

    local = local_device(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    desc.load()
    if world > 1:
        init_pg(dev)
    es, rows, cols = wl["es"], wl["rows"], wl["cols"]
    src = synth.random_bits((rows, cols), es, synth.BASE_SEED + 7 + 1000 * rank)
    x = torch.from_numpy(src.view(np.int32)).to(dev)
    v = desc.desc_view_compile((rows, cols), wl["view"])
    shape = v.dims[0]
    y = torch.empty(shape, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches = 0

    def step():
        desc.desc_view_copy(x.data_ptr(), y.data_ptr(), v, "f32", stream.cuda_stream)
        return desc.desc_last_launch_count()

    h0 = time.perf_counter()
    for _ in range(args.warmup):
        step()
    host_step = (time.perf_counter() - h0) / args.warmup
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        host_gate(torch, stream, gate_seconds(host_step, args.steps))
        e0.record(stream)
        for _ in range(args.steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        clk.region(t1 - e0.elapsed_time(e1) / 1e3 - 1e-4, t1)
    clk.extend(step, torch, dev)
    ms = e0.elapsed_time(e1)
    ms_max = reduce_scalar(ms, "max", dev)
    step_bytes = 2 * rows * cols * es
    value = step_bytes * world * args.steps / (ms_max / 1e3) / 1e9
    achieved = step_bytes / (ms / args.steps / 1e3) / 1e9
    peak, peak_src = load_peak()
    parity = None
    if rank == 0 and not args.no_oracle:
        from oracle import views as V
        exp = V.materialize(src, wl["view"])
        got = y.cpu().numpy().view(np.uint32)
        parity = "bit-exact vs oracle (views)" if got.tobytes() == exp.tobytes() else "MISMATCH"
    if rank == 0:
        shp, strd, off = v.dims
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": wl["dtype"],
            "data": "synthetic (seeded random bit patterns, host-generated)",
            "config": {"workload": wl["name"], "rows": rows, "cols": cols,
                       "view_ops": wl["view"],
                       "compiled_view": {"shape": shp, "stride": strd, "offset": off},
                       "parallelism": f"{world} independent replica(s), no collective",
                       "l2": "inputs larger than L2, no flush",
                       "timing": "CUDA events around the K launches, max over ranks"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "nominal_peak": NOMINAL_HBM_GBS,
                         "frac_of_nominal": round(achieved / NOMINAL_HBM_GBS, 4),
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": load_traffic(args.workload),
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": step_bytes},
            "parity": parity, "gpu_launches": launches, "cpu_baseline": None, "e2e": None,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def op_arm(args, wl, world, rank, local):
    """the paper's other memory-bound benchmarks -- one
    step = one desc_block_reduce / desc_scan launch over the whole array; parity vs the
    oracle (integers bit-exact, floats within the summation-order bound)."""
    import torch
    import paper_2305_03448_b200 as desc

    local = local_device(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    desc.load()
    if world > 1:
        init_pg(dev)
    n, es, op = wl["cols"], wl["es"], wl["op"]
    npdt = {"f32": np.float32, "f64": np.float64, "i32": np.int32}[wl["dtype"]]
    a = (synth.random_floats(n, npdt, synth.BASE_SEED + 11 + rank) if npdt != np.int32
         else synth.random_ints(n, npdt, synth.BASE_SEED + 11 + rank))
    x = torch.from_numpy(a).to(dev)
    stream = torch.cuda.current_stream(dev)
    if op == "reduce":
        B = wl["block"]
        y = torch.empty(-(-n // B), dtype=x.dtype, device=dev)
        step_bytes = (n + y.numel()) * es

        def step():
            desc.desc_block_reduce(x.data_ptr(), y.data_ptr(), n, B, wl["dtype"], stream.cuda_stream)
            return desc.desc_last_launch_count()
    else:
        y = torch.empty_like(x)
        ws = desc.desc_scan_workspace(n, wl["dtype"])
        work = torch.empty(ws, dtype=torch.uint8, device=dev)
        step_bytes = 2 * n * es

        def step():
            desc.desc_scan_ex(x.data_ptr(), y.data_ptr(), n, wl["dtype"], work.data_ptr(), ws,
                              args.scan_algo, stream.cuda_stream)
            return desc.desc_last_launch_count()
    h0 = time.perf_counter()
    for _ in range(args.warmup):
        step()
    host_step = (time.perf_counter() - h0) / args.warmup
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        host_gate(torch, stream, gate_seconds(host_step, args.steps))
        e0.record(stream)
        for _ in range(args.steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        clk.region(t1 - e0.elapsed_time(e1) / 1e3 - 1e-4, t1)
    clk.extend(step, torch, dev)
    ms = e0.elapsed_time(e1)
    ms_max = reduce_scalar(ms, "max", dev)
    value = step_bytes * world * args.steps / (ms_max / 1e3) / 1e9
    achieved = step_bytes / (ms / args.steps / 1e3) / 1e9
    peak, peak_src = load_peak()
    read_peak = None
    if op == "reduce":
        # the reduction reads n and writes n/B elements: its roofline is the HBM READ rate.
        # A plain read-only probe (desc_read_probe: 16-byte loads, 8 in flight per lane, 4 KB
        # per warp, 1 GiB, best of 20) is measured in this run, but the
        # reduction's L2 prefetch of the next chunk reads faster than that probe, so the
        # roofline peak is the nominal HBM3e rate (an upper bound); the probe is reported beside
        read_peak = read_only_peak(torch, desc, dev, stream)
        copy_peak, copy_src = peak, peak_src
        peak, peak_src = NOMINAL_HBM_GBS, ("nominal B200 HBM3e 8 TB/s (BASELINE.json north star): "
                                           "an upper bound for a read-only stream")
    parity = cpu_baseline = None
    if rank == 0 and not args.no_oracle:
        import oracle
        got = y.cpu().numpy()
        t0 = time.perf_counter()
        if op == "reduce":
            ref = oracle.block_reduce(a, wl["block"])
            t_oracle = time.perf_counter() - t0
            absx = oracle.block_reduce(np.abs(a).astype(np.float64), wl["block"])
            m = np.minimum(wl["block"], n - np.arange(ref.size) * wl["block"])
        else:
            ref = oracle.scan(a)
            t_oracle = time.perf_counter() - t0
            absx = oracle.scan(np.abs(a).astype(np.float64))
            m = np.arange(1, n + 1)
        if npdt != np.int32:
            tol = np.spacing(np.abs(ref).astype(npdt)).astype(np.float64) + \
                2.0 * m * 2.0 ** -53 * absx
            ok = bool(np.all(np.abs(got.astype(np.float64) - ref) <= tol))
            parity = ("within the fp summation-order bound vs oracle" if ok else "MISMATCH")
        else:
            parity = "bit-exact vs oracle" if got.tobytes() == ref.tobytes() else "MISMATCH"
        cpu_baseline = {"value": round(step_bytes / t_oracle / 1e9, 4), "unit": "GB/s", "cores": 1,
                        "kind": "oracle",
                        "sample": f"the whole workload once (the parity reference call, "
                                  f"{t_oracle:.3f} s): oracle/reduce_scan_ref.c, 1 thread, same "
                                  f"byte formula"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": wl["dtype"],
            "data": "synthetic (seeded, host-generated)",
            "config": {"workload": wl["name"], "n": n, "block": wl.get("block"),
                       "scan_algo": args.scan_algo if op == "scan" else None,
                       "parallelism": f"{world} independent replica(s), no collective",
                       "l2": "inputs larger than L2, no flush",
                       "timing": "CUDA events around the K launches, max over ranks"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "nominal_peak": NOMINAL_HBM_GBS,
                         "frac_of_nominal": round(achieved / NOMINAL_HBM_GBS, 4),
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": load_traffic(args.workload),
                         "peak_source": peak_src,
                         **({"read_probe": read_peak,
                             "frac_of_read_probe": round(achieved / read_peak, 4),
                             "read_probe_what": "desc_read_probe in this run: plain 16-byte "
                                                "ld.global.nc, 8 in flight per lane, 1 GiB, best of 20",
                             "copy_peak": copy_peak, "frac_of_copy_peak": round(achieved / copy_peak, 4),
                             "copy_peak_source": copy_src} if op == "reduce" else {}),
                         "algorithmic_bytes_per_launch": step_bytes},
            "parity": parity, "gpu_launches": launches, "cpu_baseline": cpu_baseline, "e2e": None,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def read_only_peak(torch, desc, dev, stream, nbytes: int = 1 << 30, reps: int = 20) -> float:
    """HBM read-only GB/s: the library's read probe over an nbytes buffer, best of `reps`
    back-to-back launches (each timed by its own events)."""
    buf = torch.ones(nbytes // 4, dtype=torch.int32, device=dev)
    sink = torch.empty(desc.desc_read_probe_sink_bytes(), dtype=torch.uint8, device=dev)
    sp = stream.cuda_stream
    for _ in range(3):
        desc.desc_read_probe(buf.data_ptr(), nbytes, sink.data_ptr(), sp)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for k in range(reps):
        desc.desc_read_probe(buf.data_ptr(), nbytes, sink.data_ptr(), sp)
        ev[k + 1].record(stream)
    torch.cuda.synchronize(dev)
    best = min(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))
    del buf, sink
    return round(nbytes / (best / 1e3) / 1e9, 1)


def pcie_ceiling(torch, dev, h_in, h_out, reps: int = 3) -> float:
    """GB/s (H2D + D2H bytes) of a plain pinned H2D copy of h_in concurrent with a plain D2H
    copy into h_out on two streams, per rank -- the PCIe bound of the e2e measurement."""
    d_a = torch.empty(h_in.numel(), dtype=h_in.dtype, device=dev)
    d_b = torch.empty(h_out.numel(), dtype=h_out.dtype, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    hi, ho = h_in.reshape(-1), h_out.reshape(-1)
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(s1)
        s2.wait_event(e0)
        with torch.cuda.stream(s1):
            d_a.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(d_b, non_blocking=True)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize(dev)
        ms = max(e0.elapsed_time(e1), e0.elapsed_time(e2))
        best = max(best, (hi.numel() * hi.element_size() + ho.numel() * ho.element_size())
                   / (ms / 1e3) / 1e9)
    del d_a, d_b
    return best


def measure_e2e(args, desc, torch, dev, stream, src_t, tdt, batch, rows, cols, wl, kernel, world):
    """Same metric end to end through the public host-buffer API desc_transpose_host:
    pinned host input -> (H2D band k+1 | transpose band k | D2H band k-1, pipelined on two
    internal streams) -> pinned host output, every step, inside the timed region."""
    es = wl["es"]
    h_in = src_t.pin_memory()
    h_out = torch.empty((batch, cols, rows), dtype=src_t.dtype).pin_memory()
    nbytes_ws = (desc.desc_transpose_host_workspace_batched(batch, rows, cols, wl["dtype"])
                 if batch > 1 else desc.desc_transpose_host_workspace(rows, cols, wl["dtype"]))
    work = torch.empty(nbytes_ws, dtype=torch.uint8, device=dev)
    nbytes = batch * rows * cols * es
    steps = max(3, min(args.steps, args.e2e_steps))
    launches = [0]

    def one():
        desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), batch, rows, cols, cols,
                                 rows, rows * cols if batch > 1 else 0,
                                 rows * cols if batch > 1 else 0, wl["dtype"],
                                 work.data_ptr(), nbytes_ws, stream.cuda_stream)
        launches[0] += desc.desc_last_launch_count()

    for _ in range(2):
        one()
    torch.cuda.synchronize(dev)
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = reduce_scalar(e0.elapsed_time(e1), "max", dev)
    ok = bool(torch.equal(h_out[0, :64, :64], src_t[0, :64, :64].t().contiguous()))
    ceil = pcie_ceiling(torch, dev, h_in, h_out)
    value = 2 * nbytes * world * steps / (ms / 1e3) / 1e9
    return {"value": round(value, 3), "unit": "GB/s",
            "pcie_ceiling": {"value": round(ceil * world, 3), "unit": "GB/s",
                             "frac": round(value / (ceil * world), 4),
                             "what": "the same bytes as one plain H2D copy and one plain D2H "
                                     "copy running concurrently on two streams (no "
                                     "transpose): the bound the e2e path can reach"},
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": steps,
            "gpu_launches": launches[0], "spot_check": "ok" if ok else "MISMATCH",
            "path": "desc_transpose_host (C-ABI): pinned host -> banded H2D | transpose | D2H "
                    "overlapped on 2 streams -> pinned host"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="default: 8192f32 at N = 1 (configs[2], the headline target), "
                         "dist65536 at N > 1 (configs[4], the distributed transpose)")
    ap.add_argument("--kernel", choices=["auto", "tma", "tma_st", "smem", "tiled", "tma_tile", "vtiled"],
                    default="auto")
    ap.add_argument("--scan-algo", choices=["auto", "lookback", "three_pass", "stream"],
                    default="auto")
    ap.add_argument("--oracle-seconds", type=float, default=12.0)
    ap.add_argument("--reference-seconds", type=float, default=120.0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--dist-impl", choices=["nccl", "p2p"], default="nccl")
    ap.add_argument("--dist-chunks", type=int, default=None,
                    help="pipeline depth of the NCCL slab transpose (default: dist.default_chunks)")
    ap.add_argument("--dist-n", type=int, default=65536)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-context", action="store_true",
                    help="skip the untimed same-bytes copy / graph-replay context (launch lists)")
    ap.add_argument("--l2", choices=["rotate", "flush"], default="rotate",
                    help="how a working set smaller than 2 x L2 is kept out of L2")
    ap.add_argument("--dist-e2e-n", type=int, default=16384,
                    help="matrix side of the dist workload's e2e measurement (host memory bound)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    if args.workload is None:
        args.workload = "dist65536" if world > 1 else "8192f32"
    wl = dict(WORKLOADS[args.workload])
    if wl.get("dist") and args.impl == "ours":
        return dist_arm(args, wl, world, rank, local)
    if wl.get("view") and args.impl == "ours":
        return view_arm(args, wl, world, rank, local)
    if wl.get("op") and args.impl == "ours":
        return op_arm(args, wl, world, rank, local)
    if args.impl == "reference":
        return reference_arm(args, wl, world, rank)
    return ours_arm(args, wl, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
