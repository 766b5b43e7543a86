"""Practical HBM ceiling at the transpose's byte count: a plain device-to-device copy of the
same number of bytes, timed exactly like bench.py times the transpose (back-to-back launches,
CUDA events).  Context for the roofline fraction, not a product path.

python scripts/copy_ceiling.py   (under gpurun)
"""
import json
import statistics

import torch


def time_copy(nbytes, steps=300, warmup=20, flush=False):
    x = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda").random_()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    scratch = torch.ones(2 * 126 * 2**20 // 4, dtype=torch.int32, device="cuda")
    sink = torch.empty((), dtype=torch.int64, device="cuda")
    for _ in range(warmup):
        y.copy_(x)
    torch.cuda.synchronize()
    if flush:   # same clean read-flush as bench.py, each copy timed alone
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
        for k in range(steps):
            torch.sum(scratch, dim=0, dtype=torch.int64, out=sink)
            ev[2 * k].record(s)
            y.copy_(x)
            ev[2 * k + 1].record(s)
        torch.cuda.synchronize()
        per = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(steps)]
        mean = statistics.mean(per)
    else:       # back to back, region timing like bench.py
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for k in range(steps):
            y.copy_(x)
        e1.record(s)
        torch.cuda.synchronize()
        mean = e0.elapsed_time(e1) / steps
    return {"bytes_each_way": nbytes, "flush": flush, "mean_us": round(mean * 1e3, 2),
            "GBps_read_plus_write": round(2 * nbytes / (mean / 1e3) / 1e9, 1)}


if __name__ == "__main__":
    out = {}
    for name, nb in (("2048f64", 2048 * 2048 * 8), ("3000x5000f64", 3000 * 5000 * 8),
                     ("8192f32", 8192 * 8192 * 4), ("batched", 256 * 1024 * 1024 * 4),
                     ("1GiB", 1 << 30)):
        for fl in (False, True):
            out[name] = time_copy(nb, flush=fl)
            print(name, json.dumps(out[name]), flush=True)
