"""Practical HBM ceiling at the transpose's byte count: a plain device-to-device copy of the
same number of bytes, timed exactly like bench.py times the transpose (back-to-back launches,
CUDA events).  Context for the roofline fraction, not a product path.

python scripts/copy_ceiling.py   (under gpurun)
"""
import json
import statistics

import torch


def time_copy(nbytes, steps=300, warmup=20):
    x = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda").random_()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        y.copy_(x)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(s)
    for k in range(steps):
        y.copy_(x)
        ev[k + 1].record(s)
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    med = statistics.median(per)
    return {"bytes_each_way": nbytes, "median_us": round(med * 1e3, 2),
            "GBps_read_plus_write": round(2 * nbytes / (med / 1e3) / 1e9, 1)}


if __name__ == "__main__":
    out = {}
    for name, nb in (("2048f64", 2048 * 2048 * 8), ("3000x5000f64", 3000 * 5000 * 8),
                     ("8192f32", 8192 * 8192 * 4), ("batched", 256 * 1024 * 1024 * 4),
                     ("1GiB", 1 << 30)):
        out[name] = time_copy(nb)
        print(name, json.dumps(out[name]), flush=True)
