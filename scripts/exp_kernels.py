"""A/B of transpose kernel variants the way bench.py times them (the driver's metric): K launches
back to back on the stream (PDL overlaps them), one pair of region events; working sets
smaller than 4 x L2 rotate over R (input, output) pairs so every launch starts evicted.
Also the median of 100 per-launch event times.  GB/s = 2 * bytes / t; frac vs
MEASURED_PEAKS.json.

  python scripts/exp_kernels.py [--kernels tiled,tma_tile] [--shapes 8192x8192:f32,...] [--reps N]
  DESC_LIB=build_variants/lib_x.so python scripts/exp_kernels.py ...   (compile-time variants)
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

L2 = 126 * 2**20
DT = {"u8": torch.uint8, "bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64,
      "i32": torch.int32}
DEFAULT_SHAPES = "8192x8192:f32,3000x5000:f64,2048x2048:f64,4096x4096:f64,8192x8192:f64,256x1024x1024:f32"


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def measure(kernel, batch, rows, cols, dn, K, dev):
    es = torch.empty((), dtype=DT[dn]).element_size()
    nb = batch * rows * cols * es
    R = max(1, -(-4 * L2 // (2 * nb)))
    xs = [torch.zeros((batch, rows, cols), dtype=DT[dn], device=dev) for _ in range(R)]
    ys = [torch.empty((batch, cols, rows), dtype=DT[dn], device=dev) for _ in range(R)]
    st = torch.cuda.current_stream().cuda_stream
    si, so = (rows * cols, cols * rows) if batch > 1 else (0, 0)

    def go(k):
        if kernel == "copy":    # same bytes, plain 16-byte row copy (copy_rows_kernel, PDL)
            desc.desc_copy_batched(xs[k % R].data_ptr(), ys[k % R].data_ptr(), 1, batch * rows,
                                   cols, cols, cols, 0, 0, dn, st)
            return
        desc.desc_transpose_ex(xs[k % R].data_ptr(), ys[k % R].data_ptr(), batch, rows, cols, cols,
                               rows, si, so, dn, kernel, st)
    for k in range(10):
        go(k)
    torch.cuda.synchronize()
    best = None
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(K):
            go(k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        best = ms if best is None else min(best, ms)
    per = []
    for k in range(100):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go(k)
        e1.record()
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
    del xs, ys
    return 2 * nb / (best / 1e3) / 1e9, 2 * nb / (statistics.median(per) / 1e3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default="tiled,tma_tile,tma_st")
    ap.add_argument("--shapes", default=DEFAULT_SHAPES)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    pk = peak()
    tag = os.path.basename(os.environ.get("DESC_LIB", "product"))
    for spec in a.shapes.split(","):
        shp, dn = spec.split(":")
        dims = [int(v) for v in shp.split("x")]
        batch, rows, cols = ([1] + dims) if len(dims) == 2 else dims
        for k in a.kernels.split(","):
            try:
                b2b, med = measure(k, batch, rows, cols, dn, a.reps, dev)
                print(f"{tag:24s} {shp:>16s} {dn:4s} {k:9s} b2b {b2b:7.0f} GB/s ({b2b / pk:.3f})  "
                      f"median {med:7.0f} ({med / pk:.3f})", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{tag:24s} {shp:>16s} {dn:4s} {k:9s} n/a ({str(e)[:60]})", flush=True)


if __name__ == "__main__":
    main()
