"""A/B of desc_copy_batched (copy_rows_kernel: the NCCL slab path's unpack step) on the
shapes it is used at, timed like bench.py (K launches back to back, rotating buffer pairs
for working sets < 4 x L2).  Knobs: DESC_COPY_GRID (0 persistent / 1 one row per CTA),
DESC_COPY_UNR (4 / 8 loads in flight per thread).
  python scripts/exp_copy.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

L2 = 126 * 2**20
# (name, batch, rows, cols, ld_out, es): a plain 8192^2 f32 copy, 2048^2 f64, and the unpack
# of the slab transpose at P = 2 / 4 / 8 for a 32768^2 f32 global matrix (P blocks of R x R
# landing side by side at pitch N)
SHAPES = [("8192^2 f32", 1, 8192, 8192, 8192, 4), ("2048^2 f64", 1, 2048, 2048, 2048, 8),
          ("unpack P=2 R=16384", 2, 16384, 16384, 32768, 4),
          ("unpack P=4 R=8192", 4, 8192, 8192, 32768, 4),
          ("unpack P=8 R=4096", 8, 4096, 4096, 32768, 4)]


def main():
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    tag = f"grid={os.environ.get('DESC_COPY_GRID', '0')} unr={os.environ.get('DESC_COPY_UNR', '4')}"
    st = torch.cuda.current_stream().cuda_stream
    for name, B, rows, cols, ldo, es in SHAPES:
        nb = B * rows * cols * es
        R = max(1, -(-4 * L2 // (2 * nb)))
        dt = torch.int32 if es == 4 else torch.int64
        xs = [torch.ones(B * rows * cols, dtype=dt, device="cuda") for _ in range(R)]
        ys = [torch.empty(rows * ldo if B > 1 else rows * cols, dtype=dt, device="cuda") for _ in range(R)]

        def go(k):
            x, y = xs[k % R], ys[k % R]
            # block b (rows x cols, contiguous) -> out[:, b*cols : (b+1)*cols] at pitch ldo
            desc.desc_copy_batched(x.data_ptr(), y.data_ptr(), B, rows, cols, cols, ldo,
                                   rows * cols, cols, "f32" if es == 4 else "f64", st)
        for k in range(5):
            go(k)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(30):
                go(k)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 30
            best = ms if best is None else min(best, ms)
        gbs = 2 * nb / (best / 1e3) / 1e9
        print(f"{tag:14s} {name:22s} {gbs:7.0f} GB/s ({gbs / pk:.3f})", flush=True)
        del xs, ys


if __name__ == "__main__":
    main()
