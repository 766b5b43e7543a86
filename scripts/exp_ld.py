"""Experiment: effect of padded leading dimensions / tile raster group on 8192^2 f32."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

def bench(rows, cols, ld_in, ld_out, kernel, dtype="f32", steps=200):
    es = 4 if dtype == "f32" else 8
    t = torch.int32 if es == 4 else torch.int64
    x = torch.empty(rows * ld_in, dtype=t, device="cuda").random_()
    y = torch.empty(cols * ld_out, dtype=t, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, rows, cols, ld_in, ld_out, 0, 0, dtype, kernel, s)
    for _ in range(20): f()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for k in range(steps):
        f(); ev[k + 1].record()
    torch.cuda.synchronize()
    med = statistics.median(ev[k].elapsed_time(ev[k + 1]) for k in range(steps))
    return 2 * rows * cols * es / (med / 1e3) / 1e9, med * 1e3

kernel = sys.argv[1] if len(sys.argv) > 1 else "tma_st"
for pad in (0, 16, 32, 64, 128, 256, 1024):
    g, us = bench(8192, 8192, 8192 + pad, 8192 + pad, kernel)
    print(f"8192^2 f32 ld=8192+{pad:5d}: {g:8.1f} GB/s  {us:7.1f} us", flush=True)
for n in (4096, 6144, 8000, 8192, 10000, 12288, 16384):
    g, us = bench(n, n, n, n, kernel)
    print(f"{n}^2 f32: {g:8.1f} GB/s  {us:7.1f} us", flush=True)
for r, c in ((4096, 16384), (16384, 4096), (2048, 32768), (32768, 2048)):
    g, us = bench(r, c, c, r, kernel)
    print(f"{r}x{c} f32: {g:8.1f} GB/s  {us:7.1f} us", flush=True)
