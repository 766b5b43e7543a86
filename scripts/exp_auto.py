"""A/B of the transpose variants per dtype and shape (what AUTO should pick): median of
per-launch CUDA-event times, L2 flushed (read of 2 x L2) before each launch when the
working set is < 2 x L2.  GB/s = 2 * bytes / t."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_03448_b200 as desc

L2 = 126 * 2**20
dev = torch.device("cuda", 0)
scratch = torch.ones(2 * L2 // 4, dtype=torch.int32, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)
DT = {"u8": torch.uint8, "bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}
shapes = [(8192, 8192), (1024, 1024), (16384, 1024), (1024, 16384), (3000, 5000), (256, 65536),
          (65536, 256), (8, 1 << 20), (1 << 20, 8)]
for dn in ("u8", "bf16", "f32", "f64"):
    es = torch.empty((), dtype=DT[dn]).element_size()
    for rows, cols in shapes:
        x = torch.zeros((rows, cols), dtype=DT[dn], device=dev)
        y = torch.empty((cols, rows), dtype=DT[dn], device=dev)
        nb = 2 * rows * cols * es
        flush = nb < 4 * L2
        st = torch.cuda.current_stream().cuda_stream
        res = []
        for k in ("tiled", "tma", "tma_st"):
            try:
                ts = []
                for it in range(40):
                    if flush:
                        torch.sum(scratch, dim=0, dtype=torch.int64, out=sink)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, rows, cols, cols, rows,
                                           0, 0, dn, k, st)
                    e1.record()
                    torch.cuda.synchronize()
                    if it >= 5:
                        ts.append(e0.elapsed_time(e1))
                t = statistics.median(ts)
                res.append(f"{k}={nb / t / 1e6:7.0f}")
            except Exception as e:
                res.append(f"{k}=  n/a  ")
        auto = desc.desc_select_kernel(x.data_ptr(), y.data_ptr(), 1, rows, cols, cols, rows, 0, 0, dn)
        print(f"{dn:4s} {rows:>7}x{cols:<7} {' '.join(res)}  auto={auto}", flush=True)
