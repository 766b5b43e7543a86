"""Block reduction across block sizes and dtypes (the three group widths G = 1 / 32 / CTA):
GB/s = (n + n/B) * es / t, CUDA events around 200 back-to-back launches (256 MB inputs > L2).
Run with DESC_LIB=<variant .so> for A/B."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

tag = os.path.basename(os.environ.get("DESC_LIB") or "base")
for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
    n = (256 << 20) // (4 if dt == "f32" else 8)
    x = torch.randn(n, dtype=tdt, device="cuda")
    for B in (4, 8, 16, 32, 64, 128, 256, 512, 1024, 3000, 4096, 8192, 16384, 65536, 1 << 20, 1 << 22):
        y = torch.empty(-(-n // B), dtype=tdt, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        f = lambda: desc.desc_block_reduce(x.data_ptr(), y.data_ptr(), n, B, dt, s)
        for _ in range(10): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 200
        print(f"{tag} {dt} B={B}: {(n + y.numel()) * x.element_size() / ms / 1e6:.0f} GB/s", flush=True)
