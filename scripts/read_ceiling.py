"""Context for the reduction's roofline: read-only stream rates of library kernels on the same
256 MB f32 array (torch.sum, a 1024-block torch reduction), timed like bench.py."""
import torch
n = 1 << 26
x = torch.randn(n, device="cuda")
def t(fn, reps=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: torch.sum(x)); print(f"torch.sum 256 MB: {n*4/ms/1e6:.1f} GB/s read")
ms = t(lambda: x.view(-1, 1024).sum(dim=1)); print(f"torch 1024-block sums: {(n*4 + n//1024*4)/ms/1e6:.1f} GB/s")
ms = t(lambda: torch.cumsum(x, 0)); print(f"torch.cumsum 256 MB: {2*n*4/ms/1e6:.1f} GB/s (read+write)")
