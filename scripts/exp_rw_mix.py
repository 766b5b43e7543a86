"""HBM ceilings by access mix on this B200: read-only (desc_read_probe), write-only (torch
fill_ of a 1 GiB buffer), read+write (desc_copy_batched row copy and torch copy_ of 256 MiB),
all back to back, CUDA events; GB/s counts the bytes each moves (read + write for copies).
Context for the transpose's position.
  python scripts/exp_rw_mix.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402


def region(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


st = torch.cuda.current_stream().cuda_stream
big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")         # 1 GiB
ms = region(lambda: big.fill_(7))
print(f"write-only  torch fill_ 1 GiB          {big.numel() * 4 / (ms / 1e3) / 1e9:7.0f} GB/s")
sink = torch.empty(desc.desc_read_probe_sink_bytes() // 8 + 1, dtype=torch.int64, device="cuda")
ms = region(lambda: desc.desc_read_probe(big.data_ptr(), big.numel() * 4, sink.data_ptr(), st))
print(f"read-only   desc_read_probe 1 GiB      {big.numel() * 4 / (ms / 1e3) / 1e9:7.0f} GB/s")
n = 8192
xs = [torch.ones((n, n), dtype=torch.int32, device="cuda") for _ in range(2)]
ys = [torch.empty((n, n), dtype=torch.int32, device="cuda") for _ in range(2)]
k = [0]


def own():
    i = k[0] % 2
    k[0] += 1
    desc.desc_copy_batched(xs[i].data_ptr(), ys[i].data_ptr(), 1, n, n, n, n, 0, 0, "i32", st)


ms = region(own)
print(f"read+write  desc_copy_batched 256 MiB  {2 * n * n * 4 / (ms / 1e3) / 1e9:7.0f} GB/s")
ms = region(lambda: ys[0].copy_(xs[0]))
print(f"read+write  torch copy_ 256 MiB        {2 * n * n * 4 / (ms / 1e3) / 1e9:7.0f} GB/s")


def tr():
    i = k[0] % 2
    k[0] += 1
    desc.desc_transpose(xs[i].data_ptr(), ys[i].data_ptr(), n, n, n, n, "i32", st)


ms = region(tr)
print(f"read+write  desc_transpose 8192^2 i32  {2 * n * n * 4 / (ms / 1e3) / 1e9:7.0f} GB/s")
