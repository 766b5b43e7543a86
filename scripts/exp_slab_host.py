"""The host-buffer slab pipeline (dist.slab_transpose_host) through a one-rank NCCL group on
one GPU, n x n f32 with C chunks, against the unpipelined H2D -> slab_transpose -> D2H and
the banded desc_transpose_host (GB/s = H2D + D2H bytes / time).  A one-rank all-to-all is a
device copy, so this times the PCIe / compute overlap of the pipeline, not NVLink.
  python scripts/exp_slab_host.py [n]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402
from paper_2305_03448_b200 import dist as ddist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
h_in = torch.randint(0, 1 << 30, (n, n), dtype=torch.int32).pin_memory()
h_out = torch.empty((n, n), dtype=torch.int32).pin_memory()
x = torch.empty((n, n), dtype=torch.int32, device="cuda")
out = torch.empty_like(x)
ws = (torch.empty(n * n, dtype=torch.int32, device="cuda"),
      torch.empty(n * n, dtype=torch.int32, device="cuda"))


def timed(fn, k=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 2 * n * n * 4 / (e0.elapsed_time(e1) / k / 1e3) / 1e9


def plain():
    x.copy_(h_in, non_blocking=True)
    ddist.slab_transpose(x, out, workspace=ws, chunks=4)
    h_out.copy_(out, non_blocking=True)


print(f"{n}^2 f32, one-rank NCCL group")
print(f"  H2D -> slab_transpose(C=4) -> D2H      {timed(plain):6.1f} GB/s")
for C in (2, 4, 8, 16):
    g = timed(lambda: ddist.slab_transpose_host(h_in, h_out, x, out, workspace=ws, chunks=C))
    print(f"  slab_transpose_host C={C:<2d}              {g:6.1f} GB/s")
print(f"  desc_transpose_host (banded)           "
      f"{timed(lambda: ddist.slab_transpose_host(h_in, h_out, x, out)):6.1f} GB/s")
print("  check", torch.equal(h_out[:64, :64], h_in[:64, :64].t()))
dist.destroy_process_group()
