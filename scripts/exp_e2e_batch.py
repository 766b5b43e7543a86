"""e2e of the batched workload (256 x 1024^2 f32, pinned host buffers) through
desc_transpose_host with different workspace sizes (whole-matrix batch bands need room for
nb matrices) against the zero-copy path; GB/s = 2 * bytes / time.
  python scripts/exp_e2e_batch.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

B, n = 256, 1024
h_in = torch.randint(0, 1 << 30, (B, n, n), dtype=torch.int32).pin_memory()
h_out = torch.empty((B, n, n), dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream().cuda_stream
nbytes = B * n * n * 4
for ws_mb in (16, 64, 256, 512):
    work = torch.empty(ws_mb << 20, dtype=torch.uint8, device="cuda")

    def go():
        desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), B, n, n, n, n, n * n, n * n,
                                 "i32", work.data_ptr(), work.numel(), st)
    for _ in range(2):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        go()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"workspace {ws_mb:4d} MB: {2 * nbytes / (ms / 1e3) / 1e9:6.1f} GB/s, "
          f"{desc.desc_last_launch_count()} launches per call "
          f"(DESC_HOST_BATCH={os.environ.get('DESC_HOST_BATCH', '1')})", flush=True)
    del work
ok = torch.equal(h_out[7], h_in[7].t().contiguous())
print("spot check", "ok" if ok else "MISMATCH")
