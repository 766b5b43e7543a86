"""A/B: desc_transpose_host with and without ramped band sizes (8192^2 f32, pinned), run as
two processes (DESC_HOST_RAMP is read once per process)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

n = 8192
S = n * n * 4
h_in = torch.empty(n * n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n * n, dtype=torch.int32).pin_memory()
ws = desc.desc_transpose_host_workspace(n, n, "f32")
work = torch.empty(ws, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), 1, n, n, n, n, 0, 0,
                                     "f32", work.data_ptr(), ws, st)
for _ in range(3):
    f()
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"ramp={os.environ.get('DESC_HOST_RAMP', '1')} launches={desc.desc_last_launch_count()} "
          f"{2 * S / ms / 1e6:.1f} GB/s", flush=True)
