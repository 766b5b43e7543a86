"""Experiment: PCIe ceilings vs desc_transpose_host band sizes (8192^2 f32, pinned)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

n = 8192
S = n * n * 4
h_in = torch.empty(n * n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n * n, dtype=torch.int32).pin_memory()
d_a = torch.empty(n * n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n * n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

ms = t(lambda: d_a.copy_(h_in, non_blocking=True)); print(f"H2D 268MB: {S/ms/1e6:.1f} GB/s")
ms = t(lambda: h_out.copy_(d_a, non_blocking=True)); print(f"D2H 268MB: {S/ms/1e6:.1f} GB/s")
def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event(); ev.record(cur)
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event(); e1.record(s1); e2.record(s2)
    cur.wait_event(e1); cur.wait_event(e2)
ms = t(both); print(f"H2D || D2H 268MB each: {2*S/ms/1e6:.1f} GB/s total")
for band in (256, 512, 1024, 2048, 4096):
    ws = desc.desc_transpose_host_workspace(band, n, "f32")
    work = torch.empty(ws, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), 1, n, n, n, n, 0, 0, "f32", work.data_ptr(), ws, st)
    ms = t(f); print(f"desc_transpose_host band={band}: {2*S/ms/1e6:.1f} GB/s (e2e metric)", flush=True)
