"""Experiment: back-to-back launch gaps -- region-only timing vs per-launch events, PDL on/off
(DESC_PDL env), CUDA graph replay."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

n = 8192
x = torch.empty(n * n, dtype=torch.int32, device="cuda").random_()
y = torch.empty(n * n, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
f = lambda: desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, n, n, n, n, 0, 0, "f32", "auto", st.cuda_stream)
for _ in range(50): f()
torch.cuda.synchronize()
K = 1000
for trial in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K): f()
    e1.record(); torch.cuda.synchronize()
    print(f"region only: {e0.elapsed_time(e1) / K * 1e3:.2f} us/step", flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(K):
    ev[2 * k].record(); f(); ev[2 * k + 1].record()
e1.record(); torch.cuda.synchronize()
per = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(K)]
print(f"with per-launch events: region {e0.elapsed_time(e1) / K * 1e3:.2f} us/step, mean launch {statistics.mean(per) * 1e3:.2f} us", flush=True)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, n, n, n, n, 0, 0, "f32", "auto", s.cuda_stream)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(100):
        desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, n, n, n, n, 0, 0, "f32", "auto", torch.cuda.current_stream().cuda_stream)
g.replay(); torch.cuda.synchronize()
e0.record()
for _ in range(10): g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph replay: {e0.elapsed_time(e1) / 1000 * 1e3:.2f} us/step", flush=True)
