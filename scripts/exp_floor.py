"""Experiment: what the 'launch floor' of a flushed, event-bracketed launch is made of.
Times (median of 100, CUDA events around ONE op) after an L2-flush read:
  empty torch op, 1-tile desc transpose, 2048^2 f64 transpose
each (a) as the bench does it (host enqueues op by op) and (b) behind a torch.cuda._sleep gate
so the whole sequence is queued before the GPU reaches it (host overhead excluded)."""
import os, statistics, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
L2 = 126 * 2**20
scratch = torch.ones(2 * L2 // 4, dtype=torch.int32, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)
flush = lambda: torch.sum(scratch, dim=0, dtype=torch.int64, out=sink)

def mk(rows, cols, dt):
    x = torch.zeros((rows, cols), dtype=dt, device=dev)
    y = torch.empty((cols, rows), dtype=dt, device=dev)
    name = {torch.float64: "f64", torch.float32: "f32"}[dt]
    return lambda: desc.desc_transpose_ex(x.data_ptr(), y.data_ptr(), 1, rows, cols, cols, rows, 0, 0, name, "auto", st.cuda_stream)

tiny = mk(64, 16, torch.float64)
big = mk(2048, 2048, torch.float64)
e = torch.empty(1, device=dev)
empty = lambda: e.add_(1)

def measure(fn, gate, n=100, do_flush=True):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n)]
    if gate:
        torch.cuda._sleep(int(2e9 * 0.03))   # ~30 ms at ~2 GHz: the host queues everything
    t0 = time.perf_counter()
    for k in range(n):
        if do_flush: flush()
        ev[2 * k].record(st); fn(); ev[2 * k + 1].record(st)
    host_us = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return statistics.median(ev[2*k].elapsed_time(ev[2*k+1]) for k in range(n)) * 1e3, host_us

for name, fn in (("empty torch add_", empty), ("1-tile desc", tiny), ("2048^2 f64 desc", big)):
    for gate in (False, True):
        for fl in (True, False):
            us, host = measure(fn, gate, do_flush=fl)
            print(f"{name:18s} gate={gate!s:5s} flush={fl!s:5s}: {us:7.2f} us device  (host {host:6.1f} us/iter)")
# host cost of one desc call alone
for _ in range(100): tiny()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000): tiny()
print(f"host time per desc_transpose_ex call: {(time.perf_counter()-t0):.1f} ms / 1000")
torch.cuda.synchronize()
