"""Per-tile timeline of the streaming scan from a DESC_SCAN_TRACE build (DESC_LIB=<it>):
claim -> bytes landed -> A published -> look-back start/end (+ polls) -> scan start."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_03448_b200 as desc

dt = sys.argv[1] if len(sys.argv) > 1 else "i32"
n = 1 << 26
x = (torch.arange(n, device="cuda", dtype=torch.int32) % 7) if dt == "i32" else torch.randn(n, device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    desc.scan(x, out=y, algo="stream")
torch.cuda.synchronize()
lib = desc.load()
buf = np.zeros((8, 1 << 16), dtype=np.uint64)
lib.desc_scan_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.desc_scan_trace_copy(buf.ctypes.data, buf.nbytes) == 0
nt = int((buf[0] > 0).sum())
b = buf[:, :nt].astype(np.int64)
t0 = b[0].min()
b = b - t0
def q(a):
    return " ".join(f"{np.percentile(a, p) / 1e3:7.2f}" for p in (10, 50, 90, 99))
print(f"{dt}: {nt} tiles, kernel span {(b[6].max()) / 1e3:.1f} us (percentiles 10/50/90/99, us)")
print("claim -> landed        ", q(b[1] - b[0]))
print("landed -> A published  ", q(b[2] - b[1]))
print("A -> look-back start   ", q(b[3, 1:] - b[2, 1:]))
print("look-back duration     ", q(b[4, 1:] - b[3, 1:]))
print("polls per look-back    ", " ".join(f"{np.percentile(buf[5, 1:nt], p):7.1f}" for p in (10, 50, 90, 99)))
print("look-back end -> scan  ", q(b[6, 1:] - b[4, 1:]))
print("landed -> scan start   ", q(b[6] - b[1]))
# predecessor readiness: for tile t, latest A among t-1..t-148 relative to t's A
A = b[2]
lag = np.array([A[max(0, t - 148):t].max() - A[t] for t in range(1, nt)])
print("max(A of 148 preds) - A(t)", q(lag))
np_ = (buf[7, :nt] > 0).sum()
print(f"tiles with a segment re-read from L2: {np_} of {nt}; segments: {int(buf[7, :nt].sum())}")
