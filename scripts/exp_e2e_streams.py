"""e2e (desc_transpose_host, pinned buffers) with 2 or 3 internal band buffers/streams
(DESC_HOST_STREAMS, read once per process) and workspace = recommended x {1, 1.5}.
  DESC_HOST_STREAMS=3 python scripts/exp_e2e_streams.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
for (rows, cols, dt, tdt) in ((8192, 8192, "f32", torch.int32), (3000, 5000, "f64", torch.int64),
                              (2048, 2048, "f64", torch.int64)):
    es = torch.empty((), dtype=tdt).element_size()
    h_in = torch.randint(0, 1 << 30, (rows, cols), dtype=tdt).pin_memory()
    h_out = torch.empty((cols, rows), dtype=tdt).pin_memory()
    base = desc.desc_transpose_host_workspace(rows, cols, dt)
    for f in (1.0, 1.5):
        work = torch.empty(int(base * f) // 256 * 256 + 256, dtype=torch.uint8, device="cuda")

        def go():
            desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), 1, rows, cols, cols, rows,
                                     0, 0, dt, work.data_ptr(), work.numel(), st)
        for _ in range(2):
            go()
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                go()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            best = ms if best is None else min(best, ms)
        ok = torch.equal(h_out[:64, :64], h_in[:64, :64].t())
        print(f"streams={os.environ.get('DESC_HOST_STREAMS', '2')} {rows}x{cols} {dt} ws x{f}: "
              f"{2 * rows * cols * es / (best / 1e3) / 1e9:6.1f} GB/s, "
              f"{desc.desc_last_launch_count()} bands {'ok' if ok else 'MISMATCH'}", flush=True)
        del work
