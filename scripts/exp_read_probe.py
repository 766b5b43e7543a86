"""Read-only HBM probe (desc_read_probe) at several buffer sizes: best of 20 launches, GB/s.
DESC_LIB selects a compile-time variant (e.g. without the in-loop L2 prefetch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

tag = os.path.basename(os.environ.get("DESC_LIB", "product"))
s = torch.cuda.current_stream()
sink = torch.empty(desc.desc_read_probe_sink_bytes(), dtype=torch.uint8, device="cuda")
for mb in (128, 256, 512, 1024, 2048):
    n = mb << 20
    buf = torch.ones(n // 4, dtype=torch.int32, device="cuda")
    for _ in range(3):
        desc.desc_read_probe(buf.data_ptr(), n, sink.data_ptr(), s.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
    ev[0].record()
    for k in range(20):
        desc.desc_read_probe(buf.data_ptr(), n, sink.data_ptr(), s.cuda_stream)
        ev[k + 1].record()
    torch.cuda.synchronize()
    best = min(ev[k].elapsed_time(ev[k + 1]) for k in range(20))
    print(f"{tag:24s} {mb:5d} MB  {n / best / 1e6:8.0f} GB/s", flush=True)
    del buf
