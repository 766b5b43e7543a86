"""Streaming scan of 2^28 uint8 (sums mod 2^32 into uint32... the output has the input's
type: the inclusive prefix wraps mod 256), back to back; GB/s = 2 n / time.
  DESC_LIB=... python scripts/exp_scan_u8.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

n = 1 << 28
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
work = torch.empty(desc.desc_scan_workspace(n, "u8"), dtype=torch.uint8, device="cuda")
for _ in range(3):
    desc.scan(x, out=y, work=work, algo="stream")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    desc.scan(x, out=y, work=work, algo="stream")
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
ref = torch.cumsum(x[:1 << 20].to(torch.int64), 0) % 256
ok = torch.equal(y[:1 << 20].to(torch.int64), ref)
print(f"{os.path.basename(os.environ.get('DESC_LIB', 'product'))}: u8 scan 2^28 "
      f"{2 * n / (ms / 1e3) / 1e9:.0f} GB/s ({2 * n / (ms / 1e3) / 1e9 / pk:.3f}) check {ok}")
