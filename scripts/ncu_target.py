"""Small launch target for ncu captures of kernels that bench.py does not time by default:
  python scripts/ncu_target.py u8|bf16 [n]     (AUTO transposes of an n x n matrix, 6 launches)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

dt = {"u8": torch.uint8, "bf16": torch.bfloat16, "f32": torch.float32}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
x = torch.randint(0, 100, (n, n), dtype=torch.uint8 if dt == torch.uint8 else torch.int16,
                  device="cuda").view(dt)
y = torch.empty_like(x)
for _ in range(6):
    desc.transpose(x, y)
torch.cuda.synchronize()
print("ok", torch.equal(y.view(torch.uint8 if dt == torch.uint8 else torch.int16)[:64, :64],
                        x.view(torch.uint8 if dt == torch.uint8 else torch.int16)[:64, :64].t()))
