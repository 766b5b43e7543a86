"""Stress: every transpose variant on 8192^2 f32 many times, each output compared on the
device with the definition (torch's strided view of the input as the checker -- test
infrastructure, not the product path); mismatches are located and decoded: which kernel,
which launch, how many elements, and where the wrong values came from.

  python scripts/stress_8192.py [reps] [kernels]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    kernels = sys.argv[2].split(",") if len(sys.argv) > 2 else \
        ["auto", "tma", "tma_st", "tma_tile", "smem", "tiled", "vtiled"]
    n = 8192
    a = synth.random_bits((n, n), 4, synth.BASE_SEED + 2)
    x = torch.from_numpy(a.view(np.int32)).cuda()
    ref = x.t().contiguous()
    # self-describing input too: a wrong value names its source
    sd = torch.arange(n * n, dtype=torch.int64, device="cuda").view(n, n).to(torch.int32)
    sd_ref = sd.t().contiguous()
    y = torch.empty_like(x)
    total_bad = 0
    for k in kernels:
        bad_launches = 0
        for it in range(reps):
            for src, exp, what in ((x, ref, "random"), (sd, sd_ref, "self-describing")):
                y.fill_(-0x5A5A5A5B)
                desc.transpose(src.view(torch.float32), y.view(torch.float32), kernel=k)
                torch.cuda.synchronize()
                neq = (y != exp)
                cnt = int(neq.sum())
                if cnt:
                    bad_launches += 1
                    idx = torch.nonzero(neq)[:4].tolist()
                    info = []
                    for (j, i) in idx:
                        got = int(y[j, i])
                        e = int(exp[j, i])
                        src_of = (f"in[{got // n}][{got % n}]" if what == "self-describing"
                                  and 0 <= got < n * n else f"{got & 0xffffffff:#010x}")
                        info.append(f"out[{j}][{i}] = {src_of} want {e & 0xffffffff:#010x}")
                    print(f"MISMATCH kernel={k} it={it} input={what}: {cnt} elements; "
                          + "; ".join(info), flush=True)
        total_bad += bad_launches
        print(f"{k:9s} {2 * reps} launches, {bad_launches} with mismatches", flush=True)
    print("STRESS", "FAIL" if total_bad else "PASS")


if __name__ == "__main__":
    main()
