"""Repeated-launch stress of the non-transpose paths (scan algorithms, block reduction, row
copy, view copies, the fused slab kernel): integer inputs, each result compared on the device
with a torch expression of the definition (test infrastructure, never the product path).
Intermittent races show up as a few bad launches out of hundreds (cf. stress_8192.py).

  python scripts/stress_all.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

M32 = (1 << 32) - 1


def wrap32(t):
    """int64 tensor -> the int32 with the same low 32 bits."""
    t = t & M32
    return torch.where(t >= (1 << 31), t - (1 << 32), t).to(torch.int32)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    dev = "cuda"
    res = {}

    def check(name, fn):
        bad = 0
        for it in range(reps):
            if not fn(it):
                bad += 1
        res[name] = bad
        print(f"{name:34s} {reps} launches, {bad} with mismatches", flush=True)

    # scans (every algorithm), int32 wrap-around sums
    n = (1 << 24) + 3
    x = torch.from_numpy(synth.random_ints(n, np.int32, 5)).to(dev)
    ref = wrap32(torch.cumsum(x.to(torch.int64), 0))
    work = torch.empty(desc.desc_scan_workspace(n, "i32"), dtype=torch.uint8, device=dev)
    for algo in ("stream", "lookback", "three_pass"):
        y = torch.empty_like(x)

        def f(it, algo=algo, y=y):
            y.fill_(7)
            desc.scan(x, out=y, work=work, algo=algo)
            return bool(torch.equal(y, ref))
        check(f"scan i32 {algo}", f)
    # f32 scan through the lane-contiguous TMA-store path: repeat determinism (bitwise)
    xf = torch.from_numpy(synth.random_floats(n, np.float32, 6)).to(dev)
    yf0 = desc.scan(xf, work=work, algo="stream").clone()
    yf = torch.empty_like(xf)

    def ff(it):
        yf.fill_(0)
        desc.scan(xf, out=yf, work=work, algo="stream")
        return bool(torch.equal(yf.view(torch.int32), yf0.view(torch.int32)))
    check("scan f32 stream (bitwise repeat)", ff)
    # block reduction
    for B in (16, 1024, 5000, 1 << 20):
        nn = (1 << 24) if B != 5000 else 5000 * 3000
        xr = torch.from_numpy(synth.random_ints(nn, np.int32, B)).to(dev)
        nb = -(-nn // B)
        pad = torch.zeros(nb * B, dtype=torch.int64, device=dev)
        pad[:nn] = xr.to(torch.int64)
        rref = wrap32(pad.view(nb, B).sum(1))
        yr = torch.empty(nb, dtype=torch.int32, device=dev)

        def fr(it, xr=xr, B=B, yr=yr, rref=rref):
            yr.fill_(7)
            desc.block_reduce(xr, B, out=yr)
            return bool(torch.equal(yr, rref))
        check(f"block_reduce i32 B={B}", fr)
    # row copy (unpack shape: P blocks side by side)
    P, R = 4, 4096
    xc = torch.from_numpy(synth.random_ints(P * R * R, np.int32, 9)).to(dev)
    yc = torch.empty((R, P * R), dtype=torch.int32, device=dev)
    cref = xc.view(P, R, R).permute(1, 0, 2).reshape(R, P * R)

    def fc(it):
        yc.fill_(7)
        desc.desc_copy_batched(xc.data_ptr(), yc.data_ptr(), P, R, R, R, P * R, R * R, R, "i32",
                               torch.cuda.current_stream().cuda_stream)
        return bool(torch.equal(yc, cref))
    check("copy_batched unpack P=4 R=4096", fc)
    # view copies: rot180, group_by_tile, rot90
    a = synth.random_bits((4096, 4096), 4, 10)
    xv = torch.from_numpy(a.view(np.int32)).to(dev)
    views = {"rot180": ([("reverse", 0, 0), ("reverse", 0, 1)], torch.flip(xv, [0, 1])),
             "group_by_tile<64,64>": ([("group", 64, 0), ("group", 64, 2), ("transpose", 0, 1)],
                                      xv.view(64, 64, 64, 64).permute(0, 2, 1, 3).contiguous()),
             "rot90": ([("transpose", 0, 0), ("reverse", 0, 1)], torch.flip(xv.t(), [1]))}
    for name, (ops, vref) in views.items():
        def fv(it, ops=ops, vref=vref):
            yv = desc.view_copy(xv, ops)
            return bool(torch.equal(yv.reshape(vref.shape), vref))
        check(f"view {name}", fv)
    # fused slab transpose + exchange, two slabs on this GPU
    M = N = 4096
    g = torch.from_numpy(synth.random_bits((M, N), 4, 11).view(np.int32)).to(dev)
    gt = g.t().contiguous()
    slabs = [torch.empty((N // 2, M), dtype=torch.int32, device=dev) for _ in range(2)]

    def fs(it):
        for t in slabs:
            t.fill_(7)
        for r in range(2):
            desc.desc_slab_transpose_peer(g[r * (M // 2):(r + 1) * (M // 2)].data_ptr(),
                                          [t.data_ptr() for t in slabs], r, M, N, "i32",
                                          torch.cuda.current_stream().cuda_stream)
        return all(bool(torch.equal(slabs[r], gt[r * (N // 2):(r + 1) * (N // 2)]))
                   for r in range(2))
    check("slab_transpose_peer (2 slabs)", fs)
    print("STRESS", "FAIL" if any(res.values()) else "PASS")


if __name__ == "__main__":
    main()
