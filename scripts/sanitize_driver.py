"""Small driver for compute-sanitizer gates (racecheck / synccheck / memcheck / initcheck).

Runs every kernel variant on a few small and ragged shapes through the C-ABI and checks the
result against the oracle, so a sanitizer run both exercises and validates the kernels:

  compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_driver.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: expected values)
import synth  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

CASES = [  # (batch, rows, cols, es)
    (1, 64, 64, 8), (1, 67, 131, 4), (1, 131, 67, 8), (1, 300, 500, 4), (3, 33, 65, 4),
    (2, 130, 70, 8), (1, 5, 3, 4), (1, 256, 512, 2), (1, 257, 300, 1), (1, 68, 132, 4),
]
DT = {1: "u8", 2: "f16", 4: "f32", 8: "f64"}
TI = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
NI = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def main():
    desc.load()
    bad = 0
    for batch, rows, cols, es in CASES:
        v = 16 // es
        ld_in = cols + (-cols) % v
        ld_out = rows + (-rows) % v
        src = synth.random_bits((batch, rows, cols), es, rows * 31 + cols)
        xin = torch.zeros((batch, rows, ld_in), dtype=TI[es], device="cuda")
        xin[:, :, :cols] = torch.from_numpy(src.view(NI[es])).cuda()
        ref = oracle.transpose(src)
        kernels = ["smem", "tiled", "tma"] + (["tma_st", "tma_tile"] if es in (4, 8) and rows * es >= 16 else [])
        if es in (4, 8) and rows % v == 0 and cols % v == 0:
            kernels.append("vtiled")      # 16-byte cp.async staging (rows, cols multiples of 16/es)
        for k in kernels:
            out = torch.zeros((batch, cols, ld_out), dtype=TI[es], device="cuda")
            desc.desc_transpose_ex(xin.data_ptr(), out.data_ptr(), batch, rows, cols, ld_in,
                                   ld_out, rows * ld_in, cols * ld_out, DT[es], k,
                                   torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            got = out[:, :, :rows].cpu().numpy().view(synth.UINT_OF_SIZE[es])
            ok = got.tobytes() == ref.tobytes()
            bad += not ok
            print(f"{k:7s} batch={batch} {rows}x{cols} es={es}: {'ok' if ok else 'MISMATCH'}",
                  flush=True)
    # dynamically scheduled TMA-store launches with stage reuse (run the driver with
    # DESC_DYN_MIN=1 so that this modest size takes the dynamic path)
    from oracle import views as V
    big = synth.random_bits((2048, 2048), 4, 99)
    xb = torch.from_numpy(big.view(np.int32)).cuda()
    # outputs are zero-filled first: initcheck does not see TMA bulk-tensor stores as
    # initialising writes (it would flag every byte the TMA-store kernel produced)
    yb = desc.transpose(xb, torch.zeros((2048, 2048), dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    ok = yb.cpu().numpy().view(np.uint32).tobytes() == oracle.transpose(big).tobytes()
    bad += not ok
    print(f"tma_st 2048x2048 es=4 (dynamic when DESC_DYN_MIN=1): {'ok' if ok else 'MISMATCH'}",
          flush=True)
    # view copies: every dispatch path
    small = synth.random_bits((192, 320), 4, 7)
    xs = torch.from_numpy(small.view(np.int32)).cuda()
    for ops in ([("transpose", 0, 0), ("reverse", 0, 1)],                     # mirrored TMA
                [("group", 64, 0), ("group", 64, 2), ("transpose", 0, 1)],   # 16-byte rows
                [("reverse", 0, 0), ("reverse", 0, 1)],                      # reversed vectors
                [("split_snd", 7, 1), ("reverse", 0, 0)]):                   # element gather
        shape = desc.desc_view_compile(tuple(xs.shape), ops, tuple(xs.stride())).dims[0]
        y = desc.view_copy(xs, ops, out=torch.zeros(shape, dtype=xs.dtype, device="cuda"))
        torch.cuda.synchronize()
        ok = y.cpu().numpy().view(np.uint32).tobytes() == V.materialize(small, ops).tobytes()
        bad += not ok
        print(f"view {ops}: {'ok' if ok else 'MISMATCH'}", flush=True)
    # block reduction (thread / warp / CTA groups) and scan (every algorithm; the streaming
    # one over a few tiles per CTA so that its stage ring wraps)
    for dt, n in ((np.int32, 100003), (np.float32, 70001), (np.int64, 50000), (np.uint8, 90000)):
        a = (synth.random_ints(n, dt, 5) if dt != np.float32 else synth.random_floats(n, dt, 5))
        x = torch.from_numpy(a).cuda()
        for B in (16, 1000, 20000):
            y = desc.block_reduce(x, B)
            torch.cuda.synchronize()
            ref = oracle.block_reduce(a, B)
            if dt == np.float32:
                ok = np.allclose(y.cpu().numpy(), ref, rtol=1e-6, atol=1e-6)
            else:
                ok = y.cpu().numpy().tobytes() == ref.tobytes()
            bad += not ok
            print(f"block_reduce {dt.__name__} n={n} B={B}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if dt == np.float32:
            # warp-row kernel (whole 512-byte rows per block, 1 and 2 rows) and the 8-CTA
            # cluster kernel (40 blocks of 16400 elements)
            for nn, B in ((512 * 128 * 3, 128), (512 * 256 + 256, 256), (40 * 16400 + 5, 16400)):
                aa = synth.random_floats(nn, dt, 6)
                y = desc.block_reduce(torch.from_numpy(aa).cuda(), B)
                torch.cuda.synchronize()
                ok = np.allclose(y.cpu().numpy(), oracle.block_reduce(aa, B), rtol=1e-6, atol=1e-6)
                bad += not ok
                print(f"block_reduce float32 n={nn} B={B}: {'ok' if ok else 'MISMATCH'}", flush=True)
        ref = oracle.scan(a)
        for algo in ("lookback", "three_pass", "stream"):
            y = desc.scan(x, out=torch.zeros_like(x), algo=algo)
            torch.cuda.synchronize()
            ok = (np.allclose(y.cpu().numpy(), ref, rtol=1e-5, atol=1e-3) if dt == np.float32
                  else y.cpu().numpy().tobytes() == ref.tobytes())
            bad += not ok
            print(f"scan {algo} {dt.__name__} n={n}: {'ok' if ok else 'MISMATCH'}", flush=True)
    # streaming scan, several tiles per CTA so every stage ring and TMEM slot ring wraps
    # (i32 48 KB tiles ~10 per CTA; f32 48 KB tiles ~6; f64 60 KB tiles ~5, on 148 SMs)
    for dt, n in ((np.int32, 148 * 10 * 12288 + 5), (np.float32, 148 * 6 * 12288 + 7),
                  (np.float64, 148 * 5 * 7680 + 3)):
        a = (synth.random_ints(n, dt, 6) if dt == np.int32 else synth.random_floats(n, dt, 6))
        x = torch.from_numpy(a).cuda()
        y = desc.scan(x, algo="stream")
        torch.cuda.synchronize()
        ref = oracle.scan(a)
        ok = (y.cpu().numpy().tobytes() == ref.tobytes() if dt == np.int32
              else np.allclose(y.cpu().numpy(), ref, rtol=1e-5, atol=1e-3))
        bad += not ok
        print(f"scan stream {dt.__name__} n={n}: {'ok' if ok else 'MISMATCH'}", flush=True)
    print("sanitize driver:", "PASS" if bad == 0 else f"{bad} FAILURES")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
