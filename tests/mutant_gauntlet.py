"""Parity gauntlet run in a subprocess against one library build.

`python tests/mutant_gauntlet.py` prints one JSON object {check: true|false} -- true when the
CUDA path matched the oracle byte for byte (and left every sentinel byte alone).
tests/test_mutants_gpu.py runs it once against the product library (every check must pass)
and once per defect of the test-teeth library (DESC_LIB=build_variants/libdesc_mutants.so,
DESC_MUTANT=<id>; at least one check must fail). The checks are the same comparisons the
parity tests make (self-describing inputs, guard bands, padded ld, random bits with NaN
payloads), kept small so one run takes seconds.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2305_03448_b200 as desc  # noqa: E402

SENT = -0x5A5A5A5B
NP = {4: np.int32, 8: np.int64}
TT = {4: torch.int32, 8: torch.int64}
FT = {4: torch.float32, 8: torch.float64}


def padded(kernel, rows, cols, es, ld_in, ld_out):
    """Self-describing input in a padded buffer; output region inside a buffer of sentinels
    large enough that a swapped-ld write still lands inside the allocation."""
    src = synth.self_describing(1, rows, cols, es)[0]
    xin = torch.zeros((rows, ld_in), dtype=TT[es], device="cuda")
    xin[:, :cols] = torch.from_numpy(src.view(NP[es])).cuda()
    need = cols * max(ld_in, ld_out) + 4096
    buf = torch.full((need,), SENT, dtype=TT[es], device="cuda")
    yout = buf[: cols * ld_out].view(cols, ld_out)
    desc.transpose(xin.view(FT[es])[:, :cols], yout.view(FT[es])[:, :rows], kernel=kernel)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    logical = got[: cols * ld_out].reshape(cols, ld_out)[:, :rows]
    ok = logical.view(src.dtype).tobytes() == oracle.transpose(src).tobytes()
    pad = got[: cols * ld_out].reshape(cols, ld_out)[:, rows:]
    return bool(ok and (pad == SENT).all() and (got[cols * ld_out:] == SENT).all())


def tight(kernel, rows, cols, es, seed, specials=False, reps=1):
    a = synth.random_bits((rows, cols), es, seed)
    if specials:
        a = synth.with_specials(a, es, seed)
    x = torch.from_numpy(a.view(NP[es])).cuda().view(FT[es])
    ref = oracle.transpose(a).tobytes()
    ok = True
    for _ in range(reps):
        y = desc.transpose(x, kernel=kernel)
        torch.cuda.synchronize()
        ok &= y.view(TT[es]).cpu().numpy().view(a.dtype).tobytes() == ref
    return bool(ok)


def described(kernel, rows, cols, es, reps=1):
    src = synth.self_describing(1, rows, cols, es)[0]
    x = torch.from_numpy(src.view(NP[es])).cuda().view(FT[es])
    ref = oracle.transpose(src).tobytes()
    ok = True
    for _ in range(reps):
        y = desc.transpose(x, kernel=kernel)
        torch.cuda.synchronize()
        ok &= y.view(TT[es]).cpu().numpy().view(src.dtype).tobytes() == ref
    return bool(ok)


def scan(n, algo):
    a = synth.random_ints(n, np.int32, n)
    y = desc.scan(torch.from_numpy(a).cuda(), algo=algo)
    torch.cuda.synchronize()
    return bool(y.cpu().numpy().tobytes() == oracle.scan(a).tobytes())


def reduce(n, B):
    a = synth.random_ints(n, np.int32, n + B)
    y = desc.block_reduce(torch.from_numpy(a).cuda(), B)
    torch.cuda.synchronize()
    return bool(y.cpu().numpy().tobytes() == oracle.block_reduce(a, B).tobytes())


CHECKS = {
    "smem_padded_f32": lambda: padded("smem", 67, 131, 4, 131 + 5, 67 + 3),
    "smem_described_i32": lambda: described("smem", 100, 200, 4),
    "smem_random_f64": lambda: tight("smem", 64, 96, 8, 11, specials=True),
    "tma_padded_f32": lambda: padded("tma_st", 67, 131, 4, 136, 72),
    "tma_padded_f64": lambda: padded("tma_st", 45, 70, 8, 72, 46),
    "tma_described_f32": lambda: described("tma_st", 2048, 2048, 4, reps=3),
    "tma_random_f64": lambda: tight("tma_st", 1000, 1500, 8, 12, specials=True, reps=3),
    "tiled_padded_f32": lambda: padded("tiled", 67, 131, 4, 136, 72),
    "tiled_padded_f64": lambda: padded("tiled", 130, 197, 8, 199, 131),
    "tiled_described_f32": lambda: described("tiled", 2048, 2048, 4, reps=3),
    "tiled_random_f64": lambda: tight("tiled", 1000, 1500, 8, 12, specials=True, reps=3),
    "vtiled_padded_f32": lambda: padded("vtiled", 68, 132, 4, 136, 72),
    "vtiled_described_f32": lambda: described("vtiled", 2048, 2048, 4, reps=3),
    "vtiled_random_f64": lambda: tight("vtiled", 1000, 1500, 8, 12, specials=True, reps=3),
    "scan_stream_i32": lambda: scan(1 << 22, "stream"),
    "scan_lookback_i32": lambda: scan(100003, "lookback"),
    "scan_three_pass_i32": lambda: scan(1 << 21, "three_pass"),
    "reduce_i32": lambda: reduce(1000003, 4099),
}


def main():
    desc.load()
    res = {}
    for name, fn in CHECKS.items():
        try:
            res[name] = fn()
        except Exception as e:  # a fault counts as a failed check
            res[name] = False
            res[name + "_error"] = f"{type(e).__name__}: {e}"[:200]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
