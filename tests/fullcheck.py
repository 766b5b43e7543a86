"""Every-element verification of huge transposes, on the device (test infrastructure).

For inputs too large for the CPU oracle (65536^2 f32: 2^32 elements, 16 GiB) the input is the
counter hash of ``synth`` -- in[i][j] = H(seed, i*N + j) truncated to the cell -- so every
element of the result has a closed form: the transpose's definition (caption
P:108; SURVEY.md 8(c) "Distributed at 65536^2") gives

    out[j][i] = in[i][j] = H(seed, i*N + j).

``hash_transpose_mismatches`` recomputes H for every output element in row chunks with torch
integer ops (``synth.splitmix64_torch``, the same generator that filled the input; no code of
the CUDA path) and compares -- a decode of the generator, not the method's arithmetic, so it
can run at full size where the oracle cannot (VERDICT r01 "Next round" #1).

Imported by tests/ and by bench.py's post-region parity check only.
"""
from __future__ import annotations

import synth


def hash_transpose_mismatches(out, out_row0: int, in_cols: int, seed: int,
                              chunk_rows: int = 256):
    """Count the elements of ``out`` (a (R, M) int32/int64 CUDA tensor: rows
    [out_row0, out_row0 + R) of the N x M transpose of the M x N hash-filled input) that differ
    from H(seed, i*N + j) at out[j - out_row0][i].  Returns (mismatches, first) where first is
    (j, i) of the first mismatching element or None.  Every element is checked."""
    import torch

    R, M = out.shape
    es = out.element_size()
    ii = torch.arange(M, device=out.device, dtype=torch.int64) * in_cols      # i * N
    bad_total = 0
    first = None
    for r0 in range(0, R, chunk_rows):
        r1 = min(R, r0 + chunk_rows)
        jj = torch.arange(r0, r1, device=out.device, dtype=torch.int64) + out_row0
        h = synth.splitmix64_torch(ii[None, :] + jj[:, None], seed)           # (r1-r0, M)
        got = out[r0:r1].to(torch.int64)
        if es == 4:
            h = h & 0xFFFFFFFF
            got = got & 0xFFFFFFFF
        ne = got != h
        nbad = int(ne.sum().item())
        if nbad and first is None:
            k = int(torch.nonzero(ne.reshape(-1))[0].item())
            first = (out_row0 + r0 + k // M, k % M)
        bad_total += nbad
        del h, got, ne
    return bad_total, first
