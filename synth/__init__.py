"""Seeded synthetic input generators shared by the oracle's tests and the CUDA path's tests/bench.

This module holds NONE of the method's arithmetic (no transpose, no index map of
the method): it only produces input bit patterns and decodes the self-describing
pattern it encodes.  It is the one module both sides may import
(task rule ③).

Recipes (DESIGN.md §Input recipe):
  * random_bits     -- uniform random element bit patterns (so NaN payloads,
                       signalling NaNs, +-0, infinities and subnormals all occur
                       for f32/f64 views); seed = 0x23050344 + config index.
  * with_specials   -- overwrites a few cells with hand-picked special patterns.
  * self_describing -- element bits = (b << (kr+kc)) | (i << kc) | j, with
                       kc = bits(cols), kr = bits(rows): any misplaced element
                       decodes to the coordinate it came from.
  * splitmix64 hash -- closed-form input H(seed ^ flat_index) for matrices too
                       large to materialise on the host (65536^2 f32); the same
                       counter-based generator is implemented in numpy (host) and
                       in torch integer ops (device fill), both here.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 0x23050344

# element size in bytes -> unsigned numpy type carrying the element's bits
UINT_OF_SIZE = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}
# dtype name -> (element size, numpy view type)
DTYPES = {
    "f32": (4, np.float32),
    "i32": (4, np.int32),
    "f64": (8, np.float64),
    "i64": (8, np.int64),
    "f16": (2, np.float16),
    "bf16": (2, None),  # numpy has no bf16; carried as uint16 bits
    "u8": (1, np.uint8),
}


def nbits(n: int) -> int:
    """Number of bits needed to hold values 0..n-1 (at least 1)."""
    return max(1, int(n - 1).bit_length())


def random_bits(shape, es: int, seed: int) -> np.ndarray:
    """Uniform random bit patterns of width 8*es as an unsigned array."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ut = UINT_OF_SIZE[es]
    if es == 8:
        return rng.integers(0, 2**64, size=shape, dtype=np.uint64, endpoint=False)
    return rng.integers(0, np.iinfo(ut).max, size=shape, dtype=ut, endpoint=True)


SPECIALS = {
    4: [0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00001, 0x7F800001,
        0x00000001, 0x807FFFFF, 0xFFFFFFFF, 0x3F800000],
    8: [0x0000000000000000, 0x8000000000000000, 0x7FF0000000000000,
        0xFFF0000000000000, 0x7FF8000000000001, 0x7FF0000000000001,
        0x0000000000000001, 0x800FFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF,
        0x3FF0000000000000],
    2: [0x0000, 0x8000, 0x7C00, 0xFC00, 0x7E01, 0x7C01, 0x0001, 0x83FF, 0xFFFF],
    1: [0x00, 0xFF, 0x80, 0x7F],
}


def with_specials(a: np.ndarray, es: int, seed: int) -> np.ndarray:
    """Copy of `a` with special bit patterns (NaN payloads, sNaN, -0, inf,
    subnormals) written at seeded positions."""
    a = a.copy()
    flat = a.reshape(-1)
    if flat.size == 0:
        return a
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EC1A1))
    specials = np.array(SPECIALS[es], dtype=UINT_OF_SIZE[es])
    pos = rng.integers(0, flat.size, size=min(flat.size, 4 * len(specials)))
    flat[pos] = specials[np.arange(pos.size) % len(specials)]
    return a


def self_describing(batch: int, rows: int, cols: int, es: int) -> np.ndarray:
    """Unsigned array [batch, rows, cols] with bits (b<<(kr+kc)) | (i<<kc) | j."""
    kc, kr = nbits(cols), nbits(rows)
    kb = nbits(batch) if batch > 1 else 0
    if kb + kr + kc > 8 * es:
        raise ValueError(f"self-describing pattern needs {kb+kr+kc} bits > {8*es}")
    b = np.arange(batch, dtype=np.uint64)[:, None, None]
    i = np.arange(rows, dtype=np.uint64)[None, :, None]
    j = np.arange(cols, dtype=np.uint64)[None, None, :]
    v = (b << np.uint64(kr + kc)) | (i << np.uint64(kc)) | j
    return v.astype(UINT_OF_SIZE[es])


def decode_self_describing(bits: np.ndarray, batch: int, rows: int, cols: int):
    """Inverse of self_describing: returns (b, i, j) arrays of the source coordinate."""
    kc, kr = nbits(cols), nbits(rows)
    v = bits.astype(np.uint64)
    j = v & np.uint64((1 << kc) - 1)
    i = (v >> np.uint64(kc)) & np.uint64((1 << kr) - 1)
    b = v >> np.uint64(kr + kc)
    return b, i, j


# --- counter-based hash (splitmix64 finaliser), host and device versions ---
_SM_GAMMA = 0x9E3779B97F4A7C15
_SM_M1 = 0xBF58476D1CE4E5B9
_SM_M2 = 0x94D049BB133111EB


def splitmix64_np(idx, seed: int) -> np.ndarray:
    """H(seed, idx) for uint64 idx (numpy, host)."""
    with np.errstate(over="ignore"):
        z = (np.asarray(idx, dtype=np.uint64) ^ np.uint64(seed)) + np.uint64(_SM_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM_M2)
        return z ^ (z >> np.uint64(31))


def _to_i64(u: int) -> int:
    return u - (1 << 64) if u >= (1 << 63) else u


def splitmix64_torch(idx, seed: int):
    """Same H as splitmix64_np, in torch int64 ops (wrapping mul, logical shifts).

    Works on any device; used to fill 65536^2 inputs directly in HBM."""
    import torch

    def lsr(z, k):  # logical shift right on int64
        return (z >> k) & ((1 << (64 - k)) - 1)

    z = (idx ^ _to_i64(seed)) + _to_i64(_SM_GAMMA)
    z = (z ^ lsr(z, 30)) * _to_i64(_SM_M1)
    z = (z ^ lsr(z, 27)) * _to_i64(_SM_M2)
    return z ^ lsr(z, 31)


def hash_fill_torch(out, row0: int, col0: int, global_cols: int, seed: int,
                    chunk_rows: int = 1024):
    """Fill a 2-D int tensor `out` (rows x cols, any device, int32 or int64 view)
    with H(seed, (row0+i)*global_cols + col0 + j) truncated to the element width."""
    import torch

    rows, cols = out.shape
    jj = torch.arange(cols, device=out.device, dtype=torch.int64) + col0
    for r0 in range(0, rows, chunk_rows):
        r1 = min(rows, r0 + chunk_rows)
        ii = torch.arange(r0, r1, device=out.device, dtype=torch.int64) + row0
        flat = ii[:, None] * global_cols + jj[None, :]
        h = splitmix64_torch(flat, seed)
        if out.element_size() == 4:
            h = (h & 0xFFFFFFFF)
            h = torch.where(h >= (1 << 31), h - (1 << 32), h)
        out[r0:r1].copy_(h.to(out.dtype))
    return out


def hash_expected_np(i, j, global_cols: int, seed: int, es: int) -> np.ndarray:
    """Host value of input element (i, j) of the hash-filled matrix, as unsigned bits."""
    flat = np.asarray(i, dtype=np.uint64) * np.uint64(global_cols) + np.asarray(j, dtype=np.uint64)
    h = splitmix64_np(flat, seed)
    if es == 4:
        return (h & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return h


def random_floats(n: int, dtype, seed: int, spread: int = 8) -> np.ndarray:
    """Finite floats with mixed signs and magnitudes: uniform(-1, 1) * 2^k, k uniform in
    [-spread, spread] (reduction / scan inputs: NaN/inf would make sums meaningless)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    v = rng.uniform(-1.0, 1.0, size=n) * np.exp2(rng.integers(-spread, spread + 1, size=n))
    return v.astype(dtype)


def random_ints(n: int, dtype, seed: int) -> np.ndarray:
    """Uniform integers over the whole range of `dtype` (sums wrap around)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    info = np.iinfo(dtype)
    return rng.integers(info.min, info.max, size=n, dtype=dtype, endpoint=True)
