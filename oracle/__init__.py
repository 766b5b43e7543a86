"""CPU ORACLE for the transpose -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product package
(paper_2305_03448_b200) never imports it and shares no code with it.

The arithmetic lives in oracle/transpose_ref.c (a naive loop over the plain
definition out[j][i] = in[i][j]); this
file only builds/loads it with gcc + ctypes and marshals numpy buffers.

Distributed reading (R13): rank r of P owns input rows
[rR, (r+1)R) and output rows [rR, (r+1)R) of the global transpose, R = rows/P.

Parity pins: tests/test_oracle.py.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "transpose_ref.c")
_SRCS = [_SRC, os.path.join(_HERE, "reduce_scan_ref.c")]
_LIB = os.path.join(_HERE, "liboracle_transpose.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 (plain C, no intrinsics, no threads)."""
    if force or not os.path.exists(_LIB) or any(
            os.path.getmtime(_LIB) < os.path.getmtime(src) for src in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC",
                               "-o", tmp, *_SRCS])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64 = ctypes.c_int64
        lib.oracle_transpose_batched.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                                 i64, i64, i64, i64, i64, i64, i64, i64]
        lib.oracle_transpose_batched.restype = ctypes.c_int
        lib.oracle_transpose.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                         i64, i64, i64, i64, i64]
        lib.oracle_transpose.restype = ctypes.c_int
        vp = ctypes.c_void_p
        for name in ("oracle_block_reduce_int", "oracle_block_reduce_float"):
            getattr(lib, name).argtypes = [vp, vp, i64, i64, i64]
            getattr(lib, name).restype = ctypes.c_int
        for name in ("oracle_scan_int", "oracle_scan_float"):
            getattr(lib, name).argtypes = [vp, vp, i64, i64]
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def transpose_raw(in_buf: np.ndarray, out_buf: np.ndarray, batch: int, rows: int,
                  cols: int, ld_in: int, ld_out: int, stride_in: int,
                  stride_out: int, es: int, in_offset: int = 0,
                  out_offset: int = 0) -> None:
    """out[b*stride_out + j*ld_out + i] = in[b*stride_in + i*ld_in + j] on raw
    C-contiguous buffers (element offsets given in elements of size es)."""
    assert in_buf.flags.c_contiguous and out_buf.flags.c_contiguous
    pin = in_buf.ctypes.data + in_offset * es
    pout = out_buf.ctypes.data + out_offset * es
    rc = _load().oracle_transpose_batched(pin, pout, batch, rows, cols, ld_in,
                                          ld_out, stride_in, stride_out, es)
    if rc != 0:
        raise ValueError("oracle: arguments outside the definition")


def transpose(a: np.ndarray) -> np.ndarray:
    """Transpose of a 2-D array, or of the last two dims of a 3-D array."""
    a = np.ascontiguousarray(a)
    if a.ndim == 2:
        rows, cols = a.shape
        out = np.empty((cols, rows), dtype=a.dtype)
        transpose_raw(a, out, 1, rows, cols, cols, rows, 0, 0, a.itemsize)
        return out
    if a.ndim == 3:
        batch, rows, cols = a.shape
        out = np.empty((batch, cols, rows), dtype=a.dtype)
        transpose_raw(a, out, batch, rows, cols, cols, rows, rows * cols,
                      rows * cols, a.itemsize)
        return out
    raise ValueError("oracle.transpose takes a 2-D or 3-D array")


def dist_expected_slab(global_in: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rank `rank`'s output slab of the distributed transpose: rows
    [rR, (r+1)R) of transpose(global_in), R = cols/world (R13)."""
    rows, cols = global_in.shape
    if cols % world:
        raise ValueError("cols must divide by world size (R13)")
    R = cols // world
    return transpose(global_in)[rank * R:(rank + 1) * R]


def time_transpose(in_buf: np.ndarray, out_buf: np.ndarray, batch: int, rows: int,
                   cols: int, ld_in: int, ld_out: int, stride_in: int,
                   stride_out: int, es: int, reps: int = 3):
    """Wall-clock the single-threaded oracle: returns the list of per-rep seconds."""
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        transpose_raw(in_buf, out_buf, batch, rows, cols, ld_in, ld_out,
                      stride_in, stride_out, es)
        times.append(time.perf_counter() - t0)
    return times


# ---- block-wide reduction and scan ----
def _is_float(a: np.ndarray) -> bool:
    return a.dtype.kind == "f"


def block_reduce(a: np.ndarray, block: int) -> np.ndarray:
    """out[b] = sum of a[b*B : (b+1)*B] -- integers wrap (same dtype), floats are
    sequential fp64 sums (float64 result).  oracle/reduce_scan_ref.c."""
    a = np.ascontiguousarray(a).reshape(-1)
    if block <= 0:
        raise ValueError("oracle: block must be positive")
    nb = -(-a.size // block)
    if _is_float(a):
        out = np.empty(nb, dtype=np.float64)
        rc = _load().oracle_block_reduce_float(a.ctypes.data, out.ctypes.data, a.size, block,
                                               a.itemsize)
    else:
        out = np.empty(nb, dtype=a.dtype)
        rc = _load().oracle_block_reduce_int(a.ctypes.data, out.ctypes.data, a.size, block,
                                             a.itemsize)
    if rc:
        raise ValueError("oracle: arguments outside the definition")
    return out


def scan(a: np.ndarray) -> np.ndarray:
    """Inclusive prefix sum -- integers wrap (same dtype), floats sequential fp64."""
    a = np.ascontiguousarray(a).reshape(-1)
    if _is_float(a):
        out = np.empty(a.size, dtype=np.float64)
        rc = _load().oracle_scan_float(a.ctypes.data, out.ctypes.data, a.size, a.itemsize)
    else:
        out = np.empty(a.size, dtype=a.dtype)
        rc = _load().oracle_scan_int(a.ctypes.data, out.ctypes.data, a.size, a.itemsize)
    if rc:
        raise ValueError("oracle: arguments outside the definition")
    return out
