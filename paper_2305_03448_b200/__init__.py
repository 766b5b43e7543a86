"""paper_2305_03448_b200 -- B200-native tiled matrix transpose (Descend, arxiv 2305.03448).

Thin Python binding over the C-ABI library libdesc_transpose.so
(include/desc_transpose.h).  Argument marshalling only: every byte of the
transpose is moved by the library's CUDA kernels.  There is NO CPU fallback:
if the library is missing, every call raises.

Raw entry points (same names and argument order as the C header):
    desc_transpose, desc_transpose_batched, desc_transpose_ex, desc_select_kernel
Tensor conveniences:
    transpose(x, out=None, kernel="auto")          2-D, out = x^T
    transpose_batched(x, out=None, kernel="auto")  3-D, transposes the last two dims
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "DescError", "DTYPE", "KERNEL", "lib_path", "load",
    "desc_transpose", "desc_transpose_batched", "desc_transpose_ex", "desc_select_kernel",
    "desc_status_string", "desc_last_error", "desc_dtype_size", "desc_version",
    "desc_last_launch_count", "desc_copy_batched", "desc_transpose_host",
    "desc_ipc_handle", "desc_ipc_open", "desc_ipc_close", "desc_view_compile",
    "desc_view_copy", "view_copy", "desc_block_reduce", "desc_scan", "desc_scan_ex",
    "desc_scan_workspace", "SCAN_ALGO", "desc_read_probe", "desc_read_probe_sink_bytes",
    "desc_slab_transpose_peer",
    "block_reduce", "scan", "desc_transpose_host_workspace",
    "desc_transpose_host_workspace_batched", "desc_copy2d",
    "transpose", "transpose_batched", "transpose_host",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
# DESC_LIB: another in-tree build of the same library (compile-time variants for A/B runs)
lib_path = os.environ.get("DESC_LIB") or os.path.join(_PKG, "libdesc_transpose.so")

# enums (include/desc_transpose.h)
STATUS = {0: "DESC_OK", 1: "DESC_ERR_NULL", 2: "DESC_ERR_SHAPE", 3: "DESC_ERR_DTYPE",
          4: "DESC_ERR_ALIAS", 5: "DESC_ERR_MEMSPACE", 6: "DESC_ERR_CUDA", 7: "DESC_ERR_KERNEL"}
DTYPE = {"f32": 0, "f64": 1, "i32": 2, "i64": 3, "f16": 4, "bf16": 5, "u8": 6}
KERNEL = {"auto": 0, "smem": 1, "tma": 2, "tma_st": 3, "tiled": 4, "tma_tile": 5, "vtiled": 6}
KERNEL_NAME = {v: k for k, v in KERNEL.items()}
SCAN_ALGO = {"auto": 0, "lookback": 1, "three_pass": 2, "stream": 3}

_lib = None

MAX_DIMS = 8
VIEW_KIND = {"group": 0, "transpose": 1, "split_fst": 2, "split_snd": 3, "reverse": 4}


class ViewOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("depth", ctypes.c_int32), ("k", ctypes.c_int64)]


class StridedView(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("offset", ctypes.c_int64), ("shape", ctypes.c_int64 * MAX_DIMS),
                ("stride", ctypes.c_int64 * MAX_DIMS)]

    @property
    def dims(self):
        return tuple(self.shape[:self.ndim]), tuple(self.stride[:self.ndim]), self.offset


class DescError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.status_name = STATUS.get(status, f"status {status}")
        super().__init__(f"{self.status_name}: {message}")


def load():
    """Load libdesc_transpose.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise RuntimeError(
            f"{lib_path} is missing: build it with `python -m paper_2305_03448_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(lib_path)
    i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    lib.desc_transpose.argtypes = [vp, vp, i64, i64, i64, i64, ci, vp]
    lib.desc_transpose.restype = ci
    lib.desc_transpose_batched.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ci, vp]
    lib.desc_transpose_batched.restype = ci
    lib.desc_transpose_ex.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ci, ci, vp]
    lib.desc_transpose_ex.restype = ci
    lib.desc_select_kernel.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ci]
    lib.desc_select_kernel.restype = ci
    lib.desc_transpose_host.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ci, vp,
                                        ctypes.c_size_t, vp]
    lib.desc_transpose_host.restype = ci
    lib.desc_transpose_host_workspace.argtypes = [i64, i64, ci]
    lib.desc_transpose_host_workspace.restype = ctypes.c_size_t
    lib.desc_copy2d.argtypes = [vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_size_t,
                                ctypes.c_size_t, vp]
    lib.desc_copy2d.restype = ci
    lib.desc_transpose_host_workspace_batched.argtypes = [i64, i64, i64, ci]
    lib.desc_transpose_host_workspace_batched.restype = ctypes.c_size_t
    lib.desc_copy_batched.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ci, vp]
    lib.desc_copy_batched.restype = ci
    lib.desc_ipc_handle.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
    lib.desc_ipc_handle.restype = ci
    lib.desc_ipc_open.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
    lib.desc_ipc_open.restype = ci
    lib.desc_ipc_close.argtypes = [vp]
    lib.desc_ipc_close.restype = ci
    lib.desc_view_compile.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ViewOp),
                                      ctypes.c_int32, ctypes.POINTER(StridedView)]
    lib.desc_view_compile.restype = ci
    lib.desc_view_copy.argtypes = [vp, vp, ctypes.POINTER(StridedView), ci, vp]
    lib.desc_view_copy.restype = ci
    lib.desc_block_reduce.argtypes = [vp, vp, i64, i64, ci, vp]
    lib.desc_block_reduce.restype = ci
    lib.desc_scan_workspace.argtypes = [i64, ci]
    lib.desc_scan_workspace.restype = ctypes.c_size_t
    lib.desc_scan.argtypes = [vp, vp, i64, ci, vp, ctypes.c_size_t, vp]
    lib.desc_scan.restype = ci
    lib.desc_scan_ex.argtypes = [vp, vp, i64, ci, vp, ctypes.c_size_t, ci, vp]
    lib.desc_scan_ex.restype = ci
    lib.desc_slab_transpose_peer.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                             ctypes.c_int32, i64, i64, ci, vp]
    lib.desc_slab_transpose_peer.restype = ci
    lib.desc_read_probe.argtypes = [vp, ctypes.c_size_t, vp, vp]
    lib.desc_read_probe.restype = ci
    lib.desc_read_probe_sink_bytes.argtypes = []
    lib.desc_read_probe_sink_bytes.restype = ctypes.c_size_t
    lib.desc_last_launch_count.argtypes = []
    lib.desc_last_launch_count.restype = ci
    lib.desc_status_string.argtypes = [ci]
    lib.desc_status_string.restype = ctypes.c_char_p
    lib.desc_last_error.argtypes = []
    lib.desc_last_error.restype = ctypes.c_char_p
    lib.desc_dtype_size.argtypes = [ci]
    lib.desc_dtype_size.restype = ctypes.c_size_t
    lib.desc_version.argtypes = []
    lib.desc_version.restype = ci
    _lib = lib
    return lib


def _check(status: int) -> int:
    if status != 0:
        raise DescError(status, load().desc_last_error().decode())
    return status


# ---- raw C-ABI wrappers (same names as the header) --------------------------------
def desc_transpose(in_ptr, out_ptr, rows, cols, ld_in, ld_out, dtype, stream=0):
    return _check(load().desc_transpose(in_ptr, out_ptr, rows, cols, ld_in, ld_out,
                                        _dt(dtype), stream))


def desc_transpose_batched(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out, stride_in,
                           stride_out, dtype, stream=0):
    return _check(load().desc_transpose_batched(in_ptr, out_ptr, batch, rows, cols, ld_in,
                                                ld_out, stride_in, stride_out, _dt(dtype),
                                                stream))


def desc_transpose_ex(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                      dtype, kernel="auto", stream=0):
    return _check(load().desc_transpose_ex(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out,
                                           stride_in, stride_out, _dt(dtype), _kn(kernel),
                                           stream))


def desc_select_kernel(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out, stride_in,
                       stride_out, dtype) -> str:
    k = load().desc_select_kernel(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out,
                                  stride_in, stride_out, _dt(dtype))
    return KERNEL_NAME[k]


def desc_transpose_host(h_in_ptr, h_out_ptr, batch, rows, cols, ld_in, ld_out, stride_in,
                        stride_out, dtype, d_work_ptr, work_bytes, stream=0):
    return _check(load().desc_transpose_host(h_in_ptr, h_out_ptr, batch, rows, cols, ld_in,
                                             ld_out, stride_in, stride_out, _dt(dtype),
                                             d_work_ptr, work_bytes, stream))


def desc_transpose_host_workspace(rows, cols, dtype) -> int:
    return load().desc_transpose_host_workspace(rows, cols, _dt(dtype))


def desc_copy2d(dst, dpitch, src, spitch, width, height, stream=0):
    """2-D copy of `height` rows of `width` bytes (host <-> device or device <-> device)."""
    return _check(load().desc_copy2d(dst, dpitch, src, spitch, width, height, stream))


def desc_transpose_host_workspace_batched(batch, rows, cols, dtype) -> int:
    return load().desc_transpose_host_workspace_batched(batch, rows, cols, _dt(dtype))


def desc_copy_batched(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                      dtype, stream=0):
    return _check(load().desc_copy_batched(in_ptr, out_ptr, batch, rows, cols, ld_in, ld_out,
                                           stride_in, stride_out, _dt(dtype), stream))


def desc_view_compile(shape, ops, strides=None) -> StridedView:
    """Compile a view chain [(kind, k, depth), ...] over a root of `shape` (element
    `strides`, default C-contiguous) into a strided view (host only)."""
    nd = len(shape)
    sh = (ctypes.c_int64 * max(nd, 1))(*shape)
    st = (ctypes.c_int64 * max(nd, 1))(*strides) if strides is not None else None
    arr = (ViewOp * max(len(ops), 1))(*[ViewOp(VIEW_KIND[k], d, n) for k, n, d in ops])
    out = StridedView()
    _check(load().desc_view_compile(nd, sh, st, arr, len(ops), ctypes.byref(out)))
    return out


def desc_view_copy(in_ptr, out_ptr, view: StridedView, dtype, stream=0):
    return _check(load().desc_view_copy(in_ptr, out_ptr, ctypes.byref(view), _dt(dtype), stream))


def view_copy(x, ops, out=None):
    """Materialise the view chain `ops` of the CUDA tensor x (its own strides are the root's
    layout): returns a contiguous tensor of the view's shape."""
    import torch
    v = desc_view_compile(tuple(x.shape), ops, tuple(x.stride()))
    shape = v.dims[0]
    if out is None:
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    if tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous tensor of shape {shape}")
    desc_view_copy(x.data_ptr(), out.data_ptr(), v, x.dtype, _stream_of(x))
    return out


def desc_block_reduce(in_ptr, out_ptr, n, block, dtype, stream=0):
    return _check(load().desc_block_reduce(in_ptr, out_ptr, n, block, _dt(dtype), stream))


def desc_scan_workspace(n, dtype) -> int:
    return load().desc_scan_workspace(n, _dt(dtype))


def desc_scan(in_ptr, out_ptr, n, dtype, d_work_ptr, work_bytes, stream=0):
    return _check(load().desc_scan(in_ptr, out_ptr, n, _dt(dtype), d_work_ptr, work_bytes,
                                   stream))


def desc_scan_ex(in_ptr, out_ptr, n, dtype, d_work_ptr, work_bytes, algo="auto", stream=0):
    return _check(load().desc_scan_ex(in_ptr, out_ptr, n, _dt(dtype), d_work_ptr, work_bytes,
                                      SCAN_ALGO[algo] if isinstance(algo, str) else int(algo),
                                      stream))


def _check_out(out, x, numel: int) -> None:
    """The C ABI takes no output size: a wrong `out` would be written out of bounds."""
    if (not out.is_contiguous() or out.device != x.device or out.dtype != x.dtype
            or out.numel() != numel):
        raise ValueError(f"out must be a contiguous {x.dtype} tensor of {numel} elements "
                         f"on {x.device}")


def block_reduce(x, block: int, out=None):
    """Per-block sums of a contiguous 1-D CUDA tensor (see desc_block_reduce)."""
    import torch
    x = x.reshape(-1)
    nb = -(-x.numel() // block) if block > 0 else 0
    if out is None:
        out = torch.empty(nb, dtype=x.dtype, device=x.device)
    _check_out(out, x, nb)
    desc_block_reduce(x.data_ptr(), out.data_ptr(), x.numel(), block, x.dtype, _stream_of(x))
    return out


def scan(x, out=None, work=None, algo="auto"):
    """Inclusive prefix sum of a contiguous 1-D CUDA tensor (see desc_scan / desc_scan_ex)."""
    import torch
    x = x.reshape(-1)
    if out is None:
        out = torch.empty_like(x)
    _check_out(out, x, x.numel())
    nbytes = desc_scan_workspace(x.numel(), x.dtype)
    if work is None:
        work = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=x.device)
    desc_scan_ex(x.data_ptr(), out.data_ptr(), x.numel(), x.dtype, work.data_ptr(), work.numel(),
                 algo, _stream_of(x))
    return out


def desc_slab_transpose_peer(in_ptr, out_ptrs, r, M, N, dtype, stream=0):
    """One launch: block (r, s)^T of this rank's slab into every out_ptrs[s] (see the header)."""
    P = len(out_ptrs)
    arr = (ctypes.c_void_p * max(P, 1))(*out_ptrs)
    return _check(load().desc_slab_transpose_peer(in_ptr, arr, P, r, M, N, _dt(dtype), stream))


def desc_read_probe(in_ptr, nbytes, sink_ptr, stream=0):
    """Measurement helper: read nbytes at in_ptr (the reduction's read roofline)."""
    return _check(load().desc_read_probe(in_ptr, nbytes, sink_ptr, stream))


def desc_read_probe_sink_bytes() -> int:
    return load().desc_read_probe_sink_bytes()


IPC_HANDLE_BYTES = 64


def desc_ipc_handle(dptr):
    """-> (64-byte handle of the allocation containing dptr, dptr's offset in it)"""
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = ctypes.c_uint64()
    _check(load().desc_ipc_handle(dptr, buf, ctypes.byref(off)))
    return buf.raw, off.value


def desc_ipc_open(handle: bytes) -> int:
    """Map a peer allocation; returns its BASE address (add the exported offset)."""
    if len(handle) != IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be 64 bytes")
    p = ctypes.c_void_p()
    _check(load().desc_ipc_open(handle, ctypes.byref(p)))
    return p.value


def desc_ipc_close(dptr) -> None:
    _check(load().desc_ipc_close(dptr))


def desc_status_string(status: int) -> str:
    return load().desc_status_string(status).decode()


def desc_last_error() -> str:
    return load().desc_last_error().decode()


def desc_dtype_size(dtype) -> int:
    return load().desc_dtype_size(_dt(dtype))


def desc_version() -> int:
    return load().desc_version()


def desc_last_launch_count() -> int:
    return load().desc_last_launch_count()


def _dt(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    if isinstance(dtype, str):
        return DTYPE[dtype]
    return DTYPE[torch_dtype_name(dtype)]


def _kn(kernel) -> int:
    return kernel if isinstance(kernel, int) else KERNEL[kernel]


# ---- torch tensor conveniences -------------------------------------------------------
def torch_dtype_name(dt) -> str:
    import torch
    table = {torch.float32: "f32", torch.float64: "f64", torch.int32: "i32",
             torch.int64: "i64", torch.float16: "f16", torch.bfloat16: "bf16",
             torch.uint8: "u8", torch.int8: "u8", torch.bool: "u8",
             torch.uint32: "i32", torch.uint64: "i64", torch.int16: "f16",
             torch.uint16: "f16"}
    if dt not in table:
        raise DescError(3, f"unsupported torch dtype {dt}")
    return table[dt]


def _stream_of(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def transpose(x, out=None, kernel: str = "auto"):
    """out = x^T for a 2-D CUDA tensor with unit column stride (row pitch = x.stride(0))."""
    import torch
    if x.dim() != 2:
        raise ValueError("transpose expects a 2-D tensor")
    rows, cols = x.shape
    if out is None:
        out = torch.empty((cols, rows), dtype=x.dtype, device=x.device)
    if tuple(out.shape) != (cols, rows) or out.dtype != x.dtype:
        raise ValueError(f"out must be {(cols, rows)} {x.dtype}")
    if rows and cols and (x.stride(1) != 1 or out.stride(1) != 1):
        raise ValueError("tensors need unit stride in the last dimension")
    ld_in = x.stride(0) if rows > 1 else cols
    ld_out = out.stride(0) if cols > 1 else rows
    desc_transpose_ex(x.data_ptr(), out.data_ptr(), 1, rows, cols, ld_in, ld_out, 0, 0,
                      x.dtype, kernel, _stream_of(x))
    return out


def transpose_batched(x, out=None, kernel: str = "auto"):
    """out[b] = x[b]^T for a 3-D CUDA tensor (unit stride in the last dimension)."""
    import torch
    if x.dim() != 3:
        raise ValueError("transpose_batched expects a 3-D tensor")
    batch, rows, cols = x.shape
    if out is None:
        out = torch.empty((batch, cols, rows), dtype=x.dtype, device=x.device)
    if tuple(out.shape) != (batch, cols, rows) or out.dtype != x.dtype:
        raise ValueError(f"out must be {(batch, cols, rows)} {x.dtype}")
    if batch and rows and cols and (x.stride(2) != 1 or out.stride(2) != 1):
        raise ValueError("tensors need unit stride in the last dimension")
    ld_in = x.stride(1) if rows > 1 else cols
    ld_out = out.stride(1) if cols > 1 else rows
    stride_in = x.stride(0) if batch > 1 else 0
    stride_out = out.stride(0) if batch > 1 else 0
    desc_transpose_ex(x.data_ptr(), out.data_ptr(), batch, rows, cols, ld_in, ld_out,
                      stride_in, stride_out, x.dtype, kernel, _stream_of(x))
    return out


def transpose_host(x, out=None, work=None):
    """out = x^T (or per-matrix for 3-D) for CPU tensors (pin them for PCIe overlap),
    streamed through the GPU by desc_transpose_host on the current CUDA stream.
    `work` is an optional uint8 CUDA tensor used as the device workspace."""
    import torch
    if x.device.type != "cpu":
        raise ValueError("transpose_host takes host (CPU) tensors")
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    batch, rows, cols = x3.shape
    if out is None:
        out = torch.empty((batch, cols, rows) if x.dim() == 3 else (cols, rows), dtype=x.dtype,
                          pin_memory=x.is_pinned())
    o3 = out if out.dim() == 3 else out.unsqueeze(0)
    if tuple(o3.shape) != (batch, cols, rows) or out.dtype != x.dtype:
        raise ValueError("out has the wrong shape or dtype")
    if work is None:
        nbytes = desc_transpose_host_workspace_batched(batch, rows, cols, x.dtype)
        work = torch.empty(max(nbytes, 256), dtype=torch.uint8, device="cuda")
    ld_in = x3.stride(1) if rows > 1 else cols
    ld_out = o3.stride(1) if cols > 1 else rows
    stride_in = x3.stride(0) if batch > 1 else 0
    stride_out = o3.stride(0) if batch > 1 else 0
    desc_transpose_host(x3.data_ptr(), o3.data_ptr(), batch, rows, cols, ld_in, ld_out,
                        stride_in, stride_out, x.dtype, work.data_ptr(), work.numel(),
                        torch.cuda.current_stream(work.device).cuda_stream)
    return out
