"""Distributed transpose of a row-slab-sharded matrix across the GPUs of one node.

BASELINE.json north_star (4) / SURVEY.md §8(a) a9, §8(e).  The paper has no multi-GPU
content; this is the build's extension of the transpose (reading R13):

  global input A is M x N, rank r of P owns input rows  [r*Rm, (r+1)*Rm),  Rm = M / P
  global output A^T is N x M, rank r owns output rows   [r*Rn, (r+1)*Rn),  Rn = N / P
  block (r, s) = A[r*Rm:(r+1)*Rm, s*Rn:(s+1)*Rn] travels to rank s, transposed, and lands
  at out_s[:, r*Rm:(r+1)*Rm].

Two implementations:

* ``slab_transpose`` -- NCCL path (the baseline the north star names):
    1. local transpose of the whole slab (desc kernel): T_r = in_r^T is N x Rm, and its row
       band s (rows s*Rn..) is exactly block (r, s)^T, contiguous -> the all-to-all send buffer;
    2. ``all_to_all_single`` over NCCL (NVLink 5 / NVSwitch);
    3. unpack: the P received Rn x Rm blocks are placed side by side in out_r with
       ``desc_copy_batched`` (pitch M).
  Per-rank HBM traffic ~6 S (S = slab bytes), NVLink S (P-1)/P each direction.  The three
  steps are pipelined over C row chunks of the slab so that the all-to-all (NVLink-bound)
  overlaps the local passes (HBM-bound).

* ``PeerSlabTranspose`` -- fused peer-to-peer path: every rank maps the
  other ranks' output slabs with CUDA IPC once; a call is ONE launch
  (desc_slab_transpose_peer): TILED tiles (plain coalesced loads of local HBM, 128-byte warp
  stores, over NVLink for the other GPUs' slabs; no tensor map ever addresses peer memory)
  that each pick their destination slab, writing block (r, s)^T straight into out_s (shapes
  the fused kernel cannot tile fall back to one launch per destination): one pass, no
  pack/unpack, no NCCL kernels: HBM 2 S per rank (read local S, the writes of S
  land in the peers' HBM), NVLink S (P-1)/P.  A group barrier after the kernels orders the
  writes before anyone reads its slab.

``slab_transpose_host`` is the NCCL path from and to pinned HOST buffers with the PCIe copies
inside the pipeline (column chunks: strided H2D, contiguous D2H; bench.py's N > 1 e2e).

The local steps are injectable (``local_transpose``/``local_copy``) only so the exchange
logic can be tested on CPU with the gloo backend (tests/test_dist_cpu.py); the product
default is the CUDA library, and CUDA tensors are required.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

import paper_2305_03448_b200 as desc


@dataclass(frozen=True)
class SlabLayout:
    M: int          # global rows of the input
    N: int          # global cols of the input
    P: int          # ranks
    r: int          # this rank

    def __post_init__(self):
        if self.P < 1 or not (0 <= self.r < self.P):
            raise ValueError("bad rank / world size")
        if self.M % self.P or self.N % self.P:
            raise ValueError(f"M={self.M} and N={self.N} must both divide by P={self.P} (R13)")

    @property
    def Rm(self) -> int:
        return self.M // self.P

    @property
    def Rn(self) -> int:
        return self.N // self.P

    def in_rows(self, r=None):
        r = self.r if r is None else r
        return r * self.Rm, (r + 1) * self.Rm

    def out_rows(self, r=None):
        r = self.r if r is None else r
        return r * self.Rn, (r + 1) * self.Rn

    def algorithmic_bytes(self, es: int) -> int:
        """Bytes the method must move per rank: read the slab, write the slab."""
        return 2 * self.Rm * self.N * es

    def nvlink_bytes(self, es: int) -> int:
        """Bytes per rank that must cross NVLink in each direction: S (P-1)/P."""
        return self.Rm * self.N * es * (self.P - 1) // self.P


def _cuda_transpose(src, dst):
    """dst (N x Rm) = src (Rm x N)^T with the desc kernels."""
    desc.transpose(src, dst)


def _cuda_unpack(recv, out, P, Rn, c, M, col0=0, Rm=None):
    """out[:, s*Rm + col0 : s*Rm + col0 + c] = recv[s] for s < P  (recv: P x Rn x c contiguous;
    Rm defaults to c, i.e. the unchunked exchange)."""
    Rm = c if Rm is None else Rm
    es = out.element_size()
    desc.desc_copy_batched(recv.data_ptr(), out.data_ptr() + col0 * es, P, Rn, c, c, M, Rn * c,
                           Rm, recv.dtype, torch.cuda.current_stream(recv.device).cuda_stream)


def default_chunks(Rm: int, P: int) -> int:
    """Pipeline depth of the NCCL path: 4 chunks of >= 128 slab rows when they divide Rm."""
    if P == 1:
        return 1
    for C in (4, 2):
        if Rm % C == 0 and Rm // C >= 128:
            return C
    return 1


def default_host_chunks(Rn: int, es: int) -> int:
    """Pipeline depth of the host-buffer path: the most chunks (16, 8, 4, 2) that divide the
    block width Rn and keep each block's strided H2D rows >= 2 KB
    (profiles/r02_exp_slab_host.txt)."""
    for C in (16, 8, 4, 2):
        if Rn % C == 0 and (Rn // C) * es >= 2048:
            return C
    return 1


def slab_transpose(in_slab: torch.Tensor, out_slab: torch.Tensor | None = None, group=None,
                   local_transpose=None, local_copy=None, workspace=None, chunks=None,
                   all_to_all=None):
    """Transpose the global matrix whose row slab this rank holds (NCCL all-to-all path).

    in_slab: (Rm, N) contiguous, this rank's rows of the M x N input (M = Rm * P).
    returns out_slab: (Rn, M), this rank's rows of the N x M transpose (Rn = N / P).
    workspace: optional (send, recv) pair of tensors with N * Rm elements each.
    chunks: C, the pipeline depth (default ``default_chunks``).  The slab is cut into C row
      chunks of c = Rm / C rows; chunk k is transposed into its own send buffer (N x c: its row
      band s is block (r, s)'s chunk, transposed), exchanged with an asynchronous all-to-all,
      and unpacked into out_r[:, s*Rm + k*c : ... + c].  All C transposes are issued first, so
      the all-to-all of chunk k overlaps the transposes of the later chunks and the unpacks of
      the earlier ones (the NCCL collective runs on its own stream); the result does not depend
      on C.
    all_to_all: the exchange primitive (default ``torch.distributed.all_to_all_single``); an
      injection point for the single-GPU multi-process test only.
    With one rank and ``chunks`` left at None the call is a single local transpose; an
    explicit ``chunks`` runs the whole exchange pipeline even then (a one-rank NCCL
    all-to-all is a device copy), so the NCCL code path can be exercised on one GPU."""
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    r = dist.get_rank(group) if dist.is_initialized() else 0
    Rm, N = in_slab.shape
    lay = SlabLayout(Rm * P, N, P, r)
    Rn, M = lay.Rn, lay.M
    if not in_slab.is_contiguous():
        raise ValueError("in_slab must be contiguous")
    if out_slab is None:
        out_slab = torch.empty((Rn, M), dtype=in_slab.dtype, device=in_slab.device)
    if tuple(out_slab.shape) != (Rn, M) or not out_slab.is_contiguous():
        raise ValueError(f"out_slab must be contiguous {(Rn, M)}")
    local_transpose = local_transpose or _cuda_transpose
    local_copy = local_copy or _cuda_unpack
    all_to_all = all_to_all or dist.all_to_all_single
    if P == 1 and chunks is None:
        local_transpose(in_slab, out_slab)
        return out_slab
    C = default_chunks(Rm, P) if chunks is None else int(chunks)
    if C < 1 or Rm % C:
        raise ValueError(f"chunks={C} must divide the slab rows Rm={Rm}")
    c = Rm // C
    if workspace is None:
        send = torch.empty(N * Rm, dtype=in_slab.dtype, device=in_slab.device)
        recv = torch.empty(N * Rm, dtype=in_slab.dtype, device=in_slab.device)
    else:
        send, recv = (w.view(-1) for w in workspace)
        if send.numel() < N * Rm or recv.numel() < N * Rm:
            raise ValueError("workspace tensors need N * Rm elements each")
    works = []
    for k in range(C):
        send_k = send[k * N * c:(k + 1) * N * c]
        recv_k = recv[k * N * c:(k + 1) * N * c]
        local_transpose(in_slab[k * c:(k + 1) * c], send_k.view(N, c))   # band s = (r,s)_k^T
        works.append(all_to_all(recv_k, send_k, group=group, async_op=True))
    for k in range(C):
        works[k].wait()                      # NCCL: the compute stream waits for chunk k only
        recv_k = recv[k * N * c:(k + 1) * N * c].view(P, Rn, c)
        local_copy(recv_k, out_slab, P, Rn, c, M, k * c, Rm)   # out_r[:, s*Rm + k*c ..] = recv_k[s]
    return out_slab


_HOST_STREAMS = {}


def _host_streams(device):
    """(H2D, D2H) side streams of the host-buffer pipeline, one pair per device."""
    key = device.index if device.index is not None else torch.cuda.current_device()
    if key not in _HOST_STREAMS:
        _HOST_STREAMS[key] = (torch.cuda.Stream(device), torch.cuda.Stream(device))
    return _HOST_STREAMS[key]


def slab_transpose_host(h_in: torch.Tensor, h_out: torch.Tensor, in_slab: torch.Tensor,
                        out_slab: torch.Tensor, group=None, workspace=None, chunks=None,
                        all_to_all=None, work=None):
    """``slab_transpose`` from and to HOST memory, with the PCIe copies inside the pipeline.

    h_in: (Rm, N) pinned host tensor, this rank's input rows; h_out: (Rn, M) pinned host
    tensor for this rank's output rows; in_slab / out_slab: device staging of the same shapes
    (workspace / all_to_all as in ``slab_transpose``).  The pipeline runs over C COLUMN chunks
    of every block (d = Rn / C columns of block s = input columns s*Rn + k*d ..): chunk k's
    output is rows [k*d, (k+1)*d) of this rank's output slab -- contiguous on the host -- so
    the H2D copies are 2-D (P stripes of Rm rows x d cells, the direction PCIe handles better,
    DESIGN §7 "band axis") and the D2H copy of each chunk is one contiguous block:
      side stream  : H2D of chunk k (``desc_copy2d``)                    -> event
      compute      : wait chunk k; transpose its P sub-blocks (Rm x d -> d x Rm, one batched
                     launch) into the send buffer; asynchronous all-to-all; then unpack chunk
                     k - 1 (d rows x Rm cells from every source, side by side)  -> event
      third stream : D2H of the unpacked rows of chunk k - 1 (contiguous)
    The caller's current stream waits for the last D2H: asynchronous and stream-ordered like
    the rest of the library.  chunks: C (default ``default_host_chunks``).  One rank without
    ``chunks``: the banded ``desc_transpose_host`` (work: its device workspace)."""
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    r = dist.get_rank(group) if dist.is_initialized() else 0
    Rm, N = in_slab.shape
    lay = SlabLayout(Rm * P, N, P, r)
    Rn, M = lay.Rn, lay.M
    if h_in.is_cuda or h_out.is_cuda:
        raise ValueError("h_in / h_out must be host tensors")
    if tuple(h_in.shape) != (Rm, N) or tuple(h_out.shape) != (Rn, M):
        raise ValueError(f"h_in must be {(Rm, N)} and h_out {(Rn, M)}")
    if not (h_in.is_contiguous() and h_out.is_contiguous() and in_slab.is_contiguous()
            and out_slab.is_contiguous()):
        raise ValueError("h_in, h_out, in_slab and out_slab must be contiguous")
    dev = in_slab.device
    compute = torch.cuda.current_stream(dev)
    if P == 1 and chunks is None:
        if work is None:
            work = torch.empty(desc.desc_transpose_host_workspace(Rm, N, in_slab.dtype),
                               dtype=torch.uint8, device=dev)
        desc.desc_transpose_host(h_in.data_ptr(), h_out.data_ptr(), 1, Rm, N, N, Rm, 0, 0,
                                 in_slab.dtype, work.data_ptr(), work.numel(),
                                 compute.cuda_stream)
        return h_out
    all_to_all = all_to_all or dist.all_to_all_single
    es = in_slab.element_size()
    C = default_host_chunks(Rn, es) if chunks is None else int(chunks)
    if C < 1 or Rn % C:
        raise ValueError(f"chunks={C} must divide the block width Rn={Rn}")
    d = Rn // C
    if workspace is None:
        send = torch.empty(N * Rm, dtype=in_slab.dtype, device=dev)
        recv = torch.empty(N * Rm, dtype=in_slab.dtype, device=dev)
    else:
        send, recv = (w.view(-1) for w in workspace)
        if send.numel() < N * Rm or recv.numel() < N * Rm:
            raise ValueError("workspace tensors need N * Rm elements each")
    h2d, d2h = _host_streams(dev)
    h2d.wait_stream(compute)               # stream order: everything before the call
    d2h.wait_stream(compute)
    landed = []
    for k in range(C):                     # H2D: P stripes of Rm rows x d cells per chunk
        for s_ in range(P):
            off = (s_ * Rn + k * d) * es
            desc.desc_copy2d(in_slab.data_ptr() + off, N * es, h_in.data_ptr() + off, N * es,
                             d * es, Rm, h2d.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(h2d)
        landed.append(ev)
    works = []
    piece = P * d * Rm                     # elements of one chunk's send / recv buffer

    def finish(k):                         # unpack chunk k, then its D2H on the third stream
        works[k].wait()
        # from source rank q: d x Rm cells -> out rows k*d.., columns q*Rm..
        desc.desc_copy_batched(recv.data_ptr() + k * piece * es,
                               out_slab.data_ptr() + k * d * M * es, P, d, Rm, Rm, M, d * Rm,
                               Rm, out_slab.dtype, compute.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(compute)
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            h_out[k * d:(k + 1) * d].copy_(out_slab[k * d:(k + 1) * d], non_blocking=True)

    # compute-stream order: pack k, then unpack k - 1 -- the D2H of chunk k - 1 starts while
    # chunk k + 1 is still arriving (all packs first would hold every D2H back until the last
    # H2D had landed: no overlap, profiles/r02_exp_slab_host.txt)
    for k in range(C):
        compute.wait_event(landed[k])
        send_k = send[k * piece:(k + 1) * piece]
        recv_k = recv[k * piece:(k + 1) * piece]
        # sub-block s (Rm x d at input column s*Rn + k*d) -> send_k[s] = its transpose (d x Rm)
        desc.desc_transpose_batched(in_slab.data_ptr() + k * d * es, send_k.data_ptr(), P, Rm, d,
                                    N, Rm, Rn, d * Rm, in_slab.dtype, compute.cuda_stream)
        works.append(all_to_all(recv_k, send_k, group=group, async_op=True))
        if k >= 1:
            finish(k - 1)
    finish(C - 1)
    compute.wait_stream(d2h)
    return h_out


class PeerSlabTranspose:
    """Fused peer-to-peer slab transpose over CUDA IPC (one kernel pass, no NCCL kernels).

    Construct once per output slab (collective over `group`): it exports this rank's output
    slab and maps every peer's.  ``__call__(in_slab)`` then writes block (r, s)^T straight into
    rank s's slab for every s and finishes with a group barrier (all writes complete before
    any rank reads its slab).  Works with any process-group backend for the handle exchange
    (gloo in the single-GPU two-process test, NCCL in bench.py)."""

    def __init__(self, out_slab: torch.Tensor, M: int, group=None, kernel: str = "auto",
                 remote_kernel: str = "tiled", force_remote: bool = False, fused: bool = True):
        """fused: ONE launch for all destinations (desc_slab_transpose_peer: TILED tiles that
        pick their destination slab) when P <= 8 and N/P is a multiple of the tile width;
        otherwise one launch per destination with
        kernel: for this rank's own block; remote_kernel: for blocks stored into a slab on
        another GPU.  force_remote: treat every peer's slab as remote even when it lives on
        this GPU -- the one-GPU multi-process test then runs exactly the kernel selection a
        multi-GPU run takes."""
        if not out_slab.is_cuda or not out_slab.is_contiguous():
            raise ValueError("out_slab must be a contiguous CUDA tensor")
        self.group = group
        self.P = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.out = out_slab
        self.M = M
        self.kernel = kernel
        Rn = out_slab.shape[0]
        self.lay = SlabLayout(M, Rn * self.P, self.P, self.r)
        handle, offset = desc.desc_ipc_handle(out_slab.data_ptr())
        handles = [None] * self.P
        dist.all_gather_object(handles, (handle, offset, out_slab.device.index), group=group)
        # blocks for a slab on ANOTHER GPU go through the TILED kernel (plain coalesced loads
        # of local HBM, 128-byte warp stores over NVLink; no tensor map ever addresses peer
        # memory); same-device slabs (the one-GPU test) take AUTO
        self.kernels = [kernel if s == self.r or (d == out_slab.device.index and not force_remote)
                        else remote_kernel for s, (_, _, d) in enumerate(handles)]
        es = out_slab.element_size()
        tile_w = 32 if es == 8 else 64
        self.fused = bool(fused and self.P <= 8 and es in (4, 8) and self.lay.Rn % tile_w == 0)
        self.peer_ptr = []
        self._opened = []
        for s, (h, off, _) in enumerate(handles):
            if s == self.r:
                self.peer_ptr.append(out_slab.data_ptr())
            else:
                base = desc.desc_ipc_open(h)          # allocation base in this process
                self.peer_ptr.append(base + off)
                self._opened.append(base)

    def __call__(self, in_slab: torch.Tensor, barrier: bool = True):
        lay = self.lay
        Rm, N = in_slab.shape
        if (Rm, N) != (lay.Rm, lay.N) or not in_slab.is_contiguous():
            raise ValueError(f"in_slab must be contiguous {(lay.Rm, lay.N)}")
        es = in_slab.element_size()
        stream = torch.cuda.current_stream(in_slab.device).cuda_stream
        if barrier:       # every peer finished reading its previous output
            dist.barrier(group=self.group)
        launches = 0
        if self.fused:
            desc.desc_slab_transpose_peer(in_slab.data_ptr(), self.peer_ptr, self.r, lay.M, lay.N,
                                          in_slab.dtype, stream)
            launches = desc.desc_last_launch_count()
        # start with the next rank so that the P writers spread over the P destinations
        for k in range(0 if self.fused else self.P):
            s = (self.r + k) % self.P
            src = in_slab.data_ptr() + s * lay.Rn * es                       # block (r, s)
            dst = self.peer_ptr[s] + self.r * lay.Rm * es                    # out_s[:, r*Rm]
            desc.desc_transpose_ex(src, dst, 1, lay.Rm, lay.Rn, lay.N, lay.M, 0, 0,
                                   in_slab.dtype, self.kernels[s], stream)
            launches += desc.desc_last_launch_count()
        if barrier:
            torch.cuda.current_stream(in_slab.device).synchronize()
            dist.barrier(group=self.group)
        return self.out, launches

    def close(self):
        for p in self._opened:
            desc.desc_ipc_close(p)
        self._opened = []
