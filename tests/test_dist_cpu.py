"""Host-side tests of the distributed slab transpose (no GPU): partition math, a fake-ranks
simulation of the exchange, and the real torch.distributed code path at world size 2 and 4
over gloo, with the local steps supplied on the CPU by the ORACLE (test infrastructure) so
that only the exchange logic of paper_2305_03448_b200/dist.py is under test here.  The CUDA
local steps are covered by tests/test_gpu_parity.py and tests/test_dist_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2305_03448_b200 import dist as ddist


def test_layout_math():
    lay = ddist.SlabLayout(65536, 65536, 8, 3)
    assert (lay.Rm, lay.Rn) == (8192, 8192)
    assert lay.in_rows() == (3 * 8192, 4 * 8192) and lay.out_rows(7) == (7 * 8192, 65536)
    assert lay.algorithmic_bytes(4) == 2 * 8192 * 65536 * 4
    assert lay.nvlink_bytes(4) == 8192 * 65536 * 4 * 7 // 8
    with pytest.raises(ValueError):
        ddist.SlabLayout(100, 64, 8, 0)       # R13: P must divide both dimensions
    with pytest.raises(ValueError):
        ddist.SlabLayout(64, 64, 4, 4)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(64, 64), (32, 96), (128, 40)])
def test_fake_ranks_exchange(P, shape):
    """The three steps of slab_transpose simulated with P numpy ranks and an in-memory
    all-to-all reproduce the oracle's global transpose, slab by slab."""
    M, N = shape
    if M % P or N % P:
        pytest.skip("P must divide M and N")
    A = synth.random_bits((M, N), 4, M * N + P)
    Rm, Rn = M // P, N // P
    sends = [oracle.transpose(A[r * Rm:(r + 1) * Rm]) for r in range(P)]        # step 1
    recvs = [np.stack([sends[s][r * Rn:(r + 1) * Rn] for s in range(P)]) for r in range(P)]
    for r in range(P):                                                            # step 3
        out = np.empty((Rn, M), dtype=A.dtype)
        for s in range(P):
            out[:, s * Rm:(s + 1) * Rm] = recvs[r][s]
        assert out.tobytes() == oracle.dist_expected_slab(A, r, P).tobytes()


@pytest.mark.parametrize("P,C", [(2, 1), (2, 2), (4, 4), (8, 2)])
def test_fake_ranks_chunked_exchange(P, C):
    """The pipelined variant (C row chunks per slab, an all-to-all per chunk) simulated with P
    numpy ranks: chunk k of rank s lands at out_r[:, s*Rm + k*c : s*Rm + (k+1)*c]."""
    M, N = 64 * P, 48 * P
    A = synth.random_bits((M, N), 4, 77 + P * C)
    Rm, Rn = M // P, N // P
    c = Rm // C
    outs = [np.empty((Rn, M), dtype=A.dtype) for _ in range(P)]
    for k in range(C):
        sends = [oracle.transpose(A[r * Rm + k * c:r * Rm + (k + 1) * c]) for r in range(P)]
        for r in range(P):
            for s in range(P):
                outs[r][:, s * Rm + k * c:s * Rm + (k + 1) * c] = sends[s][r * Rn:(r + 1) * Rn]
    for r in range(P):
        assert outs[r].tobytes() == oracle.dist_expected_slab(A, r, P).tobytes()


def test_default_chunks_and_bad_chunks():
    assert ddist.default_chunks(8192, 8) == 4 and ddist.default_chunks(8192, 1) == 1
    assert ddist.default_chunks(256, 2) == 2 and ddist.default_chunks(100, 2) == 1
    x = torch.zeros((6, 8), dtype=torch.int32)
    with pytest.raises(ValueError):    # P = 1 without explicit chunks: no exchange, shape still checked
        ddist.slab_transpose(x, torch.zeros((6, 6), dtype=torch.int32))


def test_fake_ranks_column_chunked_host_pipeline():
    """The host-buffer pipeline's exchange (dist.slab_transpose_host) restated on the CPU with
    fake ranks: chunk k = columns [s*Rn + k*d, +d) of every block s; each block's sub-block is
    transposed into the send buffer, exchanged, and unpacked as output rows [k*d, +d) of the
    receiver, columns q*Rm.. from source q.  Every chunk count must rebuild every rank's
    output slab exactly (oracle.dist_expected_slab)."""
    P, M, N = 4, 64, 96
    A = synth.random_bits((M, N), 4, 77)
    Rm, Rn = M // P, N // P
    for C in (1, 2, 3, 6):
        d = Rn // C
        outs = [np.zeros((Rn, M), dtype=A.dtype) for _ in range(P)]
        for k in range(C):
            # rank q's send buffer: P pieces (d x Rm), piece s = its block (q, s) sub-block^T
            sends = [[oracle.transpose(A[q * Rm:(q + 1) * Rm, s * Rn + k * d:s * Rn + (k + 1) * d])
                      for s in range(P)] for q in range(P)]
            for s in range(P):             # receiver s gets piece s from every source q
                for q in range(P):
                    outs[s][k * d:(k + 1) * d, q * Rm:(q + 1) * Rm] = sends[q][s]
        for r in range(P):
            assert outs[r].tobytes() == oracle.dist_expected_slab(A, r, P).tobytes(), (C, r)


def test_default_host_chunks():
    """Most chunks (16, 8, 4, 2) dividing the block width with >= 2 KB strided H2D rows."""
    assert ddist.default_host_chunks(16384, 4) == 16     # 1024 cells = 4 KB rows
    assert ddist.default_host_chunks(2048, 4) == 4       # 512 cells = 2 KB
    assert ddist.default_host_chunks(1000, 4) == 1       # no divisor keeps 2 KB rows
    assert ddist.default_host_chunks(8192, 8) == 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cpu_transpose(src, dst):           # oracle-backed local step (test only)
    dst.copy_(torch.from_numpy(oracle.transpose(src.numpy())))


def _cpu_unpack(recv, out, P, Rn, c, M, col0=0, Rm=None):
    Rm = c if Rm is None else Rm
    for s in range(P):
        out[:, s * Rm + col0:s * Rm + col0 + c] = recv[s]


def _worker(rank, world, port, M, N, q, chunks=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.random_bits((M, N), 4, 1234)         # every rank can build the global input
        Rm = M // world
        slab = torch.from_numpy(A[rank * Rm:(rank + 1) * Rm].view(np.int32).copy())
        exp = oracle.dist_expected_slab(A, rank, world).tobytes()
        ok = True
        for C in ([chunks] if chunks is not None else [None, 1, 2, 4]):
            out = ddist.slab_transpose(slab, local_transpose=_cpu_transpose,
                                       local_copy=_cpu_unpack, chunks=C)
            ok &= out.numpy().view(np.uint32).tobytes() == exp
        q.put((rank, ok))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,M,N", [(1, 64, 96), (2, 64, 96), (4, 128, 64), (2, 1024, 256)])
def test_gloo_slab_transpose(world, M, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}
