"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, byte for byte.

Bit-exact is the only bar (R14: a transpose moves bits, no tolerance).
Every kernel variant reachable by dispatch is run, plus each variant forced.  Outputs
live inside guard bands and padded rows filled with a sentinel, which must survive.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2305_03448_b200 as desc
from paper_2305_03448_b200 import build as desc_build

pytestmark = pytest.mark.gpu
ROOT_DIR = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GUARD = 4096  # bytes of sentinel before and after every output buffer
SENT = 0xA5


@pytest.fixture(scope="module", autouse=True)
def _lib():
    desc_build.build()
    desc.load()
    torch.cuda.set_device(0)


DT_OF_ES = {1: "u8", 2: "f16", 4: "f32", 8: "f64"}
TORCH_INT = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
NP_INT = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def _to_dev_bytes(a: np.ndarray, extra_front: int = 0) -> torch.Tensor:
    """Copy raw bytes of `a` to a fresh uint8 device buffer at byte offset extra_front
    (the buffer base itself is 256-byte aligned)."""
    raw = np.frombuffer(a.tobytes(), dtype=np.uint8)
    buf = torch.empty(raw.size + extra_front + 64, dtype=torch.uint8, device="cuda")
    buf[extra_front:extra_front + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return buf


def run_case(batch, rows, cols, es, kernel="auto", ld_in=None, ld_out=None, stride_in=None,
             stride_out=None, in_off=0, out_off=0, src=None, check=True):
    """Transpose a seeded input through desc_transpose_ex and compare with the oracle.
    Returns the kernel AUTO would select."""
    ld_in = cols if ld_in is None else ld_in
    ld_out = rows if ld_out is None else ld_out
    stride_in = rows * ld_in if stride_in is None else stride_in
    stride_out = cols * ld_out if stride_out is None else stride_out
    ut = synth.UINT_OF_SIZE[es]
    n_in = (batch - 1) * stride_in + (rows - 1) * ld_in + cols if batch and rows and cols else 0
    n_out = (batch - 1) * stride_out + (cols - 1) * ld_out + rows if batch and rows and cols else 0
    inbuf = synth.random_bits((max(n_in, 1),), es, 1234 + rows * 7 + cols)  # padding = noise
    if src is None:
        if synth.nbits(cols) + synth.nbits(rows) + (synth.nbits(batch) if batch > 1 else 0) <= 8 * es:
            src = synth.self_describing(batch, rows, cols, es)
        else:
            src = synth.with_specials(synth.random_bits((batch, rows, cols), es, 77 + rows), es, 3)
    for b in range(batch):
        for i in range(rows):
            base = b * stride_in + i * ld_in
            inbuf[base:base + cols] = src[b, i]
    d_in = _to_dev_bytes(inbuf, in_off)
    out_bytes = max(n_out, 1) * es
    d_out = torch.full((GUARD + out_bytes + GUARD + out_off,), SENT, dtype=torch.uint8, device="cuda")
    p_in = d_in.data_ptr() + in_off
    p_out = d_out.data_ptr() + GUARD + out_off
    sel = desc.desc_select_kernel(p_in, p_out, batch, rows, cols, ld_in, ld_out, stride_in,
                                  stride_out, DT_OF_ES[es])
    desc.desc_transpose_ex(p_in, p_out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                           DT_OF_ES[es], kernel, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    if not check:
        return sel
    host = d_out.cpu().numpy()
    assert (host[:GUARD + out_off] == SENT).all(), "front guard band written"
    assert (host[GUARD + out_off + out_bytes:] == SENT).all(), "back guard band written"
    body = host[GUARD + out_off:GUARD + out_off + out_bytes].view(ut)
    # expected: oracle into a sentinel-filled buffer of the same layout
    exp = np.frombuffer(bytes([SENT]) * out_bytes, dtype=ut).copy()
    if n_out:   # the oracle reads the very same raw input buffer (overlapping inputs too)
        oracle.transpose_raw(inbuf, exp, batch, rows, cols, ld_in, ld_out, stride_in,
                             stride_out, es)
    if body.tobytes() != exp.tobytes():
        bad = np.nonzero(body != exp)[0]
        raise AssertionError(f"{bad.size} mismatching elements, first at flat {bad[:8]}")
    return sel


KERNELS = ["auto", "smem", "tiled", "tma", "tma_st", "tma_tile", "vtiled"]


def _kernels_for(es, rows, cols, ld_in, ld_out):
    ks = ["auto", "smem", "tiled"]
    if (ld_in * es) % 16 == 0 and (ld_out * es) % 16 == 0:
        ks.append("tma")
        if es in (4, 8) and rows * es >= 16:
            ks += ["tma_st", "tma_tile"]
        if rows % (16 // es) == 0 and cols % (16 // es) == 0:
            ks.append("vtiled")
    return ks


# --------------------------------------------------------------- small exhaustive-ish
@pytest.mark.parametrize("es", [4, 8])
def test_small_shapes_all_kernels(es):
    """(rows, cols) over [1,40]^2 (every 3rd) with ld padded to 16-byte multiples so the
    TMA path is eligible; every kernel variant."""
    v = 16 // es
    for rows in range(1, 41, 3):
        for cols in range(1, 41, 3):
            ld_in = -(-cols // v) * v
            ld_out = -(-rows // v) * v
            for k in _kernels_for(es, rows, cols, ld_in, ld_out):
                run_case(1, rows, cols, es, k, ld_in=ld_in, ld_out=ld_out)


@pytest.mark.parametrize("es", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [31, 32, 33, 63, 64, 65, 127, 128, 129])
def test_edge_set(es, n):
    v = 16 // es
    for m in (31, 64, 129, 257):
        for rows, cols in ((n, m), (m, n)):
            ld_in = -(-cols // v) * v
            ld_out = -(-rows // v) * v
            for k in _kernels_for(es, rows, cols, ld_in, ld_out):
                run_case(1, rows, cols, es, k, ld_in=ld_in, ld_out=ld_out)


@pytest.mark.parametrize("es", [4, 8])
def test_tight_ld_odd_shapes_fall_back(es):
    """Tight ld that is not a 16-byte multiple: AUTO must pick the TILED kernel and be exact;
    the paper-schedule SMEM kernel too."""
    assert run_case(1, 67, 131, es) == "tiled"
    assert run_case(1, 3, 5, es) == "tiled"
    run_case(1, 67, 131, es, "smem")
    run_case(1, 130, 197, es, "tiled")


@pytest.mark.parametrize("es", [4, 8])
def test_padded_ld_guard_bands(es):
    """T4: 67x131 with ld_in=136, ld_out=72: padding columns and guard bands untouched."""
    for k in ("auto", "tma", "tma_st", "tma_tile", "smem", "tiled"):
        run_case(1, 67, 131, es, k, ld_in=136, ld_out=72)


@pytest.mark.parametrize("es", [4, 8])
def test_misaligned_base(es):
    """Base offsets that break 16-byte alignment route to the TILED kernel and stay exact."""
    assert run_case(1, 100, 200, es, in_off=es) == "tiled"
    assert run_case(1, 100, 200, es, out_off=es) == "tiled"
    for k in ("tma", "tma_st", "tma_tile"):
        with pytest.raises(desc.DescError, match="DESC_ERR_KERNEL"):
            run_case(1, 100, 200, es, k, in_off=es, check=False)


@pytest.mark.parametrize("es", [4, 8])
def test_batched_odd_strides(es):
    """T7: 7 x (33 x 65) with strides that leave gaps; input strides overlapping allowed."""
    v = 16 // es
    for k in ("auto", "smem", "tiled", "tma", "tma_st", "tma_tile"):
        run_case(7, 33, 65, es, k, ld_in=65 + (-65) % v, ld_out=40, stride_in=33 * 72 + v,
                 stride_out=65 * 40 + 2 * v)
    run_case(5, 20, 24, es, "smem", ld_in=24, ld_out=20, stride_in=24 * 10, stride_out=480)
    run_case(5, 20, 24, es, "tiled", ld_in=24, ld_out=20, stride_in=24 * 10, stride_out=480)
    run_case(3, 70, 99, es, "tiled", ld_in=101, ld_out=71, stride_in=101 * 75, stride_out=71 * 99)


@pytest.mark.parametrize("es", [1, 2, 4, 8])
def test_vtiled_shapes_and_rules(es):
    """DESC_KERNEL_VTILED (16-byte cp.async staging, swizzled tile, register micro-transposes;
    4x4 / 2x2 renaming for 4/8-byte cells, 8x8 / 16x16 byte permutes for 2/1-byte cells):
    ragged edge tiles in both directions, padded ld, batched strides, the BASELINE f64 shapes;
    arguments outside its rules (misaligned base, rows or cols not a multiple of 16/size,
    ld*size not a multiple of 16) are refused with DESC_ERR_KERNEL, never run."""
    v = 16 // es
    for rows, cols in ((17 * v, 33 * v), (4 * v, 65 * v), (65 * v, 4 * v), (v, v), (64, 64),
                       (6 * v, 10 * v), (1008, 1536)):
        run_case(1, rows, cols, es, "vtiled")
    run_case(1, 17 * v, 33 * v, es, "vtiled", ld_in=34 * v, ld_out=18 * v)
    run_case(7, 9 * v, 16 * v, es, "vtiled", ld_in=18 * v, ld_out=10 * v,
             stride_in=9 * v * 18 * v + v, stride_out=16 * v * 10 * v + 2 * v)
    if es == 8:
        run_case(1, 3000, 5000, es, "vtiled")
    for kw in (dict(in_off=es), dict(out_off=es)):
        with pytest.raises(desc.DescError, match="DESC_ERR_KERNEL"):
            run_case(1, 64, 64, es, "vtiled", check=False, **kw)
    for rows, cols, ld_in, ld_out in ((67, 132, 144, 80), (68, 131, 144, 80), (68, 130, 130, 68)):
        if (ld_in * es) % 16 == 0 and (ld_out * es) % 16 == 0 and rows % v == 0 and cols % v == 0:
            continue
        with pytest.raises(desc.DescError, match="DESC_ERR_KERNEL"):
            run_case(1, rows, cols, es, "vtiled", ld_in=ld_in, ld_out=ld_out, check=False)


def test_involution_and_determinism():
    x = torch.from_numpy(synth.random_bits((1000, 1536), 4, 3).view(np.int32)).cuda()
    y1 = desc.transpose(x)
    y2 = desc.transpose(x)
    z = desc.transpose(y1)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(z, x)


@pytest.mark.parametrize("kernel", ["tiled", "tma_st", "tma_tile", "vtiled", "auto"])
def test_pdl_dependent_chain(kernel):
    """Back-to-back launches with programmatic dependent launch, each reading what the
    previous one wrote (no host sync in between): 24 transposes ping-ponging between two
    buffers, a view copy and a block reduction of the result at the end -- every kernel must
    wait for its predecessor (griddepcontrol.wait) before touching memory."""
    a = synth.random_bits((1536, 2560), 4, 21)
    x = torch.from_numpy(a.view(np.int32)).cuda()
    bufs = [x.clone(), torch.empty((2560, 1536), dtype=torch.int32, device="cuda")]
    for k in range(24):
        src, dst = bufs[k % 2], bufs[(k + 1) % 2]
        desc.transpose(src, dst, kernel=kernel)
    v = desc.view_copy(bufs[0], [("transpose", 0, 0), ("reverse", 0, 1)])
    r = desc.block_reduce(bufs[0].view(-1), 4096)
    torch.cuda.synchronize()
    assert bufs[0].cpu().numpy().view(np.uint32).tobytes() == a.tobytes()
    from oracle import views as V
    assert v.cpu().numpy().view(np.uint32).tobytes() == \
        V.materialize(a, [("transpose", 0, 0), ("reverse", 0, 1)]).tobytes()
    assert r.cpu().numpy().tobytes() == oracle.block_reduce(a.view(np.int32).ravel(), 4096).tobytes()


def test_concurrent_streams_and_graph_capture():
    """Dynamically scheduled launches on two streams at once (distinct tile counters), then
    the same launches captured into and replayed from a CUDA graph."""
    a = synth.random_bits((2, 2048, 3072), 4, 11)
    xs = [torch.from_numpy(a[k].view(np.int32)).cuda() for k in range(2)]
    ys = [torch.empty((3072, 2048), dtype=torch.int32, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(5):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                desc.transpose(xs[k], ys[k])
    torch.cuda.synchronize()
    for k in range(2):
        assert ys[k].cpu().numpy().view(np.uint32).tobytes() == oracle.transpose(a[k]).tobytes()
        ys[k].zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=streams[0]):
        for _ in range(3):
            desc.transpose(xs[0], ys[0])
            desc.transpose(xs[1], ys[1])
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for k in range(2):
        assert ys[k].cpu().numpy().view(np.uint32).tobytes() == oracle.transpose(a[k]).tobytes()


def test_per_thread_default_streams_concurrent():
    """Two host threads launching dynamically scheduled TMA-store transposes on the per-thread
    default stream (the same handle, cudaStreamPerThread = 2, in both threads, but two
    different streams): each must get its own tile counter (counters were keyed
    by the handle), so no tile goes missing."""
    import threading
    R, C = 4096, 8192          # >= 16 tiles per CTA: the dynamic scheduler is on
    a = synth.random_bits((2, R, C), 4, 12)
    xs = [torch.from_numpy(a[k].view(np.int32)).cuda() for k in range(2)]
    ys = [torch.zeros((C, R), dtype=torch.int32, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    errs = []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            for _ in range(20):
                desc.desc_transpose_ex(xs[k].data_ptr(), ys[k].data_ptr(), 1, R, C, C, R, 0, 0,
                                       "i32", "tma_st", 2)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for k in range(2):
        assert ys[k].cpu().numpy().view(np.uint32).tobytes() == oracle.transpose(a[k]).tobytes()


def test_tensor_api_dtypes():
    for dt in (torch.float32, torch.float64, torch.int32, torch.int64, torch.float16,
               torch.bfloat16, torch.uint8):
        es = torch.empty(0, dtype=dt).element_size()
        a = synth.random_bits((96, 80), es, 9)
        x = torch.from_numpy(a.view(NP_INT[es])).cuda().view(dt)
        y = desc.transpose(x)
        torch.cuda.synchronize()
        got = y.view(TORCH_INT[es]).cpu().numpy().view(synth.UINT_OF_SIZE[es])
        assert got.tobytes() == oracle.transpose(a).tobytes(), dt


def test_memspace_rejects_host_pointer():
    h = torch.empty((64, 64), dtype=torch.float32).pin_memory()
    d = torch.empty((64, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(desc.DescError, match="DESC_ERR_MEMSPACE"):
        desc.desc_transpose(h.data_ptr(), d.data_ptr(), 64, 64, 64, 64, "f32")
    a = np.zeros(4096, dtype=np.float32)
    with pytest.raises(desc.DescError, match="DESC_ERR_MEMSPACE"):
        desc.desc_transpose(d.data_ptr(), a.ctypes.data, 64, 64, 64, 64, "f32")


def test_empty_is_noop():
    x = torch.empty((0, 17), dtype=torch.float32, device="cuda")
    y = desc.transpose(x)
    assert y.shape == (17, 0) and desc.desc_last_launch_count() == 0


# ------------------------------------------------------------ BASELINE.json configs
def test_config0_64x64_f64():
    for k in KERNELS:
        run_case(1, 64, 64, 8, k)


def test_config1_2048_f64():
    a = synth.random_bits((1, 2048, 2048), 8, synth.BASE_SEED + 1)
    for k in KERNELS:
        run_case(1, 2048, 2048, 8, k, src=a)


def test_config2_8192_f32_and_i32():
    a = synth.random_bits((1, 8192, 8192), 4, synth.BASE_SEED + 2)
    x = torch.from_numpy(a[0].view(np.int32)).cuda()
    ref = oracle.transpose(a[0])
    for k in ("auto", "tma", "tma_st", "tma_tile", "smem", "tiled"):
        for dt in (torch.float32, torch.int32):
            y = desc.transpose(x.view(dt), kernel=k)
            torch.cuda.synchronize()
            assert y.view(torch.int32).cpu().numpy().view(np.uint32).tobytes() == ref.tobytes()


def test_config3_3000x5000_f64_and_misaligned_ld():
    a = synth.random_bits((1, 3000, 5000), 8, synth.BASE_SEED + 3)
    assert run_case(1, 3000, 5000, 8, src=a) == "tiled"
    assert run_case(1, 3000, 5000, 8, ld_in=5001, src=a) == "tiled"
    run_case(1, 3000, 5000, 8, "smem", ld_in=5001, src=a)


def test_config4_batched_256x1024sq_f32():
    """256 x (1024 x 1024) f32: every matrix checked against the oracle (self-describing)."""
    src = synth.self_describing(256, 1024, 1024, 4)
    x = torch.from_numpy(src.view(np.int32)).cuda()
    y = desc.transpose_batched(x)
    torch.cuda.synchronize()
    assert y.cpu().numpy().view(np.uint32).tobytes() == oracle.transpose(src).tobytes()


@pytest.mark.parametrize("kernel", ["auto", "vtiled"])
def test_config5_65536_f32_every_element(kernel):
    """65536 x 65536 f32 (16 GiB in + 16 GiB out, offsets beyond 2^31) in one launch (AUTO,
    and the 16-byte cp.async kernel), hash-filled on device: ALL 2^32 output elements
    compared with the closed form out[j][i] = H(i*N + j) (tests/fullcheck.py), plus 64 x 64
    blocks at the corners and at random places against the oracle itself."""
    from tests.fullcheck import hash_transpose_mismatches
    n = 65536
    seed = synth.BASE_SEED + 5
    x = torch.empty((n, n), dtype=torch.int32, device="cuda")
    synth.hash_fill_torch(x, 0, 0, n, seed, chunk_rows=2048)
    y = torch.empty_like(x)
    desc.transpose(x.view(torch.float32), y.view(torch.float32), kernel=kernel)
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()
    bad, first = hash_transpose_mismatches(y, 0, n, seed, chunk_rows=512)
    assert bad == 0, f"{bad} of 2^32 elements differ, first at out{first}"
    rng = np.random.default_rng(seed)
    picks = [(0, 0), (n - 64, n - 64), (0, n - 64), (n - 64, 0)] + \
        [tuple(int(v) for v in rng.integers(0, n - 64, 2)) for _ in range(4)]
    for i0, j0 in picks:
        ii, jj = np.meshgrid(np.arange(i0, i0 + 64), np.arange(j0, j0 + 64), indexing="ij")
        blk = synth.hash_expected_np(ii, jj, n, seed, 4)           # in[i0:i0+64, j0:j0+64]
        exp = oracle.transpose(blk)                               # -> out[j0:, i0:]
        got = y[j0:j0 + 64, i0:i0 + 64].cpu().numpy().view(np.uint32)
        assert got.tobytes() == exp.tobytes(), (i0, j0)
    del y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kernel", ["auto", "tma_st", "tma_tile", "vtiled"])
def test_involution_full_size(kernel):
    """T6 at the BASELINE sizes: T(T(A)) == A bytewise for 8192^2 f32 and 3000 x 5000 f64."""
    for shape, es, dt in (((8192, 8192), 4, torch.float32), ((3000, 5000), 8, torch.float64)):
        a = synth.with_specials(synth.random_bits(shape, es, 31 + es), es, 5)
        x = torch.from_numpy(a.view(NP_INT[es])).cuda().view(dt)
        z = desc.transpose(desc.transpose(x, kernel=kernel), kernel=kernel)
        torch.cuda.synchronize()
        assert torch.equal(z.view(TORCH_INT[es]), x.view(TORCH_INT[es])), (shape, kernel)


# ------------------------------------------------------------ host-buffer entry point
@pytest.mark.parametrize("pinned", [True, False])
def test_transpose_host_bands(pinned):
    """desc_transpose_host: pinned and pageable host buffers, a workspace small enough to
    force many row bands, ragged shapes, f32 and f64, plus a batched case."""
    for (batch, rows, cols, es) in ((1, 1000, 777, 4), (1, 333, 1024, 8), (3, 130, 257, 4)):
        src = synth.random_bits((batch, rows, cols), es, rows + cols)
        x = torch.from_numpy(src.view(NP_INT[es]))
        if pinned:
            x = x.pin_memory()
        for work_rows in (64, 100000):
            nbytes = desc.desc_transpose_host_workspace(min(rows, work_rows), cols, DT_OF_ES[es])
            work = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            y = desc.transpose_host(x if batch > 1 else x[0], work=work)
            torch.cuda.synchronize()
            assert desc.desc_last_launch_count() >= 1
            got = y.numpy().view(synth.UINT_OF_SIZE[es])
            assert got.tobytes() == oracle.transpose(src if batch > 1 else src[0]).tobytes()


def test_transpose_host_both_band_axes():
    """The host pipeline bands by input columns by default (strided H2D, contiguous D2H) and
    by input rows with DESC_HOST_AXIS=1 (read once per process, hence the subprocess): both
    bit-exact on ragged f32 / f64 shapes with padded pitches and a batch, many bands each."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
import oracle, synth, paper_2305_03448_b200 as desc
for (batch, rows, cols, es, li, lo) in ((1, 1000, 777, 4, 780, 1003), (2, 333, 1024, 8, 1030, 340)):
    src = synth.random_bits((batch, rows, cols), es, rows + cols)
    ut = synth.UINT_OF_SIZE[es]
    hin = torch.zeros((batch, rows, li), dtype=torch.int32 if es == 4 else torch.int64).pin_memory()
    hin.numpy().view(ut)[:, :, :cols] = src
    hout = torch.full((batch, cols, lo), -1, dtype=torch.int32 if es == 4 else torch.int64).pin_memory()
    nbytes = desc.desc_transpose_host_workspace(64, 64, "f32" if es == 4 else "f64")
    work = torch.empty(nbytes * 8, dtype=torch.uint8, device="cuda")
    desc.desc_transpose_host(hin.data_ptr(), hout.data_ptr(), batch, rows, cols, li, lo,
                             rows * li if batch > 1 else 0, cols * lo if batch > 1 else 0,
                             "f32" if es == 4 else "f64", work.data_ptr(), work.numel())
    torch.cuda.synchronize()
    assert desc.desc_last_launch_count() > 2 * batch
    got = hout.numpy().view(ut)
    assert got[:, :, :rows].tobytes() == oracle.transpose(src).tobytes()
    assert (hout.numpy()[:, :, rows:] == -1).all()
print("ok")
""" % ROOT_DIR
    for axis in ("0", "1", "2"):
        env = dict(os.environ, DESC_HOST_AXIS=axis)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0 and "ok" in p.stdout, (axis, p.stderr[-2000:])


def test_transpose_host_zero_copy_many_bands():
    """> 64 bands with pinned (mapped) host buffers: one TILED launch over PCIe reads and
    writes the host buffers directly; pageable buffers keep the banded copy pipeline.  The
    output has padded rows (ld_out > rows), so the batch-band path (tight outputs only) does
    not apply, and the padding must survive."""
    src = synth.random_bits((80, 70, 50), 4, 123)
    for pinned in (True, False):
        x = torch.from_numpy(src.view(np.int32))
        big = torch.full((80, 50, 72), -1, dtype=torch.int32)
        if pinned:
            x, big = x.pin_memory(), big.pin_memory()
        nbytes = desc.desc_transpose_host_workspace(64, 50, "i32")
        work = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        desc.transpose_host(x, out=big[:, :, :70], work=work)
        torch.cuda.synchronize()
        assert desc.desc_last_launch_count() == (1 if pinned else 160)
        got = big.numpy()
        assert got[:, :, :70].view(np.uint32).tobytes() == oracle.transpose(src).tobytes()
        assert (got[:, :, 70:] == -1).all()


@pytest.mark.parametrize("pinned", [True, False])
def test_transpose_host_batch_bands(pinned):
    """Matrices stored back to back with a tight output travel whole: each band is a group of
    consecutive matrices -- one contiguous H2D copy, one batched transpose, one contiguous D2H
    copy; also with a padded input pitch (the last row's padding may lie past the buffer)."""
    # (the default workspace holds one whole tight matrix when cols <= 1024; a padded pitch or
    # a larger matrix falls back to column bands -- parity either way)
    for (batch, rows, cols, ld_in, whole) in ((80, 70, 50, 50, True), (33, 64, 96, 96, True),
                                              (33, 64, 96, 100, False),
                                              (9, 1000, 1536, 1536, False)):
        full = synth.random_bits((batch, rows, ld_in), 4, batch + rows)
        src = full[:, :, :cols]
        flat = full.reshape(-1)[:(batch * rows - 1) * ld_in + cols].copy()   # ends at the last cell
        x = torch.from_numpy(flat.view(np.int32))
        out = torch.empty((batch, cols, rows), dtype=torch.int32)
        if pinned:
            x, out = x.pin_memory(), out.pin_memory()
        nbytes = desc.desc_transpose_host_workspace(rows, cols, "i32")
        work = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        desc.desc_transpose_host(x.data_ptr(), out.data_ptr(), batch, rows, cols, ld_in, rows,
                                 rows * ld_in, cols * rows, "i32", work.data_ptr(), nbytes,
                                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        n = desc.desc_last_launch_count()
        if whole:
            assert min(batch, 8) <= n <= batch, n
        assert out.numpy().view(np.uint32).tobytes() == oracle.transpose(np.ascontiguousarray(src)).tobytes()


def test_transpose_host_rejects_device_buffers():
    d = torch.empty((64, 64), dtype=torch.float32, device="cuda")
    work = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h = torch.empty((64, 64), dtype=torch.float32)
    with pytest.raises(desc.DescError, match="DESC_ERR_MEMSPACE"):
        desc.desc_transpose_host(d.data_ptr(), h.data_ptr(), 1, 64, 64, 64, 64, 0, 0, "f32",
                                 work.data_ptr(), work.numel())
    with pytest.raises(desc.DescError, match="DESC_ERR_SHAPE"):
        desc.desc_transpose_host(h.data_ptr(), torch.empty_like(h).data_ptr(), 1, 64, 64, 64, 64,
                                 0, 0, "f32", work.data_ptr(), 16)


@pytest.mark.parametrize("kernel", ["auto", "tma", "tma_st", "tma_tile", "vtiled"])
def test_repeated_launches_8192_no_intermittent_mismatch(kernel):
    """Intermittent-race guard (r02): the persistent TMA-load kernel once released its ring
    slot without a proxy fence between its ld.shared reads and the next TMA write -- 1-2 of
    300 launches of 8192^2 f32 had wrong elements (profiles/r02_tma_release_race.txt).  300
    launches per kernel, random and self-describing inputs, each output compared on the
    device with the definition (torch's transposed view as the checker)."""
    n = 8192
    a = synth.random_bits((n, n), 4, synth.BASE_SEED + 2)
    srcs = [torch.from_numpy(a.view(np.int32)).cuda(),
            torch.arange(n * n, dtype=torch.int64, device="cuda").view(n, n).to(torch.int32)]
    refs = [s.t().contiguous() for s in srcs]
    y = torch.empty_like(srcs[0])
    bad = []
    for it in range(150):
        for s, r in zip(srcs, refs):
            y.fill_(-0x5A5A5A5B)
            desc.transpose(s.view(torch.float32), y.view(torch.float32), kernel=kernel)
            cnt = int((y != r).sum())
            if cnt:
                bad.append((it, cnt))
    assert not bad, f"{kernel}: launches with mismatching elements (iteration, count): {bad[:5]}"


def test_transpose_host_two_threads():
    """Two host threads calling desc_transpose_host at once on their own CUDA streams: the
    per-device internal streams and join events are shared, so each call's enqueue is
    serialised (HostPipe::enqueue); both results must be exact, every time."""
    import threading
    srcs = [synth.random_bits((1000, 1536), 4, 40 + k) for k in range(2)]
    errs = []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            x = torch.from_numpy(srcs[k].view(np.int32)).pin_memory()
            work = torch.empty(desc.desc_transpose_host_workspace(1000, 1536, "i32"),
                               dtype=torch.uint8, device="cuda")
            for it in range(20):
                out = torch.full((1536, 1000), -1, dtype=torch.int32).pin_memory()
                desc.desc_transpose_host(x.data_ptr(), out.data_ptr(), 1, 1000, 1536, 1536, 1000,
                                         0, 0, "i32", work.data_ptr(), work.numel(), s.cuda_stream)
                s.synchronize()
                if out.numpy().view(np.uint32).tobytes() != oracle.transpose(srcs[k]).tobytes():
                    errs.append((k, it))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
