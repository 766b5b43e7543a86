"""GPU parity of the block-wide reduction and the single-pass scan (C ABI) against the oracle
(oracle/reduce_scan_ref.c): integers bit-exact (sums mod 2^bits); floats within the bound the
arithmetic gives -- |gpu - oracle| <= ulp_out(|oracle|) (f32 output rounding) +
2 * m * 2^-53 * sum|x| (two fp64 summation orders over m terms)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2305_03448_b200 as desc

pytestmark = pytest.mark.gpu

INTS = (np.uint8, np.int32, np.int64)
FLOATS = (np.float32, np.float64)
TORCH = {np.uint8: torch.uint8, np.int32: torch.int32, np.int64: torch.int64,
         np.float32: torch.float32, np.float64: torch.float64}


def _input(n, dt, seed):
    if dt in INTS:
        return synth.random_ints(n, dt, seed)
    return synth.random_floats(n, dt, seed)


def _dev(a, offset):
    """Device copy of `a` starting `offset` elements into a fresh allocation (misalignment)."""
    t = torch.empty(a.size + offset + 16, dtype=TORCH[a.dtype.type], device="cuda")
    t[offset:offset + a.size] = torch.from_numpy(a).cuda()
    return t[offset:offset + a.size]


def _ulp(dt, ref):
    if dt == np.float32:
        return np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    return np.zeros_like(ref)


@pytest.mark.parametrize("dt", INTS + FLOATS)
@pytest.mark.parametrize("n,B", [(1, 1), (1000, 1), (1000, 3), (12345, 16), (12345, 64),
                                 (100000, 65), (100000, 1000), (1 << 20, 1024),
                                 (300000, 16384), (300000, 16385), (1000003, 100000),
                                 (50, 1000),
                                 # 1 … 16 vectors per block (segmented warp rows; a
                                 # partial last row; 3 vectors per block falls back)
                                 (64 * 5000, 64), (16 * 777, 16), (8 * 1001, 8), (4 * 999, 4),
                                 (32 * 4099, 32), (12 * 1000, 12),
                                 # whole 512-byte warp rows per block (1, 2, 4 rows; K-block
                                 # groups plus a remainder of blocks)
                                 (128 * 1000 + 128 * 7, 128), (256 * 5003, 256), (512 * 77, 512),
                                 (2048 * 33, 2048), (1024 * 301, 1024), (4000 * 300 + 7, 4000),
                                 # 3, 5, 6 … warp rows per block (not a power of two:
                                 # the warp-per-block kernel)
                                 (384 * 1000, 384), (192 * 1001, 192), (1536 * 77, 1536),
                                 (640 * 313, 640), (768 * 100, 768), (1920 * 41, 1920),
                                 # fewer blocks than CTA slots: cluster per block (ragged,
                                 # near-empty last block; more blocks than clusters)
                                 ((1 << 22) + 17, 1 << 20), (2000000, 20000),
                                 ((1 << 24) + 5, 20000), ((1 << 24) + 3, 1 << 22)])
def test_block_reduce(dt, n, B):
    for offset in (0, 1):
        a = _input(n, dt, n + B + offset)
        x = _dev(a, offset)
        y = desc.block_reduce(x, B)
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        ref = oracle.block_reduce(a, B)
        assert got.shape == ref.shape
        if dt in INTS:
            assert got.tobytes() == ref.tobytes(), (n, B, offset)
        else:
            absx = oracle.block_reduce(np.abs(a).astype(np.float64), B)
            m = np.minimum(B, n - np.arange(ref.size) * B)
            tol = _ulp(dt, ref) + 2.0 * m * 2.0 ** -53 * absx
            assert np.all(np.abs(got.astype(np.float64) - ref) <= tol), (n, B, offset)


@pytest.mark.parametrize("n,B", [(1 << 20, 16), (1 << 20, 1024), (1 << 20, 5000),
                                 ((1 << 22) + 17, 1 << 20), (2000000, 20000)])
def test_block_reduce_repeats_bitwise(n, B):
    """The summation order is fixed per (n, B, dtype, alignment): no atomics (header claim)."""
    x = _dev(synth.random_floats(n, np.float32, 17), 0)
    first = desc.block_reduce(x, B).cpu().numpy().tobytes()
    for _ in range(3):
        assert desc.block_reduce(x, B).cpu().numpy().tobytes() == first


def _check_scan(got, a, dt, what):
    ref = oracle.scan(a)
    if dt in INTS:
        assert got.tobytes() == ref.tobytes(), what
    else:
        absx = oracle.scan(np.abs(a).astype(np.float64))
        tol = _ulp(dt, ref) + 2.0 * np.arange(1, a.size + 1) * 2.0 ** -53 * absx
        assert np.all(np.abs(got.astype(np.float64) - ref) <= tol), what


@pytest.mark.parametrize("algo", ["auto", "lookback", "three_pass", "stream"])
@pytest.mark.parametrize("dt", INTS + FLOATS)
@pytest.mark.parametrize("n", [1, 15, 255, 4096, 4097, 100003, (1 << 22) + 3])
def test_scan(dt, n, algo):
    for offset in (0, 1):
        a = _input(n, dt, n + offset)
        x = _dev(a, offset)
        misaligned = (x.data_ptr() % 16) != 0
        if algo == "stream" and misaligned:
            with pytest.raises(desc.DescError, match="KERNEL"):
                desc.scan(x, algo=algo)
            continue
        y = desc.scan(x, algo=algo)
        torch.cuda.synchronize()
        _check_scan(y.cpu().numpy(), a, dt, (n, offset, algo))


@pytest.mark.parametrize("dt", INTS + FLOATS)
def test_scan_stream_many_tiles_per_cta(dt):
    """Long enough that every persistent CTA streams several tiles through each stage, with a
    ragged tail (not a multiple of 16 bytes); also the AUTO choice at this size."""
    n = (1 << 25) + 7 if np.dtype(dt).itemsize <= 4 else (1 << 24) + 7
    a = _input(n, dt, 99)
    x = torch.from_numpy(a).cuda()
    for algo in ("stream", "auto"):
        y = desc.scan(x, algo=algo)
        torch.cuda.synchronize()
        assert desc.desc_last_launch_count() == 2      # state reset + the single pass
        _check_scan(y.cpu().numpy(), a, dt, algo)


@pytest.mark.parametrize("algo", ["lookback", "three_pass", "stream"])
def test_scan_f32_special_values(algo):
    """f32 widening to the fp64 accumulator: mixed vectors of +-0, subnormals, the extreme
    normal exponents and ordinary values must still meet the bound; an inf makes every later
    prefix inf, a NaN every later prefix NaN, exactly as in the oracle."""
    n = (1 << 22) + 5
    rng = np.random.default_rng(7)
    a = synth.random_floats(n, np.float32, 8)
    kind = rng.integers(0, 8, n)
    a[kind == 0] = 0.0
    a[kind == 1] = -0.0
    sub = rng.integers(1, 1 << 23, n).astype(np.uint32).view(np.float32)   # subnormals
    a[kind == 2] = sub[kind == 2]
    tiny = np.float32(np.finfo(np.float32).tiny)
    a[kind == 3] = tiny * np.sign(rng.standard_normal(n)[kind == 3]).astype(np.float32)
    a[kind == 4] = np.float32(1e30) * np.sign(rng.standard_normal(n)[kind == 4]).astype(np.float32)
    x = torch.from_numpy(a).cuda()
    y = desc.scan(x, algo=algo)
    torch.cuda.synchronize()
    _check_scan(y.cpu().numpy(), a, np.float32, algo)
    for special in (np.inf, np.nan):
        b = a.copy()
        k = n // 3 + 1
        b[k] = special
        y = desc.scan(torch.from_numpy(b).cuda(), algo=algo).cpu().numpy()
        ref = oracle.scan(b)
        assert np.all(np.isfinite(y[:k])) and np.isnan(ref[k:]).any() == np.isnan(special)
        if np.isnan(special):
            assert np.all(np.isnan(y[k:]))
        else:   # +inf plus finite terms below the f32 overflow stays +inf
            assert np.array_equal(np.isinf(y[k:]), np.isinf(ref[k:].astype(np.float32)))
        _check_scan(y[:k], b[:k], np.float32, (algo, special))


def test_scan_in_place_and_repeat():
    a = synth.random_ints(1 << 20, np.int32, 4)
    x = torch.from_numpy(a).cuda()
    work = torch.empty(desc.desc_scan_workspace(a.size, "i32"), dtype=torch.uint8, device="cuda")
    for algo in ("auto", "lookback", "three_pass", "stream"):
        for _ in range(3):      # workspace reused: the call re-zeroes the tile state
            y = desc.scan(x, work=work, algo=algo)
    for algo in ("lookback", "three_pass", "stream"):
        z = x.clone()
        desc.scan(z, out=z, work=work, algo=algo)   # in place
        torch.cuda.synchronize()
        assert z.cpu().numpy().tobytes() == oracle.scan(a).tobytes(), algo
    desc.scan(x, out=x, work=work)     # in place
    torch.cuda.synchronize()
    assert x.cpu().numpy().tobytes() == oracle.scan(a).tobytes()
    assert y.cpu().numpy().tobytes() == oracle.scan(a).tobytes()


def test_errors():
    x = torch.zeros(100, dtype=torch.float16, device="cuda")
    with pytest.raises(desc.DescError, match="DTYPE"):
        desc.block_reduce(x, 10)
    y = torch.zeros(100, dtype=torch.float32, device="cuda")
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_block_reduce(y.data_ptr(), y.data_ptr(), 100, 0, "f32")
    work = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.scan(y, work=work)
    with pytest.raises(desc.DescError, match="ALIAS"):
        desc.desc_scan(y.data_ptr(), y.data_ptr() + 4, 50, "f32", work.data_ptr(), 1 << 20)
    big = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(desc.DescError, match="KERNEL"):
        desc.desc_scan_ex(y.data_ptr(), y.data_ptr(), 100, "f32", big.data_ptr(), 1 << 20, 9)


def test_read_probe_reads_every_byte():
    """desc_read_probe (the reduction's read-roofline helper): the XOR of the per-CTA sink words
    equals the XOR of every 16-byte word of the input, so every byte was loaded."""
    for nbytes in (16, 16 * 1001, 1 << 24):
        a = synth.random_bits((nbytes // 4,), 4, nbytes).view(np.int32)
        x = torch.from_numpy(a).cuda()
        sink = torch.zeros(desc.desc_read_probe_sink_bytes(), dtype=torch.uint8, device="cuda")
        desc.desc_read_probe(x.data_ptr(), nbytes, sink.data_ptr())
        torch.cuda.synchronize()
        got = np.bitwise_xor.reduce(sink.cpu().numpy().view(np.uint32).reshape(-1, 4), axis=0)
        exp = np.bitwise_xor.reduce(a.view(np.uint32).reshape(-1, 4), axis=0)
        assert got.tobytes() == exp.tobytes(), nbytes
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_read_probe(x.data_ptr() + 4, 16, sink.data_ptr())
