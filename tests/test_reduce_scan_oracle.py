"""Pins for the block-reduction and scan oracles (oracle/reduce_scan_ref.c), CPU only:
SPEC's printed value (golden fixture), closed forms, exact big-integer arithmetic
for the wrap-around, math.fsum (exactly rounded) within the fp64 sequential-sum bound,
the scan/reduce consistency invariant, edge cases and mutation teeth."""
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    blocks, cur = {}, None
    for line in open(os.path.join(GOLDEN, "reduce_scan_1_16.txt")):
        line = line.strip()
        if line.startswith("# "):
            key = line[2:].split()[0]
            if key in ("in", "block_reduce", "inclusive"):
                cur = key
                blocks[cur] = []
                continue
        if line and not line.startswith("#"):
            blocks[cur] += [int(v) for v in line.split()]
    return blocks


def test_golden_spec_values():
    g = _golden()
    for dt in (np.int32, np.int64, np.uint8, np.float32, np.float64):
        a = np.array(g["in"], dtype=dt)
        assert int(oracle.block_reduce(a, 16)[0]) == g["block_reduce"][0] == 136
        assert [int(v) for v in oracle.scan(a)] == g["inclusive"]


@pytest.mark.parametrize("n,B", [(1000, 64), (4096, 1024), (1001, 7), (5, 1), (5, 100), (0, 3)])
def test_closed_forms(n, B):
    a = np.arange(n, dtype=np.int64)
    out = oracle.block_reduce(a, B)
    assert out.size == -(-n // B)
    for b in range(out.size):
        lo, hi = b * B, min(n, (b + 1) * B)
        assert out[b] == (hi * (hi - 1) - lo * (lo - 1)) // 2       # sum_{i=lo}^{hi-1} i
    s = oracle.scan(a)
    assert all(s[i] == i * (i + 1) // 2 for i in range(n))
    assert np.array_equal(oracle.scan(np.ones(n, dtype=np.int32)), np.arange(1, n + 1))


@pytest.mark.parametrize("dt,bits", [(np.int32, 32), (np.int64, 64), (np.uint8, 8)])
def test_integer_wraparound_matches_exact_arithmetic(dt, bits):
    rng = np.random.default_rng(3)
    info = np.iinfo(dt)
    a = rng.integers(info.min, info.max, size=3000, dtype=dt, endpoint=True)
    B = 250
    got = oracle.block_reduce(a, B)
    mask = (1 << bits) - 1
    for b in range(got.size):
        exact = sum(int(v) for v in a[b * B:(b + 1) * B]) & mask
        assert int(got[b]) & mask == exact
    s = oracle.scan(a)
    run = 0
    for i, v in enumerate(a):
        run = (run + int(v)) & mask
        if i in (0, 1, 999, 2999):
            assert int(s[i]) & mask == run


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_float_sums_within_sequential_bound(dt):
    a = synth.random_bits((5000,), 4 if dt == np.float32 else 8, 11).view(dt)
    a = np.where(np.isfinite(a), a, 0).astype(dt)
    a = (a / np.maximum(1.0, np.abs(a).max())).astype(dt) * dt(3.0)   # finite, mixed signs
    B = 700
    got = oracle.block_reduce(a, B)
    u = 2.0 ** -53
    for b in range(got.size):
        blk = [float(v) for v in a[b * B:(b + 1) * B]]
        bound = len(blk) * u * sum(abs(v) for v in blk)
        assert abs(got[b] - math.fsum(blk)) <= bound
    s = oracle.scan(a)
    for i in (0, 10, 2500, 4999):
        pre = [float(v) for v in a[:i + 1]]
        assert abs(s[i] - math.fsum(pre)) <= (i + 1) * u * sum(abs(v) for v in pre)


def test_scan_reduce_consistency():
    a = synth.random_bits((10000,), 4, 5).view(np.int32)
    B = 300
    s = oracle.scan(a).astype(np.int64)
    r = oracle.block_reduce(a, B).astype(np.int64)
    for b in range(r.size):
        lo, hi = b * B, min(a.size, (b + 1) * B)
        assert (s[hi - 1] - (s[lo - 1] if lo else 0) - r[b]) % (1 << 32) == 0
    assert np.array_equal(oracle.block_reduce(a, 1), a)                   # B = 1: identity


def test_rejections():
    with pytest.raises(ValueError):
        oracle.block_reduce(np.zeros(4, np.int32), 0)


def _mutant_exclusive_scan(a):
    return np.concatenate([[0], np.cumsum(a)[:-1]])


def _mutant_block_off_by_one(a, B):
    return np.array([a[b * B:(b + 1) * B + 1].sum() for b in range(-(-a.size // B))])


def test_pins_catch_mutants():
    a = np.arange(1, 17, dtype=np.int64)
    g = _golden()
    assert list(_mutant_exclusive_scan(a)) != g["inclusive"]
    m = _mutant_block_off_by_one(np.arange(100, dtype=np.int64), 10)
    assert m[0] != 45
