"""Pins for the view oracle (oracle/views.py) -- CPU only.

Each basic view of Listing 3 is pinned to something other than its own numpy
expression: the values SPEC.md prints for ground examples, the golden
select-view fixture, algebraic laws (involutions, split/concat, group/flatten),
and closed-form index formulas for composed views; plus the listed side conditions, and
mutation teeth (plausible wrong views fail a pin)."""
import os

import numpy as np
import pytest

from oracle import views as V

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_ground_examples():
    # arr.group::<8>.transpose[[thread i]] index j, n = 32 -> {j*8 + i}
    x = V.index_view((32,), [("group", 8, 0), ("transpose", 0, 0)])
    assert x.shape == (8, 4)
    for i in range(8):
        for j in range(4):
            assert x[i, j] == j * 8 + i
    # reverse, n = 4 -> [3, 2, 1, 0]
    assert list(V.index_view((4,), [("reverse", 0, 0)])) == [3, 2, 1, 0]
    # split::<32> fst, n = 64 -> identity on 0..31
    assert list(V.index_view((64,), [("split_fst", 32, 0)])) == list(range(32))
    assert list(V.index_view((64,), [("split_snd", 32, 0)])) == list(range(32, 64))


def test_golden_select_view():
    golden = {}
    for line in open(os.path.join(GOLDEN, "select_view_32.txt")):
        if line.strip() and not line.startswith("#"):
            t, offs = line.split(":")
            golden[int(t)] = [int(v) for v in offs.split()]
    x = V.index_view((32,), [("group", 8, 0), ("transpose", 0, 0)])
    assert {t: list(x[t]) for t in range(8)} == golden


def test_listing3_types():
    assert V.index_view((12,), [("group", 3, 0)]).shape == (4, 3)           # [[d;k]]; n/k
    assert V.index_view((4, 6), [("transpose", 0, 0)]).shape == (6, 4)      # swap outer two
    assert V.index_view((4, 6, 5), [("transpose", 0, 0)]).shape == (6, 4, 5)  # d opaque
    assert V.index_view((10,), [("split_fst", 3, 0)]).shape == (3,)
    assert V.index_view((10,), [("split_snd", 3, 0)]).shape == (7,)
    assert V.index_view((4, 6), [("group", 2, 1)]).shape == (4, 3, 2)       # map(group)
    with pytest.raises(ValueError):
        V.index_view((10,), [("group", 3, 0)])                             # 3 does not divide 10
    with pytest.raises(ValueError):
        V.index_view((10,), [("split_fst", 11, 0)])                        # n >= k
    with pytest.raises(ValueError):
        V.index_view((10,), [("transpose", 0, 0)])
    with pytest.raises(ValueError):
        V.index_view((10,), [("reverse", 0, 1)])                           # map on a flat array


@pytest.mark.parametrize("shape", [(6,), (4, 6), (2, 3, 4)])
def test_laws(shape):
    base = V.index_view(shape, [])
    assert np.array_equal(V.index_view(shape, [("reverse", 0, 0), ("reverse", 0, 0)]), base)
    if len(shape) >= 2:
        assert np.array_equal(V.index_view(shape, [("transpose", 0, 0), ("transpose", 0, 0)]), base)
    n = shape[0]
    for k in range(n + 1):
        fst = V.index_view(shape, [("split_fst", k, 0)])
        snd = V.index_view(shape, [("split_snd", k, 0)])
        assert np.array_equal(np.concatenate([fst, snd]), base)
    for k in (1, 2, 3, 6):
        if n % k == 0:
            g = V.index_view(shape, [("group", k, 0)])
            assert np.array_equal(g.reshape(base.shape), base)


def test_closed_forms_of_compositions():
    R, C, tr, tc = 8, 12, 4, 3
    # group_by_tile<tr,tc> = group<tr>.map(map(group<tc>)).map(transpose)   (reading A11)
    t = V.index_view((R, C), [("group", tr, 0), ("group", tc, 2), ("transpose", 0, 1)])
    assert t.shape == (R // tr, C // tc, tr, tc)
    for I in range(R // tr):
        for J in range(C // tc):
            for r in range(tr):
                for c in range(tc):
                    assert t[I, J, r, c] == (I * tr + r) * C + J * tc + c
    # map(reverse) over groups reverses inside each group
    g = V.index_view((12,), [("group", 4, 0), ("reverse", 0, 1)])
    assert all(g[i, j] == i * 4 + (3 - j) for i in range(3) for j in range(4))
    # transpose of a 2-D array = the matrix transpose's index map
    tt = V.index_view((5, 7), [("transpose", 0, 0)])
    assert all(tt[j, i] == i * 7 + j for i in range(5) for j in range(7))
    # rot90: transpose.map(reverse)   out[j][i] = in[R-1-i][j]
    rot = V.index_view((5, 7), [("transpose", 0, 0), ("reverse", 0, 1)])
    assert all(rot[j, i] == (4 - i) * 7 + j for i in range(5) for j in range(7))


def test_materialize_is_gather_of_index_view():
    a = np.arange(100, 124, dtype=np.int32).reshape(4, 6)
    m = V.materialize(a, [("transpose", 0, 0)])
    assert m.flags.c_contiguous and np.array_equal(m, np.ascontiguousarray(a.T))


def _wrong_transpose(x):          # swaps the innermost two dims instead of the outer two
    return np.swapaxes(x, -1, -2)


def test_mutation_teeth():
    x = np.arange(24).reshape(2, 3, 4)
    assert _wrong_transpose(x).shape != V.transpose(x).shape
    bad = np.arange(32).reshape(8, 4)        # group<4> instead of group<8>, no transpose
    assert not np.array_equal(bad, V.index_view((32,), [("group", 8, 0), ("transpose", 0, 0)]))
