"""The host view compiler (desc_view_compile, C ABI, no GPU needed) against the view oracle:
for many random chains of Listing 3's views over small roots, the compiled strided view must
address exactly the oracle's index array (SPEC S:583's "lowering == view_permutation"
criterion, exhaustive over the enumerated chains); plus the rejection rules."""
import random

import numpy as np
import pytest

import paper_2305_03448_b200 as desc
from oracle import views as V
from paper_2305_03448_b200 import build as desc_build


@pytest.fixture(scope="module", autouse=True)
def _lib():
    desc_build.build()
    desc.load()


def _strided_index(view):
    shape, stride, offset = view.dims
    idx = np.full(shape, offset, dtype=np.int64)
    for d, (n, s) in enumerate(zip(shape, stride)):
        r = np.arange(n, dtype=np.int64) * s
        idx += r.reshape((1,) * d + (n,) + (1,) * (len(shape) - d - 1))
    return idx


def random_chain(rng: random.Random, shape, length):
    ops, cur = [], list(shape)
    for _ in range(length):
        choices = []
        for d in range(len(cur)):
            n = cur[d]
            ks = [k for k in range(1, n + 1) if n % k == 0]
            if len(cur) < 8 and ks:
                choices.append(("group", rng.choice(ks), d))
            if d + 1 < len(cur):
                choices.append(("transpose", 0, d))
            choices.append(("split_fst", rng.randint(0, n), d))
            choices.append(("split_snd", rng.randint(0, n), d))
            choices.append(("reverse", 0, d))
        kind, k, d = rng.choice(choices)
        ops.append((kind, k, d))
        if kind == "group":
            cur[d:d + 1] = [cur[d] // k, k]
        elif kind == "transpose":
            cur[d], cur[d + 1] = cur[d + 1], cur[d]
        elif kind == "split_fst":
            cur[d] = k
        elif kind == "split_snd":
            cur[d] = cur[d] - k
    return ops


@pytest.mark.parametrize("shape", [(8,), (12,), (4, 6), (8, 8), (2, 3, 4), (6, 10)])
def test_compiler_matches_oracle_random_chains(shape):
    rng = random.Random(hash(shape) & 0xFFFF)
    for trial in range(150):
        ops = random_chain(rng, shape, rng.randint(1, 4))
        ref = V.index_view(shape, ops)
        got = desc.desc_view_compile(shape, ops)
        assert got.dims[0] == ref.shape, (ops, got.dims, ref.shape)
        assert np.array_equal(_strided_index(got), ref), ops


def test_compiler_listing_views():
    # Listing 2's input place: input.group_by_tile::<32,32>.transpose (reading A11)
    ops = [("group", 32, 0), ("group", 32, 2), ("transpose", 0, 1), ("transpose", 0, 0)]
    got = desc.desc_view_compile((64, 96), ops)
    assert np.array_equal(_strided_index(got), V.index_view((64, 96), ops))
    # rot90 = transpose.map(reverse) on a padded root (ld 10 > 7 cols)
    got = desc.desc_view_compile((5, 7), [("transpose", 0, 0), ("reverse", 0, 1)], strides=(10, 1))
    assert got.dims == ((7, 5), (1, -10), 40)


def test_compiler_rejections():
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_view_compile((10,), [("group", 3, 0)])          # R12: k | n
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_view_compile((10,), [("split_fst", 11, 0)])     # n >= k
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_view_compile((10,), [("transpose", 0, 0)])      # flat array
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_view_compile((4, 4), [("reverse", 0, 2)])       # map deeper than nesting
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.desc_view_compile((256,), [("group", 2, d) for d in range(8)])   # > 8 dims
