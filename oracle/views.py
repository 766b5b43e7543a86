"""CPU ORACLE for view-composed copies -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Ground semantics of Descend's basic views, Listing 3 and §3.2
(P:504-548): a view reshapes or reorders the way an array is accessed; "the memory layout of
the original array stays the same".  Here a view is applied to an INDEX ARRAY --
an ndarray whose entries are flat element offsets into the root array (the ground semantics
SPEC.md calls place_index_map / view_permutation) -- so every function
below is the definition written out with numpy reshapes / slices, nothing else:

  group<k>    [[d;n]] -> [[ [[d;k]]; n/k ]]        P:517-519, P:537-538 (k | n, reading R12)
  transpose   [[ [[d;n]]; m ]] -> [[ [[d;m]]; n ]] P:521, P:539-540 (outer two dims only)
  split<k>    [[d;n]] -> ([[d;k]], [[d;n-k]])      P:514-516, P:535-536 (n >= k)
  reverse     [[d;n]] -> [[d;n]] reversed
  map(v)      applies v to every element

A chain of views is a list of (kind, k, depth) triples: kind in {"group", "transpose",
"split_fst", "split_snd", "reverse"}, k its nat argument (group/split), depth the number of
enclosing map(...) wrappers (depth 1 = map(v), depth 2 = map(map(v)), ...).  This encoding is
shared with the C ABI's desc_view_op (include/desc_transpose.h) as DATA only.

materialize(a, ops) returns the elements the place `a.v1.v2...` denotes, in the view's
row-major order -- what a view copy must produce.  Pins: tests/test_views_oracle.py.
"""
from __future__ import annotations

import numpy as np

KINDS = ("group", "transpose", "split_fst", "split_snd", "reverse")


def group(x: np.ndarray, k: int) -> np.ndarray:
    n = x.shape[0]
    if k <= 0 or n % k:
        raise ValueError(f"group<{k}>: n={n} must be divisible by k (R12)")
    return x.reshape((n // k, k) + x.shape[1:])


def transpose(x: np.ndarray) -> np.ndarray:
    if x.ndim < 2:
        raise ValueError("transpose needs a nested (2-D) array")
    return np.swapaxes(x, 0, 1)


def split(x: np.ndarray, k: int):
    if not (0 <= k <= x.shape[0]):
        raise ValueError(f"split<{k}>: n={x.shape[0]} must be >= k")
    return x[:k], x[k:]


def reverse(x: np.ndarray) -> np.ndarray:
    return x[::-1]


def vmap(v, x: np.ndarray) -> np.ndarray:
    """map(v): v applied to each element of the outer array (stacked back together)."""
    if x.shape[0] == 0:
        probe = v(np.zeros(x.shape[1:], dtype=x.dtype))
        return np.zeros((0,) + probe.shape, dtype=x.dtype)
    return np.stack([v(x[i]) for i in range(x.shape[0])])


def apply_op(x: np.ndarray, kind: str, k: int = 0, depth: int = 0) -> np.ndarray:
    if depth > 0:
        if x.ndim <= depth:
            raise ValueError("map depth exceeds the nesting of the array")
        return vmap(lambda e: apply_op(e, kind, k, depth - 1), x)
    if kind == "group":
        return group(x, k)
    if kind == "transpose":
        return transpose(x)
    if kind == "split_fst":
        return split(x, k)[0]
    if kind == "split_snd":
        return split(x, k)[1]
    if kind == "reverse":
        return reverse(x)
    raise ValueError(f"unknown view {kind}")


def index_view(shape, ops) -> np.ndarray:
    """The place's flat element offsets into a C-contiguous root array of `shape`."""
    x = np.arange(int(np.prod(shape)), dtype=np.int64).reshape(shape)
    for kind, k, depth in ops:
        x = apply_op(x, kind, k, depth)
    return x


def materialize(a: np.ndarray, ops) -> np.ndarray:
    """Elements of the view of the (C-contiguous) root array `a`, in view order."""
    idx = index_view(a.shape, ops)
    return np.ascontiguousarray(a.reshape(-1)[idx])
