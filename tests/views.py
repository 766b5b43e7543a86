"""Test-only simulations of the paper's two transpose listings (Listing 1 thread by
thread, Listing 2 through the view algebra of Listing 3 -- the basic views come from
oracle/views.py), used to PIN the oracle against the paper's own worked example.

A view is modelled as an index array: an ndarray whose entries are flat
offsets into the root array (SPEC S:293-301 `place_index_map` /
`view_permutation` idea).  Views reshape/reorder that index array; the memory
layout of the root never changes.
"""
from __future__ import annotations

import numpy as np


# ---- basic views, Listing 3: the oracle's definitions (oracle/views.py) ----
from oracle.views import group, transpose, split, reverse, vmap  # noqa: E402,F401


def group_by_row(x: np.ndarray, row_size: int, num_rows: int) -> np.ndarray:
    """group_by_row<row_size,num_rows> = group::<row_size/num_rows>.map(transpose)
    exactly as defined at P:526-531 (finding 3: shape [4][32][8] on a 32x32 tile)."""
    return vmap(transpose, group(x, row_size // num_rows))


def group_by_row_reading_a(x: np.ndarray, num_rows: int) -> np.ndarray:
    """Reading R2(a): group::<num_rows>.map(transpose) -> [ty][tx][i] = tile[4ty+i][tx]."""
    return vmap(transpose, group(x, num_rows))


def group_by_row_reading_b(x: np.ndarray, row_size: int, num_rows: int) -> np.ndarray:
    """Reading R2(b): group::<row_size/num_rows>.transpose.map(transpose)
    -> [ty][tx][i] = tile[ty + 8i][tx]  (Listing 1's pattern)."""
    return vmap(transpose, transpose(group(x, row_size // num_rows)))


def group_by_tile(x: np.ndarray, tr: int, tc: int) -> np.ndarray:
    """group_by_tile<tr,tc> (used at P:98/P:102, never defined; reading A11):
    [R][C] -> [R/tr][C/tc][tr][tc] = group::<tr>.map(map(group::<tc>)).map(transpose)."""
    g = group(x, tr)                                   # [R/tr][tr][C]
    g = vmap(lambda t: vmap(lambda row: group(row, tc), t), g)  # [R/tr][tr][C/tc][tc]
    return vmap(transpose, g)                          # [R/tr][C/tc][tr][tc]


# ---- the paper's listings, simulated ------------------------------------------
def listing2_transpose(inp: np.ndarray, tile: int = 32, threads_y: int = 8,
                       literal: bool = False, row_reading: str = "b") -> np.ndarray:
    """Simulate Listing 2 on a square n x n matrix with the view
    semantics above.  literal=True follows the listing character for character
    (copy-out uses the same intra-tile view on both sides: finding 2, only tiles
    are permuted).  literal=False adds the intra-tile `.transpose` on the tmp
    side of the copy-out (reading R1, the intended full transpose)."""
    n = inp.shape[0]
    assert inp.shape == (n, n) and n % tile == 0
    k = tile // threads_y   # iterations per thread (4)
    flat_in = inp.reshape(-1)
    out = np.zeros(n * n, dtype=inp.dtype)
    idx_in = np.arange(n * n).reshape(n, n)
    idx_out = np.arange(n * n).reshape(n, n)

    def gbr(t):
        if row_reading == "a":
            return group_by_row_reading_a(t, k)
        return group_by_row_reading_b(t, tile, k)

    in_blocks = transpose(group_by_tile(idx_in, tile, tile))    # input.group_by_tile.transpose
    out_blocks = group_by_tile(idx_out, tile, tile)              # output.group_by_tile
    nb = n // tile
    for by in range(nb):                 # sched(Y,X) block in grid
        for bx in range(nb):
            tmp = np.zeros(tile * tile, dtype=inp.dtype)         # alloc gpu.shared
            tmp_idx = np.arange(tile * tile).reshape(tile, tile)
            src = gbr(in_blocks[by][bx])                         # [ty][tx][i]
            dst_tmp = gbr(tmp_idx)
            for ty in range(threads_y):  # sched(Y,X) thread in block
                for tx in range(tile):
                    for i in range(k):
                        tmp[dst_tmp[ty][tx][i]] = flat_in[src[ty][tx][i]]
            # sync
            src_tmp = gbr(tmp_idx if literal else transpose(tmp_idx))
            dst = gbr(out_blocks[by][bx])
            for ty in range(threads_y):
                for tx in range(tile):
                    for i in range(k):
                        out[dst[ty][tx][i]] = tmp[src_tmp[ty][tx][i]]
    return out.reshape(n, n)


def listing1_transpose(inp: np.ndarray, fixed: bool = True, float_tmp: bool = False):
    """Simulate Listing 1 on an n x n f64 matrix (2048 -> n).

    fixed=True applies the paper's fix (`threadIdx.y+j` parenthesised).
    float_tmp=True reproduces `__shared__ float tmp[1024]` staging f64
    through f32.  Threads run sequentially in canonical order (last writer wins).
    Returns (out, writers) where writers[b][slot] counts writes to each tmp slot."""
    n = inp.shape[0]
    assert inp.shape == (n, n) and n % 32 == 0 and inp.dtype == np.float64
    flat_in = inp.reshape(-1)
    out = np.zeros(n * n, dtype=np.float64)
    nb = n // 32
    writers = np.zeros((nb * nb, 1024), dtype=np.int64)
    for by in range(nb):
        for bx in range(nb):
            tmp = np.zeros(1024, dtype=np.float32 if float_tmp else np.float64)
            for ty in range(8):
                for tx in range(32):
                    for j in range(0, 32, 8):
                        slot = (ty + j) * 32 + tx if fixed else ty + j * 32 + tx
                        writers[by * nb + bx][slot] += 1
                        tmp[slot] = flat_in[(by * 32 + ty + j) * n + bx * 32 + tx]
            # __syncthreads()
            for ty in range(8):
                for tx in range(32):
                    for j in range(0, 32, 8):
                        out[(bx * 32 + ty + j) * n + by * 32 + tx] = tmp[tx * 32 + ty + j]
    return out.reshape(n, n), writers
