"""Host bijection / coverage / race check of every kernel's index map (no GPU; VERDICT r01
"missing" #1).  tests/index_maps.py restates each kernel's (CTA, thread, k) -> (src, dst)
map from csrc/*.cuh and executes a launch on element ids; here every variant must be a
race-free bijection onto the logical output carrying the transpose's values (P:40, P:163,
P:596-599), on small grids with edge tiles, padded pitches and batches -- and the restated
defects of csrc/mutants.cuh, plus the paper's own racy kernels (Listing 1 as printed,
P:44-45; rev_per_block), must each be rejected."""
import numpy as np
import pytest

from tests import index_maps as IM

# (batch, rows, cols, ld_in, ld_out, stride_in, stride_out): tight, ragged, padded, batched
SHAPES = [
    (1, 64, 64, 64, 64, 0, 0),
    (1, 67, 131, 131, 67, 0, 0),
    (1, 131, 67, 72, 136, 0, 0),
    (1, 3, 5, 5, 3, 0, 0),
    (1, 1, 200, 200, 1, 0, 0),
    (1, 200, 1, 1, 200, 0, 0),
    (3, 33, 65, 68, 40, 33 * 72 + 4, 65 * 40 + 8),
    (2, 100, 70, 70, 100, 7000, 7000),
]


def _check(L, shape):
    return IM.check_launch(L, *shape)


@pytest.mark.parametrize("es", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", SHAPES)
def test_tiled_map_is_a_race_free_bijection(shape, es):
    assert _check(IM.tiled_launch(*shape, es), shape) == []


# the TILED tile shapes desc_transpose.cu run_tiled can launch (DESC_TILED_CFG 1-3)
TILED_SHAPES = {4: [(32, 64, 128), (32, 128, 256), (16, 128, 128)],
                8: [(16, 64, 128), (16, 128, 256), (32, 64, 256)]}


@pytest.mark.parametrize("es", [4, 8])
@pytest.mark.parametrize("shape", SHAPES[1:4] + SHAPES[6:])
def test_tiled_alternative_shapes_are_race_free_bijections(shape, es):
    for TR, TC, NT in TILED_SHAPES[es]:
        assert _check(IM.tiled_launch(*shape, es, TR=TR, TC=TC, NT=NT), shape) == [], (TR, TC, NT)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("grid", [None, 3])
def test_smem_map_is_a_race_free_bijection(shape, grid):
    """The corrected Listing 1 schedule, one tile per CTA and a persistent grid of 3 CTAs."""
    assert _check(IM.smem_launch(*shape, 4, grid=grid), shape) == []


def _tma_shapes(es):
    """TMA needs 16-byte pitches: pad ld_in / ld_out / strides to 16 bytes."""
    v = 16 // es
    out = []
    for (b, r, c, *_ ) in SHAPES:
        li, lo = -(-c // v) * v, -(-r // v) * v + v
        out.append((b, r, c, li, lo, r * li if b > 1 else 0, c * lo if b > 1 else 0))
    return out


TMA2_CFGS = {4: [(128, 2, 8), (64, 2, 8)], 8: [(128, 1, 16), (64, 2, 8)]}   # (TR, NB, CW)


@pytest.mark.parametrize("es", [4, 8])
def test_tma_store_map_is_a_race_free_bijection(es):
    """transpose_tma2_kernel, both tuned configurations per cell size (desc_transpose.cu
    run_tma2), static persistent schedule on a small grid, raster groups of 1 and all rows;
    includes rows % VEC != 0 (the ragged tail the lanes write themselves)."""
    for shape in _tma_shapes(es):
        for TR, NB, CW in TMA2_CFGS[es]:
            for grid, group in ((None, None), (2, 1)):
                L = IM.tma_launch(*shape, es, TR=TR, NB=NB, CW=CW, grid=grid, group=group)
                assert _check(L, shape) == [], (shape, TR, NB, CW, grid, group)


@pytest.mark.parametrize("es", [4, 8])
def test_tma_tile_map_is_a_race_free_bijection(es):
    """transpose_tma_tile_kernel (csrc/tma_tile_transpose.cuh): the TMA-store kernel's lane
    maps with 4 warps and one tile per CTA (64 x 64 for 4-byte cells: TR 64, 2 boxes; 32 x 64
    for 8-byte cells: TR 32, 4 boxes); the transposed rows are written back into the input
    buffer after a barrier, which the model's separate read / write intervals express."""
    TR, NB = (64, 2) if es == 4 else (32, 4)
    for shape in _tma_shapes(es):
        for group in (None, 1):
            L = IM.tma_launch(*shape, es, TR=TR, NB=NB, CW=4, grid=None, group=group)
            assert _check(L, shape) == [], (shape, group)


@pytest.mark.parametrize("es", [1, 2, 4, 8])
def test_tma_load_map_is_a_race_free_bijection(es):
    """transpose_tma_kernel (TMA load + 16-byte st.global), the default configuration per
    cell size (desc_transpose.cu run_tma: TR 128, 1 box; 8 or 16 / 4 / 2 consumer warps)."""
    CW = {1: 2, 2: 4, 4: 8, 8: 16}[es]
    for shape in _tma_shapes(es):
        L = IM.tma_launch(*shape, es, TR=128, NB=1, CW=CW, store=False, grid=2)
        assert _check(L, shape) == [], shape


def _vtiled_shapes(es):
    """The vector tile kernel's rules: 16-byte pitches and rows, cols multiples of 16/es."""
    v = 16 // es
    out = []
    for (b, r, c, *_) in SHAPES + [(1, 132, 68, 0, 0, 0, 0), (2, 96, 200, 0, 0, 0, 0)]:
        r, c = -(-r // v) * v, -(-c // v) * v
        li, lo = c + (v if b > 1 else 0), r + v
        out.append((b, r, c, li, lo, r * li + v if b > 1 else 0, c * lo + 2 * v if b > 1 else 0))
    return out


@pytest.mark.parametrize("es", [1, 2, 4, 8])
def test_vtiled_map_is_a_race_free_conflict_free_bijection(es):
    """transpose_vtiled_kernel (csrc/vtiled_transpose.cuh), default tile per cell size and the
    DESC_VTILED_CFG alternatives: every output element once with its transpose source, no
    shared-memory race, every 8-lane phase of the 16-byte copy-in and copy-out conflict-free
    (the 16-byte XOR swizzle)."""
    cfgs = {4: [(16, 128), (16, 256), (32, 256), (8, 128), (16, 64), (32, 128), (8, 64)],
            8: [(16, 64), (16, 256), (32, 256), (8, 128), (16, 128), (32, 128), (32, 64)],
            2: [(8, 128), (16, 256), (8, 64)], 1: [(8, 128), (8, 64)]}
    for shape in _vtiled_shapes(es):
        for TCH, NT in cfgs[es]:
            L = IM.vtiled_launch(*shape, es, TCH=TCH, NT=NT)
            assert _check(L, shape) == [], (shape, TCH, NT)


def test_vtiled_mutants_and_unswizzled_layout_rejected():
    shape = (1, 100, 132, 132, 104, 0, 0)
    for mutant, what in (("tile_only", "wrong source"), ("no_sync", "race")):
        errs = _check(IM.vtiled_launch(*shape, 4, mutant=mutant), shape)
        assert errs and any(what in e for e in errs), (mutant, errs)
    for es in (4, 8):       # without the XOR swizzle the micro-block reads conflict
        errs = _check(IM.vtiled_launch(*shape, es, swizzle=False), shape)
        assert errs and all("bank conflict" in e for e in errs), errs


# ------------------------------------------------------------------ teeth
def test_tiled_mutants_rejected():
    shape = (1, 100, 131, 131, 100, 0, 0)        # edge tiles in both directions
    for mutant, what in (("tile_only", "wrong source"), ("edge", "outside"),
                         ("no_sync", "race")):
        errs = _check(IM.tiled_launch(*shape, 4, mutant=mutant), shape)
        assert errs and any(what in e for e in errs), (mutant, errs)


def test_smem_mutants_rejected():
    """Listing 1 as printed (several threads write one tmp slot) is a shared-memory
    race; the literal Listing 2 (tile permutation only) carries wrong sources; the edge
    off-by-one writes padding."""
    shape = (1, 96, 70, 70, 96, 0, 0)
    errs = _check(IM.smem_launch(*shape, 4, mutant="no_paren"), shape)
    assert any("race" in e for e in errs), errs
    errs = _check(IM.smem_launch(*shape, 4, mutant="tile_only"), shape)
    assert any("wrong source" in e for e in errs), errs
    errs = _check(IM.smem_launch(1, 90, 70, 70, 100, 0, 0, 4, mutant="edge"),
                  (1, 90, 70, 70, 100, 0, 0))
    assert any("outside" in e for e in errs), errs


def test_tma_store_mutants_rejected():
    shape = (1, 67, 131, 132, 72, 0, 0)          # rows % 4 = 3: a ragged tail
    for mutant, what in (("no_micro", "wrong source"), ("no_tail", "never written"),
                         ("no_swizzle", "wrong source")):
        errs = _check(IM.tma_launch(*shape, 4, TR=64, NB=2, CW=8, mutant=mutant), shape)
        assert errs and any(what in e for e in errs), (mutant, errs)


def test_swizzle_is_what_makes_tma_phases_conflict_free():
    """Reading the 128-byte-swizzled stage linearly (mutant 8) also costs bank conflicts: the
    conflict-freedom claim depends on the swizzle, and the checker sees it."""
    shape = (1, 64, 64, 64, 64, 0, 0)
    errs = _check(IM.tma_launch(*shape, 4, TR=64, NB=2, CW=8, mutant="no_swizzle"), shape)
    assert any("bank conflict" in e for e in errs), errs


# ------------------------------------------------------------------ views: access safety
def test_rev_per_block_is_a_race():
    """block_part[tid] = block_part[blockDim-1-tid] -- reads through `rev` what other
    threads write in the same phase: rejected (what Descend's checker reports at P:176-182);
    racecheck cannot see it (global memory, scripts/sanitizer_controls.py rev_global)."""
    n = 256
    cells = np.arange(n)
    assert IM.thread_conflicts(cells, cells[::-1]) == n        # every cell but... all of them
    assert IM.thread_conflicts(np.arange(1), np.arange(1)) == 0   # one thread: no race
    # the race-free version: write through the identity view into ANOTHER buffer
    assert IM.thread_conflicts(cells, n + cells[::-1]) == 0


def test_listing1_printed_index_is_a_waw_race():
    """tmp[threadIdx.y + j*32 + threadIdx.x] (j = 0, 8, 16, 24) -- in one phase
    threads with equal ty + tx write the same slot; with the parentheses, (ty + j) * 32 + tx,
    every slot of every phase has exactly one writer."""
    tx, ty = np.meshgrid(np.arange(32), np.arange(8))
    for j in (0, 8, 16, 24):
        assert IM.thread_conflicts(((ty + j) * 32 + tx).ravel()) == 0
        assert IM.thread_conflicts((ty + j * 32 + tx).ravel()) > 0


@pytest.mark.parametrize("seed", range(40))
def test_views_are_injective_so_writes_through_them_are_race_free(seed):
    """Every basic view of Listing 3 (group, transpose, split, reverse, map) is injective, so
    a composition of them gives each thread of a flat schedule a distinct cell (narrowing,
    P:596-599): writing through any random chain is race-free; reading the SAME buffer
    through `reverse` while writing it (rev_per_block's pattern) is not."""
    rng = np.random.default_rng(seed)
    shape = (int(rng.choice([4, 6, 8, 12])), int(rng.choice([4, 8, 10, 16])))
    ops = []
    nd = 2
    cur = list(shape)
    for _ in range(int(rng.integers(1, 5))):
        kind = str(rng.choice(["group", "transpose", "reverse", "split_fst", "split_snd"]))
        depth = int(rng.integers(0, nd))
        n = cur[depth]
        if kind == "group":
            ks = [k for k in (2, 3, 4) if n % k == 0]
            if not ks or nd >= 5:
                continue
            k = int(rng.choice(ks))
            ops.append(("group", k, depth))
            cur[depth:depth + 1] = [n // k, k]
            nd += 1
        elif kind == "transpose":
            if depth + 1 >= nd:
                continue
            ops.append(("transpose", 0, depth))
            cur[depth], cur[depth + 1] = cur[depth + 1], cur[depth]
        elif kind == "reverse":
            ops.append(("reverse", 0, depth))
        else:
            k = int(rng.integers(1, n)) if n > 1 else 0
            ops.append((kind, k, depth))
            cur[depth] = k if kind == "split_fst" else n - k
    cells = IM.view_thread_cells(shape, ops)
    assert np.unique(cells).size == cells.size                     # injective
    assert IM.thread_conflicts(cells) == 0
    if cells.size > 1:
        assert IM.thread_conflicts(cells, cells[::-1]) > 0 or np.array_equal(cells, cells[::-1])


def test_group_by_tile_blocks_own_disjoint_parts():
    """Narrowing: with group_by_tile<32,32> and one block per tile, the
    blocks' cell sets partition the matrix."""
    from tests import views as TV
    n = 128
    tiles = TV.group_by_tile(np.arange(n * n).reshape(n, n), 32, 32)   # [4][4][32][32]
    owner = np.full(n * n, -1)
    for bi in range(4):
        for bj in range(4):
            cells = tiles[bi, bj].ravel()
            assert (owner[cells] == -1).all()
            owner[cells] = bi * 4 + bj
    assert (owner >= 0).all()


@pytest.mark.parametrize("P,M,N,es", [(2, 128, 256, 4), (4, 96, 512, 4), (8, 64, 512, 8),
                                      (2, 70, 128, 8), (3, 90, 192, 4)])
def test_slab_peer_scatter_covers_every_slab_exactly_once(P, M, N, es):
    """desc_slab_transpose_peer over all P ranks: the union of the P launches writes every
    element of every rank's output slab exactly once, with the global transpose's source
    (out_s[j][i] = A[i][s*Rn + j]), and no tile straddles two destinations when N/P is a
    multiple of the tile width (the C ABI rejects other shapes)."""
    Rm, Rn = M // P, N // P
    per, straddle = IM.slab_peer_launches(P, M, N, es)
    assert straddle == 0
    for s in range(P):
        dst, gid = per[s]
        assert np.array_equal(np.sort(dst), np.arange(Rn * M)), s          # exactly once
        j, i = dst // M, dst % M
        assert np.array_equal(gid, i * N + s * Rn + j), s                  # the transpose


def test_slab_peer_scatter_needs_tile_aligned_segments():
    """Why the C ABI requires N/P to be a multiple of the tile width: with N/P = 48 and 64-wide
    tiles, tiles straddle two destination slabs and the per-tile routing misplaces columns."""
    per, straddle = IM.slab_peer_launches(2, 64, 96, 4)
    assert straddle > 0
