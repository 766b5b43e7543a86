"""Pins for the CPU oracle (oracle/transpose_ref.c) -- runs without a GPU.

Each pin checks the oracle against something other than its own formula:
  * a library routine  (numpy's transpose copy, bit-exact on raw bit patterns),
  * the paper's worked example (Listing 1 with the P:44 fix, simulated; Listing 2
    through the view algebra of Listing 3, reading R1),
  * golden fixtures under tests/golden/ (cited),
  * closed forms / invariants (self-describing decode, involution, block identity,
    1xN memcpy, symmetric fixed point, permutation multiset),
  * guard bands (padding and out-of-range bytes never written).
The mutation tests at the end prove the pins have teeth: plausible wrong
transposes (copy without transpose, swapped ld, tile-only permutation, f32
staging of f64, off-by-one edge) each fail at least one pin.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from tests import views

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ES_ALL = (1, 2, 4, 8)


def _T(a):
    return oracle.transpose(a)


# ---------------------------------------------------------------- library pin
@pytest.mark.parametrize("es", ES_ALL)
@pytest.mark.parametrize("shape", [(64, 64), (1, 4097), (4097, 1), (300, 500),
                                   (33, 65), (129, 127), (2048, 2048)])
def test_matches_numpy_transpose_copy(es, shape):
    if shape == (2048, 2048) and es < 4:
        pytest.skip("large shape only for 4/8-byte elements")
    a = synth.with_specials(synth.random_bits(shape, es, synth.BASE_SEED + 1), es, 7)
    got = _T(a)
    ref = np.ascontiguousarray(a.T)
    assert got.shape == (shape[1], shape[0])
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("es", (4, 8))
def test_batched_matches_numpy(es):
    a = synth.random_bits((7, 33, 65), es, synth.BASE_SEED + 3)
    got = _T(a)
    assert got.tobytes() == np.ascontiguousarray(np.swapaxes(a, 1, 2)).tobytes()


def test_float_views_bit_exact_specials():
    """f64 NaN payloads, sNaN, -0.0 and subnormals survive (reading R4/R11)."""
    a = synth.with_specials(synth.random_bits((40, 24), 8, 11), 8, 12)
    f = a.view(np.float64)
    assert np.isnan(f).any()
    got = _T(f)
    assert got.view(np.uint64).tobytes() == np.ascontiguousarray(a.T).tobytes()


# ------------------------------------------------------------- golden fixtures
def _read_golden_matrix(name):
    blocks, cur = {}, None
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line in ("# in", "# out"):
            cur = line[2:]
            blocks[cur] = []
        elif line and not line.startswith("#"):
            blocks[cur].append([int(v) for v in line.split()])
    return np.array(blocks["in"], dtype=np.int32), np.array(blocks["out"], dtype=np.int32)


def test_golden_textbook_3x4():
    a, expected = _read_golden_matrix("transpose_3x4.txt")
    assert np.array_equal(_T(a), expected)
    assert np.array_equal(_T(a.astype(np.float64)), expected.astype(np.float64))


def test_golden_select_view_is_what_the_view_model_computes():
    """Pins tests/views.py (used by the Listing 2 pin below) to Fig. select-view."""
    golden = {}
    for line in open(os.path.join(GOLDEN, "select_view_32.txt")):
        if line.strip() and not line.startswith("#"):
            t, offs = line.split(":")
            golden[int(t)] = [int(v) for v in offs.split()]
    v = views.transpose(views.group(np.arange(32), 8))   # array.group::<8>.transpose
    assert v.shape == (8, 4)
    for t in range(8):
        assert list(v[t]) == golden[t]


# ------------------------------------------------- the paper's worked examples
@pytest.mark.parametrize("n", [32, 64, 128])
def test_corrected_listing1_equals_oracle(n):
    """Listing 1 with the P:44 fix, simulated thread by thread."""
    a = synth.random_bits((n, n), 8, 99).view(np.float64)
    out, writers = views.listing1_transpose(a, fixed=True)
    assert (writers == 1).all(), "fixed listing writes each tmp slot exactly once"
    assert out.view(np.uint64).tobytes() == _T(a).view(np.uint64).tobytes()


def test_buggy_listing1_races_and_differs():
    """The printed Listing 1 (missing parentheses) makes several threads
    write one tmp slot: a data race; its result is not the transpose."""
    a = synth.random_bits((64, 64), 8, 5).view(np.float64)
    out, writers = views.listing1_transpose(a, fixed=False)
    assert writers.max() > 1                      # "multiple threads will write ... the same memory location"
    assert (writers[0] > 0).sum() < 1024          # and some slots are never written
    assert out.view(np.uint64).tobytes() != _T(a).view(np.uint64).tobytes()


def test_float_tmp_listing1_not_bit_exact():
    """`__shared__ float tmp[1024]` staging f64 through f32 loses bits (reading R4)."""
    a = synth.random_bits((64, 64), 8, 6).view(np.float64)
    out, _ = views.listing1_transpose(a, fixed=True, float_tmp=True)
    assert out.view(np.uint64).tobytes() != _T(a).view(np.uint64).tobytes()


@pytest.mark.parametrize("reading", ["a", "b"])
@pytest.mark.parametrize("n", [32, 64, 96])
def test_listing2_intended_equals_oracle(n, reading):
    """Listing 2 through Listing 3's views with reading R1 (intra-tile
    transpose on the copy-out) and either reading R2 of group_by_row."""
    a = synth.random_bits((n, n), 8, 17)
    got = views.listing2_transpose(a, literal=False, row_reading=reading)
    assert got.tobytes() == _T(a).tobytes()


def test_listing2_literal_only_permutes_tiles():
    """Finding 2 / reading R1: the literal listing moves tile (I,J) to (J,I) but
    does not transpose inside a tile -- so it is NOT the oracle's result."""
    n = 64
    a = synth.self_describing(1, n, n, 4)[0]
    lit = views.listing2_transpose(a, literal=True)
    assert lit.tobytes() != _T(a).tobytes()
    for I in range(2):
        for J in range(2):
            assert np.array_equal(lit[32 * J:32 * J + 32, 32 * I:32 * I + 32],
                                  a[32 * I:32 * I + 32, 32 * J:32 * J + 32])


def test_group_by_row_as_printed_has_wrong_shape():
    """Finding 3: group::<8>.map(transpose) on a 32x32 tile is [4][32][8],
    not the [8][32][4] Listing 2 needs for XY<32,8> threads x 4 iterations."""
    t = np.arange(1024).reshape(32, 32)
    assert views.group_by_row(t, 32, 4).shape == (4, 32, 8)
    assert views.group_by_row_reading_a(t, 4).shape == (8, 32, 4)
    assert views.group_by_row_reading_b(t, 32, 4).shape == (8, 32, 4)


# ------------------------------------------------------ closed forms, invariants
@pytest.mark.parametrize("es", (4, 8))
def test_self_describing_exhaustive_small(es):
    """All (rows, cols) in [1,40]^2: out[j][i] must decode to source (i, j)."""
    for rows in range(1, 41):
        for cols in range(1, 41):
            a = synth.self_describing(1, rows, cols, es)[0]
            out = _T(a)
            b, i, j = synth.decode_self_describing(out, 1, rows, cols)
            jj, ii = np.meshgrid(np.arange(cols), np.arange(rows), indexing="ij")
            assert (i == ii).all() and (j == jj).all() and (b == 0).all()


@pytest.mark.parametrize("shape", [(31, 32), (33, 63), (64, 65), (127, 129), (129, 128)])
@pytest.mark.parametrize("es", (4, 8))
def test_self_describing_edges(shape, es):
    rows, cols = shape
    a = synth.self_describing(3, rows, cols, es)
    out = _T(a)
    b, i, j = synth.decode_self_describing(out, 3, rows, cols)
    bb, jj, ii = np.meshgrid(np.arange(3), np.arange(cols), np.arange(rows), indexing="ij")
    assert (b == bb).all() and (i == ii).all() and (j == jj).all()


@pytest.mark.parametrize("es", ES_ALL)
@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (40, 3), (65, 129)])
def test_involution(es, shape):
    a = synth.random_bits(shape, es, 23)
    assert _T(_T(a)).tobytes() == a.tobytes()


@pytest.mark.parametrize("es", (4, 8))
def test_row_vector_is_memcpy(es):
    a = synth.random_bits((1, 4097), es, 29)
    assert _T(a).tobytes() == a.tobytes()
    assert _T(a.reshape(4097, 1)).tobytes() == a.tobytes()


def test_symmetric_fixed_point():
    r = synth.random_bits((64, 64), 8, 31)
    s = np.triu(r) + np.triu(r, 1).T
    assert _T(s).tobytes() == s.tobytes()


def test_block_identity():
    """[[A, B], [C, D]]^T == [[A^T, C^T], [B^T, D^T]] (blocks of unequal size)."""
    m = synth.random_bits((50, 70), 4, 37)
    A, B, C, D = m[:20, :45], m[:20, 45:], m[20:, :45], m[20:, 45:]
    top = np.concatenate([_T(A), _T(C)], axis=1)
    bot = np.concatenate([_T(B), _T(D)], axis=1)
    assert _T(m).tobytes() == np.concatenate([top, bot], axis=0).tobytes()


def test_permutation_multiset():
    a = synth.random_bits((123, 77), 4, 41)
    assert np.array_equal(np.sort(_T(a).ravel()), np.sort(a.ravel()))


@pytest.mark.parametrize("es", (4, 8))
def test_padded_ld_and_guard_bands(es):
    """T4: 67x131 with ld_in=136, ld_out=70 and 4 KiB sentinel bands: only the
    logical cols x rows region of out is written (reading R8)."""
    rows, cols, ld_in, ld_out = 67, 131, 136, 70
    guard = 4096 // es
    ut = synth.UINT_OF_SIZE[es]
    src = synth.self_describing(1, rows, cols, es)[0]
    inb = np.zeros(rows * ld_in, dtype=ut)
    inb.reshape(rows, ld_in)[:, :cols] = src
    outb = np.full(guard + cols * ld_out + guard, 0xA5A5A5A5A5A5A5A5 & ((1 << (8 * es)) - 1), dtype=ut)
    sentinel = outb[0]
    oracle.transpose_raw(inb, outb, 1, rows, cols, ld_in, ld_out, 0, 0, es, out_offset=guard)
    body = outb[guard:guard + cols * ld_out].reshape(cols, ld_out)
    assert body[:, :rows].tobytes() == np.ascontiguousarray(src.T).tobytes()
    assert (body[:, rows:] == sentinel).all()
    assert (outb[:guard] == sentinel).all() and (outb[guard + cols * ld_out:] == sentinel).all()


def test_empty_and_invalid():
    a = np.zeros((0, 5), dtype=np.float32)
    assert _T(a).shape == (5, 0)
    buf = np.zeros(16, dtype=np.uint32)
    with pytest.raises(ValueError):
        oracle.transpose_raw(buf, buf.copy(), 1, 4, 4, 3, 4, 0, 0, 4)   # ld_in < cols


def test_dist_expected_slab_partition():
    """R13: rank slabs of the distributed transpose concatenate to the global transpose."""
    g = synth.random_bits((64, 64), 4, 43)
    for P in (1, 2, 4, 8):
        slabs = [oracle.dist_expected_slab(g, r, P) for r in range(P)]
        assert np.concatenate(slabs, axis=0).tobytes() == np.ascontiguousarray(g.T).tobytes()


# --------------------------------------------------------------- mutation teeth
def _mutant_copy(a):           # forgets to transpose (shape fixed up)
    return np.ascontiguousarray(a).reshape(a.shape[1], a.shape[0])


def _mutant_offbyone(a):       # drops the last source column
    out = np.ascontiguousarray(a.T).copy()
    out[-1, :] = 0
    return out


def _mutant_swapped_ld(a):     # reads with ld_out instead of ld_in
    rows, cols = a.shape
    flat = np.ascontiguousarray(a).reshape(-1)
    out = np.empty((cols, rows), dtype=a.dtype)
    for i in range(rows):
        for j in range(cols):
            out[j, i] = flat[(i * rows + j) % flat.size]
    return out


@pytest.mark.parametrize("mutant", [_mutant_copy, _mutant_offbyone, _mutant_swapped_ld,
                                    lambda a: views.listing2_transpose(a, literal=True)])
def test_pins_catch_mutants(mutant):
    rows = cols = 64
    a = synth.self_describing(1, rows, cols, 4)[0]
    if mutant is _mutant_swapped_ld:
        a = synth.self_describing(1, 48, 64, 4)[0]
        rows, cols = 48, 64
    got = mutant(a)
    b, i, j = synth.decode_self_describing(got, 1, rows, cols)
    jj, ii = np.meshgrid(np.arange(cols), np.arange(rows), indexing="ij")
    decode_ok = got.shape == (cols, rows) and (i == ii).all() and (j == jj).all()
    numpy_ok = got.tobytes() == np.ascontiguousarray(a.T).tobytes()
    assert not decode_ok and not numpy_ok


def test_fullcheck_closed_form_pinned_to_oracle():
    """tests/fullcheck.py (the every-element check used at 65536^2) agrees with the oracle on
    small hash-filled matrices: 0 mismatches for the oracle's transpose (whole matrix and a
    row slab of it), exactly the planted ones otherwise, and a copy without transpose fails."""
    import torch
    from tests.fullcheck import hash_transpose_mismatches
    seed = synth.BASE_SEED + 5
    for M, N, es in ((96, 160, 4), (64, 40, 8), (1, 7, 4)):
        x = torch.empty((M, N), dtype=torch.int32 if es == 4 else torch.int64)
        synth.hash_fill_torch(x, 0, 0, N, seed)
        a = x.numpy().view(synth.UINT_OF_SIZE[es])
        ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
        assert a.tobytes() == synth.hash_expected_np(ii, jj, N, seed, es).tobytes()
        t = oracle.transpose(a)                                  # N x M
        y = torch.from_numpy(t.view(np.int32 if es == 4 else np.int64).copy())
        assert hash_transpose_mismatches(y, 0, N, seed, chunk_rows=7) == (0, None)
        r0 = N // 3
        assert hash_transpose_mismatches(y[r0:], r0, N, seed, chunk_rows=5) == (0, None)
        if M > 1:
            y2 = y.clone()
            y2[N - 1, M // 2] ^= 1 << 5
            assert hash_transpose_mismatches(y2, 0, N, seed) == (1, (N - 1, M // 2))
            wrong = torch.from_numpy(np.ascontiguousarray(
                a.view(np.int32 if es == 4 else np.int64).reshape(N, M)))   # copy, no transpose
            assert hash_transpose_mismatches(wrong, 0, N, seed)[0] > 0
