"""Host restatements of the CUDA kernels' index maps, and the checks run on them (tests only).

The executable analog of Descend's access-safety check (§3.3 "Narrowing", P:596-599:
each block / thread a distinct part of the output; §4 typing, access_safety_check,
P:1006-1011) and of the race definition of §2.2: for every kernel variant the (CTA,
thread, k) -> (source, destination) maps of csrc/*.cuh are restated below in numpy, line by
line (each function cites the lines it mirrors), a launch is "executed" on element ids, and
``check_launch`` asserts

  * global: every logical output element (b, j, i) is written EXACTLY once, with the id of
    input element (b, i, j) (the transpose), and no padding / guard element is
    written -- the write-after-write race on global memory that racecheck cannot see
    (P:165-175);
  * shared memory: inside every barrier interval, a cell that one thread writes is touched by
    no other thread (no WAW / RAW / WAR hazard), and every cell read was written
    (by a thread or by the TMA unit) before the barrier that precedes the read;
  * TMA kernels: every 8-lane phase of each 16-byte shared-memory access hits 8 distinct
    16-byte bank groups (DESIGN.md §6 "bank-conflict freedom"), and the swizzled addresses
    of a tile form a bijection.

Element ids: input element at flat offset o has id o; -1 = never written; -2 = a TMA
zero-fill (out-of-range box element).
"""
from __future__ import annotations

import numpy as np

from oracle import views as V

UNWRITTEN = -1
ZERO_FILL = -2


class Launch:
    """What one launch did: global writes and shared-memory events (per CTA interval)."""

    def __init__(self):
        self.dst = []      # flat output offsets written
        self.val = []      # id written there
        self.smem = []     # (interval key, thread ids, cell ids, is_write)
        self.unwritten_reads = 0
        self.bank_conflicts = 0

    def write(self, dst, val):
        self.dst.append(np.asarray(dst, dtype=np.int64).ravel())
        self.val.append(np.asarray(val, dtype=np.int64).ravel())

    def sm(self, key, thread, cell, is_write):
        thread, cell = np.broadcast_arrays(np.asarray(thread), np.asarray(cell))
        self.smem.append((key, thread.ravel().astype(np.int64), cell.ravel().astype(np.int64),
                          bool(is_write)))


def expected_output(batch, rows, cols, ld_in, ld_out, stride_in, stride_out):
    """(dst offsets, input ids) of the transpose definition: out[b][j][i] = in[b][i][j]."""
    b, i, j = np.meshgrid(np.arange(batch), np.arange(rows), np.arange(cols), indexing="ij")
    return (b * stride_out + j * ld_out + i).ravel(), (b * stride_in + i * ld_in + j).ravel()


def check_launch(L: Launch, batch, rows, cols, ld_in, ld_out, stride_in, stride_out):
    """Returns a list of violations (empty = the launch is a race-free bijection onto the
    logical output with the transpose's values)."""
    errs = []
    dst = np.concatenate(L.dst) if L.dst else np.zeros(0, np.int64)
    val = np.concatenate(L.val) if L.val else np.zeros(0, np.int64)
    edst, eval_ = expected_output(batch, rows, cols, ld_in, ld_out, stride_in, stride_out)
    logical = np.zeros(0, np.int64) if edst.size == 0 else edst
    inside = np.isin(dst, logical)
    if (~inside).any():
        errs.append(f"{int((~inside).sum())} writes outside the logical output (padding / guard), "
                    f"first at {dst[~inside][:4]}")
    uniq, counts = np.unique(dst, return_counts=True)
    if (counts > 1).any():
        errs.append(f"{int((counts > 1).sum())} output elements written more than once "
                    f"(global WAW), first at {uniq[counts > 1][:4]}")
    missing = np.setdiff1d(logical, dst)
    if missing.size:
        errs.append(f"{missing.size} output elements never written, first at {missing[:4]}")
    exp = dict(zip(edst.tolist(), eval_.tolist()))
    wrong = [(d, v) for d, v in zip(dst.tolist(), val.tolist()) if d in exp and exp[d] != v]
    if wrong:
        errs.append(f"{len(wrong)} elements carry the wrong source, first (dst, id) {wrong[:3]}")
    errs += smem_hazards(L)
    if L.unwritten_reads:
        errs.append(f"{L.unwritten_reads} shared-memory reads of never-written cells")
    if L.bank_conflicts:
        errs.append(f"{L.bank_conflicts} 16-byte shared-memory phases with a bank conflict")
    return errs


def smem_hazards(L: Launch):
    """within one barrier interval of one CTA, a cell written by a thread must not be
    read or written by any other thread."""
    by_key = {}
    for key, th, cell, w in L.smem:
        by_key.setdefault(key, []).append((th, cell, np.full(th.shape, w)))
    bad = 0
    for key, evs in by_key.items():
        th = np.concatenate([e[0] for e in evs])
        cell = np.concatenate([e[1] for e in evs])
        w = np.concatenate([e[2] for e in evs])
        wc = np.unique(cell[w])
        sel = np.isin(cell, wc)
        if not sel.any():
            continue
        c, t = cell[sel], th[sel]
        order = np.lexsort((t, c))
        c, t = c[order], t[order]
        starts = np.r_[True, c[1:] != c[:-1]]
        first_t = t[np.maximum.accumulate(np.where(starts, np.arange(c.size), 0))]
        bad += int(np.unique(c[t != first_t]).size)
    return [f"{bad} shared-memory cells accessed by two threads in one barrier interval "
            "with at least one write (race, P:163)"] if bad else []


# ------------------------------------------------------------------ TILED (AUTO's kernel)
def tiled_cfg(es):
    """desc_transpose.cu run_tiled defaults: 32 x 32 tiles with 128 threads for 8-byte cells,
    64 x 64 with 256 threads otherwise -> (TR, TC, NT)."""
    return (32, 32, 128) if es == 8 else (64, 64, 256)


def tiled_launch(batch, rows, cols, ld_in, ld_out, stride_in, stride_out, es, mutant=None,
                 TR=None, TC=None, NT=256):
    """csrc/tiled_transpose.cuh transpose_tiled_kernel restated.  One NT-thread CTA per tile
    (launcher desc_transpose.cu launch_tiled: grid = ntiles); mutant in {None, "tile_only"
    (12), "edge" (13), "no_sync" (14)}."""
    if TR is None:
        TR, TC, NT = tiled_cfg(es)
    NW = NT // 32
    CW, RK = TC // 32, TR // NW
    LPR = min(TR, 32)
    RPI = 32 // LPR
    OK, OH = TC // (RPI * NW), TR // LPR
    tiles_r, tiles_c = -(-rows // TR), -(-cols // TC)
    L = Launch()
    tid = np.arange(NT)
    tx, ty = tid & 31, tid >> 5
    ox, oy = tx % LPR, tx // LPR
    k = np.arange(RK)
    g = np.arange(CW)
    r = (ty[:, None, None] + NW * k[None, :, None]) + 0 * g[None, None, :]     # rows ty + NW k
    c = (tx[:, None, None] + 32 * g[None, None, :]) + 0 * k[None, :, None]     # cols tx + 32g
    th_l = np.broadcast_to(tid[:, None, None], r.shape)
    m = np.arange(OK)
    h = np.arange(OH)
    oc = (RPI * (ty[:, None, None] + NW * m[None, :, None]) + oy[:, None, None]) + 0 * h[None, None, :]
    orr = (ox[:, None, None] + LPR * h[None, None, :]) + 0 * m[None, :, None]
    th_o = np.broadcast_to(tid[:, None, None], oc.shape)
    for t in range(tiles_r * tiles_c * batch):
        bt, rem = divmod(t, tiles_r * tiles_c)
        ti, tj = divmod(rem, tiles_c)
        r0, c0 = ti * TR, tj * TC
        full = r0 + TR <= rows and c0 + TC <= cols
        nr, nc = min(rows - r0, TR), min(cols - c0, TC)
        tile = np.full((TR, TC + 1), UNWRITTEN, dtype=np.int64)
        mask = np.ones(r.shape, bool) if full else (r < nr) & (c < nc)
        src = bt * stride_in + (r0 + r) * ld_in + c0 + c
        tile[r[mask], c[mask]] = src[mask]
        L.sm((t, 0), th_l[mask], r[mask] * (TC + 1) + c[mask], True)
        iv = 0 if mutant == "no_sync" else 1                      # the staging barrier
        lim_r = nr + (1 if mutant == "edge" else 0)
        mo = np.ones(oc.shape, bool) if full else (oc < nc) & (orr < lim_r)
        rr, cc = (oc, orr) if mutant == "tile_only" else (orr, oc)
        rr_m, cc_m = rr[mo], cc[mo]
        inb = (rr_m < TR) & (cc_m < TC + 1)
        vals = np.full(rr_m.shape, UNWRITTEN, dtype=np.int64)
        vals[inb] = tile[rr_m[inb], cc_m[inb]]
        L.unwritten_reads += int((vals == UNWRITTEN).sum())
        L.sm((t, iv), th_o[mo], rr_m * (TC + 1) + cc_m, False)
        L.write(bt * stride_out + (c0 + oc[mo]) * ld_out + r0 + orr[mo], vals)
    return L


# ------------------------------------------------------------------ VTILED (16-byte vectors)
def vtiled_launch(batch, rows, cols, ld_in, ld_out, stride_in, stride_out, es, TCH=None, NT=None,
                  mutant=None, swizzle=True):
    """csrc/vtiled_transpose.cuh transpose_vtiled_kernel restated at element granularity.
    Tile TR = 16 VEC rows x TCH 16-byte chunks (VEC = 16 / es cells each), one NT-thread CTA
    per tile (desc_transpose.cu run_vtiled defaults: 64 x 64 cells / 128 threads for 4-byte
    cells, 32 x 32 / 64 for 8-byte, 128 x 64 / 128 for 2-byte, 256 x 128 / 128 for 1-byte).  Copy-in: chunk q = tid + NT k -> row q / TCH, chunk
    q % TCH, stored at chunk (q % TCH) ^ ((row / VEC) & 7); copy-out: micro-block b = tid +
    NT m -> (mr, mc) = (b % 16, b / 16), VEC 16-byte reads of rows VEC mr + k at chunk
    mc ^ (mr & 7), output row VEC mc + j gets cells x[k][j].  mutant in {None, "tile_only"
    (12: o = x[j], untransposed), "no_sync" (14)}; swizzle=False drops the XOR (a teeth check
    for the conflict counter); requires rows, cols multiples of VEC."""
    sw = 1 if swizzle else 0
    VEC = 16 // es
    if TCH is None:
        TCH, NT = {8: (16, 64), 4: (16, 128), 2: (8, 128), 1: (8, 128)}[es]
    TR, TC = 16 * VEC, TCH * VEC
    assert rows % VEC == 0 and cols % VEC == 0
    tiles_r, tiles_c = -(-rows // TR), -(-cols // TC)
    L = Launch()
    tid = np.arange(NT)
    e = np.arange(VEC)
    for t in range(tiles_r * tiles_c * batch):
        bt, rem = divmod(t, tiles_r * tiles_c)
        ti, tj = divmod(rem, tiles_c)
        r0, c0 = ti * TR, tj * TC
        full = r0 + TR <= rows and c0 + TC <= cols
        nr, nc = min(rows - r0, TR), min(cols - c0, TC)
        tile = np.full(TR * TCH * VEC, UNWRITTEN, dtype=np.int64)
        for k in range(TR * TCH // NT):                                    # copy-in
            q = tid + NT * k
            w, c = q // TCH, q % TCH
            mk = np.ones(NT, bool) if full else (w < nr) & (c * VEC < nc)
            phys = w * TCH + (c ^ (sw * ((w // VEC) & 7)))
            for p in range(NT // 8):                                       # 8-lane phases
                sel = slice(8 * p, 8 * p + 8)
                if mk[sel].all() and np.unique(phys[sel] & 7).size != 8:
                    L.bank_conflicts += 1
            cells = phys[mk][:, None] * VEC + e[None, :]
            src = bt * stride_in + (r0 + w[mk])[:, None] * ld_in + c0 + (c[mk] * VEC)[:, None] + e[None, :]
            tile[cells] = src
            L.sm((t, 0), np.broadcast_to(tid[mk][:, None], cells.shape), cells, True)
        iv = 0 if mutant == "no_sync" else 1
        for m in range(16 * TCH // NT):                                    # copy-out
            b = tid + NT * m
            mr, mc = b & 15, b >> 4
            mk = np.ones(NT, bool) if full else (VEC * mr < nr) & (VEC * mc < nc)
            x = np.zeros((NT, VEC, VEC), dtype=np.int64)                   # [thread][k][cell]
            for k in range(VEC):
                phys = (VEC * mr + k) * TCH + (mc ^ (sw * (mr & 7)))
                for p in range(NT // 8):
                    sel = slice(8 * p, 8 * p + 8)
                    if mk[sel].all() and np.unique(phys[sel] & 7).size != 8:
                        L.bank_conflicts += 1
                cells = phys[:, None] * VEC + e[None, :]
                x[:, k, :] = tile[cells]
                L.unwritten_reads += int((x[mk, k, :] == UNWRITTEN).sum())
                L.sm((t, iv), np.broadcast_to(tid[mk][:, None], cells[mk].shape), cells[mk], False)
            for j in range(VEC):
                mj = mk & ((VEC * mc + j < nc) | full)
                o = x[:, j, :] if mutant == "tile_only" else x[:, :, j]    # o[k] = x[k][j]
                dst = (bt * stride_out + (c0 + VEC * mc + j)[:, None] * ld_out + r0
                       + (VEC * mr)[:, None] + e[None, :])
                L.write(dst[mj], o[mj])
    return L


# ------------------------------------------------------------------ SMEM (Listing 1 schedule)
def smem_launch(batch, rows, cols, ld_in, ld_out, stride_in, stride_out, es, grid=None,
                mutant=None):
    """csrc/smem_transpose.cuh:18-57 restated (the corrected Listing 1, P:49-60 with the P:44
    fix).  grid CTAs of 32 x 8 threads loop over the tiles (t += gridDim.x); mutant in
    {None, "tile_only" (1), "no_paren" (2: Listing 1 as printed, tmp[ty + j*32 + tx]),
    "edge" (4)}."""
    tiles_r, tiles_c = -(-rows // 32), -(-cols // 32)
    ntiles = tiles_r * tiles_c * batch
    grid = ntiles if grid is None else grid
    L = Launch()
    tx, ty = np.meshgrid(np.arange(32), np.arange(8), indexing="xy")           # [ty][tx]
    tid = (ty * 32 + tx)
    for blk in range(grid):
        for n_it, t in enumerate(range(blk, ntiles, grid)):                     # :26
            bt, rem = divmod(t, tiles_r * tiles_c)
            ti, tj = divmod(rem, tiles_c)
            tile = np.full(32 * 33, UNWRITTEN, dtype=np.int64)
            key = (blk, n_it)
            for j in range(0, 32, 8):                                           # :34-45
                i, c = ti * 32 + ty + j, tj * 32 + tx
                mk = (i < rows) & (c < cols)
                cell = (ty + j * 33 + tx) if mutant == "no_paren" else (ty + j) * 33 + tx
                src = bt * stride_in + i * ld_in + c
                tile[cell[mk]] = src[mk]
                L.sm(key + (0,), tid[mk], cell[mk], True)
            for j in range(0, 32, 8):                                           # :48-54 after :46
                orow, ocol = tj * 32 + ty + j, ti * 32 + tx
                lim = rows + (1 if mutant == "edge" else 0)
                mk = (orow < cols) & (ocol < lim)
                cell = (ty + j) * 33 + tx if mutant == "tile_only" else tx * 33 + ty + j
                vals = tile[cell[mk]]
                L.unwritten_reads += int((vals == UNWRITTEN).sum())
                L.sm(key + (1,), tid[mk], cell[mk], False)
                L.write(bt * stride_out + orow[mk] * ld_out + ocol[mk], vals)
    return L


# ------------------------------------------------------------------ TMA kernels
def _swz(row, chunk):
    """CU_TENSOR_MAP_SWIZZLE_128B: 16-byte chunk c of box row r sits at chunk c ^ (r & 7)."""
    return chunk ^ (row & 7)


def _tile_coords(t, tiles_r, tiles_c, group):
    """csrc/tma_transpose.cuh:71-84 (tile_coords)."""
    per_mat = tiles_r * tiles_c
    bt, rem = divmod(t, per_mat)
    per_group = group * tiles_c
    gi, in_g = divmod(rem, per_group)
    g0 = gi * group
    gsz = min(group, tiles_r - g0)
    tj, off = divmod(in_g, gsz)
    return bt, g0 + off, tj


def _box_load(stage, box, ld_in, stride_in, bt, r0, c0, TR, TC, VEC, rows, cols):
    """A TMA box load (TR rows x 128 bytes) into `stage` (element granularity, swizzled):
    elements outside [0, rows) x [0, cols) are zero-filled (TMA OOB fill)."""
    rr, cc = np.meshgrid(np.arange(TR), np.arange(TC), indexing="ij")
    gi, gj = r0 + rr, c0 + cc
    ids = np.where((gi < rows) & (gj < cols) & (gi >= 0), bt * stride_in + gi * ld_in + gj, ZERO_FILL)
    phys = box * TR * TC + rr * TC + _swz(rr, cc // VEC) * VEC + cc % VEC
    stage[phys] = ids


class _Lanes:
    """Lane maps: StoreLane<ES> (csrc/tma_store_transpose.cuh:34-59) for the TMA-store kernel,
    the generic a/b split (csrc/tma_transpose.cuh:255-258) for the TMA-load kernel."""

    def __init__(self, es, store: bool):
        lane = np.arange(32)
        self.VEC = 16 // es
        if store:
            self.b = lane & 3
            if es == 4:
                self.a, self.flip = lane >> 2, lane & 2
            else:
                self.a = ((lane >> 3) & 1) | (((lane >> 2) & 1) << 1) | (((lane >> 4) & 1) << 2)
                self.flip = lane & 1
            self.cpw, self.apw = 4, 8
        else:
            logvec = {16: 4, 8: 3, 4: 2, 2: 1}[self.VEC]
            BB = min(logvec, 3)
            self.b = lane & ((1 << BB) - 1)
            self.a = (lane >> 3) * (1 << (3 - BB)) + ((lane >> BB) & ((1 << (3 - BB)) - 1))
            self.flip = np.zeros(32, dtype=np.int64)
            self.cpw, self.apw = 1 << BB, 1 << (5 - BB)


def _phase_conflicts(chunks_phys):
    """Per 8-lane phase of a 16-byte access: the 8 physical chunk slots (addr / 16 mod 8) must
    be distinct."""
    bad = 0
    for p in range(4):
        if np.unique(chunks_phys[8 * p:8 * p + 8] & 7).size != 8:
            bad += 1
    return bad


def tma_launch(batch, rows, cols, ld_in, ld_out, stride_in, stride_out, es, TR=128, NB=1,
               CW=8, grid=None, group=None, store=True, mutant=None):
    """The persistent TMA kernels restated at element granularity.

    store=True : transpose_tma2_kernel, csrc/tma_store_transpose.cuh:96-276 (TMA load, register
                 micro-transpose, swizzled output staging, TMA store clipped at rows_main,
                 ragged tail by the lanes that own it); mutant in {None, "no_micro" (6),
                 "no_tail" (7), "no_swizzle" (8)}.
    store=False: transpose_tma_kernel, csrc/tma_transpose.cuh:198-309 (TMA load, 16-byte
                 st.global of the micro-transposed rows, partial edge chunks)."""
    Ln = _Lanes(es, store)
    VEC, TC = Ln.VEC, 128 // es
    TILE_COLS = NB * TC
    RPW = Ln.apw * VEC                      # input rows per warp-task
    CG = 8 // Ln.cpw                        # chunk groups
    TPB = (TR // RPW) * CG                  # tasks per box
    TASKS = TPB * NB
    TPW = TASKS // CW
    assert TASKS % CW == 0 and TR % RPW == 0
    tiles_r, tiles_c = -(-rows // TR), -(-cols // TILE_COLS)
    ntiles = tiles_r * tiles_c * batch
    group = tiles_r if group is None else min(group, tiles_r)
    grid = ntiles if grid is None else grid
    rows_main = rows - rows % VEC
    OBOXES = TR * es // 128
    L = Launch()
    lane = np.arange(32)
    seen_tiles = []
    for blk in range(grid):
        for it, t in enumerate(range(blk, ntiles, grid)):                     # static schedule
            seen_tiles.append(t)
            bt, ti, tj = _tile_coords(t, tiles_r, tiles_c, group)
            stage = np.full(NB * TR * TC, UNWRITTEN, dtype=np.int64)
            for nb in range(NB):                                               # producer
                _box_load(stage, nb, ld_in, stride_in, bt, ti * TR, tj * TILE_COLS + nb * TC,
                          TR, TC, VEC, rows, cols)
            ostage = np.full(OBOXES * TILE_COLS * TC, UNWRITTEN, dtype=np.int64)
            key = (blk, it)
            for cw in range(CW):
                for q in range(TPW):
                    T = cw + q * CW
                    box, tib = divmod(T, TPB)
                    rgrp = tib // CG
                    chunk = (tib % CG) * Ln.cpw + Ln.b
                    row0 = VEC * (rgrp * Ln.apw + Ln.a)
                    # consumer reads: r[k] = 16-byte chunk `chunk` of box row row0+k
                    rk = np.zeros((32, VEC, VEC), dtype=np.int64)               # [lane][k][e]
                    for k in range(VEC):
                        row = row0 + k
                        sw = 0 if mutant == "no_swizzle" else (row & 7)
                        pch = chunk ^ sw
                        L.bank_conflicts += _phase_conflicts(pch)
                        base = box * TR * TC + row * TC + pch * VEC
                        rk[:, k, :] = stage[base[:, None] + np.arange(VEC)[None, :]]
                        L.unwritten_reads += int((rk[:, k, :] == UNWRITTEN).sum())
                    # micro-transpose: output row J, element e = r[e][J]  (micro_row)
                    mic = np.transpose(rk, (0, 2, 1))                           # [lane][J][e]
                    if mutant == "no_micro":
                        mic = rk
                    orow0 = VEC * (box * 8 + chunk)     # output row in tile (input column)
                    if store:
                        for JJ in range(VEC):          # store instruction JJ (:228-238):
                            Jl = JJ ^ Ln.flip              # lane writes row orow0 + (JJ ^ f)
                            row = orow0 + Jl               # with rotated_row<JJ> = micro row
                            c = Ln.a                       # JJ ^ f; 16-byte chunk a in box
                            pch = c ^ (row & 7)
                            L.bank_conflicts += _phase_conflicts(pch)
                            base = rgrp * TILE_COLS * TC + row * TC + pch * VEC
                            idx = base[:, None] + np.arange(VEC)[None, :]
                            ostage[idx] = mic[lane, Jl, :]
                            L.sm(key + (1,), np.repeat(cw * 32 + lane, VEC), idx.ravel(), True)
                        # ragged tail (rows % VEC): the lanes at in_row0 == rows_main
                        in_row0 = ti * TR + row0
                        if rows_main != rows and mutant != "no_tail":
                            sel = np.nonzero(in_row0 == rows_main)[0]
                            for ln in sel:
                                _emit(L, mic[ln], bt, stride_out, ld_out,
                                      tj * TILE_COLS + orow0[ln], in_row0[ln], cols,
                                      rows - rows_main, VEC)
                    else:
                        in_row0 = ti * TR + row0
                        for ln in range(32):
                            nvalid = min(rows - in_row0[ln], VEC)
                            if nvalid > 0:
                                _emit(L, mic[ln], bt, stride_out, ld_out,
                                      tj * TILE_COLS + box * TC + VEC * chunk[ln], in_row0[ln],
                                      cols, nvalid, VEC)
            if store:
                # TMA stores (after fence + named barrier): box o -> output columns
                # ti*TR + o*TC .. (input rows), output rows tj*TILE_COLS .., clipped at
                # rows_main x cols (tma_store_transpose.cuh:263-272; out_map in
                # desc_transpose.cu clips at rows rounded down to 16 bytes)
                for o in range(OBOXES):
                    rr, cc = np.meshgrid(np.arange(TILE_COLS), np.arange(TC), indexing="ij")
                    orow_g, ocol_g = tj * TILE_COLS + rr, ti * TR + o * TC + cc
                    ok = (orow_g < cols) & (ocol_g < rows_main)
                    phys = o * TILE_COLS * TC + rr * TC + _swz(rr, cc // VEC) * VEC + cc % VEC
                    vals = ostage[phys[ok]]
                    L.unwritten_reads += int((vals == UNWRITTEN).sum())
                    L.sm(key + (2,), np.full(vals.shape, -100), phys[ok], False)
                    L.write(bt * stride_out + orow_g[ok] * ld_out + ocol_g[ok], vals)
    if sorted(seen_tiles) != list(range(ntiles)):
        L.dst.append(np.array([-1]))          # a tile scheduled twice / never: flagged
        L.val.append(np.array([-1]))
    return L


def _emit(L, mic, bt, stride_out, ld_out, orow0, in_row0, cols, nvalid, VEC):
    """emit_rows / emit_row / store_partial (csrc/tma_transpose.cuh:137-175): output row
    orow0 + J (if < cols) gets the first nvalid elements of micro row J at column in_row0."""
    for J in range(VEC):
        orow = orow0 + J
        if orow < cols:
            e = np.arange(nvalid)
            L.write(bt * stride_out + orow * ld_out + in_row0 + e, mic[J, :nvalid])


# ------------------------------------------------------------------ views (Listing 3)
def thread_conflicts(writes: np.ndarray, reads: np.ndarray | None = None) -> int:
    """writes[t], reads[t]: the memory cell thread t writes / reads in one phase.  Returns the
    number of cells written by one thread and read or written by another."""
    writes = np.asarray(writes).ravel()
    n = writes.size
    ev_cell = writes
    ev_thr = np.arange(n)
    ev_w = np.ones(n, bool)
    if reads is not None:
        reads = np.asarray(reads).ravel()
        ev_cell = np.r_[ev_cell, reads]
        ev_thr = np.r_[ev_thr, np.arange(reads.size)]
        ev_w = np.r_[ev_w, np.zeros(reads.size, bool)]
    L = Launch()
    L.sm(0, ev_thr[ev_w], ev_cell[ev_w], True)
    if reads is not None:
        L.sm(0, ev_thr[~ev_w], ev_cell[~ev_w], False)
    h = smem_hazards(L)
    return int(h[0].split()[0]) if h else 0


def view_thread_cells(shape, ops):
    """The cells of a root array of `shape` that thread t of a flat schedule over the view
    `ops` (one element per thread, in the view's row-major order) accesses: the view's
    index array from the oracle's definitions (oracle/views.py)."""
    return V.index_view(shape, ops).ravel()


def slab_peer_launches(P, M, N, es, TR=None, TC=None, NT=256):
    """desc_slab_transpose_peer (csrc/desc_transpose.cu run_slab_peer + the SCATTER branch of
    csrc/tiled_transpose.cuh) restated for every rank r of P: rank r's TILED launch over its
    Rm x N slab, each tile routed to destination s = c0 / Rn at column (c - s*Rn), output
    column offset r*Rm.  Returns {s: (dst offsets in slab s, global input ids)} over all
    ranks, plus the number of tiles whose columns straddle two destinations."""
    if TR is None:
        TR, TC, NT = tiled_cfg(es)
    Rm, Rn = M // P, N // P
    per = {s: ([], []) for s in range(P)}
    straddle = 0
    for r in range(P):
        L = tiled_launch(1, Rm, N, N, M, 0, 0, es, TR=TR, TC=TC, NT=NT)
        d = np.concatenate(L.dst)
        v = np.concatenate(L.val)
        c, row = d // M, d % M                     # unscattered: out[c][row], c = input column
        c0 = (c // TC) * TC                         # the tile's first column
        s_tile = c0 // Rn                           # destination the kernel picks (per tile)
        straddle += int((s_tile != c // Rn).sum())
        gid = v + r * Rm * N                        # local ids -> global input ids
        for s in range(P):
            m = s_tile == s
            per[s][0].append((c[m] - s * Rn) * M + r * Rm + row[m])
            per[s][1].append(gid[m])
    return {s: (np.concatenate(a), np.concatenate(b)) for s, (a, b) in per.items()}, straddle
