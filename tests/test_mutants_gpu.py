"""Test teeth on the GPU: the parity checks must FAIL on each deliberately
broken build of the CUDA path, and pass on the product build.

The defects (paper_2305_03448_b200/csrc/mutants.cuh) are compiled only into a variant library
(-DDESC_MUTANTS -> build_variants/libdesc_mutants.so); DESC_MUTANT=<id> picks one at run time.
Each run is a subprocess executing tests/mutant_gauntlet.py, so a defect that faults the
context cannot take the test process down with it.

Deterministic defects must fail at least one check, and the check families that must catch
them are named below.  MUT_TMA2_NO_FENCE (a missing proxy fence / WAR wait) is a race that
may or may not manifest: its outcome is recorded, never asserted.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

MUTANT_LIB = os.path.join(ROOT, "build_variants", "libdesc_mutants.so")
GAUNTLET = os.path.join(ROOT, "tests", "mutant_gauntlet.py")

# id -> (name, checks of which at least one must fail); ids as in mutants.cuh
DETERMINISTIC = {
    1: ("SMEM_TILE_ONLY (Listing 2 read literally)", ["smem_padded_f32", "smem_described_i32"]),
    2: ("SMEM_NO_PAREN (P:44 missing parentheses)", ["smem_padded_f32", "smem_described_i32"]),
    3: ("SMEM_FLOAT_TMP (float staging of f64, P:51)", ["smem_random_f64"]),
    4: ("SMEM_EDGE (copy-out predicate off by one)", ["smem_padded_f32"]),
    5: ("SWAP_LD (ld_in / ld_out swapped)", ["smem_padded_f32", "tma_padded_f32"]),
    6: ("TMA2_NO_MICRO (chunks not transposed)", ["tma_described_f32", "tma_random_f64"]),
    7: ("TMA2_NO_TAIL (ragged columns dropped)", ["tma_padded_f32", "tma_padded_f64"]),
    8: ("TMA2_NO_SWIZZLE (swizzled stage read linearly)", ["tma_described_f32", "tma_random_f64"]),
    10: ("SCAN_NO_LOOKBACK (tile prefixes dropped)",
         ["scan_stream_i32", "scan_lookback_i32", "scan_three_pass_i32"]),
    11: ("REDUCE_NO_TAIL (scalar tail dropped)", ["reduce_i32"]),
    12: ("TILED_TILE_ONLY (tile copied out untransposed)", ["tiled_described_f32", "tiled_random_f64"]),
    13: ("TILED_EDGE (edge store predicate off by one)", ["tiled_padded_f32", "tiled_padded_f64"]),
    15: ("SCAN_LC_NO_SWIZZLE (TMA-store staging written linearly)", ["scan_stream_i32"]),
}
RACE_ONLY = {9: "TMA2_NO_FENCE (proxy fence and WAR wait removed)",
             14: "TILED_NO_SYNC (staging / copy-out barrier removed; TILED and VTILED)",
             16: "SCAN_LC_NO_WAIT (staging rewritten before the TMA store read it; no proxy fence)"}
# the TILED defects compiled into the 16-byte vector tile kernel too (csrc/vtiled_transpose.cuh):
# a second family that must catch them independently
ALSO = {12: ["vtiled_described_f32", "vtiled_random_f64"]}


def _mutant_lib():
    from paper_2305_03448_b200 import build as b
    srcs = b.sources()
    if not os.path.exists(MUTANT_LIB) or any(os.path.getmtime(s) > os.path.getmtime(MUTANT_LIB)
                                             for s in srcs):
        os.makedirs(os.path.dirname(MUTANT_LIB), exist_ok=True)
        b.build(defines=["DESC_MUTANTS"], out=MUTANT_LIB)
    return MUTANT_LIB


def _run(lib=None, mutant=None):
    env = dict(os.environ)
    env.pop("DESC_LIB", None)
    env.pop("DESC_MUTANT", None)
    if lib:
        env["DESC_LIB"] = lib
    if mutant is not None:
        env["DESC_MUTANT"] = str(mutant)
    p = subprocess.run([sys.executable, GAUNTLET], env=env, capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    if not lines:   # the process died: every check counts as failed
        return {"_died": True, "_stderr": p.stderr[-2000:]}
    return json.loads(lines[-1])


@pytest.fixture(scope="module")
def mutant_lib():
    return _mutant_lib()


def _checks(res):
    return {k: v for k, v in res.items() if not k.startswith("_") and not k.endswith("_error")}


def test_product_build_passes_gauntlet():
    res = _run()
    assert not res.get("_died"), res
    failed = [k for k, v in _checks(res).items() if not v]
    assert not failed, res


def test_mutant_build_without_defect_passes(mutant_lib):
    res = _run(mutant_lib, 0)
    assert not res.get("_died"), res
    failed = [k for k, v in _checks(res).items() if not v]
    assert not failed, res


@pytest.mark.parametrize("mid", sorted(DETERMINISTIC))
def test_defect_is_caught(mutant_lib, mid):
    name, must = DETERMINISTIC[mid]
    res = _run(mutant_lib, mid)
    if res.get("_died"):
        return      # the defect crashed the process: caught
    checks = _checks(res)
    for fam in [must] + ([ALSO[mid]] if mid in ALSO else []):
        caught = [k for k in fam if not checks.get(k, False)]
        assert caught, f"{name}: none of {fam} failed: {res}"


@pytest.mark.parametrize("mid", sorted(RACE_ONLY))
def test_race_defect_recorded(mutant_lib, mid):
    res = _run(mutant_lib, mid)
    failed = [k for k, v in _checks(res).items() if not v]
    print(f"{RACE_ONLY[mid]}: failed checks {failed or 'none (race did not manifest)'}")
