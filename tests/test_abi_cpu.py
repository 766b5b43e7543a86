"""Host-side tests of the C-ABI library (no GPU needed, no compute calls).

* the library builds for sm_100a, loads, and exports every symbol include/*.h declares;
* the cubin inside is sm_100a SASS with the TMA instruction (UTMALDG) in the TMA kernel;
* argument validation (performed before any CUDA call) returns the documented status codes;
* the product package does not import the oracle and has no CPU fallback.
"""
import ctypes
import glob
import os
import re
import subprocess

import pytest

import paper_2305_03448_b200 as desc
from paper_2305_03448_b200 import build as desc_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    desc_build.build()
    return desc.load()


def _header_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(desc_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(lib):
    names = _header_functions()
    assert {"desc_transpose", "desc_transpose_batched", "desc_transpose_ex"} <= names
    out = subprocess.run(["nm", "-D", "--defined-only", desc.lib_path], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = names - exported
    assert not missing, f"declared but not exported: {missing}"
    for n in names:
        assert getattr(lib, n) is not None


def test_sass_is_sm100a_with_tma(lib):
    out = subprocess.run(["cuobjdump", "-sass", desc.lib_path], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    blocks = out.split("Function : ")[1:]
    tma = [b for b in blocks if "transpose_tma_kernel" in b[:200]]
    tma2 = [b for b in blocks if "transpose_tma2_kernel" in b[:200]]
    assert tma and tma2, "TMA kernels missing from the cubin"
    tile = [b for b in blocks if "transpose_tma_tile_kernel" in b[:200]]
    assert tile, "TMA tile kernel missing from the cubin"
    for blk in tma + tma2 + tile:
        assert "UTMALDG" in blk, "TMA kernel does not issue cp.async.bulk.tensor loads"
        assert "SYNCS" in blk, "TMA kernel does not use mbarriers"
    for blk in tma2 + tile:
        assert "UTMASTG" in blk, "TMA-store kernels must store with cp.async.bulk.tensor"
    for blk in tma2:
        assert "UTMASTG" in blk, "TMA-store kernel does not issue bulk tensor stores"


def test_sass_vtiled_is_16_byte_cp_async(lib):
    """DESC_KERNEL_VTILED (csrc/vtiled_transpose.cuh): every global and shared access 16 bytes
    wide -- cp.async.cg 16-byte copies (LDGSTS.E.BYPASS.128) into shared memory, LDS.128
    micro-block reads, STG.E.128 stores; no 4-byte global access."""
    out = subprocess.run(["cuobjdump", "-sass", desc.lib_path], capture_output=True, text=True,
                         check=True).stdout
    blocks = [b for b in out.split("Function : ")[1:] if "transpose_vtiled_kernel" in b[:200]]
    assert len(blocks) >= 2, "vector tile kernels missing from the cubin"
    for blk in blocks:
        assert "LDGSTS.E.BYPASS.128" in blk and "LDGDEPBAR" in blk
        assert "LDS.128" in blk and "STG.E.128" in blk
        assert "STG.E " not in blk and "LDG.E " not in blk


def test_product_build_carries_no_test_defects(lib):
    """The test-teeth defects (csrc/mutants.cuh) exist only in the -DDESC_MUTANTS variant."""
    with open(desc.lib_path, "rb") as f:
        assert b"g_desc_mutant" not in f.read()


def test_host_helpers(lib):
    assert desc.desc_version() >= 100
    assert desc.desc_dtype_size("f32") == 4 and desc.desc_dtype_size("f64") == 8
    assert desc.desc_dtype_size("i32") == 4 and desc.desc_dtype_size("u8") == 1
    assert desc.desc_dtype_size(99) == 0
    assert desc.desc_status_string(4) == "DESC_ERR_ALIAS"


FAKE_IN, FAKE_OUT = 0x7f0000000000, 0x7f1000000000   # never dereferenced


def _status(fn, *args):
    return getattr(desc.load(), fn)(*args)


def test_validation_codes(lib):
    i, o = FAKE_IN, FAKE_OUT
    # empty shapes: success, no launch (R10)
    assert _status("desc_transpose", i, o, 0, 5, 5, 0, 0, None) == 0
    assert desc.desc_last_launch_count() == 0
    assert _status("desc_transpose_batched", i, o, 0, 4, 4, 4, 4, 16, 16, 0, None) == 0
    # null pointers
    assert _status("desc_transpose", None, o, 4, 4, 4, 4, 0, None) == 1
    assert _status("desc_transpose", i, None, 4, 4, 4, 4, 0, None) == 1
    # shapes
    assert _status("desc_transpose", i, o, 4, 4, 3, 4, 0, None) == 2       # ld_in < cols
    assert _status("desc_transpose", i, o, 4, 4, 4, 3, 0, None) == 2       # ld_out < rows
    assert _status("desc_transpose", i, o, -1, 4, 4, 4, 0, None) == 2
    assert _status("desc_transpose", i, o, 1 << 40, 1 << 40, 1 << 40, 1 << 40, 0, None) == 2
    # batched outputs must be disjoint (narrowing)
    assert _status("desc_transpose_batched", i, o, 2, 4, 8, 8, 4, 32, 31, 0, None) == 2
    # side-by-side batched outputs are disjoint too (the distributed unpack layout)
    assert _status("desc_transpose_batched", i, o, 2, 4, 8, 8, 8, 32, 4, 0, None) in (5, 6)
    assert _status("desc_transpose_batched", i, o, 2, 4, 8, 8, 8, 32, 3, 0, None) == 2
    assert _status("desc_copy_batched", i, o, 4, 8, 16, 16, 64, 128, 16, 0, None) in (5, 6)
    assert _status("desc_copy_batched", i, o, 4, 8, 16, 16, 63, 128, 16, 0, None) == 2
    # dtype
    assert _status("desc_transpose", i, o, 4, 4, 4, 4, 42, None) == 3
    # aliasing: &uniq out overlapping & in
    assert _status("desc_transpose", i, i + 32, 4, 4, 4, 4, 0, None) == 4
    assert _status("desc_transpose", i, i, 4, 4, 4, 4, 0, None) == 4
    assert "overlap" in desc.desc_last_error()
    # unknown kernel variant / TMA on misaligned args are reported, not silently rerouted
    assert _status("desc_transpose_ex", i, o, 1, 4, 4, 4, 4, 0, 0, 0, 2, None) in (5, 6)


def test_host_entry_validation(lib):
    import numpy as np
    h_in = np.zeros(64, dtype=np.float32)
    h_out = np.zeros(64, dtype=np.float32)
    f = "desc_transpose_host"
    args = (h_in.ctypes.data, h_out.ctypes.data)
    assert _status(f, *args, 1, 0, 8, 8, 8, 0, 0, 0, FAKE_OUT, 4096, None) == 0     # empty
    assert _status(f, None, h_out.ctypes.data, 1, 8, 8, 8, 8, 0, 0, 0, FAKE_OUT, 4096, None) == 1
    assert _status(f, *args, 1, 8, 8, 8, 8, 0, 0, 0, None, 4096, None) == 1         # no workspace
    assert _status(f, *args, 1, 8, 8, 7, 8, 0, 0, 0, FAKE_OUT, 4096, None) == 2     # ld_in < cols
    assert _status(f, *args, 1, 8, 8, 8, 8, 0, 0, 42, FAKE_OUT, 4096, None) == 3    # dtype
    assert _status(f, h_in.ctypes.data, h_in.ctypes.data, 1, 8, 8, 8, 8, 0, 0, 0, FAKE_OUT,
                   4096, None) == 4                                                # alias
    # double-buffered 1024-column bands (in: 8192 x 1024, out: 1024 x 8192), r02 band axis
    assert desc.desc_transpose_host_workspace(8192, 8192, "f32") == 2 * 2 * 1024 * 8192 * 4
    assert desc.desc_transpose_host_workspace(0, 8, "f32") == 0
    # batched: ~32 MB of input per whole-matrix band, >= 8 bands, never below the 1-matrix size
    assert desc.desc_transpose_host_workspace_batched(256, 1024, 1024, "f32") == 2 * 8 * 2 * (4 << 20)
    assert desc.desc_transpose_host_workspace_batched(16, 1024, 1024, "f32") == 2 * 2 * 2 * (4 << 20)
    assert desc.desc_transpose_host_workspace_batched(1, 1024, 1024, "f32") == \
        desc.desc_transpose_host_workspace(1024, 1024, "f32")
    # matrices above 32 MB travel one per band (in + out, double-buffered)
    assert desc.desc_transpose_host_workspace_batched(64, 8192, 8192, "f32") == 2 * 2 * (256 << 20)


def test_select_kernel_alignment_rules(lib):
    i, o = FAKE_IN, FAKE_OUT
    assert desc.desc_select_kernel(i, o, 1, 64, 64, 64, 64, 0, 0, "f32") == "tiled"
    assert desc.desc_select_kernel(i, o, 1, 64, 64, 64, 64, 0, 0, "u8") == "vtiled"
    assert desc.desc_select_kernel(i, o, 1, 56, 64, 64, 64, 0, 0, "u8") == "tma"     # 56 % 16
    assert desc.desc_select_kernel(i, o, 1, 2, 64, 64, 4, 0, 0, "f32") == "tma"
    assert desc.desc_select_kernel(i, o, 1, 32, 64, 64, 32, 0, 0, "f32") == "tma_st"   # skinny
    assert desc.desc_select_kernel(i, o, 1, 64, 48, 48, 64, 0, 0, "f64") == "tma_st"
    assert desc.desc_select_kernel(i, o, 1, 64, 64, 64, 64, 0, 0, "bf16") == "vtiled"
    assert desc.desc_select_kernel(i, o, 1, 60, 64, 64, 64, 0, 0, "bf16") == "tma"   # 60 % 8
    assert desc.desc_select_kernel(i + 4, o, 1, 64, 64, 64, 64, 0, 0, "f32") == "tiled"
    assert desc.desc_select_kernel(i, o, 1, 3000, 5001, 5001, 3000, 0, 0, "f64") == "tiled"
    assert desc.desc_select_kernel(i, o, 1, 3000, 5000, 5000, 3000, 0, 0, "f64") == "tiled"
    assert desc.desc_select_kernel(i, o, 1, 3, 5, 5, 3, 0, 0, "f32") == "tiled"
    assert desc.desc_select_kernel(i, o, 2, 64, 64, 64, 64, 4096, 4096, "f32") == "tiled"
    assert desc.desc_select_kernel(i, o, 2, 64, 64, 64, 64, 4097, 4096, "f32") == "tiled"


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2305_03448_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if os.path.isfile(path) and path.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            text = open(path).read()
            assert not re.search(r"^\s*(import|from)\s+oracle\b", text, flags=re.M), path
            assert "transpose_ref" not in text, path
            assert "liboracle" not in text, path


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(desc, "_lib", None)
    monkeypatch.setattr(desc, "lib_path", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        desc.load()


def test_tensor_wrappers_validate_out():
    """block_reduce / scan hand out.data_ptr() to a C ABI that takes no output size: a wrong
    `out` must be refused before any call."""
    import torch
    x = torch.zeros(100, dtype=torch.float32)
    for bad in (torch.zeros(9, dtype=torch.float32), torch.zeros(10, dtype=torch.float64),
                torch.zeros(20, dtype=torch.float32)[::2]):
        with pytest.raises(ValueError, match="out must be"):
            desc.block_reduce(x, 10, out=bad)
    for bad in (torch.zeros(99, dtype=torch.float32), torch.zeros(100, dtype=torch.int32),
                torch.zeros(200, dtype=torch.float32)[::2]):
        with pytest.raises(ValueError, match="out must be"):
            desc.scan(x, out=bad)


def test_slab_peer_validation_codes(lib):
    """desc_slab_transpose_peer argument checks (all before any CUDA call)."""
    import ctypes
    f = lib.desc_slab_transpose_peer
    outs = (ctypes.c_void_p * 2)(FAKE_OUT, FAKE_OUT + (1 << 30))
    assert f(None, outs, 2, 0, 256, 256, 0, None) == 1                 # null in_slab
    assert f(FAKE_IN, None, 2, 0, 256, 256, 0, None) == 1              # null out array
    assert f(FAKE_IN, outs, 0, 0, 256, 256, 0, None) == 2              # P < 1
    assert f(FAKE_IN, outs, 9, 0, 256, 256, 0, None) == 2              # P > 8
    assert f(FAKE_IN, outs, 2, 2, 256, 256, 0, None) == 2              # r >= P
    assert f(FAKE_IN, outs, 2, 0, 255, 256, 0, None) == 2              # P does not divide M
    assert f(FAKE_IN, outs, 2, 0, 256, 96, 0, None) == 2               # N/P = 48: not tile-wide
    assert "tile width" in desc.desc_last_error()
    assert f(FAKE_IN, outs, 2, 0, 256, 256, 4, None) == 3              # 2-byte cells
