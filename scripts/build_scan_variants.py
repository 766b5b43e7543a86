"""Compile-time variants of the streaming scan for A/B runs (DESC_LIB=<path>)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_03448_b200 import build as B

VARIANTS = {
    "lb2": ["DESC_SCAN_LB_WARPS=2"],
    "qt4": ["DESC_SCAN_TMEM_SLOTS=4"],
    "v10": ["DESC_SCAN_VPT=10"],
    "v16s3q4": ["DESC_SCAN_VPT=16", "DESC_SCAN_STAGES=3", "DESC_SCAN_TMEM_SLOTS=4"],
    "diag1": ["DESC_SCAN_DIAG=1"],
    "diag3": ["DESC_SCAN_DIAG=3"],
    # r02 (session 2): f32 lane-contiguous layout with TMA-store staging
    "lc": ["DESC_SCAN_LC_F32=1"],
    "lc_diag1": ["DESC_SCAN_LC_F32=1", "DESC_SCAN_DIAG=1"],
    "nolc": ["DESC_SCAN_LC_F32=0"],
    "lc_i32": ["DESC_SCAN_LC_I32=1"],
    "lc_i32_nr8": ["DESC_SCAN_LC_I32=1", "DESC_SCAN_LC_I32_NR=8"],
    "lc_f64": ["DESC_SCAN_LC_F64=1"],
    "relnofence": ["DESC_SCAN_REL_FENCE=0"],
    "lc_u8": ["DESC_SCAN_LC_U8=1"],
    # look-back knobs on the lane-contiguous kernels
    "lbw2": ["DESC_SCAN_LB_WINDOW=2"],
    "sleep64": ["DESC_SCAN_SLEEP_CAP=64"],
    "sleep512": ["DESC_SCAN_SLEEP_CAP=512"],
}
out_dir = os.path.join(B.ROOT, "build_variants")
os.makedirs(out_dir, exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
with ThreadPoolExecutor(8) as ex:
    for name, p in zip(names, ex.map(lambda n: B.build(defines=VARIANTS[n], out=os.path.join(out_dir, f"lib_{n}.so")), names)):
        print(name, p)
