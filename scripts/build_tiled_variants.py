"""Compile-time variants of the TILED transpose kernel for A/B runs (DESC_LIB=<path>).

  python scripts/build_tiled_variants.py [name ...]     (default: every variant below)
"""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_03448_b200 import build as B

VARIANTS = {
    # r02 tile-shape sweep (8-byte cells)
    "s1": ["DESC_TILED_TR8=32", "DESC_TILED_TC8=64"],
    "s2": ["DESC_TILED_TR8=64", "DESC_TILED_TC8=32"],
    "s3": ["DESC_TILED_TR8=32", "DESC_TILED_TC8=32"],
    # (r02 session 2: the TILED knobs for cp.async staging, banded raster orders, load / store
    # cache hints and 6 CTAs/SM were measured -- profiles/r02_tiled_variants_cpasync_raster_hints.txt
    # -- none won, and they were removed from tiled_transpose.cuh again)
    # r02 (session 2): the 16-byte vector tile kernel without cp.async (LDG.128 -> STS.128)
    "vt_nocpa": ["DESC_VT_CPA=0"],
    # TMA ring slot release after ld.shared without the proxy fence (ptx.cuh)
    "rel0": ["DESC_REL_MODE=0"],
    # view copies: first-item prefetch compiled into the plain 16-byte mode
    # (viewpf1, DESC_VIEW_PF1=1: the first-item prefetch in the plain view mode -- lost,
    #  profiles/r02_view_tiles_pf1.txt -- the knob was removed again)
    "viewunr8": ["DESC_VIEW_UNR=8"],
    # (tiledpf2, DESC_TILED_PF2=1: second-tile prefetch -- lost, removed again;
    #  profiles/r02_tiled_tiles_per_cta.txt)
    "vtminb10": ["DESC_VT_MINB=10"],
    "vtminb12": ["DESC_VT_MINB=12"],
    "viewunr2": ["DESC_VIEW_UNR=2"],
}
names = sys.argv[1:] or [n for n in VARIANTS if n not in ("s1", "s2", "s3")]
out_dir = os.path.join(B.ROOT, "build_variants")
os.makedirs(out_dir, exist_ok=True)
with ThreadPoolExecutor(8) as ex:
    for name, p in zip(names, ex.map(lambda n: B.build(defines=VARIANTS[n], out=os.path.join(out_dir, f"lib_tiled_{n}.so")), names)):
        print(name, p)
