"""Compile-time variants of the library for A/B runs on the GPU (load with DESC_LIB=<path>).

    python scripts/build_variants.py NAME=DEF1,DEF2 [NAME=...]
e.g. python scripts/build_variants.py tt10=DESC_TMA_TILE_MINB=10 tt12=DESC_TMA_TILE_MINB=12
Builds build_variants/lib_<NAME>.so in parallel."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_03448_b200 import build as B  # noqa: E402

out_dir = os.path.join(B.ROOT, "build_variants")
os.makedirs(out_dir, exist_ok=True)
specs = dict(a.split("=", 1) for a in sys.argv[1:])
with ThreadPoolExecutor(max(1, len(specs))) as ex:
    futs = {n: ex.submit(B.build, defines=d.split(","), out=os.path.join(out_dir, f"lib_{n}.so"))
            for n, d in specs.items()}
    for n, f in futs.items():
        print(n, f.result())
