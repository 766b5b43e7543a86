"""Compile-time variants of the block reduction for A/B runs (DESC_LIB=<path>)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_03448_b200 import build as B

VARIANTS = {
    "ct256": ["DESC_REDUCE_CLUSTER_THREADS=256"],
    "ct512": ["DESC_REDUCE_CLUSTER_THREADS=512"],
}
out_dir = os.path.join(B.ROOT, "build_variants")
os.makedirs(out_dir, exist_ok=True)
with ThreadPoolExecutor(len(VARIANTS)) as ex:
    for name, p in zip(VARIANTS, ex.map(lambda kv: B.build(defines=kv[1], out=os.path.join(out_dir, f"lib_{kv[0]}.so")), VARIANTS.items())):
        print(name, p)
