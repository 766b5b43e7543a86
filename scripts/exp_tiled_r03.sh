#!/bin/bash
# r03 TILED A/B: product vs compile-time variants (scripts/build_tiled_variants.py), interleaved
#   bash scripts/exp_tiled_r03.sh "<variants>" "<shapes>" <rounds>
V=${1:-"cpa5 cpa8 r4 r8 r16 r32 ldcs ldlu stcs stcg ldcs_stcs minb6"}
S=${2:-"8192x8192:f32,3000x5000:f64,2048x2048:f64,4096x4096:f64,8192x8192:f64,256x1024x1024:f32"}
R=${3:-2}
for r in $(seq $R); do
  echo "## round $r"
  python scripts/exp_kernels.py --kernels tiled --shapes $S
  for v in $V; do
    DESC_LIB=build_variants/lib_tiled_$v.so python scripts/exp_kernels.py --kernels tiled --shapes $S
  done
done
