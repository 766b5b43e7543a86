#!/bin/bash
# r02 (session 2): DESC_KERNEL_VTILED A/B against TILED (exp_kernels.py timing), tile configs
#   bash scripts/exp_vtiled.sh "<cfgs>" "<shapes>" <rounds>
C=${1:-"1 2 3"}
S=${2:-"8192x8192:f32,3000x5000:f64,2048x2048:f64,4096x4096:f64,8192x8192:f64,256x1024x1024:f32,4096x4096:f32"}
R=${3:-2}
for r in $(seq $R); do
  echo "## round $r"
  python scripts/exp_kernels.py --kernels tiled,vtiled --shapes $S
  for c in $C; do DESC_VTILED_CFG=$c python scripts/exp_kernels.py --kernels vtiled --shapes $S | sed "s/^/cfg$c /"; done
done
