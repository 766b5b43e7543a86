#!/bin/bash
# r02 (session 2): TMA ring slot release after ld.shared -- stress (mismatch count) and speed
for v in rel0 rel1 rel2; do
  echo "## $v"
  DESC_LIB=build_variants/lib_tiled_$v.so timeout 900 python scripts/stress_8192.py 150 tma,tma_st 2>&1 | grep -v "^MISMATCH" 
  DESC_LIB=build_variants/lib_tiled_$v.so python scripts/exp_kernels.py --kernels tma,tma_st --shapes 8192x8192:f32,3000x5000:f64 | sed "s/^/$v /"
done
