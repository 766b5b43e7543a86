# block reduction: segmented warp rows for 1 … 16 vectors per block
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -x 2>&1 | tail -3
for v in base noseg; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py
done
