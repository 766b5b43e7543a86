# cluster-per-block reduction: threads per CTA adaptive (base, one wave) vs 256, twice
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -x 2>&1 | tail -1
for rnd in 1 2; do for v in base ct256; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py | grep -E "B=(16384|65536|1048576|4194304):" | sed "s/^/$v /"
done; done
