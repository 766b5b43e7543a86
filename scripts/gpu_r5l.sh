# warp-per-block reduction kernel: grid cap 8 / 16 / 32 CTAs per SM
for v in base w8 w32; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py | grep -E "B=(3000|4096|8192|16384|65536):"
done
