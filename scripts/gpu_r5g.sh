# block reduction: warp-row kernel with 16 loads in flight and 4 / 8 KB blocks
for v in base l16m4k l8m4k l16m8k; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py | grep -E "B=(64|128|256|512|1024|2048|4096):"
  DESC_LIB=$L timeout 300 python bench.py --workload reduce64M_f32 --no-oracle --no-e2e --steps 1000 --warmup 50 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench $v', d['value'], d['roofline']['frac'])"
done
