# block reduction: new default (8 loads in flight, 8 CTAs/SM) vs the earlier one, all group widths
for v in base ru4c16 ru16c8; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py
done
for rnd in 1 2; do
  timeout 300 python bench.py --workload reduce64M_f32 --steps 1000 --warmup 50 > gpurun_out/bench_reduce_$rnd.json 2>/dev/null; tail -1 gpurun_out/bench_reduce_$rnd.json | cut -c1-200
done
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu 2>&1 | tail -2
