# block reduction: cluster-per-block path (few long blocks) + warp-row path (short blocks)
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -x 2>&1 | tail -3
for v in base norows ru4c16; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python scripts/exp_reduce_blocks.py
done
timeout 300 python bench.py --workload reduce64M_f32 --steps 1000 --warmup 50 > gpurun_out/bench_reduce.json 2>/dev/null; tail -1 gpurun_out/bench_reduce.json | cut -c1-200
