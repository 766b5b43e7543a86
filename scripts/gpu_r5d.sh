# block reduction: 16-CTA clusters for very few blocks, CTA kernel back for nb >= 2 x SMs
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python scripts/exp_reduce_blocks.py
timeout 300 python bench.py --workload reduce64M_f32 --steps 1000 --warmup 50 > gpurun_out/bench_reduce.json 2>/dev/null; tail -1 gpurun_out/bench_reduce.json | cut -c1-200
timeout 600 python -m pytest tests/test_mutants_gpu.py -q -m gpu -x 2>&1 | tail -3
