set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sweep_cfg.py 2>&1 | tee gpurun_out/sweep.txt
timeout 300 python bench.py --workload 8192f32 --steps 300 --warmup 20 --no-oracle --no-e2e --kernel smem | tail -1 > gpurun_out/bench_smem.json
# launch list (cold, serialised) and one full capture of the top kernel
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tma -s 3 -c 1 -o gpurun_out/prof_tma_8192f32 python bench.py --steps 5 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full.log
