set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 300 python bench.py --kernel smem --no-oracle --no-e2e > gpurun_out/bench_smem.log 2>&1; echo bench smem rc=$?
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.log gpurun_out/bench_smem.log | tail -4
