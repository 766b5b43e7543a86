set -x
timeout 1200 python -m pytest tests/test_mutants_gpu.py -v -s > gpurun_out/pytest_mutants.log 2>&1; echo mutants rc=$?
tail -25 gpurun_out/pytest_mutants.log
timeout 300 python scripts/exp_e2e.py > gpurun_out/exp_e2e.txt 2>&1; echo e2e rc=$?
cat gpurun_out/exp_e2e.txt
