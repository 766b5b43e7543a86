timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --workload dist65536 --steps 10 --warmup 3 > gpurun_out/bench_dist1.json 2>gpurun_out/bench_dist1.err; echo dist rc=$?; cat gpurun_out/bench_dist1.json; tail -3 gpurun_out/bench_dist1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 --reference-seconds 30 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?; tail -2 gpurun_out/bench_ref.json
