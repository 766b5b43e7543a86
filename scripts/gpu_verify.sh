# round re-entry verification: smoke, GPU parity suite, default bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json
for w in scan64M_f32 scan64M_i32; do timeout 300 python bench.py --workload $w --no-oracle --no-e2e 2>/dev/null | tail -1 | cut -c1-300; done
