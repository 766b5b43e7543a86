timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for pdl in 0 1; do echo "PDL=$pdl"; DESC_PDL=$pdl timeout 600 python scripts/sweep_cfg.py --kernel auto --cfgs 0 --workloads 8192f32,2048f64,3000x5000f64,batched 2>&1; done | tee gpurun_out/sweep_pdl.txt
