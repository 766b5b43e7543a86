timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for d in 0 1; do echo "DYN=$d"; DESC_DYN=$d timeout 600 python scripts/sweep_cfg.py --kernel auto --cfgs 0 --workloads 8192f32,2048f64,3000x5000f64,batched 2>&1; done | tee gpurun_out/sweep_dyn.txt
for d in 0 1; do echo "DYN=$d"; DESC_DYN=$d timeout 300 python scripts/exp_region.py; done 2>&1 | tee gpurun_out/exp_region_dyn.txt
