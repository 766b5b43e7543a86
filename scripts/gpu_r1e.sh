timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for ev in 0 1; do
  echo "evict_first=$ev promo=0"
  DESC_TMA_EVICT=$ev DESC_TMA_PROMO=0 timeout 900 python scripts/sweep_cfg.py --kernel tma_st --cfgs 0,1,5,6,7,8,9,10,11 --workloads 8192f32,3000x5000f64,batched 2>&1
done | tee gpurun_out/sweep_tma_st2.txt
