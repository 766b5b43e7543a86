timeout 900 python -m pytest tests -x -q -m gpu -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for ev in 0 1; do for pr in 0 2; do
  echo "evict_first=$ev promo=$pr"
  DESC_TMA_EVICT=$ev DESC_TMA_PROMO=$pr timeout 600 python scripts/sweep_cfg.py --kernel tma_st --cfgs 0,1,2,3,4,5 --workloads 8192f32,3000x5000f64 2>&1
done; done | tee gpurun_out/sweep_tma_st.txt
