for g in 0 1 2 4 8 16 64 1000; do
  echo "group=$g"; DESC_TMA_CFG=9 DESC_TMA_GROUP=$g timeout 300 python scripts/sweep_cfg.py --kernel tma_st --cfgs 9 --workloads 8192f32 2>&1
done | tee gpurun_out/sweep_group2.txt
DESC_TMA_CFG=9 timeout 600 python scripts/exp_ld.py tma_st 2>&1 | tee gpurun_out/exp_ld.txt
