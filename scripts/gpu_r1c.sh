timeout 300 python scripts/copy_ceiling.py 2>&1 | tee gpurun_out/copy_ceiling.txt
for g in 1 4 8 11 16 32; do for ev in 0 1; do for pr in 0 2; do
  echo "group=$g evict_first=$ev promo=$pr"
  DESC_TMA_GROUP=$g DESC_TMA_EVICT=$ev DESC_TMA_PROMO=$pr timeout 300 python scripts/sweep_cfg.py --cfgs 0,1 --workloads 8192f32 2>&1
done; done; done | tee gpurun_out/sweep_group.txt
