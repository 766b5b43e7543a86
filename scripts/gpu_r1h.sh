timeout 900 python scripts/sweep_cfg.py --kernel tma_st --cfgs 0,1,2,3,4,5,6,7,8,9,10,11,12 --workloads 2048f64,3000x5000f64 2>&1 | tee gpurun_out/sweep_small_tma_st.txt
timeout 900 python scripts/sweep_cfg.py --kernel tma --cfgs 0,1,2,3,4,5,6,7,8 --workloads 2048f64,3000x5000f64 2>&1 | tee gpurun_out/sweep_small_tma.txt
