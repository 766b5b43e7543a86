for pdl in 0 1; do echo PDL=$pdl; DESC_PDL=$pdl timeout 300 python scripts/exp_region.py; done 2>&1 | tee gpurun_out/exp_region.txt
