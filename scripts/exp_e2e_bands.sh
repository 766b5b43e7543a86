#!/bin/bash
# r02 (session 2): e2e with at least DESC_HOST_BANDS bands per matrix (0 = largest band that fits)
for r in 1 2; do
for nb in 0 8 16; do
  for w in 8192f32 2048f64 3000x5000f64; do
    DESC_HOST_BANDS=$nb python bench.py --workload $w --steps 20 --warmup 5 --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('bands>=$nb', '$w', e['value'], e['pcie_ceiling']['frac'], e['spot_check'], e['gpu_launches'])"
  done
done
done
