#!/bin/bash
# Regression A/B: every bench workload (but dist65536), a reference library build vs the
# current one, interleaved, two rounds.   bash scripts/exp_regress.sh <reference .so>
REF=${1:-build_variants/lib_f69d7a8.so}
W="8192f32 2048f64 3000x5000f64 4096f64 8192i32 8192f64 3000x5000f64_ld5001 8192f32_ld8193 batched view_tiles8192f32 view_transpose8192f32 view_rot90_8192f32 view_flip8192f32 reduce64M_f32 scan64M_f32 scan64M_i32 scan32M_f64"
for r in 1 2; do
  for w in $W; do
    for lib in $REF paper_2305_03448_b200/libdesc_transpose.so; do
      DESC_LIB=$lib python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%-44s %-22s %9.1f %.4f' % ('$lib', '$w', d['value'], d['roofline']['frac']))"
    done
  done
done
