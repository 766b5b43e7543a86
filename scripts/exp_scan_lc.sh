#!/bin/bash
# r02 scan A/B: lane-contiguous layout with TMA-store staging (scripts/build_scan_variants.py)
#   bash scripts/exp_scan_lc.sh "<variant:workload ...>" <rounds>
# parity (the scan GPU tests) for each non-diagnostic variant, then bench lines interleaved
V=${1:-"nolc:scan64M_f32 lc_i32:scan64M_i32 lc_i32_nr8:scan64M_i32 lc_f64:scan32M_f64"}
R=${2:-2}
for vw in $V; do
  v=${vw%%:*}
  case $v in *diag*) continue;; esac     # diagnostics builds compute wrong results by design
  echo "## parity $v"
  DESC_LIB=build_variants/lib_$v.so timeout 600 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -k "scan" -x 2>&1 | tail -1
done
line() {  # label workload [env]
  python bench.py --workload $2 --steps 20 --warmup 5 --no-oracle --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', '$2', d['value'], d['roofline']['frac'])"
}
for r in $(seq $R); do
  echo "## round $r"
  for w in $(for vw in $V; do echo ${vw#*:}; done | sort -u); do line product $w; done
  for vw in $V; do v=${vw%%:*}; w=${vw#*:}; DESC_LIB=build_variants/lib_$v.so line $v $w; done
done
