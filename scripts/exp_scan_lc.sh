#!/bin/bash
# r02 scan A/B: lane-contiguous f32 layout variants (scripts/build_scan_variants.py)
#   bash scripts/exp_scan_lc.sh "<variants>" <rounds>
V=${1:-"lc lc_pad4_qt4 lc_diag1 diag1"}
R=${2:-2}
for v in $V; do
  case $v in *diag*) continue;; esac     # diagnostics builds compute wrong results by design
  echo "## parity $v"
  DESC_LIB=build_variants/lib_$v.so timeout 600 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -k "scan and not diag" -x 2>&1 | tail -2
done
for r in $(seq $R); do
  echo "## round $r"
  for w in scan64M_f32; do
    python bench.py --workload $w --steps 20 --warmup 5 --no-oracle --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('product', d['config']['workload'][:30], d['value'], d['roofline']['frac'])"
    for v in $V; do
      DESC_LIB=build_variants/lib_$v.so python bench.py --workload $w --steps 20 --warmup 5 --no-oracle --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['config']['workload'][:30], d['value'], d['roofline']['frac'])"
    done
  done
done
