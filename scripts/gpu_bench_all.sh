#!/bin/bash
# every bench workload line (default steps) -> gpurun_out/ev/bench_<w>.json, one summary line each
mkdir -p gpurun_out/ev
for w in ${1:-8192f32 2048f64 3000x5000f64 4096f64 8192i32 8192f64 3000x5000f64_ld5001 8192f32_ld8193 batched view_tiles8192f32 view_transpose8192f32 view_rot90_8192f32 view_flip8192f32 reduce64M_f32 scan64M_f32 scan64M_i32 scan32M_f64 dist65536}; do
  st=20; wu=5; [ $w = dist65536 ] && st=10 && wu=3
  timeout 600 python bench.py --workload $w --steps $st --warmup $wu > gpurun_out/ev/bench_$w.json 2> gpurun_out/ev/bench_$w.err
  echo "bench $w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/ev/bench_$w.json').readline()); e=d.get('e2e') or {}; print(d['value'], d['roofline']['frac'], 'e2e', e.get('value'), '|', d.get('parity'))" 2>/dev/null)"
done
