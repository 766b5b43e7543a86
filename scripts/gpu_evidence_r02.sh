#!/bin/bash
# r02 (session 2) evidence refresh: every bench workload line, launch list of the default
# bench command, ncu --set full of the kernels changed this session
mkdir -p gpurun_out/ev
for w in 8192f32 2048f64 3000x5000f64 4096f64 8192i32 8192f64 3000x5000f64_ld5001 8192f32_ld8193 batched view_tiles8192f32 view_transpose8192f32 view_rot90_8192f32 view_flip8192f32 reduce64M_f32 scan64M_f32 scan64M_i32 scan32M_f64; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/ev/bench_$w.json 2> gpurun_out/ev/bench_$w.err
  echo "bench $w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/ev/bench_$w.json').readline()); print(d['value'], d['roofline']['frac'], d.get('parity'))" 2>/dev/null)"
done
timeout 600 python bench.py --workload dist65536 --steps 10 --warmup 3 > gpurun_out/ev/bench_dist65536.json 2> gpurun_out/ev/bench_dist65536.err
echo "dist65536 rc=$?"
timeout 600 python bench.py --kernel vtiled --steps 20 --warmup 5 > gpurun_out/ev/bench_vtiled_8192f32.json 2>/dev/null; echo "vtiled rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 20 --warmup 5 --no-oracle --no-e2e > gpurun_out/ev/launches_bench.log 2>&1; echo "launches rc=$?"
python scripts/ncu_summary.py --launches gpurun_out/ev/launches.csv gpurun_out/ev/launches_8192f32.md > /dev/null 2>&1; echo "launch summary rc=$?"
for spec in view_flip8192f32:view_tiles_kernel 8192f32:transpose_tiled; do
  w=${spec%%:*}; k=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o gpurun_out/ev/prof_${w}_$k -f python bench.py --workload $w --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ev/ncu_${w}_$k.log 2>&1
  echo "ncu $w $k rc=$?"
  python scripts/ncu_summary.py gpurun_out/ev/prof_${w}_$k.ncu-rep gpurun_out/ev/ncu_${w}_$k.md > /dev/null 2>&1
  rm -f gpurun_out/ev/prof_${w}_$k.ncu-rep
done
# the row copy at the slab-unpack shape
timeout 900 ncu --set full --clock-control none -k regex:copy_rows -s 3 -c 1 -o gpurun_out/ev/prof_copy -f python scripts/exp_copy.py > gpurun_out/ev/ncu_copy.log 2>&1
echo "ncu copy rc=$?"
python scripts/ncu_summary.py gpurun_out/ev/prof_copy.ncu-rep gpurun_out/ev/ncu_copy_rows.md > /dev/null 2>&1
rm -f gpurun_out/ev/prof_copy.ncu-rep
