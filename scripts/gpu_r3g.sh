# TILED as AUTO for 4/8-byte cells: full GPU suite, sanitizers, bench lines, ncu captures
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
for w in 3000x5000f64 2048f64 4096f64 8192f64 batched 3000x5000f64_ld5001 8192f32_ld8193; do
  timeout 600 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
done
timeout 600 python bench.py --workload dist65536 --steps 5 --warmup 3 > gpurun_out/bench_dist65536.json 2>gpurun_out/bench_dist65536.err; echo dist rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_8192f32 python bench.py --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_3000x5000f64 python bench.py --workload 3000x5000f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_2048f64 python bench.py --workload 2048f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full3.log 2>&1; echo ncu3 rc=$?
for t in racecheck synccheck memcheck initcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
for f in gpurun_out/bench*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), (d.get('roofline') or {}).get('frac'), d['config'].get('kernel'), d.get('parity'))"; done
