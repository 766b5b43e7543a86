# f64 TILED at 32x64: parity, sanitizers, mutants, f64 bench lines, ncu
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
for t in racecheck synccheck memcheck initcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
for w in 2048f64 3000x5000f64 4096f64 8192f64 3000x5000f64_ld5001; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['parity'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_3000x5000f64 python bench.py --workload 3000x5000f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_2048f64 python bench.py --workload 2048f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full3.log 2>&1; echo ncu3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_8192f64 python bench.py --workload 8192f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_f64.log 2>&1; echo ncu f64 rc=$?
