# per-type streaming-scan configs: parity, sanitizers on the scan paths, bench lines, ncu
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py tests/test_mutants_gpu.py -x -q > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_scan.log
for t in racecheck synccheck memcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|sanitize driver" gpurun_out/sanitizer_$t.log | head -3
done
for w in scan64M_f32 scan32M_f64 scan64M_i32; do
  timeout 300 python bench.py --workload $w > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; echo $w rc=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['parity'], d['clocks'])"
done
for w in scan64M_f32 scan32M_f64; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 3 -c 1 -o gpurun_out/prof_$w python bench.py --workload $w --scan-algo stream --steps 3 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_$w.log 2>&1; echo ncu $w rc=$?
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_scan64M_f32.csv python bench.py --workload scan64M_f32 --steps 10 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches rc=$?
