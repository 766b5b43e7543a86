# scan parity, racecheck, bench lines; view copy rot180 check
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py tests/test_views_gpu.py -q > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_scan.log
for w in scan64M_f32 scan64M_i32; do
  timeout 600 python bench.py --workload $w --no-oracle --steps 300 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'])"
done
for w in view_flip8192f32 view_tiles8192f32; do
  timeout 600 python bench.py --workload $w --no-oracle --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'])"
done
DESC_DYN_MIN=1 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "SUMMARY|Race reported|PASS|FAIL" gpurun_out/sanitizer_racecheck.log | head -5
