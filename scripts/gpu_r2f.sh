for c in 1 0 1 0; do
  echo "DESC_STATIC_CLUSTER=$c"
  for w in 2048f64 3000x5000f64; do
    DESC_STATIC_CLUSTER=$c timeout 600 python bench.py --workload $w --no-oracle --no-e2e --steps 300 --warmup 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  $w', d['value'], d['roofline']['frac'], d['roofline']['launch_ms_median'], d['small_problem']['launch_floor_ms'])"
  done
done
DESC_STATIC_CLUSTER=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_views_gpu.py -x -q 2>&1 | tail -2
DESC_STATIC_CLUSTER=0 DESC_DYN=0 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/san_nocluster.log 2>&1; echo "racecheck static no-cluster rc=$?"; grep -E "SUMMARY|Race" gpurun_out/san_nocluster.log | head -3
