# wide-accumulator scan split (12 + 12 warps): parity, then A/B vs variants (DESC_LIB), 2 rounds
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -x -q > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_scan.log
for rnd in 1 2; do
for v in base old8 w10s3q4 w8q4 w8p4 w8p3; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  for w in scan64M_f32 scan32M_f64 scan64M_i32; do
    NO=--no-oracle; if [ $rnd = 1 ] && [ $v = base ]; then NO=""; fi
    DESC_LIB=$L timeout 300 python bench.py --workload $w --scan-algo stream $NO --no-e2e --steps 300 --warmup 20 2>gpurun_out/r4b_err_$v.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rnd $v', '$w', d['value'], d['roofline']['frac'], d.get('parity'))"
  done
done
done
