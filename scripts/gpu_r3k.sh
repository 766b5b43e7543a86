# PDL on every memory-bound kernel: full GPU suite, sanitizers, mutants, bench lines
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for t in racecheck synccheck memcheck initcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
for w in 2048f64 3000x5000f64 4096f64 8192f64 batched 3000x5000f64_ld5001 8192f32_ld8193 view_rot90_8192f32 view_transpose8192f32 view_tiles8192f32 view_flip8192f32 reduce64M_f32; do
  timeout 600 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
done
timeout 600 python bench.py --workload dist65536 --steps 5 --warmup 3 > gpurun_out/bench_dist65536.json 2>gpurun_out/bench_dist65536.err; echo dist rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches rc=$?
for f in gpurun_out/bench*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), (d.get('roofline') or {}).get('frac'), d['config'].get('kernel'), d.get('parity'))"; done
