# alignment-agnostic TILED kernel: parity + measurement next to the paper-schedule SMEM kernel
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_parity.log
for w in 3000x5000f64_ld5001 8192f32_ld8193; do
  timeout 300 python bench.py --workload $w --no-e2e --steps 100 --warmup 5 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; echo $w rc=$?
done
for k in tiled smem tma_st; do for w in 8192f32 3000x5000f64 2048f64 8192f64; do
  echo "$k $w $(timeout 300 python bench.py --workload $w --kernel $k --no-e2e --no-oracle --steps 100 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
done; done
for w in 3000x5000f64_ld5001 8192f32_ld8193; do python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['config']['kernel'], d['parity'], d['cpu_baseline']['value'])"; done
