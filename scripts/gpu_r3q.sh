# round-1 refresh: full GPU suite, smoke, sanitizers, mutants, every bench line, ncu launch lists
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for t in racecheck synccheck memcheck initcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
for w in 2048f64 3000x5000f64 4096f64 8192f64 8192i32 batched 3000x5000f64_ld5001 8192f32_ld8193 view_rot90_8192f32 view_transpose8192f32 view_tiles8192f32 view_flip8192f32 reduce64M_f32 scan64M_f32 scan64M_i32; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
done
timeout 600 python bench.py --workload dist65536 --steps 5 --warmup 3 > gpurun_out/bench_dist65536.json 2>gpurun_out/bench_dist65536.err; echo dist rc=$?
DESC_BENCH_BACKEND=gloo DESC_BENCH_EXCHANGE_P2P=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 100 --warmup 5 --exchange-n 16384 --no-e2e > gpurun_out/bench_n2_shared_gpu_gloo.json 2> gpurun_out/bench_n2.err; echo n2 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_scan.csv python bench.py --workload scan64M_f32 --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches scan rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 5 -c 1 -o gpurun_out/prof_scan_stream_f32 python bench.py --workload scan64M_f32 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_scan.log 2>&1; echo ncu scan rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_8192f64 python bench.py --workload 8192f64 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_f64.log 2>&1; echo ncu f64 rc=$?
timeout 900 python -m pytest tests/test_mutants_gpu.py -q -rA > gpurun_out/mutants_gpu.log 2>&1; echo mutants rc=$?
for f in gpurun_out/bench*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), (d.get('roofline') or {}).get('frac'), d.get('config',{}).get('kernel'), d.get('parity'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))"; done
