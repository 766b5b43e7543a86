timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json
for w in 2048f64 3000x5000f64 batched; do timeout 300 python bench.py --workload $w --no-oracle --no-e2e --steps 300 --warmup 20 | tail -1 > gpurun_out/bench_$w.json; done
for t in racecheck synccheck memcheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_$t.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tma2 -s 3 -c 1 -o gpurun_out/prof_tma2_8192f32 python bench.py --steps 5 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tma2 -s 3 -c 1 -o gpurun_out/prof_tma2_3000x5000f64 python bench.py --workload 3000x5000f64 --steps 5 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncu3 rc=$?
