timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json
for t in racecheck synccheck memcheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_$t.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tma2 -s 5 -c 1 -o gpurun_out/prof_tma2_8192f32_dyn python bench.py --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:view_tiles -s 3 -c 1 -o gpurun_out/prof_view_tiles python bench.py --workload view_tiles8192f32 --steps 5 --warmup 3 --no-oracle > gpurun_out/ncu_full3.log 2>&1; echo ncu3 rc=$?
