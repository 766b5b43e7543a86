# tiled mutants, reversed-row views through TILED, batched ncu capture, view benches
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_mutants_gpu.py -q -rA > gpurun_out/mutants_gpu.log 2>&1; echo mutants rc=$?
tail -25 gpurun_out/mutants_gpu.log
for w in view_rot90_8192f32 view_transpose8192f32 view_tiles8192f32 view_flip8192f32; do
  echo "$w $(timeout 300 python bench.py --workload $w --steps 200 --warmup 5 2>/dev/null | tee gpurun_out/bench_$w.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], d.get("parity"))')"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_batched python bench.py --workload batched --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_b.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_tiled -s 5 -c 1 -o gpurun_out/prof_tiled_rot90 python bench.py --workload view_rot90_8192f32 --steps 8 --warmup 3 --no-oracle > gpurun_out/ncu_r.log 2>&1; echo ncu rc=$?
