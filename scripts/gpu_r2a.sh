set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log
for w in 2048f64 3000x5000f64 batched scan64M_f32 scan64M_i32 reduce64M_f32 view_flip8192f32 view_tiles8192f32; do
  timeout 600 python bench.py --workload $w --no-oracle --no-e2e 2>/dev/null | tail -1 > gpurun_out/bench_$w.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d.get('clocks'))"
done
