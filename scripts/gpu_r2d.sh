for w in 2048f64 3000x5000f64 4096f64; do
  timeout 600 python bench.py --workload $w --no-oracle --no-e2e --steps 300 --warmup 10 2>&1 | tail -1 > gpurun_out/bench_d_$w.json
  python -c "import json; d=json.load(open('gpurun_out/bench_d_$w.json')); print('$w', d['value'], d['roofline']['frac'], d.get('small_problem'))"
done
