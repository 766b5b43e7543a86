# rotating-buffer L2 mode for small workloads vs the per-launch flush
for w in 2048f64 3000x5000f64 8192f32; do
  timeout 600 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['config']['l2']); print(d.get('small_problem'))"
  echo "flush: $(timeout 600 python bench.py --workload $w --no-e2e --no-oracle --l2 flush 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
done
