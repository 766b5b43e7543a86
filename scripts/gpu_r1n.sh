for w in view_tiles8192f32 view_transpose8192f32 view_rot90_8192f32 view_flip8192f32; do
  timeout 300 python bench.py --workload $w --steps 200 --warmup 10 | tail -1 > gpurun_out/bench_$w.json; echo "$w rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print(d['value'], d['roofline']['frac'], d['parity'], d['config']['compiled_view'])"
done
