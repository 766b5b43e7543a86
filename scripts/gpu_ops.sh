for w in reduce64M_f32 scan64M_f32 scan64M_i32; do
  timeout 300 python bench.py --workload $w --steps 200 --warmup 10 | tail -1 > gpurun_out/bench_$w.json; echo "$w rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print(d['value'], d['roofline']['frac'], d['parity'], d['ms_per_step'])"
done
