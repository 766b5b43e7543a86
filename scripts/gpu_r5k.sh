# bench lines of the reduction / scan / a view workload after the cpu_baseline change
for w in reduce64M_f32 scan64M_f32 scan64M_i32 scan32M_f64 view_rot90_8192f32; do timeout 300 python bench.py --workload $w --steps 1000 --warmup 50 --no-e2e > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; echo "$w rc=$?"; tail -1 gpurun_out/bench_$w.json | cut -c1-100; done
