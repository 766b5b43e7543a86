# bench with the PCIe ceiling, then one ncu --set full capture per workload's dominant kernel
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_c.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c.log
prof() {  # workload kernel-regex name extra...
  w=$1; k=$2; n=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o gpurun_out/prof_$n python bench.py --workload $w --steps 8 --warmup 3 --no-oracle --no-e2e "$@" > gpurun_out/ncu_$n.log 2>&1; echo "$n rc=$?"
}
prof 2048f64 transpose_tma2 tma2_2048f64
prof batched transpose_tma2 tma2_batched
prof scan64M_f32 scan_stream scan_stream_f32
prof scan64M_i32 scan_stream scan_stream_i32
prof reduce64M_f32 block_reduce reduce_f32
prof view_flip8192f32 view_tiles view_flip8192f32
prof view_rot90_8192f32 transpose_tma2 view_rot90_8192f32
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_scan.csv python bench.py --workload scan64M_f32 --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1; echo launches rc=$?
ls -la gpurun_out/
