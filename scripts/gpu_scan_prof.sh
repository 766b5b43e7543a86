# ncu captures of the streaming scan kernel (one launch each), for stall attribution
for w in f32 i32; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 3 -c 1 -o gpurun_out/prof_scan_stream_$w python bench.py --workload scan64M_$w --scan-algo stream --steps 3 --warmup 3 --no-oracle > gpurun_out/ncu_scan_$w.log 2>&1; echo $w rc=$?
done
