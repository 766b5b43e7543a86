# r02 (session 2): view workloads, pre-session library (f69d7a8) vs the current one
for r in 1 2; do
for lib in build_variants/lib_f69d7a8.so paper_2305_03448_b200/libdesc_transpose.so; do
  for w in view_tiles8192f32 view_flip8192f32 view_transpose8192f32 view_rot90_8192f32; do
    DESC_LIB=$lib python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', '$w', d['value'], d['roofline']['frac'])"
  done
done
done
