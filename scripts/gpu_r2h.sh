timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -x -q 2>&1 | tail -3
for i in 1 2; do
for v in head new; do
  L=build_variants/lib_head.so; [ $v = new ] && L=paper_2305_03448_b200/libdesc_transpose.so
  for w in scan64M_f32 scan64M_i32; do
  DESC_LIB=$L timeout 600 python bench.py --workload $w --no-oracle --no-e2e --steps 300 --warmup 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
done
done
