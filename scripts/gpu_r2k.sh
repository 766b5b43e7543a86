for i in 1 2; do
for v in head scan_c0_p2 scan_c1_p2 scan_c1_p3 scan_c1_p4; do
  for w in scan64M_f32 scan64M_i32; do
  DESC_LIB=build_variants/lib_$v.so timeout 600 python bench.py --workload $w --no-oracle --no-e2e --steps 300 --warmup 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
done
done
