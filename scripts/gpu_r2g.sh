for i in 1 2 3; do
for v in head static; do
  DESC_LIB=build_variants/lib_$v.so DESC_STATIC_CLUSTER=1 timeout 600 python bench.py --workload 2048f64 --no-oracle --no-e2e --steps 300 --warmup 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['frac'], d['roofline']['launch_ms_median'])"
done
DESC_LIB=build_variants/lib_static.so DESC_STATIC_CLUSTER=0 timeout 600 python bench.py --workload 2048f64 --no-oracle --no-e2e --steps 300 --warmup 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('static-nocluster', d['value'], d['roofline']['frac'], d['roofline']['launch_ms_median'])"
done
