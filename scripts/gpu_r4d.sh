# streaming scan with the per-type warp split: where the remaining time goes (diagnostic builds)
for rnd in 1 2; do
for v in base lb2 diag1 diag3; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  for w in scan64M_f32 scan32M_f64 scan64M_i32; do
    DESC_LIB=$L timeout 300 python bench.py --workload $w --scan-algo stream --no-oracle --no-e2e --steps 300 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rnd $v', '$w', d['value'], d['roofline']['frac'])"
  done
done
done
