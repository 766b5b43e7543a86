# block reduction: loads in flight per lane x CTAs per SM (compile-time variants), 2 rounds
for rnd in 1 2; do
for v in base ru8 rc8 ru8c8 ru8c4 rc32; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  DESC_LIB=$L timeout 300 python bench.py --workload reduce64M_f32 --no-oracle --no-e2e --steps 500 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rnd $v', d['value'], d['roofline']['frac'])"
done
done
