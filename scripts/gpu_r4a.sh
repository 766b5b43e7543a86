# NR (reduce/scan warp count) sweep of the streaming scan: A/B builds via DESC_LIB, 2 rounds
for rnd in 1 2; do
for v in base nr12v8 nr12v8p1 nr12v6q6 nr4v24; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  for w in scan64M_f32 scan64M_i32; do
    DESC_LIB=$L timeout 300 python bench.py --workload $w --scan-algo stream --no-oracle --no-e2e --steps 300 --warmup 20 2>gpurun_out/r4a_err_$v.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rnd $v', '$w', d['value'], d['roofline']['frac'], d.get('parity'))"
  done
done
done
