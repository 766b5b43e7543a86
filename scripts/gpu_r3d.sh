# TILED vs TMA_ST across the workloads (3 repeats), and TILED compile-time variants
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --workload $1 --kernel $2 --no-e2e --no-oracle --steps 200 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])'; }
for w in 8192f32 batched 3000x5000f64 2048f64 4096f64 8192f64; do for k in tiled tma_st; do
  echo "$w $k $(b $w $k) $(b $w $k) $(b $w $k)"
done; done
for v in tc8_64 tr32 tr128; do for w in 8192f32 3000x5000f64 8192f64 2048f64; do
  echo "variant $v $w $(DESC_LIB=build_variants/lib_tiled_$v.so b $w tiled)"
done; done
