# TILED tile-shape sweep (compile-time variants via DESC_LIB)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --workload $1 --kernel tiled --no-e2e --no-oracle --steps 200 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])'; }
for w in 8192f32 batched 3000x5000f64 8192f64 4096f64 2048f64; do
  echo "default $w $(b $w) $(b $w)"
  for v in a b c d; do echo "$v $w $(DESC_LIB=build_variants/lib_tiled_$v.so b $w)"; done
done
