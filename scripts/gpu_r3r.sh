# f64 TILED tile shapes for small problems (rotating buffers + PDL)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --workload $1 --no-e2e --no-oracle --steps 500 --warmup 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["ms_per_step"])'; }
for w in 2048f64 3000x5000f64 4096f64 8192f64; do
  echo "$w head $(b $w) $(b $w)"
  for v in s1 s2 s3; do echo "$w $v $(DESC_LIB=build_variants/lib_tiled_$v.so b $w) $(DESC_LIB=build_variants/lib_tiled_$v.so b $w)"; done
done
