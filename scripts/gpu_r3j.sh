# PDL on the TILED launch: back-to-back (rotating buffers) A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --workload $1 --no-e2e --no-oracle --steps 500 --warmup 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["ms_per_step"])'; }
for w in 2048f64 3000x5000f64 8192f32 8192f64 batched; do
  for p in 0 1; do echo "$w PDL=$p $(DESC_PDL=$p b $w) $(DESC_PDL=$p b $w)"; done
done
