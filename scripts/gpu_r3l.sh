# scan algorithms on 2^26 (A/B), 4096^2 f64 with and without PDL
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --workload $1 --no-e2e --no-oracle --steps 300 --warmup 10 ${@:2} 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["ms_per_step"])'; }
for w in scan64M_f32 scan64M_i32; do for a in stream lookback three_pass; do echo "$w $a $(b $w --scan-algo $a)"; done; done
for p in 0 1; do echo "4096f64 PDL=$p $(DESC_PDL=$p b 4096f64) $(DESC_PDL=$p b 4096f64)"; done
echo "reduce PDL=0 $(DESC_PDL=0 b reduce64M_f32)  PDL=1 $(b reduce64M_f32)"
