# scan: state reset as a PDL-chained kernel instead of cudaMemsetAsync
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py tests/test_mutants_gpu.py -x -q 2>&1 | tail -2
b() { timeout 300 python bench.py --workload $1 --no-e2e --steps 300 --warmup 10 ${@:2} 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["ms_per_step"], d.get("parity"), d.get("gpu_launches"))'; }
for w in scan64M_f32 scan64M_i32; do echo "$w PDL=1 $(b $w) $(b $w --no-oracle)"; echo "$w PDL=0 $(DESC_PDL=0 b $w --no-oracle)"; done
for t in racecheck synccheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
