# e2e host path: banded copies vs zero-copy kernel over PCIe
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
e() { timeout 300 python bench.py --workload $1 --no-oracle --steps 50 --warmup 5 --e2e-steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); x=d["e2e"]; print(x["value"], x["pcie_ceiling"]["value"], x["spot_check"], x["gpu_launches"])'; }
for w in 8192f32 3000x5000f64 batched; do for m in 1 2; do echo "$w HOST_MODE=$m $(DESC_HOST_MODE=$m e $w) $(DESC_HOST_MODE=$m e $w)"; done; done
DESC_HOST_MODE=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "host" 2>&1 | tail -2
