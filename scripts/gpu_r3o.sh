python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "host" 2>&1 | tail -2
timeout 300 python bench.py --workload batched --no-oracle --steps 50 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); x=d["e2e"]; print("batched e2e", x["value"], x["pcie_ceiling"]["value"], x["gpu_launches"], x["spot_check"])'
