# cluster-per-block reduction: 8-CTA clusters down to nb = SMs / 8, adaptive CTA size
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -x 2>&1 | tail -1
for rnd in 1 2; do timeout 300 python scripts/exp_reduce_blocks.py | grep -E "B=(16384|65536|1048576|4194304):"; done
