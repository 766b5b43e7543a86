for ax in 1 2 1 2; do
  echo "## DESC_HOST_AXIS=$ax"
  DESC_HOST_AXIS=$ax python scripts/exp_e2e.py 2>&1 | grep desc_transpose_host
  DESC_HOST_AXIS=$ax python bench.py --steps 20 --warmup 5 --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench e2e', d['e2e']['value'], d['e2e']['pcie_ceiling'], d['e2e']['spot_check'], 'value', d['value'])"
done
