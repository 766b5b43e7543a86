# parity of the default build, then A/B of compile-time streaming-scan variants (DESC_LIB)
timeout 120 python -c "
import torch, paper_2305_03448_b200 as d
x=torch.arange(1<<24, device='cuda', dtype=torch.int32)
y=d.scan(x, algo='stream'); torch.cuda.synchronize(); print('stream quick', (x.long().cumsum(0).int()==y).all().item())
" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -x -q > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_scan.log
for v in base lb2 qt4 v10 v16s3q4 diag1 diag3; do
  if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
  for w in scan64M_f32 scan64M_i32; do
    DESC_LIB=$L timeout 300 python bench.py --workload $w --scan-algo stream --no-oracle --steps 300 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', d['value'], d['roofline']['frac'])"
  done
done
