# streaming scan: quick sanity, parity suite, A/B against the other scan algorithms
timeout 120 python -c "
import torch, numpy as np, paper_2305_03448_b200 as d
x=torch.arange(1<<24, device='cuda', dtype=torch.int32)
y=d.scan(x, algo='stream'); torch.cuda.synchronize(); print('stream ok', y[-1].item(), (x.long().cumsum(0).int()==y).all().item())
" 2>&1 | tail -3; echo quick rc=$?
timeout 900 python -m pytest tests/test_reduce_scan_gpu.py -x -q > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_scan.log
for a in stream three_pass lookback; do for w in scan64M_f32 scan64M_i32; do
 timeout 300 python bench.py --workload $w --scan-algo $a --no-oracle --steps 200 --warmup 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', '$w', d['value'], d['roofline']['frac'], d['gpu_launches'])"
done; done
