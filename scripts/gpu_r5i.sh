# ncu --set full of the block reduction's warp-row kernel (bench workload) + the cluster kernel (B = 2^20)
: timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_reduce_rows -s 5 -c 1 -o gpurun_out/prof_reduce_rows_f32 python bench.py --workload reduce64M_f32 --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_reduce.log 2>&1; echo rows rc=$?
cat > gpurun_out/red_cluster.py <<'PY'
import torch, paper_2305_03448_b200 as desc
x = torch.randn(1 << 26, device="cuda")
for _ in range(8): desc.block_reduce(x, 1 << 20)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_reduce_cluster -s 5 -c 1 -o gpurun_out/prof_reduce_cluster_f32 env PYTHONPATH=. python gpurun_out/red_cluster.py > gpurun_out/ncu_reduce2.log 2>&1; echo cluster rc=$?
for w in reduce64M_f32 scan64M_f32; do timeout 300 python bench.py --workload $w --steps 1000 --warmup 50 --no-e2e > gpurun_out/bench_$w.json 2>/dev/null; tail -1 gpurun_out/bench_$w.json | cut -c1-100; done
