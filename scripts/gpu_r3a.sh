# re-entry verification: build state from the restored checkpoint, on B200
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
DESC_BENCH_BACKEND=gloo DESC_BENCH_EXCHANGE_P2P=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 50 --warmup 5 --exchange-n 16384 > gpurun_out/bench_n2x.json 2> gpurun_out/bench_n2x.err; echo n2 rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.json | cut -c1-1500
tail -c 1500 gpurun_out/bench_n2x.json; tail -3 gpurun_out/bench_n2x.err
cat gpurun_out/bench_ref.json | cut -c1-600
