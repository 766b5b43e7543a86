# chunked NCCL-path local steps (multi-process, one GPU) and the peer exchange object
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_dist.log
DESC_BENCH_BACKEND=gloo DESC_BENCH_EXCHANGE_P2P=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 50 --warmup 5 --exchange-n 16384 --no-oracle > gpurun_out/bench_n2x.json 2> gpurun_out/bench_n2x.err; echo n2 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_n2x.json')); print(d['value'], d.get('exchange'), d.get('exchange_p2p'))"; tail -3 gpurun_out/bench_n2x.err
timeout 600 python bench.py --workload dist65536 --dist-n 32768 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-400
