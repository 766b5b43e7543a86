# refactored distributed measurement: 1 rank, and 2 ranks sharing the GPU (gloo + IPC peer path)
timeout 600 python bench.py --workload dist65536 --dist-n 32768 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-600
DESC_BENCH_BACKEND=gloo DESC_BENCH_EXCHANGE_P2P=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 100 --warmup 10 --exchange-n 16384 > gpurun_out/bench_n2x.json 2> gpurun_out/bench_n2x.err; echo n2 rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_n2x.json')); print(d['value'], d.get('exchange'))"; tail -3 gpurun_out/bench_n2x.err
DESC_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 2 --workload dist65536 --dist-impl p2p --dist-n 16384 --steps 10 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
