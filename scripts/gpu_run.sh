#!/bin/bash
# One parameterised GPU driver (replaces the round-1 one-off gpu_r*.sh launchers).
#   gpurun --timeout S -- 'bash scripts/gpu_run.sh <stage> [<stage> ...]'
# Every stage is bounded by `timeout`, writes its log under gpurun_out/ and prints one
# status line; later stages still run when one fails.
#   smoke      __graft_entry__.smoke()
#   tests      pytest -m gpu (whole suite)          tests:<pytest -k expr>  a subset
#   bench      default bench line (8192^2 f32, N = 1)   -> gpurun_out/bench.json
#   bench:<w>  bench.py --workload <w>                  -> gpurun_out/bench_<w>.json
#   dist1      configs[4] on one GPU: 65536^2 f32, every element verified
#   gloo2      the N > 1 code path with 2 ranks sharing the GPU (gloo, host-staged
#              all-to-all, peer path through CUDA IPC), 16384^2
#   sanitize   product sanitizer gates + positive controls (scripts/gpu_sanitize.sh; the
#              pool has refused compute-sanitizer since r02 session 2 -> exits 3, SKIPPED)
#   launches   ncu launch list (gpu__time_duration) of the default bench command
#   ncu:<w>:<kernel regex>   one ncu --set full capture of that kernel in that workload
#   exp:<script args>        python scripts/<script> <args>
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv,noheader
for st in "$@"; do
  t0=$(date +%s)
  case "$st" in
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)";;
    tests)
      timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
      echo "tests rc=$? $(tail -1 gpurun_out/pytest_gpu.log)";;
    tests:*)
      timeout 2400 python -m pytest tests -q -m gpu -k "${st#tests:}" > gpurun_out/pytest_sub.log 2>&1
      echo "tests[${st#tests:}] rc=$? $(tail -1 gpurun_out/pytest_sub.log)";;
    bench)
      timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
      echo "bench rc=$?"; cut -c1-400 gpurun_out/bench.json;;
    bench:*)
      w=${st#bench:}
      timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
      echo "bench $w rc=$?"; cut -c1-300 gpurun_out/bench_$w.json;;
    dist1)
      timeout 900 python bench.py --workload dist65536 --steps 10 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
      echo "dist1 rc=$?"; cut -c1-600 gpurun_out/bench_dist1.json;;
    gloo2)
      DESC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
          --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 \
          --dist-n 16384 --dist-e2e-n 8192 > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err
      echo "gloo2 rc=$?"; cut -c1-600 gpurun_out/bench_gloo2.json;;
    sanitize)
      timeout 3000 bash scripts/gpu_sanitize.sh > gpurun_out/sanitize.log 2>&1
      echo "sanitize rc=$?"; cat gpurun_out/sanitize.log;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-oracle --no-e2e --no-context \
          > gpurun_out/launches_bench.log 2>&1
      echo "launches rc=$?";;
    ncu:*)
      # summarised ON THE BOX (reports are ~12 MB each and gpurun copies back <= 64 MiB):
      # gpurun_out/ncu_<w>_<k>.md + the traffic entry in gpurun_out/ncu_traffic.json;
      # KEEP_REP=1 keeps the .ncu-rep too
      rest=${st#ncu:}; w=${rest%%:*}; k=${rest#*:}
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 \
          -o gpurun_out/prof_${w}_${k} -f python bench.py --workload $w --steps 8 --warmup 3 \
          --no-oracle --no-e2e --no-context > gpurun_out/ncu_${w}_${k}.log 2>&1
      echo "ncu $w $k rc=$?"
      python scripts/ncu_summary.py gpurun_out/prof_${w}_${k}.ncu-rep gpurun_out/ncu_${w}_${k}.md $w > /dev/null 2>&1
      cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
      [ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/prof_${w}_${k}.ncu-rep;;
    exp:*)
      timeout 1200 python scripts/${st#exp:} > gpurun_out/exp.log 2>&1
      echo "exp ${st#exp:} rc=$?"; tail -40 gpurun_out/exp.log;;
    *) echo "unknown stage $st";;
  esac
  echo "   [$st took $(( $(date +%s) - t0 )) s]"
done
nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu --format=csv,noheader
