#!/bin/bash
# r02 (session 2): the paper's listing shape (2048^2 f64) in the bench's own timing: TILED tile
# shapes (DESC_TILED_CFG) and VTILED configs (DESC_VTILED_CFG), 2 rounds
line() { python bench.py --workload 2048f64 --steps 20 --warmup 5 --no-oracle --no-e2e --no-context $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$2', d['value'], d['roofline']['frac'])"; }
for r in 1 2; do
  for c in 0 1 2 3 4 5 6; do DESC_TILED_CFG=$c line "" "tiled cfg$c"; done
  for c in 0 1 2 3 4 5 6; do DESC_VTILED_CFG=$c line "--kernel vtiled" "vtiled cfg$c"; done
done
