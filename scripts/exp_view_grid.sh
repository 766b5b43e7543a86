#!/bin/bash
# r02 (session 2): view_tiles kernel A/B -- persistent vs one item per CTA (DESC_VIEW_GRID),
# L2 prefetch of the first item before the dependency wait (DESC_VIEW_PF)
for r in 1 2; do
  for g in 0 1; do for pf in 0 1; do for w in view_tiles8192f32 view_flip8192f32; do
    DESC_VIEW_GRID=$g DESC_VIEW_PF=$pf python bench.py --workload $w --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('grid=$g pf=$pf', '$w', d['value'], d['roofline']['frac'], d['parity'])"
  done; done; done
done
