#!/bin/bash
# r02 (session 2): the plain 16-byte view mode (group_by_tile) with the first-item L2 prefetch
# compiled in (viewpf1 build), persistent vs one item per CTA
for r in 1 2; do
  for g in 0 1; do for pf in 0 1; do
    DESC_LIB=build_variants/lib_tiled_viewpf1.so DESC_VIEW_GRID=$g DESC_VIEW_PF=$pf python bench.py --workload view_tiles8192f32 --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('viewpf1 grid=$g pf=$pf', d['value'], d['roofline']['frac'], d['parity'])"
  done; done
  python bench.py --workload view_tiles8192f32 --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('product', d['value'], d['roofline']['frac'], d['parity'])"
done
