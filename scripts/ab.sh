#!/bin/bash
# Named A/B experiments of round 2 (each was a one-off driver; folded here).
#   bash scripts/ab.sh <name> [args...]      names: tiled_tpc tiled_128rows vtiled_minb view_unroll e2e_batch tiled_variants vtiled vtiled_narrow scan_variants release e2e_axis e2e_bands copy view_grid view_pf1 view_old regress f64_2048
# Compile-time variants come from scripts/build_{tiled,scan}_variants.py (DESC_LIB=...);
# each experiment prints the lines its profiles/r02_*.txt record holds.

tiled_variants() {
  # (the TILED knobs these variants used were removed after the recorded run; see
  #  scripts/build_tiled_variants.py)
  # r03 TILED A/B: product vs compile-time variants (scripts/build_tiled_variants.py), interleaved
  #   bash scripts/ab.sh tiled_variants "<variants>" "<shapes>" <rounds>
  V=${1:-"cpa5 cpa8 r4 r8 r16 r32 ldcs ldlu stcs stcg ldcs_stcs minb6"}
  S=${2:-"8192x8192:f32,3000x5000:f64,2048x2048:f64,4096x4096:f64,8192x8192:f64,256x1024x1024:f32"}
  R=${3:-2}
  for r in $(seq $R); do
    echo "## round $r"
    python scripts/exp_kernels.py --kernels tiled --shapes $S
    for v in $V; do
      DESC_LIB=build_variants/lib_tiled_$v.so python scripts/exp_kernels.py --kernels tiled --shapes $S
    done
  done
}

vtiled() {
  # r02 (session 2): DESC_KERNEL_VTILED A/B against TILED (exp_kernels.py timing), tile configs
  #   bash scripts/ab.sh vtiled "<cfgs>" "<shapes>" <rounds>
  C=${1:-"1 2 3"}
  S=${2:-"8192x8192:f32,3000x5000:f64,2048x2048:f64,4096x4096:f64,8192x8192:f64,256x1024x1024:f32,4096x4096:f32"}
  R=${3:-2}
  for r in $(seq $R); do
    echo "## round $r"
    python scripts/exp_kernels.py --kernels tiled,vtiled --shapes $S
    for c in $C; do DESC_VTILED_CFG=$c python scripts/exp_kernels.py --kernels vtiled --shapes $S | sed "s/^/cfg$c /"; done
  done
}

vtiled_narrow() {
  # r02 (session 2): 1/2-byte cells -- the TMA-load kernel (AUTO's choice so far) vs VTILED
  # (16x16 / 8x8 byte-permute micro-transposes) vs TILED (cell-wide accesses), tile configs
  S=${1:-"8192x8192:u8,16384x16384:u8,8192x8192:bf16,4096x4096:bf16,2048x2048:u8,256x1024x1024:bf16"}
  for r in 1 2; do
    python scripts/exp_kernels.py --kernels tma,vtiled,tiled --shapes $S
    for c in 1 2; do DESC_VTILED_CFG=$c python scripts/exp_kernels.py --kernels vtiled --shapes $S | sed "s/^/cfg$c /"; done
  done
}

scan_variants() {
  # r02 scan A/B: lane-contiguous layout with TMA-store staging (scripts/build_scan_variants.py)
  #   bash scripts/ab.sh scan_variants "<variant:workload ...>" <rounds>
  # parity (the scan GPU tests) for each non-diagnostic variant, then bench lines interleaved
  V=${1:-"nolc:scan64M_f32 lc_i32:scan64M_i32 lc_i32_nr8:scan64M_i32 lc_f64:scan32M_f64"}
  R=${2:-2}
  for vw in $V; do
    v=${vw%%:*}
    case $v in *diag*) continue;; esac     # diagnostics builds compute wrong results by design
    echo "## parity $v"
    DESC_LIB=build_variants/lib_$v.so timeout 600 python -m pytest tests/test_reduce_scan_gpu.py -q -m gpu -k "scan" -x 2>&1 | tail -1
  done
  line() {  # label workload [env]
    python bench.py --workload $2 --steps 20 --warmup 5 --no-oracle --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', '$2', d['value'], d['roofline']['frac'])"
  }
  for r in $(seq $R); do
    echo "## round $r"
    for w in $(for vw in $V; do echo ${vw#*:}; done | sort -u); do line product $w; done
    for vw in $V; do v=${vw%%:*}; w=${vw#*:}; DESC_LIB=build_variants/lib_$v.so line $v $w; done
  done
}

release() {
  # r02 (session 2): TMA ring slot release after ld.shared -- stress (mismatch count) and speed
  # (the recorded run also had rel1 / rel2 builds; rel1 -- the fence -- is now the product)
  for lib in build_variants/lib_tiled_rel0.so paper_2305_03448_b200/libdesc_transpose.so; do
    v=$(basename $lib .so)
    echo "## $v"
    DESC_LIB=$lib timeout 900 python scripts/stress_8192.py 150 tma,tma_st 2>&1 | grep -v "^MISMATCH"
    DESC_LIB=$lib python scripts/exp_kernels.py --kernels tma,tma_st --shapes 8192x8192:f32,3000x5000:f64 | sed "s/^/$v /"
  done
}

e2e_axis() {
  for ax in 1 2 1 2; do
    echo "## DESC_HOST_AXIS=$ax"
    DESC_HOST_AXIS=$ax python scripts/exp_e2e.py 2>&1 | grep desc_transpose_host
    DESC_HOST_AXIS=$ax python bench.py --steps 20 --warmup 5 --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench e2e', d['e2e']['value'], d['e2e']['pcie_ceiling'], d['e2e']['spot_check'], 'value', d['value'])"
  done
}

e2e_bands() {
  # r02 (session 2): e2e with at least DESC_HOST_BANDS bands per matrix (0 = largest band that fits)
  for r in 1 2; do
  for nb in 0 8 16; do
    for w in 8192f32 2048f64 3000x5000f64; do
      DESC_HOST_BANDS=$nb python bench.py --workload $w --steps 20 --warmup 5 --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('bands>=$nb', '$w', e['value'], e['pcie_ceiling']['frac'], e['spot_check'], e['gpu_launches'])"
    done
  done
  done
}

copy() {
  for r in 1 2; do for g in 0 1; do for u in 4 8; do DESC_COPY_GRID=$g DESC_COPY_UNR=$u python scripts/exp_copy.py; done; done; done
}

view_grid() {
  # r02 (session 2): view_tiles kernel A/B -- persistent vs one item per CTA (DESC_VIEW_GRID),
  # L2 prefetch of the first item before the dependency wait (DESC_VIEW_PF)
  for r in 1 2; do
    for g in 0 1; do for pf in 0 1; do for w in view_tiles8192f32 view_flip8192f32; do
      DESC_VIEW_GRID=$g DESC_VIEW_PF=$pf python bench.py --workload $w --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('grid=$g pf=$pf', '$w', d['value'], d['roofline']['frac'], d['parity'])"
    done; done; done
  done
}

view_pf1() {
  # (the viewpf1 build's knob was removed after the recorded run: scripts/build_tiled_variants.py)
  # r02 (session 2): the plain 16-byte view mode (group_by_tile) with the first-item L2 prefetch
  # compiled in (viewpf1 build), persistent vs one item per CTA
  for r in 1 2; do
    for g in 0 1; do for pf in 0 1; do
      DESC_LIB=build_variants/lib_tiled_viewpf1.so DESC_VIEW_GRID=$g DESC_VIEW_PF=$pf python bench.py --workload view_tiles8192f32 --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('viewpf1 grid=$g pf=$pf', d['value'], d['roofline']['frac'], d['parity'])"
    done; done
    python bench.py --workload view_tiles8192f32 --steps 20 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('product', d['value'], d['roofline']['frac'], d['parity'])"
  done
}

view_old() {
  # r02 (session 2): view workloads, pre-session library (f69d7a8) vs the current one
  for r in 1 2; do
  for lib in build_variants/lib_f69d7a8.so paper_2305_03448_b200/libdesc_transpose.so; do
    for w in view_tiles8192f32 view_flip8192f32 view_transpose8192f32 view_rot90_8192f32; do
      DESC_LIB=$lib python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', '$w', d['value'], d['roofline']['frac'])"
    done
  done
  done
}

regress() {
  # Regression A/B: every bench workload (but dist65536), a reference library build vs the
  # current one, interleaved, two rounds.   bash scripts/ab.sh regress <reference .so>
  REF=${1:-build_variants/lib_f69d7a8.so}
  W="8192f32 2048f64 3000x5000f64 4096f64 8192i32 8192f64 3000x5000f64_ld5001 8192f32_ld8193 batched view_tiles8192f32 view_transpose8192f32 view_rot90_8192f32 view_flip8192f32 reduce64M_f32 scan64M_f32 scan64M_i32 scan32M_f64"
  for r in 1 2; do
    for w in $W; do
      for lib in $REF paper_2305_03448_b200/libdesc_transpose.so; do
        DESC_LIB=$lib python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-oracle 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%-44s %-22s %9.1f %.4f' % ('$lib', '$w', d['value'], d['roofline']['frac']))"
      done
    done
  done
}

f64_2048() {
  # r02 (session 2): the paper's listing shape (2048^2 f64) in the bench's own timing: TILED tile
  # shapes (DESC_TILED_CFG) and VTILED configs (DESC_VTILED_CFG), 2 rounds
  line() { python bench.py --workload 2048f64 --steps 20 --warmup 5 --no-oracle --no-e2e --no-context $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$2', d['value'], d['roofline']['frac'])"; }
  for r in 1 2; do
    for c in 0 1 2 3 4 5 6; do DESC_TILED_CFG=$c line "" "tiled cfg$c"; done
    for c in 0 1 2 3 4 5 6; do DESC_VTILED_CFG=$c line "--kernel vtiled" "vtiled cfg$c"; done
  done
}

e2e_batch() {
  # r02 (session 2): batched e2e -- whole-matrix bands (contiguous copies) vs the previous
  # zero-copy path (DESC_HOST_BATCH=0)
  for r in 1 2; do for b in 1 0; do
    DESC_HOST_BATCH=$b python bench.py --workload batched --steps 20 --warmup 5 --no-oracle --no-context 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('batch_bands=$b', e['value'], e['pcie_ceiling']['frac'], e['spot_check'], e['gpu_launches'])"
  done; done
}

view_unroll() {
  # r02 (session 2): view copies, loads in flight per thread in the short-row path (4 default)
  for r in 1 2; do
    for lib in paper_2305_03448_b200/libdesc_transpose.so build_variants/lib_tiled_viewunr8.so build_variants/lib_tiled_viewunr2.so; do
      for w in view_tiles8192f32 view_flip8192f32; do
        DESC_LIB=$lib python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-context 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $lib .so)', '$w', d['value'], d['roofline']['frac'], d['parity'])"
      done
    done
  done
}

vtiled_minb() {
  # r02 (session 2): VTILED residency (register caps via __launch_bounds__ min blocks)
  S=8192x8192:f32,4096x4096:f32,256x1024x1024:f32,8192x8192:f64,3000x5000:f64
  for r in 1 2; do
    python scripts/exp_kernels.py --kernels tiled,vtiled --shapes $S
    for v in vtminb10 vtminb12; do DESC_LIB=build_variants/lib_tiled_$v.so python scripts/exp_kernels.py --kernels vtiled --shapes $S; done
  done
}

tiled_128rows() {
  # r02 (session 2): TILED f32 tiles with 128 rows (512-byte output row segments): cfg 7 =
  # 128x64/256 thr, 8 = 128x128/512, 9 = 128x32/128 against the 64x64/256 default
  # (needs those cases back in run_tiled, desc_transpose.cu; removed after the recorded run)
  for r in 1 2; do for c in 0 7 8 9; do
    DESC_TILED_CFG=$c python bench.py --steps 20 --warmup 5 --no-oracle --no-e2e --no-context 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cfg$c 8192f32', d['value'], d['roofline']['frac'], d['parity'])"
    DESC_TILED_CFG=$c python scripts/exp_kernels.py --kernels tiled --shapes 4096x4096:f32,256x1024x1024:f32 | sed "s/^/cfg$c /"
  done; done
}

tiled_tpc() {
  # r02 (session 2): TILED with k tiles per CTA (DESC_TILED_TPC) and the second tile prefetched
  # before the dependency wait too (tiledpf2 build; its knob was removed after the run)
  line() { python bench.py --workload $1 --steps 20 --warmup 5 --no-oracle --no-e2e --no-context 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$2', '$1', d['value'], d['roofline']['frac'])"; }
  for r in 1 2; do for w in 8192f32 2048f64 batched; do
    line $w "product tpc1"
    DESC_TILED_TPC=2 line $w "product tpc2"
    DESC_LIB=build_variants/lib_tiled_tiledpf2.so DESC_TILED_TPC=2 line $w "pf2 tpc2"
    DESC_LIB=build_variants/lib_tiled_tiledpf2.so DESC_TILED_TPC=4 line $w "pf2 tpc4"
  done; done
}

name=$1; shift
case " tiled_tpc tiled_128rows vtiled_minb view_unroll e2e_batch tiled_variants vtiled vtiled_narrow scan_variants release e2e_axis e2e_bands copy view_grid view_pf1 view_old regress f64_2048 " in *" $name "*) "$name" "$@";; *) echo "unknown experiment: $name"; exit 2;; esac
