#!/bin/bash
# r02 (session 2): 1/2-byte cells -- the TMA-load kernel (AUTO's choice so far) vs VTILED
# (16x16 / 8x8 byte-permute micro-transposes) vs TILED (cell-wide accesses), tile configs
S=${1:-"8192x8192:u8,16384x16384:u8,8192x8192:bf16,4096x4096:bf16,2048x2048:u8,256x1024x1024:bf16"}
for r in 1 2; do
  python scripts/exp_kernels.py --kernels tma,vtiled,tiled --shapes $S
  for c in 1 2; do DESC_VTILED_CFG=$c python scripts/exp_kernels.py --kernels vtiled --shapes $S | sed "s/^/cfg$c /"; done
done
