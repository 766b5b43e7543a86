// mutants.cuh -- deliberate, plausible defects for the "tests have teeth" gate
// (tests/test_mutants_gpu.py).
//
// The defects are compiled ONLY into a variant library built with -DDESC_MUTANTS
// (build_variants/libdesc_mutants.so, loaded by the test through DESC_LIB); there the
// environment variable DESC_MUTANT=<id> picks one of them at run time.  In the product build
// DESC_MUTANT(k) is the constant `false`, so none of this code reaches its SASS.
//
// Each id names the bug it models:
//   1 SMEM_TILE_ONLY     Listing 2 read literally: tiles permuted, not transposed
//   2 SMEM_NO_PAREN      Listing 1 as printed: tmp[ty + j*32 + tx] (a write race)
//   3 SMEM_FLOAT_TMP     Listing 1's `__shared__ float tmp` staging f64 data
//   4 SMEM_EDGE          copy-out edge predicate off by one (writes one padding column)
//   5 SWAP_LD            ld_in and ld_out swapped inside the library
//   6 TMA2_NO_MICRO      TMA kernel stores the 16-byte chunks untransposed (tile-only again)
//   7 TMA2_NO_TAIL       TMA kernel forgets the ragged output columns (rows % VEC)
//   8 TMA2_NO_SWIZZLE    TMA kernel reads the 128B-swizzled stage as if it were linear
//   9 TMA2_NO_FENCE      no fence.proxy.async / wait_group.read (a race; may not manifest)
//  10 SCAN_NO_LOOKBACK   scan tiles skip the decoupled look-back (prefix 0)
//  11 REDUCE_NO_TAIL     block reduction drops the scalar tail after the 16-byte body
//  12 TILED_TILE_ONLY    TILED kernel copies the tile out untransposed (Listing 2 literally)
//  13 TILED_EDGE         TILED edge-tile store predicate off by one (one padding cell written)
//  14 TILED_NO_SYNC      TILED kernel without the barrier between staging and copy-out (race)
//  15 SCAN_LC_NO_SWIZZLE streaming scan writes its TMA-store staging linearly (the tensor map
//                        unswizzles it: chunks land in the wrong places)
//  16 SCAN_LC_NO_WAIT    streaming scan rewrites its staging without waiting for the previous
//                        TMA store's reads and without the proxy fence (a race; may not manifest)
#pragma once

namespace desc {

enum DescMutant : int {
    MUT_NONE = 0,
    MUT_SMEM_TILE_ONLY = 1,
    MUT_SMEM_NO_PAREN = 2,
    MUT_SMEM_FLOAT_TMP = 3,
    MUT_SMEM_EDGE = 4,
    MUT_SWAP_LD = 5,
    MUT_TMA2_NO_MICRO = 6,
    MUT_TMA2_NO_TAIL = 7,
    MUT_TMA2_NO_SWIZZLE = 8,
    MUT_TMA2_NO_FENCE = 9,
    MUT_SCAN_NO_LOOKBACK = 10,
    MUT_REDUCE_NO_TAIL = 11,
    MUT_TILED_TILE_ONLY = 12,
    MUT_TILED_EDGE = 13,
    MUT_TILED_NO_SYNC = 14,
    MUT_SCAN_LC_NO_SWIZZLE = 15,
    MUT_SCAN_LC_NO_WAIT = 16,
};

#ifdef DESC_MUTANTS
__device__ int g_desc_mutant;
#define DESC_MUTANT(k) (::desc::g_desc_mutant == (k))
#else
#define DESC_MUTANT(k) false
#endif

}  // namespace desc
