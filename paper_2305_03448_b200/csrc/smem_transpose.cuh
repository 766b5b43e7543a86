// smem_transpose.cuh -- the alignment-agnostic shared-memory tile transpose.
//
// This is the paper's Listing 1 schedule with the fix the paper
// states (`(threadIdx.y+j)*32`), generalised per DESIGN.md R4-R8:
//   * 32x32 tile, 32x8 threads, each thread moves 4 elements per phase,
//   * staging buffer of the element's own width (never `float` for f64: R4),
//   * padded to [32][33] so the column read is bank-conflict free,
//   * predicated edges (R6), leading dimensions and batch strides (R8),
//   * 64-bit offsets (65536^2 has 2^32 elements).
// Used for any alignment the TMA path cannot take (odd ld, unaligned base).
#pragma once
#include <cstdint>

#include "mutants.cuh"

namespace desc {

template <typename Cell>
__global__ void __launch_bounds__(256)
transpose_smem_kernel(const Cell *__restrict__ in, Cell *__restrict__ out, int64_t rows,
                      int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                      int64_t stride_out, int64_t tiles_r, int64_t tiles_c, int64_t ntiles) {
    __shared__ Cell tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t tiles_per_mat = tiles_r * tiles_c;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t bt = t / tiles_per_mat;
        const int64_t rem = t - bt * tiles_per_mat;
        const int64_t ti = rem / tiles_c;                 // tile row  (blockIdx.y in P:54)
        const int64_t tj = rem - ti * tiles_c;            // tile col  (blockIdx.x in P:55)
        const Cell *src = in + bt * stride_in;
        Cell *dst = out + bt * stride_out;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {                 // copy-in, P:52-55 (fixed)
            const int64_t i = ti * 32 + ty + j, c = tj * 32 + tx;
            if (i < rows && c < cols) {
                Cell v = src[i * ld_in + c];
                if constexpr (sizeof(Cell) == 8) {             // test-teeth variant only
                    if (DESC_MUTANT(MUT_SMEM_FLOAT_TMP))
                        v = (Cell)__double_as_longlong((double)(float)__longlong_as_double((long long)v));
                }
                if (DESC_MUTANT(MUT_SMEM_NO_PAREN)) (&tile[0][0])[ty + j * 33 + tx] = v;
                else tile[ty + j][tx] = v;
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {                 // copy-out
            const int64_t orow = tj * 32 + ty + j, ocol = ti * 32 + tx;
            const int64_t ocol_lim = rows + (DESC_MUTANT(MUT_SMEM_EDGE) ? 1 : 0);
            if (orow < cols && ocol < ocol_lim)
                dst[orow * ld_out + ocol] = DESC_MUTANT(MUT_SMEM_TILE_ONLY) ? tile[ty + j][tx]
                                                                           : tile[tx][ty + j];
        }
        __syncthreads();                                  // tile reused by the next iteration
    }
}

}  // namespace desc
