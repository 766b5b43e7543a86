// tiled_transpose.cuh -- the alignment-agnostic transpose for B200 (DESC_KERNEL_TILED).
//
// Same operation as every other variant (caption P:108): out[j][i] = in[i][j].
// Taken by AUTO whenever the TMA rules reject the arguments (a base that is not 16-byte
// aligned, ld*size or stride*size not a multiple of 16 -- e.g. 3000 x 5000 f64 with
// ld_in = 5001, BASELINE configs[2] variant), where no vector or bulk access is legal, so the
// kernel has to reach HBM bandwidth with cell-wide accesses.  What differs from the paper's
// Listing 1 schedule (transpose_smem_kernel, kept as the faithful baseline):
//   * a TR x TC tile (64 x 64 cells for 1/2/4-byte cells, 32 x 64 for 8-byte cells), so a
//     warp row is 128 / 256 contiguous bytes on both sides,
//   * every thread issues all of its TR*TC/256 loads (16 for f32, 8 for f64) back to back into
//     registers before touching shared memory: 16 independent HBM requests in flight per
//     thread instead of Listing 1's one-at-a-time load/store pairs (B200 needs ~40 KB in
//     flight per SM to cover HBM latency at 6.5 TB/s),
//   * the staging tile is padded to TC + 1 cells: the column read of the copy-out hits 32
//     distinct banks (4-byte cells: lane*(TC+1) = lane mod 32; 8-byte cells: per half-warp
//     2*lane mod 32, each access covering two banks),
//   * one tile per CTA, 1-D grid (the block scheduler balances the SMs), interior tiles with
//     no predicates, edge tiles predicated (R6).
#pragma once
#include <cstdint>

#include "mutants.cuh"
#include "ptx.cuh"

namespace desc {

// A/B knobs (scripts/build_tiled_variants.py): tile rows / cols for 8-byte and narrower cells
#ifndef DESC_TILED_TR8           // 8-byte cells: 32 x 64 (sweep with PDL)
#define DESC_TILED_TR8 32
#endif
#ifndef DESC_TILED_TC8
#define DESC_TILED_TC8 64
#endif
#ifndef DESC_TILED_TR4
#define DESC_TILED_TR4 64
#endif
#ifndef DESC_TILED_TC4
#define DESC_TILED_TC4 64
#endif
#ifndef DESC_TILED_L2PF          // L2 prefetch of the first tile before griddepcontrol.wait
#define DESC_TILED_L2PF 1
#endif

// Tile TR x TC cells, NT threads (NW = NT/32 warps).  Loads: lane tx takes columns tx + 32g
// (g < TC/32) of rows ty + NW*k (k < TR/NW), all issued before the first shared store.
// Copy-out: LPR = min(TR, 32) lanes per output row, RPI = 32/LPR output rows per warp
// instruction: lane tx writes output row oc = RPI*(ty + NW*m) + tx/LPR, column
// orr = tx%LPR + LPR*h (each row segment = LPR cells = 128 / 256 contiguous bytes).
template <typename Cell, int TR_ = 0, int TC_ = 0, int NT_ = 256>
struct TiledCfg {
    static constexpr bool W8 = sizeof(Cell) == 8;
    static constexpr int TR = TR_ ? TR_ : (W8 ? DESC_TILED_TR8 : DESC_TILED_TR4);   // tile rows (input)
    static constexpr int TC = TC_ ? TC_ : (W8 ? DESC_TILED_TC8 : DESC_TILED_TC4);   // tile cols (input)
    static constexpr int NT = NT_;                          // threads
    static constexpr int NW = NT / 32;                      // warps
    static constexpr int CW = TC / 32;                      // column groups per lane
    static constexpr int RK = TR / NW;                      // rows per warp
    static constexpr int LPR = TR < 32 ? TR : 32;           // lanes per output row segment
    static constexpr int RPI = 32 / LPR;                    // output rows per warp instruction
    static constexpr int OK = TC / (RPI * NW);              // output row groups per warp
    static constexpr int OH = TR / LPR;                     // segments per output row
    static constexpr int SMEM = TR * (TC + 1) * (int)sizeof(Cell);   // padded staging tile
    static_assert(TC % 32 == 0 && TR % NW == 0 && TC % (RPI * NW) == 0 && 32 % LPR == 0,
                  "tile / thread shape");
};

// Scatter destinations of the fused peer-to-peer slab transpose (desc_slab_transpose_peer):
// input column c goes to destination s = c / seg, at column (c - s*seg) of that destination's
// rows, output column offset col_off (rank r's block of every destination slab).  seg is a
// multiple of the tile width, so a tile never straddles two destinations.
constexpr int kMaxScatter = 8;
struct TiledScatter {
    void *dst[kMaxScatter];
    int64_t seg;
    int64_t col_off;
};

// Register budget: 256-thread CTAs keep 5 resident per SM (<= 51 registers; the L2
// prefetch block would otherwise push the 4-byte kernel to 62 registers = 4 CTAs/SM and cost
// 3-4% at 8192^2); 128-thread CTAs: DESC_TILED_MINB128 (A/B; 0 = no constraint, 56 regs).
#ifndef DESC_TILED_MINB128
#define DESC_TILED_MINB128 0
#endif
template <typename Cell, int TR_ = 0, int TC_ = 0, int NT_ = 256, bool SCATTER = false>
__global__ void __launch_bounds__(NT_, NT_ >= 256 ? 5 : DESC_TILED_MINB128)
transpose_tiled_kernel(const Cell *__restrict__ in, Cell *__restrict__ out, int64_t rows,
                       int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                       int64_t stride_out, int64_t tiles_r, int64_t tiles_c, int64_t ntiles,
                       int64_t pf_ctas, const __grid_constant__ TiledScatter sc) {
    using C = TiledCfg<Cell, TR_, TC_, NT_>;
    constexpr int TR = C::TR, TC = C::TC, CW = C::CW, RK = C::RK, NW = C::NW;
    constexpr int LPR = C::LPR, RPI = C::RPI, OK = C::OK, OH = C::OH;
    extern __shared__ __align__(16) unsigned char tiled_smem[];
    Cell(*tile)[TC + 1] = reinterpret_cast<Cell(*)[TC + 1]>(tiled_smem);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ox = tx % LPR, oy = tx / LPR;                 // copy-out lane split
    const int64_t tiles_per_mat = tiles_r * tiles_c;
    // this CTA's first tile (computed once: used by the prefetch and the first iteration)
    int64_t t = blockIdx.x;
    int64_t bt = t / tiles_per_mat;
    int64_t ti = (t - bt * tiles_per_mat) / tiles_c;
    int64_t tj = t - bt * tiles_per_mat - ti * tiles_c;
#if DESC_TILED_L2PF
    // While a previous grid may still run (PDL), warm L2 with this CTA's first input tile:
    // one prefetch per 128-byte line of its rows, no data to the SM, no ordering needed --
    // L2 is the point of coherence, so lines a previous grid still writes stay correct for
    // the loads after griddepcontrol.wait.  Hides the ramp of a back-to-back launch behind
    // the previous launch's tail, and puts the whole tile's requests in flight at once --
    // more than the registers of the cell loads below can hold.  pf_ctas
    // limits it to the first pf_ctas CTAs (desc_transpose.cu launch_tiled: all by default).
    {
        constexpr int LPRow = (TC * (int)sizeof(Cell) + 127) / 128;    // lines per tile row
        if (t < pf_ctas && t < ntiles && (int)threadIdx.x < TR * LPRow) {
            const int r = threadIdx.x / LPRow, l = threadIdx.x % LPRow;
            const int64_t row = ti * TR + r, col = tj * TC + l * (128 / (int)sizeof(Cell));
            if (row < rows && col < cols)
                ptx::prefetch_l2(in + bt * stride_in + row * ld_in + col);
        }
    }
#endif
    // PDL: the next kernel in the stream may be scheduled into the slots our last wave
    // frees, but nothing here touches global memory before the previous grid has completed
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();
    for (; t < ntiles; t += gridDim.x) {
        if (t != (int64_t)blockIdx.x) {
            bt = t / tiles_per_mat;
            ti = (t - bt * tiles_per_mat) / tiles_c;
            tj = t - bt * tiles_per_mat - ti * tiles_c;
        }
        const int64_t r0 = ti * TR, c0 = tj * TC;
        const Cell *src = in + bt * stride_in + r0 * ld_in + c0;
        Cell *dst;
        if constexpr (SCATTER) {              // block (r, s)^T lands in destination s
            const int64_t sd = c0 / sc.seg;
            dst = static_cast<Cell *>(sc.dst[sd]) + (c0 - sd * sc.seg) * ld_out + sc.col_off + r0;
        } else {
            dst = out + bt * stride_out + c0 * ld_out + r0;
        }
        const bool full = r0 + TR <= rows && c0 + TC <= cols;
        Cell v[RK][CW];
        if (full) {
#pragma unroll
            for (int k = 0; k < RK; ++k)
#pragma unroll
                for (int g = 0; g < CW; ++g) v[k][g] = src[(int64_t)(ty + NW * k) * ld_in + tx + 32 * g];
#pragma unroll
            for (int k = 0; k < RK; ++k)
#pragma unroll
                for (int g = 0; g < CW; ++g) tile[ty + NW * k][tx + 32 * g] = v[k][g];
        } else {
            const int nr = (int)(rows - r0 < TR ? rows - r0 : TR);
            const int nc = (int)(cols - c0 < TC ? cols - c0 : TC);
#pragma unroll
            for (int k = 0; k < RK; ++k)
#pragma unroll
                for (int g = 0; g < CW; ++g) {
                    const int r = ty + NW * k, c = tx + 32 * g;
                    if (r < nr && c < nc) v[k][g] = src[(int64_t)r * ld_in + c];
                }
#pragma unroll
            for (int k = 0; k < RK; ++k)
#pragma unroll
                for (int g = 0; g < CW; ++g) {
                    const int r = ty + NW * k, c = tx + 32 * g;
                    if (r < nr && c < nc) tile[r][c] = v[k][g];
                }
        }
        if (!DESC_MUTANT(MUT_TILED_NO_SYNC)) __syncthreads();   // block-uniform condition
        // copy-out: output row c0 + oc (= input column), LPR lanes x OH segments contiguous
        if (full) {
#pragma unroll
            for (int m = 0; m < OK; ++m)
#pragma unroll
                for (int h = 0; h < OH; ++h) {
                    const int oc = RPI * (ty + NW * m) + oy, orr = ox + LPR * h;
                    dst[(int64_t)oc * ld_out + orr] =
                        DESC_MUTANT(MUT_TILED_TILE_ONLY) ? tile[oc][orr] : tile[orr][oc];
                }
        } else {
            const int nr = (int)(rows - r0 < TR ? rows - r0 : TR);
            const int nc = (int)(cols - c0 < TC ? cols - c0 : TC);
#pragma unroll
            for (int m = 0; m < OK; ++m)
#pragma unroll
                for (int h = 0; h < OH; ++h) {
                    const int oc = RPI * (ty + NW * m) + oy, orr = ox + LPR * h;
                    if (oc < nc && orr < nr + (DESC_MUTANT(MUT_TILED_EDGE) ? 1 : 0))
                        dst[(int64_t)oc * ld_out + orr] =
                            DESC_MUTANT(MUT_TILED_TILE_ONLY) ? tile[oc][orr] : tile[orr][oc];
                }
        }
        __syncthreads();                                  // tile reused by the next iteration
    }
}

}  // namespace desc
