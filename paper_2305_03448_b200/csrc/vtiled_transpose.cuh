// vtiled_transpose.cuh -- the 16-byte-vector tile transpose (DESC_KERNEL_VTILED).
//
// Same operation as every other variant (caption P:108): out[j][i] = in[i][j].
// Listing 1's shape (one tile per block, the tile staged through shared memory, one barrier
// between the two copies, P:49-60 with the P:44 fix) with every global and shared access
// 16 bytes wide, as north_star (3) describes:
//   * the tile (TR rows x TCH 16-byte chunks) is staged with cp.async.cg 16-byte copies
//     (LDGSTS: global -> shared without registers, L1 bypassed), DESC_VT_CPA=0 for
//     LDG.128 -> STS.128 (A/B); all of a thread's copies are in flight before it waits,
//   * the staging layout is XOR-swizzled at 16-byte granularity -- chunk c of tile row w
//     sits at chunk c ^ ((w / VEC) & 7) -- so the row-major copy-in (8 lanes of a phase:
//     one row, 8 chunks) and the micro-block reads of the copy-out (8 lanes: 8 micro-rows,
//     one chunk) both touch 8 distinct 16-byte bank groups: no conflicts, no padding,
//   * each thread reads VEC x VEC micro-blocks (VEC = 16 / cell size: 4x4 f32, 2x2 f64,
//     8x8 16-bit, 16x16 bytes) with VEC ld.shared.v4, transposes them in registers (renaming
//     for 4/8-byte cells, byte permutes for 1/2-byte cells) and writes VEC 16-byte stores;
//     16 lanes cover one 256-byte output row segment, so every warp store instruction writes
//     two fully coalesced 256-byte segments,
//   * one tile per CTA in a 1-D grid, PDL with the L2 prefetch of the CTA's tile before
//     griddepcontrol.wait (as TILED, tiled_transpose.cuh), predicated edge tiles.
// Eligibility (host, vtiled_ok): 16-byte aligned bases, ld_in, ld_out (and the batch
// strides) and rows, cols multiples of VEC -- edge tiles then hold whole chunks and whole
// micro-blocks.  Tile: TR = 16 VEC rows (64 f32, 32 f64, 128 16-bit, 256 bytes).
#pragma once
#include <cstdint>

#include <utility>

#include "mutants.cuh"
#include "ptx.cuh"
#include "tma_transpose.cuh"      // micro_row: the VEC x VEC register micro-transposes

namespace desc {

#ifndef DESC_VT_CPA              // 1: cp.async.cg staging (default), 0: LDG.128 + STS.128
#define DESC_VT_CPA 1
#endif
#ifndef DESC_VT_MINB             // __launch_bounds__ min blocks (0: none)
#define DESC_VT_MINB 0
#endif

// TR tile rows x TCH 16-byte chunks per row (TC = TCH * VEC cells), NT threads.
// Micro-block b = tid + NT * m: micro-row mr = b % 16 (input rows VEC*mr .. +VEC-1), chunk
// mc = b / 16 (input cells VEC*mc .. +VEC-1); 16 micro-rows per tile (TR = 16 * VEC).
template <int ES, int TCH_, int NT_>
struct VTiledCfg {
    static constexpr int VEC = 16 / ES;                 // cells per 16-byte chunk
    static constexpr int TR = 16 * VEC;                 // tile rows: 64 (4-byte), 32 (8-byte), ...
    static constexpr int TCH = TCH_;                    // chunks per tile row
    static constexpr int TC = TCH * VEC;                // tile cols (cells)
    static constexpr int NT = NT_;
    static constexpr int LPT = TR * TCH / NT;           // chunk copies per thread
    static constexpr int MPT = 16 * TCH / NT;           // micro-blocks per thread
    static constexpr int SMEM = TR * TCH * 16;
    static_assert(TCH >= 8 && (TCH & (TCH - 1)) == 0, "swizzle spans 8 chunks");
    static_assert(LPT * NT == TR * TCH && MPT * NT == 16 * TCH && MPT >= 1, "thread shape");
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ uint4 ldg128(const void *p) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int ES, int J>
__device__ __forceinline__ void vt_emit_row(const uint4 (&x)[16 / ES], char *drow, int64_t ld_b,
                                            int jmax) {
    if (J < jmax) {
        uint4 o = micro_row<ES, J>(x);
        if (DESC_MUTANT(MUT_TILED_TILE_ONLY)) o = x[J];
        ptx::stg128(drow + (int64_t)J * ld_b, o);
    }
}

template <int ES, int... J>
__device__ __forceinline__ void vt_emit(const uint4 (&x)[16 / ES], char *drow, int64_t ld_b,
                                        int jmax, std::integer_sequence<int, J...>) {
    (vt_emit_row<ES, J>(x, drow, ld_b, jmax), ...);
}

template <int ES, int TCH_, int NT_>
__global__ void __launch_bounds__(NT_, DESC_VT_MINB)
transpose_vtiled_kernel(const char *__restrict__ in, char *__restrict__ out, int64_t rows,
                        int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                        int64_t stride_out, int64_t tiles_r, int64_t tiles_c, int64_t ntiles) {
    using C = VTiledCfg<ES, TCH_, NT_>;
    constexpr int VEC = C::VEC, TR = C::TR, TCH = C::TCH, TC = C::TC, NT = C::NT;
    extern __shared__ __align__(128) unsigned char vt_smem[];
    const uint32_t sbase = ptx::smem_u32(vt_smem);
    const int tid = threadIdx.x;
    const int64_t per = tiles_r * tiles_c;
    int64_t t = blockIdx.x;
    int64_t bt = t / per, ti = (t - bt * per) / tiles_c, tj = t - bt * per - ti * tiles_c;
    {   // L2 prefetch of this CTA's first tile, one per 128-byte line, before the wait (PDL)
        constexpr int LPRow = TCH * 16 / 128;
        if (t < ntiles && tid < TR * LPRow) {
            const int64_t row = ti * TR + tid / LPRow;
            const int64_t col = tj * TC + (tid % LPRow) * (128 / ES);
            if (row < rows && col < cols)
                ptx::prefetch_l2(in + (bt * stride_in + row * ld_in + col) * ES);
        }
    }
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();
    for (; t < ntiles; t += gridDim.x) {
        if (t != (int64_t)blockIdx.x) {
            bt = t / per;
            ti = (t - bt * per) / tiles_c;
            tj = t - bt * per - ti * tiles_c;
        }
        const int64_t r0 = ti * TR, c0 = tj * TC;
        const char *src = in + (bt * stride_in + r0 * ld_in + c0) * ES;
        char *dst = out + (bt * stride_out + c0 * ld_out + r0) * ES;
        const bool full = r0 + TR <= rows && c0 + TC <= cols;
        const int nr = (int)(rows - r0 < TR ? rows - r0 : TR);     // multiples of VEC
        const int nc = (int)(cols - c0 < TC ? cols - c0 : TC);
        // ---- copy-in: chunk q = tid + NT k -> tile row q / TCH, chunk q % TCH
#if DESC_VT_CPA
#pragma unroll
        for (int k = 0; k < C::LPT; ++k) {
            const int q = tid + NT * k, w = q / TCH, c = q % TCH;
            if (full || (w < nr && c * VEC < nc))
                cp_async16(sbase + (uint32_t)(w * TCH + (c ^ ((w / VEC) & 7))) * 16u,
                           src + ((int64_t)w * ld_in + c * VEC) * ES);
        }
        cp_async_wait_all();
#else
        {
            uint4 v[C::LPT];
#pragma unroll
            for (int k = 0; k < C::LPT; ++k) {
                const int q = tid + NT * k, w = q / TCH, c = q % TCH;
                if (full || (w < nr && c * VEC < nc))
                    v[k] = ldg128(src + ((int64_t)w * ld_in + c * VEC) * ES);
            }
#pragma unroll
            for (int k = 0; k < C::LPT; ++k) {
                const int q = tid + NT * k, w = q / TCH, c = q % TCH;
                if (full || (w < nr && c * VEC < nc))
                    ptx::sts128(sbase + (uint32_t)(w * TCH + (c ^ ((w / VEC) & 7))) * 16u, v[k]);
            }
        }
#endif
        if (!DESC_MUTANT(MUT_TILED_NO_SYNC)) __syncthreads();   // block-uniform condition
        // ---- copy-out: micro-block (mr, mc) -> VEC output rows c0 + VEC mc + j, cells
        // r0 + VEC mr .. + VEC - 1 of each
#pragma unroll
        for (int m = 0; m < C::MPT; ++m) {
            const int b = tid + NT * m, mr = b & 15, mc = b >> 4;
            if (!full && !(VEC * mr < nr && VEC * mc < nc)) continue;
            uint4 x[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                x[k] = ptx::lds128(sbase + (uint32_t)((VEC * mr + k) * TCH + (mc ^ (mr & 7))) * 16u);
            // output row VEC mc + j = column j of the VEC x VEC block (micro_row,
            // tma_transpose.cuh: register renaming for 4/8-byte cells, PRMT for 1/2-byte)
            const int jmax = full ? VEC : min(VEC, nc - VEC * mc);
            char *drow = dst + ((int64_t)(VEC * mc) * ld_out + VEC * mr) * ES;
            vt_emit<ES>(x, drow, ld_out * ES, jmax, std::make_integer_sequence<int, VEC>{});
        }
        __syncthreads();                                  // staging reused by the next tile
    }
}

}  // namespace desc
