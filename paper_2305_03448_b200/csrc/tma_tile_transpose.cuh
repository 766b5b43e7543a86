// tma_tile_transpose.cuh -- TMA in, TMA out, ONE tile per CTA (DESC_KERNEL_TMA_TILE).
//
// Same operation as every variant (caption P:108): out[j][i] = in[i][j].  The
// paper's schedule is one 32x32 tile per block with a block barrier between the copies
// (Listing 1/2); this kernel keeps that shape -- one tile per CTA, many
// CTAs resident per SM, the hardware block scheduler as the tile scheduler -- and moves both
// copies onto the Tensor Memory Accelerator:
//
//   a4 load     : one elected thread issues the tile's TMA box loads (128-byte swizzle) on
//                 one mbarrier (complete_tx); everyone waits on its phase 0
//   a6 transpose: the 4 warps read their VEC x VEC micro-blocks with conflict-free
//                 ld.shared.v4 into registers (the lane maps of the TMA-store kernel,
//                 StoreLane<ES>), __syncthreads, and write the transposed rows back INTO THE
//                 SAME buffer in the output tensor map's swizzled layout (the tile has been
//                 consumed, so no second buffer is needed: 16 KB of smem per CTA)
//   a5 barrier  : fence.proxy.async (generic writes -> async proxy) + __syncthreads
//   store       : the elected thread issues the TMA stores, then waits until they have read
//                 shared memory (cp.async.bulk.wait_group.read 0) before the CTA exits
//   a7 edges    : loads zero-fill out of range, stores clip at rows_main x cols; the ragged
//                 columns (rows % VEC) are written by the lanes that own them (R6, R8)
//
// Why this shape on B200: HBM bandwidth is set by bytes in flight per SM.  A
// persistent warp-specialised pipeline (transpose_tma2_kernel) caps them at its ring depth
// (2 x 32 KB with 1 CTA/SM); with 16 KB per CTA and 128 threads, up to 12 CTAs -- 192 KB of
// loads -- can be in flight per SM, issued by one instruction each, with no register
// staging of the loads at all.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "ptx.cuh"
#include "tma_transpose.cuh"
#include "tma_store_transpose.cuh"

namespace desc {

// ES: cell bytes; TR: input rows per tile; NB: 128-byte input boxes per tile (TILE_COLS =
// NB * 128 / ES input columns = output rows); CW warps; TPC tiles per CTA (all their loads
// are issued up front, one buffer and one mbarrier each, processed in order).
template <int ES, int TR, int NB, int CW_ = 4, int TPC_ = 1>
struct TmaTileConfig {
    using L = StoreLane<ES>;
    static constexpr int CW = CW_;                              // warps
    static constexpr int TPC = TPC_;
    static constexpr int THREADS = 32 * CW;
    static constexpr int TC = 128 / ES;
    static constexpr int BOX_BYTES = TR * 128;
    static constexpr int TILE_BYTES = BOX_BYTES * NB;
    static constexpr int TILE_COLS = NB * TC;
    static constexpr int OBOXES = TR * ES / 128;
    static constexpr int OBOX_BYTES = TILE_COLS * 128;
    static constexpr int CHUNK_GROUPS = 8 / L::CHUNKS_PER_WARP;
    static constexpr int TASKS_PER_BOX = (TR / L::ROWS_PER_WARP) * CHUNK_GROUPS;
    static constexpr int TASKS = TASKS_PER_BOX * NB;
    static constexpr int TPW = TASKS / CW;
    static constexpr int SMEM_BYTES = TPC * TILE_BYTES + 1024;   // + 1024-byte alignment slack
    static_assert(OBOXES * OBOX_BYTES == TILE_BYTES, "output staging aliases the tile");
    static_assert(TR % L::ROWS_PER_WARP == 0 && TASKS % CW == 0, "whole warp tasks");
    static_assert(TR <= 256 && TILE_COLS <= 256, "TMA box dimension <= 256");
};

#ifndef DESC_TMA_TILE_PF      // L2 prefetch of the CTA's boxes before griddepcontrol.wait
#define DESC_TMA_TILE_PF 1
#endif

// minimum resident CTAs per SM the register allocation must allow (A/B builds; 0 = none:
// ~62 registers, 8 CTAs/SM)
#ifndef DESC_TMA_TILE_MINB
#define DESC_TMA_TILE_MINB 0
#endif

template <int ES, int TR, int NB, int CW, int TPC>
__global__ void __launch_bounds__(TmaTileConfig<ES, TR, NB, CW, TPC>::THREADS, DESC_TMA_TILE_MINB)
transpose_tma_tile_kernel(const __grid_constant__ CUtensorMap map_in,
                          const __grid_constant__ CUtensorMap map_out, const TmaParams p) {
    using C = TmaTileConfig<ES, TR, NB, CW, TPC>;
    using L = StoreLane<ES>;
    constexpr int VEC = L::VEC;
    constexpr int TPW = C::TPW;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[TPC];
    const uint32_t base0 = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < TPC; ++i) ptx::mbar_init(ptx::smem_u32(&full_bar[i]), 1);
        ptx::fence_mbarrier_init();
    }
    const int64_t t0 = (int64_t)blockIdx.x * TPC;
#if DESC_TMA_TILE_PF
    // L2 prefetch of this CTA's boxes before griddepcontrol.wait (as in the TILED kernel:
    // L2 is the point of coherence, so this is safe while a previous grid still runs)
    if (threadIdx.x == 0) {
        ptx::prefetch_tensormap(&map_in);
        for (int i = 0; i < TPC; ++i) {
            if (t0 + i >= p.ntiles) break;
            const TileCoord tc = tile_coords(t0 + i, p);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const int32_t c0 = tc.tj * C::TILE_COLS + nb * C::TC;
                if (p.rank3) ptx::tma_prefetch_3d(&map_in, c0, tc.ti * TR, (int32_t)tc.bt);
                else ptx::tma_prefetch_2d(&map_in, c0, tc.ti * TR);
            }
        }
    }
#endif
    __syncthreads();
    // PDL: the prologue may overlap the previous kernel's tail; no global access before
    // every prerequisite grid has completed.
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();

    if (threadIdx.x == 0) {
        ptx::prefetch_tensormap(&map_in);
        ptx::prefetch_tensormap(&map_out);
        const uint64_t policy = p.evict_first ? ptx::policy_evict_first()
                                              : ptx::policy_evict_normal();
#pragma unroll
        for (int i = 0; i < TPC; ++i) {
            if (t0 + i >= p.ntiles) break;
            const TileCoord tc = tile_coords(t0 + i, p);
            const uint32_t fb = ptx::smem_u32(&full_bar[i]);
            const uint32_t base = base0 + i * C::TILE_BYTES;
            ptx::mbar_arrive_expect_tx(fb, C::TILE_BYTES);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const int32_t c0 = tc.tj * C::TILE_COLS + nb * C::TC;
                if (p.rank3) ptx::tma_load_3d(base + nb * C::BOX_BYTES, &map_in, fb, c0, tc.ti * TR, (int32_t)tc.bt, policy);
                else ptx::tma_load_2d(base + nb * C::BOX_BYTES, &map_in, fb, c0, tc.ti * TR, policy);
            }
        }
    }
    const int b_lane = L::b(lane), a_lane = L::a(lane), flip = L::flip(lane);
    auto task_box = [&](int q) { return (warp + q * CW) / C::TASKS_PER_BOX; };
    auto task_rgrp = [&](int q) { return ((warp + q * CW) % C::TASKS_PER_BOX) / C::CHUNK_GROUPS; };
    auto task_chunk = [&](int q) {
        return (((warp + q * CW) % C::TASKS_PER_BOX) % C::CHUNK_GROUPS) * L::CHUNKS_PER_WARP + b_lane;
    };

#pragma unroll 1
    for (int i = 0; i < TPC; ++i) {
        const int64_t t = t0 + i;
        if (t >= p.ntiles) break;                       // block-uniform
        const TileCoord tc = tile_coords(t, p);
        const uint32_t base = base0 + i * C::TILE_BYTES;
        ptx::mbar_wait(ptx::smem_u32(&full_bar[i]), 0);                // the tile landed

        uint4 r[TPW][VEC];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int row0 = VEC * (task_rgrp(q) * L::A_PER_WARP + a_lane);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const int row = row0 + k;
                r[q][k] = ptx::lds128(base + task_box(q) * C::BOX_BYTES + row * 128 +
                                      ((task_chunk(q) ^ (row & 7)) << 4));
            }
        }
        __syncthreads();                    // the whole tile is in registers: reuse its buffer

#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int orow0 = VEC * (task_box(q) * 8 + task_chunk(q));      // output row in tile
            const uint32_t ob = base + task_rgrp(q) * C::OBOX_BYTES;         // output box
            const int c = a_lane;                                            // 16-byte chunk
            const int f = flip;
            if constexpr (ES == 4) {
                const uint4 o0 = rotated_row<4, 0>(r[q], f), o1 = rotated_row<4, 1>(r[q], f);
                const uint4 o2 = rotated_row<4, 2>(r[q], f), o3 = rotated_row<4, 3>(r[q], f);
                int row;
                row = orow0 + (0 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o0);
                row = orow0 + (1 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o1);
                row = orow0 + (2 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o2);
                row = orow0 + (3 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o3);
            } else {
                const uint4 o0 = rotated_row<8, 0>(r[q], f), o1 = rotated_row<8, 1>(r[q], f);
                int row;
                row = orow0 + (0 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o0);
                row = orow0 + (1 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o1);
            }
        }
        // ragged tail: TMA stores clip only at 16-byte granularity (rows_main); the lanes
        // whose micro-block straddles `rows` write the remaining output columns themselves
        if (p.rows_main != p.rows) {
#pragma unroll
            for (int q = 0; q < TPW; ++q) {
                const int64_t in_row0 = (int64_t)tc.ti * TR + VEC * (task_rgrp(q) * L::A_PER_WARP + a_lane);
                if (in_row0 == p.rows_main) {
                    const int64_t orow0 = (int64_t)tc.tj * C::TILE_COLS + VEC * (task_box(q) * 8 + task_chunk(q));
                    char *out = reinterpret_cast<char *>(p.out) + (tc.bt * p.stride_out + in_row0) * ES;
                    emit_rows<ES>(r[q], out, p.ld_out * ES, orow0, p.cols, p.rows - p.rows_main,
                                  std::make_integer_sequence<int, VEC>{});
                }
            }
        }
        ptx::fence_proxy_async_shared();    // generic smem writes -> visible to the TMA unit
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int o = 0; o < C::OBOXES; ++o) {
                const int32_t c0 = tc.ti * TR + o * (128 / ES);   // output column (input row)
                const int32_t c1 = tc.tj * C::TILE_COLS;          // output row (input column)
                if (p.rank3) ptx::tma_store_3d(&map_out, base + o * C::OBOX_BYTES, c0, c1, (int32_t)tc.bt);
                else ptx::tma_store_2d(&map_out, base + o * C::OBOX_BYTES, c0, c1);
            }
            ptx::bulk_commit_group();
        }
    }
    if (threadIdx.x == 0) ptx::bulk_wait_group_read<0>();   // smem outlives the stores' reads
}

}  // namespace desc
