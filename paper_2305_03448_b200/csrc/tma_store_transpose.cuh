// tma_store_transpose.cuh -- TMA in, TMA out: persistent warp-specialised transpose for
// sm_100a with both directions of the copy on the Tensor Memory Accelerator.
//
// Same paper mapping as tma_transpose.cuh (Listing 2; steps a2-a8 of SURVEY §8a),
// but step a6 ("copy-out") stages the transposed tile in shared memory and writes it with
// cp.async.bulk.tensor stores instead of per-lane st.global:
//
//   producer warp : TMA box loads (128-byte swizzle) into an S-stage ring, mbarrier complete_tx
//   consumer warps: wait full[s] -> ld.shared.v4 (conflict-free) -> release empty[s]
//                   -> VEC x VEC register transpose -> st.shared.v4 into a 128-byte-swizzled
//                   output staging tile (conflict-free via a per-lane row rotation)
//                   -> fence.proxy.async -> named barrier -> one thread issues TMA stores
//   output staging: OBUF buffers; before the barrier of tile it the issuing thread waits
//                   (cp.async.bulk.wait_group.read OBUF-2) until the store that last used
//                   buffer (it+1)%OBUF has finished reading it (WAR through the async proxy).
//   edges         : loads zero-fill out of range, stores are clipped by the tensor map, so
//                   padding and guard bytes are never written (R6, R8).
//
// Lane maps (ES = element size, VEC = 16/ES; a = micro-row group, b = 16-byte chunk):
//   ES=4: b = lane[1:0], a = lane[4:2];               store row j = jj ^ (lane & 2)
//   ES=8: b = lane[1:0], a = {lane[4], lane[2], lane[3]}; store row j = jj ^ (lane & 1)
// For every 8-lane phase both the loads (chunk b ^ ((VEC*a+k) & 7)) and the stores
// (chunk a ^ ((VEC*b+j) & 7)) hit 8 distinct 16-byte bank groups.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "mutants.cuh"
#include "ptx.cuh"
#include "tma_transpose.cuh"

namespace desc {

template <int ES>
struct StoreLane;

template <>
struct StoreLane<4> {
    static constexpr int VEC = 4;
    static constexpr int A_PER_WARP = 8;
    static constexpr int CHUNKS_PER_WARP = 4;
    static constexpr int ROWS_PER_WARP = 32;
    __device__ static int b(int lane) { return lane & 3; }
    __device__ static int a(int lane) { return lane >> 2; }
    __device__ static int flip(int lane) { return lane & 2; }   // XOR applied to j
};

template <>
struct StoreLane<8> {
    static constexpr int VEC = 2;
    static constexpr int A_PER_WARP = 8;
    static constexpr int CHUNKS_PER_WARP = 4;
    static constexpr int ROWS_PER_WARP = 16;
    __device__ static int b(int lane) { return lane & 3; }
    __device__ static int a(int lane) {
        return ((lane >> 3) & 1) | (((lane >> 2) & 1) << 1) | (((lane >> 4) & 1) << 2);
    }
    __device__ static int flip(int lane) { return lane & 1; }
};

template <int ES, int TR, int NB, int STAGES, int CW, int OBUF>
struct Tma2Config {
    using L = StoreLane<ES>;
    static constexpr int TC = 128 / ES;                      // columns per input box
    static constexpr int BOX_BYTES = TR * 128;
    static constexpr int STAGE_BYTES = BOX_BYTES * NB;
    static constexpr int TILE_COLS = NB * TC;                // = output rows per tile
    static constexpr int OBOXES = TR * ES / 128;             // output boxes per tile
    static constexpr int OBOX_BYTES = TILE_COLS * 128;
    static constexpr int OUT_BYTES = OBOXES * OBOX_BYTES;    // == STAGE_BYTES
    static constexpr int CHUNK_GROUPS = 8 / L::CHUNKS_PER_WARP;
    static constexpr int TASKS_PER_BOX = (TR / L::ROWS_PER_WARP) * CHUNK_GROUPS;
    static constexpr int TASKS = TASKS_PER_BOX * NB;
    static constexpr int TPW = TASKS / CW;
    static constexpr int THREADS = 32 * (1 + CW);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OBUF * OUT_BYTES + 1024;
    static_assert(TR % L::ROWS_PER_WARP == 0, "TR must cover whole warp tasks");
    static_assert(TASKS % CW == 0, "tasks must split evenly over consumer warps");
    static_assert(TR <= 256 && TILE_COLS <= 256, "TMA box dimension <= 256");
    static_assert(OBUF >= 2, "need at least double-buffered output staging");
    static_assert(THREADS <= 1024, "block too large");
};

// Output row JJ of the lane's micro-block, rotated by `flip` (compile-time JJ, runtime flip).
template <int ES, int JJ>
__device__ __forceinline__ uint4 rotated_row(const uint4 (&r)[16 / ES], int flip) {
    if constexpr (ES == 4) {
        const uint4 x = micro_row<4, JJ>(r), y = micro_row<4, JJ ^ 2>(r);
        return flip ? y : x;
    } else {
        const uint4 x = micro_row<8, JJ>(r), y = micro_row<8, JJ ^ 1>(r);
        return flip ? y : x;
    }
}

template <int ES, int TR, int NB, int STAGES, int CW, int OBUF>
__global__ void __launch_bounds__(Tma2Config<ES, TR, NB, STAGES, CW, OBUF>::THREADS)
transpose_tma2_kernel(const __grid_constant__ CUtensorMap map_in,
                      const __grid_constant__ CUtensorMap map_out, const TmaParams p) {
    using C = Tma2Config<ES, TR, NB, STAGES, CW, OBUF>;
    using L = StoreLane<ES>;
    constexpr int VEC = L::VEC;
    constexpr int TPW = C::TPW;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ __align__(8) uint64_t empty_bar[STAGES];
    __shared__ __align__(8) int64_t tile_id[STAGES];

    const uint32_t in_base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t out_base = in_base + STAGES * C::STAGE_BYTES;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(ptx::smem_u32(&full_bar[s]), 1);
            ptx::mbar_init(ptx::smem_u32(&empty_bar[s]), CW);
        }
        ptx::fence_mbarrier_init();
    }
    __syncthreads();
    // PDL: the prologue above may overlap the previous kernel's tail; nothing below touches
    // global memory before every prerequisite grid has completed.
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();

    if (warp == 0) {
        // ------------------------------ producer: one elected lane issues TMA loads
        if (lane == 0) {
            ptx::prefetch_tensormap(&map_in);
            const uint64_t policy = p.evict_first ? ptx::policy_evict_first() : ptx::policy_evict_normal();
            // Tile ids: static round robin, or (p.sched != nullptr) fetched from a global
            // counter so that faster SMs take more tiles (dynamic scheduling).  The next id
            // is fetched one tile ahead to hide the atomic's latency.  The id reaches the
            // consumers through tile_id[s], written with st.async completing on full[s].
            auto fetch = [&](int it) -> int64_t {
                return p.sched ? (int64_t)atomicAdd(p.sched, 1ull)
                               : (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
            };
            int64_t t_next = fetch(0);
            for (int it = 0;; ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
                const int64_t t = t_next;
                if (t < p.ntiles) t_next = fetch(it + 1);
                ptx::mbar_wait(ptx::smem_u32(&empty_bar[s]), ph ^ 1u);
                // the tile id travels like the tile: an async store completing on full[s]
                const uint32_t fb = ptx::smem_u32(&full_bar[s]);
                const uint32_t ta = ptx::smem_u32(&tile_id[s]);
                if (t >= p.ntiles) {                   // no more work: tell the consumers
                    ptx::mbar_arrive_expect_tx(fb, 8);
                    ptx::st_async_b64(ta, (uint64_t)t, fb);
                    break;
                }
                const TileCoord tc = tile_coords(t, p);
                ptx::mbar_arrive_expect_tx(fb, C::STAGE_BYTES + 8);
                ptx::st_async_b64(ta, (uint64_t)t, fb);
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const uint32_t dst = in_base + s * C::STAGE_BYTES + nb * C::BOX_BYTES;
                    const int32_t c0 = tc.tj * C::TILE_COLS + nb * C::TC;
                    // rev_rows: logical rows [ti*TR, ti*TR+TR) are physical rows
                    // [rows - (ti+1)*TR, rows - ti*TR): a box that may start above row 0
                    // (zero-filled, never read back as data)
                    const int32_t r0 = p.rev_rows ? p.rows - (tc.ti + 1) * TR : tc.ti * TR;
                    if (p.rank3) ptx::tma_load_3d(dst, &map_in, fb, c0, r0, (int32_t)tc.bt, policy);
                    else ptx::tma_load_2d(dst, &map_in, fb, c0, r0, policy);
                }
            }
            if (p.sched) sched_release(p);             // this CTA fetched its last id
        }
        return;
    }

    // ------------------------------------ consumers
    const int cw = warp - 1;
    const bool issuer = (cw == 0 && lane == 0);
    if (issuer) ptx::prefetch_tensormap(&map_out);
    const int b_lane = L::b(lane), a_lane = L::a(lane), flip = L::flip(lane);
    auto task_box = [&](int q) { return (cw + q * CW) / C::TASKS_PER_BOX; };
    auto task_rgrp = [&](int q) { return ((cw + q * CW) % C::TASKS_PER_BOX) / C::CHUNK_GROUPS; };
    auto task_chunk = [&](int q) {
        return (((cw + q * CW) % C::TASKS_PER_BOX) % C::CHUNK_GROUPS) * L::CHUNKS_PER_WARP + b_lane;
    };

    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
        ptx::mbar_wait(ptx::smem_u32(&full_bar[s]), ph);           // TMA bytes landed
        const int64_t t = tile_id[s];
        if (t >= p.ntiles) break;

        const uint32_t sbase = in_base + s * C::STAGE_BYTES;
        uint4 r[TPW][VEC];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int row0 = VEC * (task_rgrp(q) * L::A_PER_WARP + a_lane);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                // logical row row0+k lives in physical box row TR-1-(row0+k) when reversed;
                // (TR-1-x) & 7 == 7 ^ (x & 7), so the phase stays conflict-free
                const int row = p.rev_rows ? TR - 1 - (row0 + k) : row0 + k;
                const int sw = DESC_MUTANT(MUT_TMA2_NO_SWIZZLE) ? 0 : (row & 7);
                r[q][k] = ptx::lds128(sbase + task_box(q) * C::BOX_BYTES + row * 128 +
                                      ((task_chunk(q) ^ sw) << 4));
            }
        }
        // release the slot: proxy fence (generic reads before the next TMA write), arrive
        ptx::release_slot_after_lds(ptx::smem_u32(&empty_bar[s]), lane);

        // transposed micro-blocks -> output staging (swizzled like the output tensor map)
        const uint32_t obase = out_base + (it % OBUF) * C::OUT_BYTES;
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int orow0 = VEC * (task_box(q) * 8 + task_chunk(q));    // output row in tile
            const uint32_t ob = obase + task_rgrp(q) * C::OBOX_BYTES;      // output box
            const int c = a_lane;                                          // 16-byte chunk in box
            if constexpr (ES == 4) {
                uint4 o0 = rotated_row<4, 0>(r[q], flip), o1 = rotated_row<4, 1>(r[q], flip);
                uint4 o2 = rotated_row<4, 2>(r[q], flip), o3 = rotated_row<4, 3>(r[q], flip);
                const int f = flip;
                if (DESC_MUTANT(MUT_TMA2_NO_MICRO)) {           // chunks stored untransposed
                    o0 = f ? r[q][2] : r[q][0]; o1 = f ? r[q][3] : r[q][1];
                    o2 = f ? r[q][0] : r[q][2]; o3 = f ? r[q][1] : r[q][3];
                }
                int row;
                row = orow0 + (0 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o0);
                row = orow0 + (1 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o1);
                row = orow0 + (2 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o2);
                row = orow0 + (3 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o3);
            } else {
                uint4 o0 = rotated_row<8, 0>(r[q], flip), o1 = rotated_row<8, 1>(r[q], flip);
                const int f = flip;
                if (DESC_MUTANT(MUT_TMA2_NO_MICRO)) { o0 = f ? r[q][1] : r[q][0]; o1 = f ? r[q][0] : r[q][1]; }
                int row;
                row = orow0 + (0 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o0);
                row = orow0 + (1 ^ f); ptx::sts128(ob + row * 128 + ((c ^ (row & 7)) << 4), o1);
            }
        }
        // Ragged tail (rows % VEC != 0): TMA stores clip only at 16-byte granularity, so the
        // output tensor map stops at rows_main = rows rounded down to VEC and the lanes whose
        // micro-block straddles `rows` write the remaining columns themselves (R6, R8).
        if (p.rows_main != p.rows && !DESC_MUTANT(MUT_TMA2_NO_TAIL)) {
            const TileCoord tc = tile_coords(t, p);
#pragma unroll
            for (int q = 0; q < TPW; ++q) {
                const int64_t in_row0 = (int64_t)tc.ti * TR + VEC * (task_rgrp(q) * L::A_PER_WARP + a_lane);
                if (in_row0 == p.rows_main) {
                    const int nvalid = p.rows - p.rows_main;
                    const int64_t orow0 = (int64_t)tc.tj * C::TILE_COLS + VEC * (task_box(q) * 8 + task_chunk(q));
                    char *out = reinterpret_cast<char *>(p.out) + (tc.bt * p.stride_out + in_row0) * ES;
                    emit_rows<ES>(r[q], out, p.ld_out * ES, orow0, p.cols, nvalid,
                                  std::make_integer_sequence<int, VEC>{});
                }
            }
        }
        if (!DESC_MUTANT(MUT_TMA2_NO_FENCE)) {
            ptx::fence_proxy_async_shared();             // generic writes -> async proxy
            if (issuer) ptx::bulk_wait_group_read<OBUF - 2>();   // buffer (it+1)%OBUF reusable
        }
        ptx::named_bar_sync(1, 32 * CW);
        if (issuer) {
            const TileCoord tc = tile_coords(t, p);
#pragma unroll
            for (int o = 0; o < C::OBOXES; ++o) {
                const int32_t c0 = tc.ti * TR + o * (128 / ES);    // output column
                const int32_t c1 = tc.tj * C::TILE_COLS;           // output row
                if (p.rank3) ptx::tma_store_3d(&map_out, obase + o * C::OBOX_BYTES, c0, c1, (int32_t)tc.bt);
                else ptx::tma_store_2d(&map_out, obase + o * C::OBOX_BYTES, c0, c1);
            }
            ptx::bulk_commit_group();
        }
    }
    if (issuer) ptx::bulk_wait_group<0>();              // all stores done before smem is freed
}

}  // namespace desc
