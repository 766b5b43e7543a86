// tma_transpose.cuh -- persistent, warp-specialised TMA transpose for sm_100a.
//
// Paper mapping (Listing 2):
//   a2 tiling / CTA schedule  : `group_by_tile` + `sched(Y,X) block in grid` become a
//                               persistent tile loop (tile t = blockIdx.x + k*gridDim.x)
//   a3 tile-grid transpose    : the CTA that reads input tile (I,J) writes output tile (J,I)
//   a4 load global->shared    : ONE TMA box load (cp.async.bulk.tensor) per 128-byte column
//                               slice of the tile, 128-byte swizzle, into an S-stage ring
//   a5 barrier ("sync"): mbarrier complete_tx (full) / consumer arrive (empty) --
//                               the "synchronization releases borrows" rule
//   a6 intra-tile transpose   : each lane reads VEC rows x 16 bytes with conflict-free
//                               ld.shared.v4, transposes VEC x VEC in registers (renaming /
//                               PRMT), and writes VEC coalesced 16-byte output rows
//   a7 edges                  : TMA zero-fills out-of-range loads; stores are predicated
//   a8 batch                  : third tensor-map dimension
//
// Shared-memory layout of one box: [TR rows][128 bytes], 16-byte chunk c of row r stored
// at chunk c ^ (r & 7) (CU_TENSOR_MAP_SWIZZLE_128B; box base 1024-byte aligned).
//
// Lane -> micro-block map (conflict-free for every element size):
//   VEC = 16/ES elements per chunk.  A lane owns the VEC x VEC micro-block at rows
//   VEC*a .. VEC*a+VEC-1, chunk b.  lane bits [0, BB) -> low bits of b, [BB, 3) -> low bits
//   of a, [3, 5) -> high bits of a, with BB = min(log2 VEC, 3).  In every 8-lane phase of a
//   ld.shared.v4 the physical chunks b ^ ((VEC*a+k) & 7) are all distinct.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda.h>

#include "ptx.cuh"

namespace desc {

struct TmaParams {
    void *out;
    int64_t ld_out;      // elements
    int64_t stride_out;  // elements
    int32_t rows, cols, batch;
    int32_t rows_main;   // rows rounded down to 16 bytes (TMA-store map extent)
    int32_t tiles_r, tiles_c;
    int32_t rank3;       // 1 => 3-D tensor map (batch > 1)
    int32_t group;       // tile rows per raster group (>= 1), see tile_coords
    int32_t evict_first; // 1 => L2 evict_first hint on the TMA loads
    int32_t rev_rows;    // 1 => logical input row i is physical row rows-1-i (TMA-store kernel)
    int64_t ntiles;
    unsigned long long *sched;  // dynamic tile counter {next, done} (nullptr: static)
};

// End of a dynamically scheduled launch, called by each CTA's producer thread after it
// fetched its terminal tile id (it never touches the counter again): the last CTA to check
// in resets {next, done} for the next launch on the stream, which cannot read the counter
// before this grid has completed (griddepcontrol.wait / stream order).
__device__ __forceinline__ void sched_release(const TmaParams &p) {
    __threadfence();
    if (atomicAdd(p.sched + 1, 1ull) == gridDim.x - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
    }
}

// Linear tile id -> (matrix, tile row, tile col).  Tiles are rastered in groups of
// `group` tile rows walked column by column, so the tiles in flight at any moment
// (one per CTA) form a near-square window of the matrix: both the rows read and the
// rows written are touched in long contiguous runs (DRAM page locality on both sides
// of the transpose).
struct TileCoord {
    int64_t bt;
    int32_t ti, tj;
};
__device__ __forceinline__ TileCoord tile_coords(int64_t t, const TmaParams &p) {
    const int64_t per_mat = (int64_t)p.tiles_r * p.tiles_c;
    TileCoord c;
    c.bt = t / per_mat;
    const int64_t rem = t - c.bt * per_mat;
    const int64_t per_group = (int64_t)p.group * p.tiles_c;
    const int32_t g = (int32_t)(rem / per_group);
    const int32_t in_g = (int32_t)(rem - (int64_t)g * per_group);
    const int32_t g0 = g * p.group;
    const int32_t gsz = min(p.group, p.tiles_r - g0);
    c.tj = in_g / gsz;
    c.ti = g0 + (in_g - c.tj * gsz);
    return c;
}

template <int ES>
struct TmaTraits {
    static constexpr int VEC = 16 / ES;                       // elements per 16-byte chunk
    static constexpr int LOGVEC = (VEC == 16) ? 4 : (VEC == 8) ? 3 : (VEC == 4) ? 2 : 1;
    static constexpr int BB = LOGVEC < 3 ? LOGVEC : 3;         // lane bits selecting chunk
    static constexpr int CHUNKS_PER_WARP = 1 << BB;
    static constexpr int A_PER_WARP = 1 << (5 - BB);           // micro-row groups per warp
    static constexpr int ROWS_PER_WARP = A_PER_WARP * VEC;     // input rows a warp covers
    static constexpr int TC = 128 / ES;                        // columns of one swizzled box
};

// VEC x VEC register micro-transpose: r[k] = input row k (16 bytes), returns output row j.
template <int ES, int J>
__device__ __forceinline__ uint4 micro_row(const uint4 (&r)[16 / ES]) {
    uint4 o;
    if constexpr (ES == 4) {
        const uint32_t *c0 = &r[0].x, *c1 = &r[1].x, *c2 = &r[2].x, *c3 = &r[3].x;
        o.x = c0[J]; o.y = c1[J]; o.z = c2[J]; o.w = c3[J];
    } else if constexpr (ES == 8) {
        const uint32_t *c0 = &r[0].x, *c1 = &r[1].x;
        o.x = c0[2 * J]; o.y = c0[2 * J + 1]; o.z = c1[2 * J]; o.w = c1[2 * J + 1];
    } else if constexpr (ES == 2) {
        constexpr uint32_t sel = (J & 1) ? 0x7632u : 0x5410u;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t a = (&r[2 * q].x)[J / 2];
            const uint32_t b = (&r[2 * q + 1].x)[J / 2];
            w[q] = __byte_perm(a, b, sel);
        }
        o = make_uint4(w[0], w[1], w[2], w[3]);
    } else {  // ES == 1
        constexpr uint32_t byte = J & 3;
        constexpr uint32_t sel2 = byte | ((4 + byte) << 4);   // bytes {a.byte, b.byte} -> [0,1]
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t lo = __byte_perm((&r[4 * q + 0].x)[J / 4], (&r[4 * q + 1].x)[J / 4], sel2);
            const uint32_t hi = __byte_perm((&r[4 * q + 2].x)[J / 4], (&r[4 * q + 3].x)[J / 4], sel2);
            w[q] = __byte_perm(lo, hi, 0x5410u);
        }
        o = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return o;
}

// 32-bit word w of a uint4 (w is a compile-time constant after unrolling).
__device__ __forceinline__ uint32_t word(const uint4 &v, int w) {
    return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}

// Store the first n (< 16/ES) elements of v at dst (edge micro-block, R6/R8).
template <int ES>
__device__ __forceinline__ void store_partial(char *dst, const uint4 &v, int n) {
#pragma unroll
    for (int e = 0; e < 16 / ES; ++e) {
        if (e < n) {
            if constexpr (ES == 8) {
                const uint64_t d = ((uint64_t)word(v, 2 * e + 1) << 32) | word(v, 2 * e);
                *reinterpret_cast<uint64_t *>(dst + 8 * e) = d;
            } else if constexpr (ES == 4) {
                *reinterpret_cast<uint32_t *>(dst + 4 * e) = word(v, e);
            } else if constexpr (ES == 2) {
                *reinterpret_cast<uint16_t *>(dst + 2 * e) = (uint16_t)(word(v, e / 2) >> (16 * (e & 1)));
            } else {
                dst[e] = (char)(word(v, e / 4) >> (8 * (e & 3)));
            }
        }
    }
}

template <int J, int ES>
__device__ __forceinline__ void emit_row(const uint4 (&r)[16 / ES], char *out, int64_t ld_out_b,
                                         int64_t orow0, int cols, int nvalid) {
    constexpr int VEC = 16 / ES;
    const int64_t orow = orow0 + J;
    if (orow < cols) {
        const uint4 o = micro_row<ES, J>(r);
        char *p = out + orow * ld_out_b;
        if (nvalid >= VEC) ptx::stg128(p, o);
        else store_partial<ES>(p, o, nvalid);
    }
}

template <int ES, int... J>
__device__ __forceinline__ void emit_rows(const uint4 (&r)[16 / ES], char *out, int64_t ld_out_b,
                                          int64_t orow0, int cols, int nvalid,
                                          std::integer_sequence<int, J...>) {
    (emit_row<J, ES>(r, out, ld_out_b, orow0, cols, nvalid), ...);
}

// TR: input rows per tile; NB: 128-byte column boxes per tile; STAGES: ring depth;
// CW: consumer warps (each handles TASKS/CW warp-tasks of every tile).
template <int ES, int TR, int NB, int STAGES, int CW>
struct TmaConfig {
    using T = TmaTraits<ES>;
    static constexpr int BOX_BYTES = TR * 128;
    static constexpr int STAGE_BYTES = BOX_BYTES * NB;
    static constexpr int CHUNK_GROUPS = 8 / T::CHUNKS_PER_WARP;
    static constexpr int TASKS_PER_BOX = (TR / T::ROWS_PER_WARP) * CHUNK_GROUPS;
    static constexpr int TASKS = TASKS_PER_BOX * NB;
    static constexpr int CONSUMERS = CW;
    static constexpr int TPW = TASKS / CW;           // warp-tasks per consumer warp per tile
    static constexpr int THREADS = 32 * (1 + CONSUMERS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;  // +1024 for alignment
    static constexpr int TILE_COLS = NB * T::TC;
    static_assert(TR % T::ROWS_PER_WARP == 0, "TR must cover whole warp tasks");
    static_assert(TASKS % CW == 0, "tasks must split evenly over consumer warps");
    static_assert(TR <= 256, "TMA box dimension <= 256");
    static_assert(THREADS <= 1024, "block too large");
};

template <int ES, int TR, int NB, int STAGES, int CW>
__global__ void __launch_bounds__(TmaConfig<ES, TR, NB, STAGES, CW>::THREADS)
transpose_tma_kernel(const __grid_constant__ CUtensorMap map, const TmaParams p) {
    using C = TmaConfig<ES, TR, NB, STAGES, CW>;
    using T = TmaTraits<ES>;
    constexpr int VEC = T::VEC;
    constexpr int TPW = C::TPW;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ __align__(8) uint64_t empty_bar[STAGES];

    const uint32_t smem_base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(ptx::smem_u32(&full_bar[s]), 1);
            ptx::mbar_init(ptx::smem_u32(&empty_bar[s]), C::CONSUMERS);
        }
        ptx::fence_mbarrier_init();
    }
    __syncthreads();
    // PDL: the prologue above may overlap the previous kernel's tail; nothing below touches
    // global memory before every prerequisite grid has completed.
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();

    if (warp == 0) {
        // ------------------------------ producer: one elected lane issues TMA
        if (lane == 0) {
            ptx::prefetch_tensormap(&map);
            const uint64_t policy = p.evict_first ? ptx::policy_evict_first() : ptx::policy_evict_normal();
            int it = 0;
            for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
                ptx::mbar_wait(ptx::smem_u32(&empty_bar[s]), ph ^ 1u);   // slot released
                const TileCoord tc = tile_coords(t, p);
                const int64_t bt = tc.bt;
                const int32_t ti = tc.ti, tj = tc.tj;
                const uint32_t fb = ptx::smem_u32(&full_bar[s]);
                ptx::mbar_arrive_expect_tx(fb, C::STAGE_BYTES);
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const uint32_t dst = smem_base + s * C::STAGE_BYTES + nb * C::BOX_BYTES;
                    const int32_t c0 = tj * C::TILE_COLS + nb * T::TC;
                    if (p.rank3) ptx::tma_load_3d(dst, &map, fb, c0, ti * TR, (int32_t)bt, policy);
                    else ptx::tma_load_2d(dst, &map, fb, c0, ti * TR, policy);
                }
            }
        }
        return;
    }

    // ------------------------------------ consumers: smem -> registers -> global
    const int cw = warp - 1;
    // lane -> (a, b) inside one warp-task (see the header comment)
    const int b_lane = lane & ((1 << T::BB) - 1);
    const int a_lane = (lane >> 3) * (1 << (3 - T::BB)) + ((lane >> T::BB) & ((1 << (3 - T::BB)) - 1));
    // warp-task q of this warp: box, first input row of the lane's micro-block, chunk
    auto task_box = [&](int q) { return (cw + q * CW) / C::TASKS_PER_BOX; };
    auto task_row = [&](int q) {
        const int tib = (cw + q * CW) % C::TASKS_PER_BOX;
        return VEC * ((tib / C::CHUNK_GROUPS) * T::A_PER_WARP + a_lane);
    };
    auto task_chunk = [&](int q) {
        const int tib = (cw + q * CW) % C::TASKS_PER_BOX;
        return (tib % C::CHUNK_GROUPS) * T::CHUNKS_PER_WARP + b_lane;
    };
    const int64_t ld_out_b = p.ld_out * ES;

    int it = 0;
    for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
        const TileCoord tc = tile_coords(t, p);
        const int64_t bt = tc.bt;
        const int32_t ti = tc.ti, tj = tc.tj;

        ptx::mbar_wait(ptx::smem_u32(&full_bar[s]), ph);           // TMA bytes landed

        const uint32_t sbase = smem_base + s * C::STAGE_BYTES;
        uint4 r[TPW][VEC];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const int row = task_row(q) + k;
                r[q][k] = ptx::lds128(sbase + task_box(q) * C::BOX_BYTES + row * 128 +
                                      ((task_chunk(q) ^ (row & 7)) << 4));
            }
        }
        // release the slot: proxy fence (generic reads before the next TMA write), arrive
        ptx::release_slot_after_lds(ptx::smem_u32(&empty_bar[s]), lane);

#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int64_t in_row0 = (int64_t)ti * TR + task_row(q);     // = output column
            const int64_t left = (int64_t)p.rows - in_row0;
            const int nvalid = (int)(left < VEC ? left : VEC);
            if (nvalid > 0) {
                const int64_t orow0 = (int64_t)tj * C::TILE_COLS + task_box(q) * T::TC +
                                      VEC * task_chunk(q);
                char *out = reinterpret_cast<char *>(p.out) + (bt * p.stride_out + in_row0) * ES;
                emit_rows<ES>(r[q], out, ld_out_b, orow0, p.cols, nvalid,
                              std::make_integer_sequence<int, VEC>{});
            }
        }
    }
}

}  // namespace desc
