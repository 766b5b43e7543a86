// reduce_scan.cuh -- the paper's two other memory-bound evaluation kernels (PAPER.md P:1047:
// "block-wide parallel reduction ... scan"), B200-native:
//
//   block reduction   out[b] = sum(in[b*B .. min(n, (b+1)*B)))        (read-bound)
//   inclusive scan    out[i] = sum(in[0 .. i])                          (read + write)
//
// Integers are summed modulo 2^bits (unsigned wrap-around; bit-exact); f32 is accumulated in
// fp64 and rounded once on output; f64 in fp64.
//
// Reduction: the group that sums one output block is chosen by B and the block count (host
// dispatch in desc_transpose.cu): lane groups of a warp (tiny blocks, segmented shuffles), a
// warp per 1-8 blocks of whole 512-byte rows, a thread / warp / 256-thread CTA per block
// (16-byte read-only loads, 8 in flight per lane, scalar head/tail around the aligned body),
// or an 8- / 16-CTA cluster per block (DSMEM combine) when there are few long blocks.
//
// Scans (three algorithms, desc_scan_ex):
//  * LOOKBACK: one 256 x ITEMS tile per CTA, tiles claimed in order from an atomic counter
//    (so every predecessor is resident or done), registers + shuffles, then decoupled
//    look-back: publish the aggregate (A), sum predecessors' A back to the nearest
//    inclusive prefix (P), publish P, write the outputs.
//  * THREE_PASS: tile aggregates -> one-CTA aggregate scan -> tile scans (3 n bytes).
//  * STREAM: persistent CTAs stream 32-96 KB tiles through a shared-memory ring with TMA
//    loads, same look-back (2 n bytes); 4- and 8-byte types use lane-contiguous tiles whose
//    results leave through swizzled staging and TMA tensor stores (scan_stream_kernel, LC).
// Tile descriptors are single-copy-atomic 64-bit {value, status} words: no fences (below).
#pragma once
#include <cstdint>
#include <cstring>
#include <type_traits>

#include <cooperative_groups.h>

#include "mutants.cuh"
#include "ptx.cuh"

namespace desc {

// ---- element <-> accumulator -----------------------------------------------------------
template <typename In> struct AccOf;
template <> struct AccOf<uint8_t> { using T = uint32_t; };
template <> struct AccOf<uint32_t> { using T = uint32_t; };
template <> struct AccOf<uint64_t> { using T = uint64_t; };
template <> struct AccOf<float> { using T = double; };
template <> struct AccOf<double> { using T = double; };

template <typename Acc, typename In>
__device__ __forceinline__ Acc to_acc(In v) { return (Acc)v; }

__device__ __forceinline__ uint32_t word_of(const uint4 &v, int w) {
    return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}

// element j (compile-time after unrolling) of the 16/sizeof(In) elements packed in a uint4
template <typename In>
__device__ __forceinline__ In unpack(const uint4 &v, int j) {
    if constexpr (sizeof(In) == 8) {
        const uint32_t lo = word_of(v, 2 * j), hi = word_of(v, 2 * j + 1);
        if constexpr (std::is_same<In, double>::value) return __hiloint2double((int)hi, (int)lo);
        else return ((uint64_t)hi << 32) | lo;
    } else if constexpr (sizeof(In) == 4) {
        if constexpr (std::is_same<In, float>::value) return __uint_as_float(word_of(v, j));
        else return word_of(v, j);
    } else {
        return (In)((word_of(v, j >> 2) >> (8 * (j & 3))) & 0xFF);
    }
}

// sum of the elements packed in a uint4
template <typename In, typename Acc>
__device__ __forceinline__ Acc vec_sum(const uint4 &v) {
    Acc s = 0;
#pragma unroll
    for (int j = 0; j < (int)(16 / sizeof(In)); ++j) s += to_acc<Acc>(unpack<In>(v, j));
    return s;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

#ifndef DESC_REDUCE_L2PF       // warp-row kernel: L2 prefetch of the first work item before
#define DESC_REDUCE_L2PF 2      // griddepcontrol.wait (1), and of the next one inside the loop (2)
#endif
#ifndef DESC_PROBE_PF          // read probe: L2 prefetch one chunk ahead (A/B only: costs the
#define DESC_PROBE_PF 0         // tight probe loop 15%, profiles/r02_reduce_prefetch.txt)
#endif

// 16-byte loads in flight per lane in the reduction's body loop
#ifndef DESC_REDUCE_UNROLL
#define DESC_REDUCE_UNROLL 8
#endif

template <typename Acc>
__device__ __forceinline__ Acc warp_sum(Acc v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum of in[lo, hi) by `nl` cooperating lanes (this one is `lane`); 16-byte vectors over the
// aligned body when `vec` (base pointer 16-byte aligned), scalar head / tail.
template <typename In, typename Acc>
__device__ __forceinline__ Acc range_sum(const In *__restrict__ in, int64_t lo, int64_t hi,
                                         int lane, int nl, bool vec) {
    constexpr int V = 16 / sizeof(In);
    Acc acc = 0;
    int64_t a = hi, nv = 0;
    if (vec) {
        a = (lo + V - 1) / V * V;
        if (a > hi) a = hi;
        nv = (hi - a) / V;
    }
    for (int64_t i = lo + lane; i < a; i += nl) acc += to_acc<Acc>(in[i]);
    const uint4 *vp = reinterpret_cast<const uint4 *>(in + a);
    int64_t k = lane;
    for (; k + (DESC_REDUCE_UNROLL - 1) * nl < nv; k += DESC_REDUCE_UNROLL * nl) {
        uint4 v[DESC_REDUCE_UNROLL];
#pragma unroll
        for (int u = 0; u < DESC_REDUCE_UNROLL; ++u) v[u] = ld_nc_v4(vp + k + u * nl);
#pragma unroll
        for (int u = 0; u < DESC_REDUCE_UNROLL; ++u) acc += vec_sum<In, Acc>(v[u]);
    }
    if constexpr (DESC_REDUCE_UNROLL > 4) {   // short blocks: 4 loads in flight per lane
        for (; k + 3 * nl < nv; k += 4 * nl) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = ld_nc_v4(vp + k + u * nl);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += vec_sum<In, Acc>(v[u]);
        }
    }
    for (; k < nv; k += nl) acc += vec_sum<In, Acc>(ld_nc_v4(vp + k));
    if (DESC_MUTANT(MUT_REDUCE_NO_TAIL)) return acc;
    for (int64_t i = a + nv * V + lane; i < hi; i += nl) acc += to_acc<Acc>(in[i]);
    return acc;
}

// G = 1: one thread per output block;  G = 32: one warp per block.
template <typename In, typename Out, int G>
__global__ void __launch_bounds__(256)
block_reduce_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n, int64_t B,
                    int64_t nblocks, bool vec) {
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    using Acc = typename AccOf<In>::T;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t groups = (int64_t)gridDim.x * blockDim.x / G;
    const int lane = G == 1 ? 0 : (threadIdx.x & 31);
    for (int64_t b = gid / G; b < nblocks; b += groups) {
        const int64_t lo = b * B, hi = lo + B < n ? lo + B : n;
        Acc s = range_sum<In, Acc>(in, lo, hi, lane, G, vec);
        if constexpr (G == 32) s = warp_sum(s);
        if (lane == 0) out[b] = (Out)s;
    }
}

// Blocks of whole 512-byte warp rows (B * sizeof(In) = 512 P, P = 1 … 16, base 16-byte
// aligned): one warp per K = L / P consecutive blocks, all L loads of a lane in flight at
// once, then the K warp sums interleaved (independent shuffle chains).
template <typename In, typename Out, int P, int L = 8>
__global__ void __launch_bounds__(256)
block_reduce_rows_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t nblocks) {
    using Acc = typename AccOf<In>::T;
    constexpr int K = L / P;           // blocks per warp iteration, L loads in flight per lane
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *vp = reinterpret_cast<const uint4 *>(in);
    const int64_t full = nblocks / K * K;   // the rest go through the per-block loop below
#if DESC_REDUCE_L2PF
    {   // the warp's first K blocks into L2 before the dependency wait (as in the TILED
        // transpose: L2 is the point of coherence; one prefetch per 128-byte line)
        const int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * K;
        if (b0 < full && (lane & 7) == 0)
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int p = 0; p < P; ++p) ptx::prefetch_l2(vp + ((b0 + k) * P + p) * 32 + lane);
    }
#endif
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    for (int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * K; b0 < full;
         b0 += warps * K) {
#if DESC_REDUCE_L2PF >= 2
        if ((lane & 7) == 0 && b0 + warps * K < full)
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int p = 0; p < P; ++p)
                    ptx::prefetch_l2(vp + ((b0 + warps * K + k) * P + p) * 32 + lane);
#endif
        uint4 v[K][P];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int p = 0; p < P; ++p) v[k][p] = ld_nc_v4(vp + ((b0 + k) * P + p) * 32 + lane);
        Acc s[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            s[k] = 0;
#pragma unroll
            for (int p = 0; p < P; ++p) s[k] += vec_sum<In, Acc>(v[k][p]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int k = 0; k < K; ++k) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
        if (lane < K) {
            static_assert(K <= 32, "one lane writes each block");
            Acc t = s[0];
#pragma unroll
            for (int k = 1; k < K; ++k) if (lane == k) t = s[k];
            out[b0 + lane] = (Out)t;
        }
    }
    for (int64_t b = full + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; b < nblocks;
         b += warps) {
        Acc t = 0;
#pragma unroll
        for (int p = 0; p < P; ++p) t += vec_sum<In, Acc>(ld_nc_v4(vp + (b * P + p) * 32 + lane));
        t = warp_sum(t);
        if (lane == 0) out[b] = (Out)t;
    }
}

// Tiny blocks of VB = 1 … 16 16-byte vectors (B * sizeof(In) = 16 VB, no ragged block, base
// 16-byte aligned): a warp reads 8 contiguous 512-byte rows at once (coalesced, unlike one
// thread per block, whose lanes sit B elements apart), each lane sums its vector, and
// xor-shuffles inside aligned groups of VB lanes finish each block (8 independent chains).
template <typename In, typename Out, int VB>
__global__ void __launch_bounds__(256)
block_reduce_seg_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t nblocks) {
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    using Acc = typename AccOf<In>::T;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint4 *vp = reinterpret_cast<const uint4 *>(in);
    const int64_t nv = nblocks * VB, full = nv / 256 * 256;
    for (int64_t c = w * 256; c < full; c += warps * 256) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_nc_v4(vp + c + u * 32 + lane);
        Acc s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = vec_sum<In, Acc>(v[u]);
#pragma unroll
        for (int o = VB / 2; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
        if ((lane & (VB - 1)) == 0) {
#pragma unroll
            for (int u = 0; u < 8; ++u) out[(c + u * 32 + lane) / VB] = (Out)s[u];
        }
    }
    // the last < 256 vectors, one 512-byte row per warp (VB divides 32: a block is wholly
    // inside or wholly outside the array)
    for (int64_t c = full + w * 32; c < nv; c += warps * 32) {
        const bool live = c + lane < nv;
        Acc s = live ? vec_sum<In, Acc>(ld_nc_v4(vp + c + lane)) : Acc(0);
#pragma unroll
        for (int o = VB / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (live && (lane & (VB - 1)) == 0) out[(c + lane) / VB] = (Out)s;
    }
}

// one 256-thread CTA per output block (large B)
template <typename In, typename Out>
__global__ void __launch_bounds__(256)
block_reduce_cta_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n, int64_t B,
                        int64_t nblocks, bool vec) {
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    using Acc = typename AccOf<In>::T;
    __shared__ Acc part[8];
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int64_t lo = b * B, hi = lo + B < n ? lo + B : n;
        Acc s = warp_sum(range_sum<In, Acc>(in, lo, hi, threadIdx.x, blockDim.x, vec));
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            Acc t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : Acc(0);
            t = warp_sum(t);
            if (threadIdx.x == 0) out[b] = (Out)t;
        }
        __syncthreads();
    }
}

// Few, long output blocks (fewer than one 256-thread CTA per SM slot): a cluster of CL CTAs
// per output block, each summing a contiguous 1/CL slice; rank 0 adds the CL CTA sums in
// rank order through distributed shared memory (deterministic, no workspace, no atomics).
template <typename In, typename Out, int CL>
__global__ void __launch_bounds__(1024)
block_reduce_cluster_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n,
                            int64_t B, int64_t nblocks, bool vec) {
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    using Acc = typename AccOf<In>::T;
    constexpr int64_t V = 16 / sizeof(In);
    __shared__ Acc part[32];
    __shared__ Acc cta_sum;
    const int r = (int)cl.block_rank();
    const int64_t nclusters = gridDim.x / CL;
    for (int64_t b = blockIdx.x / CL; b < nblocks; b += nclusters) {
        const int64_t lo = b * B, hi = lo + B < n ? lo + B : n;
        const int64_t chunk = ((hi - lo + CL - 1) / CL + V - 1) / V * V;   // slices of whole vectors
        int64_t slo = lo + r * chunk, shi = slo + chunk;
        if (slo > hi) slo = hi;
        if (shi > hi) shi = hi;
        Acc s = warp_sum(range_sum<In, Acc>(in, slo, shi, threadIdx.x, blockDim.x, vec));
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            Acc t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : Acc(0);
            t = warp_sum(t);
            if (threadIdx.x == 0) cta_sum = t;
        }
        cl.sync();                     // every CTA sum visible cluster-wide
        if (r == 0 && threadIdx.x == 0) {
            Acc t = 0;
#pragma unroll
            for (int q = 0; q < CL; ++q) t += *cl.map_shared_rank(&cta_sum, q);
            out[b] = (Out)t;
        }
        cl.sync();                     // rank 0 has read every cta_sum before the next block
    }
}

// ---- read-only HBM probe (measurement helper: the reduction's read roofline) --------------
// A plain read-only stream: each warp reads 4 KB contiguous chunks (8 x 512-byte rows, one
// 16-byte load per lane per row, all 8 in flight) grid-striding over the buffer, 16 CTAs of
// 256 threads per SM.  XOR-folded; one 16-byte word per CTA is written so the loads cannot
// be elided.  (The reduction itself, with its L2 prefetch of the next chunk, reads faster:
// the probe context, not the ceiling; bench.py reports both against the nominal HBM3e rate.)
__global__ void __launch_bounds__(256) read_probe_kernel(const uint4 *__restrict__ in, int64_t nv,
                                                         uint4 *__restrict__ sink) {
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();
    uint4 acc = make_uint4(0, 0, 0, 0);
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nchunks = nv / 256;                      // 256 vectors = 4 KB per chunk
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; c < nchunks; c += warps) {
#if DESC_PROBE_PF
        if ((lane & 7) == 0 && c + warps < nchunks)
#pragma unroll
            for (int u = 0; u < 8; ++u) ptx::prefetch_l2(in + (c + warps) * 256 + u * 32 + lane);
#endif
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_nc_v4(in + c * 256 + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w;
        }
    }
    // ragged tail (< 4 KB): the first warp of the grid
    for (int64_t i = nchunks * 256 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = ld_nc_v4(in + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x ^= __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z ^= __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w ^= __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    __shared__ uint4 part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint4 t = part[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) { t.x ^= part[w].x; t.y ^= part[w].y; t.z ^= part[w].z; t.w ^= part[w].w; }
        sink[blockIdx.x] = t;
    }
}

// ---- scan ---------------------------------------------------------------------------------
// Tile descriptors of the single-pass scans are 64-bit words {value bits : 32, status : 32}
// (status 0 = not ready, 1 = aggregate A, 2 = inclusive prefix P), written and read with
// relaxed gpu-scope 8-byte accesses, which are single-copy atomic: a reader that sees a
// status also sees its value, so no fence sits on the look-back's critical path (a gpu-scope
// fence waits for the thread's outstanding stores, microseconds under a full HBM stream).
// 64-bit values are split over two adjacent words (lo, hi) that carry the same status and
// move as one 16-byte access; a reader that sees two different statuses (a torn A -> P
// update) treats the tile as not ready and polls again.
template <typename Acc>
struct ScanState {
    uint32_t *counter;   // tile claim counter (64-bit for the streaming scan)
    uint64_t *dlo;       // single pass: descriptor words; 32-bit values: {value, status} at
                         // [t]; 64-bit values: {value[31:0], status}, {value[63:32], status}
                         // at [2t], [2t+1] (one 16-byte access each way)
    uint64_t *dhi;       // unused (kept for the workspace layout)
    Acc *agg;            // three-launch: per-tile aggregate
    Acc *incl;           // three-launch: per-tile exclusive prefix
};

__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// 16-byte relaxed accesses: each 8-byte half is single-copy atomic (all the protocol needs:
// a torn pair shows two different statuses and is read again)
__device__ __forceinline__ void st_relaxed_v2u64(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void ld_relaxed_v2u64(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

template <typename Acc>
__device__ __forceinline__ uint64_t acc_bits(Acc v) {
    if constexpr (sizeof(Acc) == 8) {
        uint64_t b;
        memcpy(&b, &v, 8);
        return b;
    } else {
        uint32_t b;
        memcpy(&b, &v, 4);
        return b;
    }
}

template <typename Acc>
__device__ __forceinline__ Acc acc_from_bits(uint64_t b) {
    Acc v;
    if constexpr (sizeof(Acc) == 8) {
        memcpy(&v, &b, 8);
    } else {
        const uint32_t w = (uint32_t)b;
        memcpy(&v, &w, 4);
    }
    return v;
}

template <typename Acc>
__device__ __forceinline__ void publish(const ScanState<Acc> &st, int64_t t, Acc v,
                                        uint32_t status) {
    const uint64_t b = acc_bits(v);
    if constexpr (sizeof(Acc) == 8)
        st_relaxed_v2u64(&st.dlo[2 * t], (b << 32) | status, (b & 0xFFFFFFFF00000000ull) | status);
    else
        st_relaxed_u64(&st.dlo[t], (b << 32) | status);
}

// status of tile t (0 while not ready or torn between A and P) and its value
template <typename Acc>
__device__ __forceinline__ uint32_t read_desc(const ScanState<Acc> &st, int64_t t, Acc &v) {
    if constexpr (sizeof(Acc) == 8) {
        uint64_t lo, hi;
        ld_relaxed_v2u64(&st.dlo[2 * t], lo, hi);
        if ((uint32_t)lo != (uint32_t)hi) return 0u;
        v = acc_from_bits<Acc>((hi & 0xFFFFFFFF00000000ull) | (lo >> 32));
        return (uint32_t)lo;
    } else {
        const uint64_t lo = ld_relaxed_u64(&st.dlo[t]);
        v = acc_from_bits<Acc>(lo >> 32);
        return (uint32_t)lo;
    }
}

template <typename Acc>
__device__ __forceinline__ Acc warp_incl_scan(Acc v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Acc t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// N independent inclusive warp scans, level by level (N shuffle chains in flight at once)
template <typename Acc, int N>
__device__ __forceinline__ void warp_incl_scan_n(Acc (&v)[N], int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Acc t[N];
#pragma unroll
        for (int i = 0; i < N; ++i) t[i] = __shfl_up_sync(0xffffffffu, v[i], o);
#pragma unroll
        for (int i = 0; i < N; ++i)
            if (lane >= o) v[i] += t[i];
    }
}

// exclusive warp prefix from the inclusive one (a shuffle, not incl - own: no cancellation)
template <typename Acc>
__device__ __forceinline__ Acc warp_excl_from_incl(Acc incl, int lane) {
    const Acc e = __shfl_up_sync(0xffffffffu, incl, 1);
    return lane == 0 ? Acc(0) : e;
}

// Look-back by one warp: exclusive prefix of `tile` = nearest inclusive prefix (P) plus the
// aggregates (A) of the tiles after it.  Lane l reads descriptors j - 32 m - l (m < LB), so
// every poll is LB coalesced requests and a window covers 32 * LB predecessors; while a
// needed predecessor is not ready the warp sleeps briefly and polls again.
#ifndef DESC_SCAN_LB_WINDOW   // streaming scan: look-back window, x32 predecessors per poll
#define DESC_SCAN_LB_WINDOW 1
#endif
#ifndef DESC_SCAN_SLEEP_CAP   // longest back-off between look-back polls, ns
#define DESC_SCAN_SLEEP_CAP 256
#endif

template <typename Acc, int LB>
__device__ Acc look_back(const ScanState<Acc> &st, int64_t tile, int lane, int *polls = nullptr) {
    constexpr int W = 32 * LB;
    Acc prefix = 0;
    int64_t j = tile - 1;                                   // newest predecessor of the window
    uint32_t ns = 32;
    while (true) {
        if (polls) ++*polls;
        uint32_t f[LB];
        Acc v[LB];
#pragma unroll
        for (int m = 0; m < LB; ++m) {
            const int64_t t = j - (m * 32 + lane);
            v[m] = 0;
            f[m] = t >= 0 ? read_desc(st, t, v[m]) : 2u;
        }
        int dp = W;                                         // distance of the nearest P
#pragma unroll
        for (int m = LB - 1; m >= 0; --m)
            if (f[m] == 2u) dp = m * 32 + lane;
        dp = (int)__reduce_min_sync(0xffffffffu, (uint32_t)dp);
        bool missing = false;
#pragma unroll
        for (int m = 0; m < LB; ++m)
            if (m * 32 + lane <= dp && f[m] == 0u) missing = true;
        if (__any_sync(0xffffffffu, missing)) {
            __nanosleep(ns);
            if (ns < DESC_SCAN_SLEEP_CAP) ns <<= 1;
            continue;
        }
        Acc sum = 0;
#pragma unroll
        for (int m = 0; m < LB; ++m)
            if (m * 32 + lane <= dp) sum += v[m];
        prefix += warp_sum(sum);
        if (dp < W) return prefix;
        j -= W;
    }
}

// set element j (compile-time after unrolling) of a packed uint4
template <typename In>
__device__ __forceinline__ void set_elem(uint4 &v, int j, In e) {
    uint32_t *w = &v.x;   // registers after full unrolling
    if constexpr (sizeof(In) == 8) {
        uint64_t b;
        memcpy(&b, &e, 8);
        w[2 * j] = (uint32_t)b;
        w[2 * j + 1] = (uint32_t)(b >> 32);
    } else if constexpr (sizeof(In) == 4) {
        uint32_t b;
        memcpy(&b, &e, 4);
        w[j] = b;
    } else {
        const int sh = 8 * (j & 3);
        w[j >> 2] = (w[j >> 2] & ~(0xFFu << sh)) | ((uint32_t)(uint8_t)e << sh);
    }
}

// The tile's elements stay packed in 16-byte registers (ITEMS * sizeof(In) / 16 of them):
// half the registers of an accumulator-typed copy for f32 -> more resident tiles per SM,
// which is what hides the look-back latency.
// Zeroes the single-pass scans' state (tile counter + descriptors) in stream order; a kernel
// rather than cudaMemsetAsync so that it and the scan after it chain with PDL.
__global__ void __launch_bounds__(256) scan_reset_kernel(uint4 *__restrict__ p, int64_t n16) {
    ptx::grid_dependency_wait();
    ptx::grid_launch_dependents();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0, 0, 0, 0);
}

template <typename In, typename Out, int ITEMS>
__global__ void __launch_bounds__(256, 4)
scan_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n,
            ScanState<typename AccOf<In>::T> st, bool vec) {
    using Acc = typename AccOf<In>::T;
    constexpr int T = 256 * ITEMS;
    constexpr int V = 16 / sizeof(In);
    constexpr int NV = ITEMS / V;
    static_assert(sizeof(In) == sizeof(Out), "scan output has the input's type");
    ptx::grid_dependency_wait();       // PDL: the state reset (and anything before) is done
    ptx::grid_launch_dependents();
    __shared__ Acc warp_tot[8];
    __shared__ Acc tile_prefix;
    __shared__ uint32_t tile_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) tile_s = atomicAdd(st.counter, 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t base = tile * T + (int64_t)tid * ITEMS;
    const bool full = vec && base + ITEMS <= n;

    uint4 raw[NV];
    if (full) {
#pragma unroll
        for (int k = 0; k < NV; ++k) raw[k] = ld_nc_v4(in + base + k * V);
    } else {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            raw[k] = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (base + k * V + j < n) set_elem<In>(raw[k], j, in[base + k * V + j]);
        }
    }
    Acc tsum = 0;                                              // thread total
#pragma unroll
    for (int k = 0; k < NV; ++k) tsum += vec_sum<In, Acc>(raw[k]);

    const Acc wincl = warp_incl_scan(tsum, lane);
    if (lane == 31) warp_tot[warp] = wincl;
    __syncthreads();
    Acc wpre = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        if (w < warp) wpre += warp_tot[w];
        agg += warp_tot[w];
    }
    const Acc texcl = wpre + warp_excl_from_incl(wincl, lane);  // exclusive prefix in the tile

    if (warp == 0) {
        Acc prefix = 0;
        if (tile == 0) {
            if (lane == 0) publish(st, 0, agg, 2u);
        } else {
            if (lane == 0) publish(st, tile, agg, 1u);
            if (!DESC_MUTANT(MUT_SCAN_NO_LOOKBACK))
                prefix = look_back<Acc, 4>(st, tile, lane);  // 4: no spills at 64 registers
            if (lane == 0) publish(st, tile, prefix + agg, 2u);
        }
        if (lane == 0) tile_prefix = prefix;
    }
    __syncthreads();
    Acc run = tile_prefix + texcl;                             // running inclusive prefix
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        uint4 o = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            run += to_acc<Acc>(unpack<In>(raw[k], j));
            set_elem<Out>(o, j, (Out)run);
        }
        if (full) {
            *reinterpret_cast<uint4 *>(out + base + k * V) = o;
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (base + k * V + j < n) out[base + k * V + j] = unpack<Out>(o, j);
        }
    }
}

// ---- reduce-then-scan (three launches; the default for long arrays) -----------------------
// Measured: the single-pass look-back spends ~20 us per tile waiting on predecessors when
// ~600 tiles are in flight (profiles/r01_scan_*), so long scans take the paper's multi-kernel
// route: tile aggregates (block_reduce_kernel with the scan's tile, fp64/u64
// accumulators) -> one CTA scans the aggregates (exclusive) -> every tile scans its elements
// from its exclusive prefix.  3 n bytes of traffic instead of 2 n, but no inter-CTA waiting,
// and deterministic float results.
template <typename Acc>
__global__ void __launch_bounds__(1024)
scan_aggregates_kernel(const Acc *__restrict__ agg, Acc *__restrict__ excl, int64_t ntiles) {
    // one CTA; chunks of 1024 threads x 16 consecutive aggregates (8192 f32 tiles = 1 chunk)
    constexpr int IT = 16;
    __shared__ Acc wt[32];
    __shared__ Acc carry_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry_s = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < ntiles; c0 += 1024 * IT) {
        const int64_t i0 = c0 + (int64_t)tid * IT;
        Acc v[IT];
        Acc tsum = 0;
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            v[k] = i0 + k < ntiles ? agg[i0 + k] : Acc(0);
            tsum += v[k];
        }
        const Acc wi = warp_incl_scan(tsum, lane);
        if (lane == 31) wt[warp] = wi;
        __syncthreads();
        if (warp == 0) wt[lane] = warp_incl_scan(wt[lane], lane);   // inclusive over warps
        __syncthreads();
        // exclusive prefix by a shuffle of the inclusive one, never wi - tsum (an inf or NaN
        // aggregate would poison the tiles before it: inf - inf, NaN - NaN)
        Acc run = carry_s + (warp ? wt[warp - 1] : Acc(0)) + warp_excl_from_incl(wi, lane);
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            if (i0 + k < ntiles) excl[i0 + k] = run;
            run += v[k];
        }
        __syncthreads();
        if (tid == 0) carry_s += wt[31];
        __syncthreads();
    }
}

// final pass: tile = blockIdx.x (256 threads x ITEMS elements), its exclusive prefix from
// scan_aggregates_kernel.  Warp w owns the contiguous segment [w*32*ITEMS, (w+1)*32*ITEMS) of
// the tile and walks it in ITEMS/V rounds of one 16-byte vector per lane, so every load and
// store instruction of a warp covers 512 contiguous bytes (coalesced); a round's warp scan
// carries into the next; one barrier combines the 8 warp totals.
template <typename In, int ITEMS>
__global__ void __launch_bounds__(256, 3)
scan_tiles_kernel(const In *__restrict__ in, In *__restrict__ out, int64_t n,
                  const typename AccOf<In>::T *__restrict__ excl, bool vec) {
    using Acc = typename AccOf<In>::T;
    constexpr int V = 16 / sizeof(In);
    constexpr int R = ITEMS / V;                   // rounds per warp
    constexpr int SEG = 32 * ITEMS;                // elements per warp
    constexpr int T = 8 * SEG;                     // elements per tile
    __shared__ Acc warp_tot[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    const int64_t wbase = tile * T + (int64_t)warp * SEG;
    uint4 raw[R];
    Acc carry = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e0 = wbase + (int64_t)k * 32 * V + (int64_t)lane * V;
        if (vec && e0 + V <= n) {
            raw[k] = ld_nc_v4(in + e0);
        } else {
            raw[k] = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (e0 + j < n) set_elem<In>(raw[k], j, in[e0 + j]);
        }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) carry += warp_sum(vec_sum<In, Acc>(raw[k]));
    if (lane == 0) warp_tot[warp] = carry;
    __syncthreads();
    Acc wpre = DESC_MUTANT(MUT_SCAN_NO_LOOKBACK) ? Acc(0) : excl[tile];
#pragma unroll
    for (int w = 0; w < 8; ++w)
        if (w < warp) wpre += warp_tot[w];
    Acc rcarry = wpre;                             // prefix before the current round
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e0 = wbase + (int64_t)k * 32 * V + (int64_t)lane * V;
        const Acc ls = vec_sum<In, Acc>(raw[k]);     // recomputed: saves R accumulators
        const Acc wi = warp_incl_scan(ls, lane);
        Acc run = rcarry + warp_excl_from_incl(wi, lane);
        rcarry += __shfl_sync(0xffffffffu, wi, 31);
        uint4 o = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            run += to_acc<Acc>(unpack<In>(raw[k], j));
            set_elem<In>(o, j, (In)run);
        }
        if (vec && e0 + V <= n) {
            *reinterpret_cast<uint4 *>(out + e0) = o;
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (e0 + j < n) out[e0 + j] = unpack<In>(o, j);
        }
    }
}

// ---- streaming single-pass scan (the default for long, 16-byte aligned arrays) ------------
// Persistent, warp-specialised, one CTA per SM.  Tiles of NR * 32 * VPT 16-byte vectors are
// claimed in order from an atomic counter and read from HBM exactly once, through an S-stage
// shared-memory ring of 1-D TMA bulk copies.  Two warp groups handle every tile:
//
//   reduce warps (NR) : stage -> registers -> warp totals (st.async onto wsum[q]); the
//                       registers are parked in tensor memory (TMEM, 256 KB per SM, idle in
//                       this kernel otherwise) and the stage is released at once
//   scan warps (NR)   : wait the tile's exclusive prefix, TMEM -> registers -> scan ->
//                       16-byte coalesced stores (2 n bytes of HBM traffic in all)
//   producer warp     : claim tile, st.async its tag + bulk-copy its bytes onto full[s]
//   aggregator warp   : wait wsum[q], aggregate, publish A (P for tile 0), forward on aggb[q]
//   look-back warps   : wait aggb[q], look back, publish P, st.async the prefix onto pfx[q]
//
// The reduce warps only wait for bytes (and a free TMEM slot), so every aggregate is
// published as soon as its tile lands and up to QT tiles can wait for their look-backs at
// once: the critical path is the HBM stream, not the inter-CTA signalling latency, which
// under a saturated memory system is several microseconds.  Measured on the way here: a
// look-back on the critical path held single-pass scans to 0.3-0.5 of peak; re-reading the
// waiting tiles from L2 instead of TMEM cost ~15%; one warp group doing both phases coupled
// each aggregate to an older tile's look-back.
//
// Reduce warp r and scan warp NR + r own the same 32 * VPT vectors of a tile (512 contiguous
// bytes per warp instruction) and the same TMEM lane quarter (r % 4) and column block.
// Values that cross warps travel by st.async on the mbarrier their reader waits on (what
// racecheck tracks), hence the 2-CTA cluster launch; TMEM hand-offs use parked[qt] / freed[qt]
// with the tcgen05 thread-sync fences.  Metadata slots q = k mod Q, Q = QT + S + 2: reduce
// warps run at most QT tiles ahead of the scan warps (TMEM slots) and S ring items ahead of
// each other, so a slot is never rewritten while it is read.  Progress: tiles are claimed in
// order by running CTAs and aggregates depend on nothing but their own bytes.
// LC = 1: lane-contiguous tile layout (lane owns VPT = 8 consecutive vectors, one 128-byte
// row), the lane's exclusive prefix inside its warp parked in TMEM by the reduce warp (2
// columns), the scan warps' results staged in a 128-byte-swizzled 4 KB buffer per warp and
// written by one TMA tensor store (32 rows x 128 bytes) -- no shuffles in the scan warps and
// fully coalesced stores.
template <int NR, int VPT, int S, int QT, int NLB, int LC = 0>
struct ScanStreamCfg {
    static constexpr int THREADS = 32 * (2 * NR + 2 + NLB);
    static constexpr int TB = NR * 32 * VPT * 16;      // tile bytes
    static constexpr int ROWS = TB / 128;              // 128-byte rows per tile (TMA view)
    static constexpr int NBOX = (ROWS + 255) / 256;    // boxes of <= 256 rows per tile
    static constexpr int BOX_ROWS = ROWS / NBOX;
    static constexpr int WSEG = 32 * VPT * 16;         // bytes of one warp's segment
    static constexpr int SMEM = S * TB + 1024 + (LC ? NR * WSEG : 0);   // + LC staging
    static_assert(!LC || VPT == 8, "lane-contiguous layout: one 128-byte row per lane");
    static_assert(ROWS % NBOX == 0, "tile rows must split into equal TMA boxes");
    static constexpr int Q = QT + S + 2;               // tile metadata slots
    static constexpr int WCOLS = 4 * VPT + (LC ? 2 : 0);   // TMEM cols per warp per tile (+ LC prefix)
    static constexpr int TCOLS = (NR / 4) * WCOLS;     // TMEM columns per tile
#ifndef DESC_SCAN_PASS
#define DESC_SCAN_PASS 2          // scan warps: register passes per tile (A/B knob)
#endif
    static constexpr int HALF = (VPT + DESC_SCAN_PASS - 1) / DESC_SCAN_PASS;   // vectors per pass
    static_assert(QT >= 2 && S >= 2, "need TMEM slack and a double-buffered ring");
    static_assert(NR % 4 == 0, "warp groups cover the four TMEM lane quarters evenly");
    static_assert(QT * TCOLS <= 512, "parked tiles must fit the 512 TMEM columns");
    static_assert(NLB >= 1 && NLB <= S + 1, "sentinel fan-out reuses only retired slots");
};

constexpr uint64_t kScanSentinel = ~0ull;              // "no more tiles" tag

#ifdef DESC_SCAN_TRACE        // diagnostics builds only: per-tile globaltimer stamps
constexpr int kTraceTiles = 1 << 16;
// 0 claim, 1 bytes landed (reduce warp 0), 2 A published, 3 look-back start, 4 look-back end,
// 5 polls, 6 scan start (prefix in hand), 7 scan end
__device__ uint64_t g_scan_trace[8][kTraceTiles];
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SCAN_TRACE(f, t, v) do { if ((uint64_t)(t) < (uint64_t)kTraceTiles) g_scan_trace[f][t] = (v); } while (0)
#else
#define SCAN_TRACE(f, t, v) do { } while (0)
#endif

#ifndef DESC_SCAN_REL_FENCE   // proxy fence before a reduce warp releases its ring stage
#define DESC_SCAN_REL_FENCE 1
#endif

#ifndef DESC_SCAN_DIAG        // diagnostics builds only (wrong results): 1 = no look-back,
#define DESC_SCAN_DIAG 0      // 2 = outputs are the inputs (no scan arithmetic)
#endif

template <typename In, int NR, int VPT, int S, int QT, int NLB, int LC = 0>
__global__ void __launch_bounds__(ScanStreamCfg<NR, VPT, S, QT, NLB, LC>::THREADS, 1)
scan_stream_kernel(const __grid_constant__ CUtensorMap map_in,
                   const __grid_constant__ CUtensorMap map_out, const In *__restrict__ in,
                   In *__restrict__ out, int64_t n, int64_t ntiles, int64_t bulk_rows,
                   ScanState<typename AccOf<In>::T> st) {
    using Acc = typename AccOf<In>::T;
    using C = ScanStreamCfg<NR, VPT, S, QT, NLB, LC>;
    constexpr int V = 16 / sizeof(In);              // elements per 16-byte vector
    constexpr int TB = C::TB;
    constexpr int Q = C::Q;
    constexpr int64_t T = TB / sizeof(In);          // tile elements
    constexpr int PROD = 2 * NR, AGGR = 2 * NR + 1, LB0 = 2 * NR + 2;   // warp roles
    extern __shared__ __align__(128) uint8_t smem_raw[];
    // the input is seen by TMA as rows of 128 bytes (bulk_rows of them; the < 128-byte tail
    // is read directly), loaded with the 128-byte swizzle: 16-byte chunk c of row w of a
    // stage sits at chunk c ^ (w & 7), so the warp-striped reads below are conflict-free
    const uint32_t ring = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int64_t n_bulk = bulk_rows * (128 / (int64_t)sizeof(In));
    __shared__ __align__(8) uint64_t full[S], empty[S];          // data ring
    __shared__ __align__(8) uint64_t tag[S];                     // tile id of each ring item
    __shared__ __align__(8) uint64_t parked[QT], freed[QT];      // TMEM slots
    __shared__ __align__(8) uint64_t wsum[Q], aggb[Q], pfx[Q];   // per tile slot
    __shared__ __align__(8) uint64_t wtot[Q][NR + 1];            // warp totals + tile id
    __shared__ __align__(8) uint64_t tagg[Q][2];                 // aggregate, tile id
    __shared__ __align__(8) uint64_t tpre[Q];                    // exclusive prefix
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    ptx::grid_dependency_wait();       // PDL: the state reset (and anything before) is done
    ptx::grid_launch_dependents();

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(ptx::smem_u32(&full[s]), 1);
            ptx::mbar_init(ptx::smem_u32(&empty[s]), NR);
        }
#pragma unroll
        for (int i = 0; i < QT; ++i) {
            ptx::mbar_init(ptx::smem_u32(&parked[i]), NR);
            ptx::mbar_init(ptx::smem_u32(&freed[i]), NR);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            ptx::mbar_init(ptx::smem_u32(&wsum[q]), 1);
            ptx::mbar_init(ptx::smem_u32(&aggb[q]), 1);
            ptx::mbar_init(ptx::smem_u32(&pfx[q]), 1);
        }
        ptx::fence_mbarrier_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 512);
    ptx::tmem_fence_before_sync();
    __syncthreads();
    ptx::tmem_fence_after_sync();

    if (warp == PROD) {
        // ------------------------------------------------------------------ producer
        if (lane != 0) return;
        const uint64_t pol = ptx::policy_evict_first();
        ptx::prefetch_tensormap(&map_in);
        for (int64_t k = 0;; ++k) {
            const int s = (int)(k % S);
            const uint32_t ph = (uint32_t)(k / S) & 1u;
            ptx::mbar_wait(ptx::smem_u32(&empty[s]), ph ^ 1u);
            const int64_t t =
                (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(st.counter), 1ull);
            const uint32_t fb = ptx::smem_u32(&full[s]);
            if (t >= ntiles) {                           // no more tiles: tell the consumers
                ptx::mbar_arrive_expect_tx(fb, 8);
                ptx::st_async_b64(ptx::smem_u32(&tag[s]), kScanSentinel, fb);
                return;
            }
            SCAN_TRACE(0, t, gtimer());
            // boxes that start inside the TMA view (rows past its end are zero-filled and
            // never read back: the reduce warps take those vectors from global memory)
            const int64_t row0 = t * C::ROWS;
            int nb = 0;
            while (nb < C::NBOX && row0 + (int64_t)nb * C::BOX_ROWS < bulk_rows) ++nb;
            ptx::mbar_arrive_expect_tx(fb, (uint32_t)(nb * C::BOX_ROWS * 128) + 8);
            ptx::st_async_b64(ptx::smem_u32(&tag[s]), (uint64_t)t, fb);
            const uint32_t dst = ring + (uint32_t)s * TB;
            for (int b = 0; b < nb; ++b)
                ptx::tma_load_2d(dst + b * C::BOX_ROWS * 128, &map_in, fb, 0,
                                 (int32_t)(row0 + (int64_t)b * C::BOX_ROWS), pol);
        }
    }

    if (warp == AGGR) {
        // ------------------------------------------------------------------ aggregator
        for (int64_t k = 0;; ++k) {
            const int q = (int)(k % Q);
            const uint32_t ph = (uint32_t)(k / Q) & 1u;
            const uint32_t wb = ptx::smem_u32(&wsum[q]);
            if (lane == 0) ptx::mbar_arrive_expect_tx(wb, (NR + 1) * 8);
            ptx::mbar_wait(wb, ph);
            const uint64_t tg = wtot[q][NR];
            Acc agg = 0;
#pragma unroll
            for (int w = 0; w < NR; ++w) agg += acc_from_bits<Acc>(wtot[q][w]);
            if (lane == 0) {
                if (tg != kScanSentinel) publish(st, (int64_t)tg, agg, tg == 0 ? 2u : 1u);
                if (tg != kScanSentinel) SCAN_TRACE(2, tg, gtimer());
                // the sentinel goes to the next NLB slots: one per look-back warp
                for (int i = 0; i < (tg == kScanSentinel ? NLB : 1); ++i) {
                    const int qi = (int)((k + i) % Q);
                    const uint32_t ab = ptx::smem_u32(&aggb[qi]);
                    ptx::mbar_arrive_expect_tx(ab, 16);
                    ptx::st_async_b64(ptx::smem_u32(&tagg[qi][0]), acc_bits(agg), ab);
                    ptx::st_async_b64(ptx::smem_u32(&tagg[qi][1]), tg, ab);
                }
            }
            if (tg == kScanSentinel) return;
        }
    }

    if (warp >= LB0) {
        // ------------------------------------------------------------------ look-back
        for (int64_t k = warp - LB0;; k += NLB) {
            const int q = (int)(k % Q);
            const uint32_t ph = (uint32_t)(k / Q) & 1u;
            ptx::mbar_wait(ptx::smem_u32(&aggb[q]), ph);
            const uint64_t tg = tagg[q][1];
            if (tg == kScanSentinel) return;
            const int64_t t = (int64_t)tg;
            const Acc agg = acc_from_bits<Acc>(tagg[q][0]);
            Acc prefix = 0;
#if !(DESC_SCAN_DIAG & 1)
            if (t > 0 && !DESC_MUTANT(MUT_SCAN_NO_LOOKBACK)) {
#ifdef DESC_SCAN_TRACE
                int polls = 0;
                if (lane == 0) SCAN_TRACE(3, t, gtimer());
                prefix = look_back<Acc, DESC_SCAN_LB_WINDOW>(st, t, lane, &polls);
                if (lane == 0) { SCAN_TRACE(4, t, gtimer()); SCAN_TRACE(5, t, polls); }
#else
                prefix = look_back<Acc, DESC_SCAN_LB_WINDOW>(st, t, lane);
#endif
                if (lane == 0) publish(st, t, prefix + agg, 2u);
            }
#endif
            if (lane == 0) {
                const uint32_t pb = ptx::smem_u32(&pfx[q]);
                ptx::mbar_arrive_expect_tx(pb, 8);
                ptx::st_async_b64(ptx::smem_u32(&tpre[q]), acc_bits(prefix), pb);
            }
        }
    }

    // segment r of a tile: vectors [r*32*VPT, (r+1)*32*VPT), round v = vectors r*32*VPT +
    // v*32 + lane; TMEM: lane quarter r % 4, column block (r / 4) * WCOLS of each slot
    const int r = warp < NR ? warp : warp - NR;
    const uint32_t tmem_w = tmem_base + ((uint32_t)(32 * (r & 3)) << 16) +
                            (uint32_t)((r >> 2) * C::WCOLS);
    if (warp < NR) {
        // ------------------------------------------------------------------ reduce warps
        for (int64_t k = 0;; ++k) {
            const int s = (int)(k % S);
            const uint32_t ph = (uint32_t)(k / S) & 1u;
            const int q = (int)(k % Q);
            const int qt = (int)(k % QT);
            ptx::mbar_wait(ptx::smem_u32(&full[s]), ph);
            const uint64_t tg = tag[s];
            Acc wsum_v = 0, lex = 0;
            uint4 x[VPT];
            if (tg != kScanSentinel) {
                if (r == 0 && lane == 0) SCAN_TRACE(1, tg, gtimer());
                const int64_t tbase = (int64_t)tg * T;
                const uint32_t sbase = ring + (uint32_t)s * TB;
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    // round layout: vector v*32 + lane of the warp's segment; LC: vector
                    // lane*VPT + v (row `lane` of the segment: under the 128-byte swizzle an
                    // 8-lane phase reads 8 rows at 8 distinct chunks v ^ (lane & 7))
                    const int vi = LC ? (r * 32 + lane) * VPT + v : (r * VPT + v) * 32 + lane;
                    const int64_t e0 = tbase + (int64_t)vi * V;
                    if (e0 + V <= n_bulk) {
                        const int w = vi >> 3;
                        x[v] = ptx::lds128(sbase + w * 128 + (((vi & 7) ^ (w & 7)) << 4));
                    } else {                             // tail: not in the TMA view
                        x[v] = make_uint4(0, 0, 0, 0);
#pragma unroll
                        for (int e = 0; e < V; ++e)
                            if (e0 + e < n) set_elem<In>(x[v], e, in[e0 + e]);
                    }
                    wsum_v += vec_sum<In, Acc>(x[v]);
                }
                if constexpr (LC) {   // lanes' exclusive prefixes go to the scan warps via TMEM
                    const Acc incl = warp_incl_scan(wsum_v, lane);
                    lex = warp_excl_from_incl(incl, lane);
                    wsum_v = __shfl_sync(0xffffffffu, incl, 31);
                } else {
                    wsum_v = warp_sum(wsum_v);
                }
            }
            // the warp total goes out before the TMEM slot is awaited: a tile's aggregate
            // depends on nothing but its bytes
            if (lane == 0) {
                const uint32_t wb = ptx::smem_u32(&wsum[q]);
                ptx::st_async_b64(ptx::smem_u32(&wtot[q][r]), acc_bits(wsum_v), wb);
                if (r == 0) ptx::st_async_b64(ptx::smem_u32(&wtot[q][NR]), tg, wb);
            }
            if (tg != kScanSentinel) {
                ptx::mbar_wait(ptx::smem_u32(&freed[qt]), ((uint32_t)(k / QT) & 1u) ^ 1u);
                ptx::tmem_fence_after_sync();
                const uint32_t tm = tmem_w + (uint32_t)(qt * C::TCOLS);
#pragma unroll
                for (int v = 0; v < VPT; ++v) ptx::tmem_st4(tm + 4 * v, x[v]);
                if constexpr (LC) {
                    const uint64_t b = acc_bits(lex);
                    ptx::tmem_st2(tm + 4 * VPT, (uint32_t)b, (uint32_t)(b >> 32));
                }
                ptx::tmem_wait_st();
                ptx::tmem_fence_before_sync();
            }
#if DESC_SCAN_REL_FENCE
            // the next TMA load into this stage is an async-proxy write after the ld.shared
            // reads above (ptx.cuh release_slot_after_lds; here the reads have also been
            // consumed -- sums, TMEM stores -- before the arrive)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(ptx::smem_u32(&empty[s]));             // stage reusable
                if (tg != kScanSentinel) ptx::mbar_arrive(ptx::smem_u32(&parked[qt]));
            }
            if (tg == kScanSentinel) break;
        }
    } else if (warp < 2 * NR) {
        // ------------------------------------------------------------------ scan warps
        const uint64_t drop = ptx::policy_evict_first();
        for (int64_t j = 0;; ++j) {
            const int q = (int)(j % Q);
            const uint32_t qph = (uint32_t)(j / Q) & 1u;
            const int qt = (int)(j % QT);
            ptx::mbar_wait(ptx::smem_u32(&wsum[q]), qph);   // warp totals + tile id
            const uint64_t tg = wtot[q][NR];
            if (tg == kScanSentinel) break;
            ptx::mbar_wait(ptx::smem_u32(&pfx[q]), qph);
            if (r == 0 && lane == 0) SCAN_TRACE(6, tg, gtimer());
            const int64_t tbase = (int64_t)tg * T;
            Acc rcarry = acc_from_bits<Acc>(tpre[q]);
#pragma unroll
            for (int w = 0; w < NR; ++w)
                if (w < r) rcarry += acc_from_bits<Acc>(wtot[q][w]);
            ptx::mbar_wait(ptx::smem_u32(&parked[qt]), (uint32_t)(j / QT) & 1u);
            ptx::tmem_fence_after_sync();
            const uint32_t tm = tmem_w + (uint32_t)(qt * C::TCOLS);
            if constexpr (LC) {
                // lane-contiguous: start = tile prefix + warps before + the lane's exclusive
                // prefix (parked by the reduce warp); vector sums, their running prefix, then
                // each vector's elements from its own base; results into the swizzled staging
                // row `lane`, one TMA tensor store of the warp's 4 KB segment
                uint32_t plo, phi;
                ptx::tmem_ld2(tm + 4 * VPT, plo, phi);
                ptx::tmem_wait_ld();
                asm volatile("" : "+r"(plo), "+r"(phi));
                Acc run = rcarry + acc_from_bits<Acc>(((uint64_t)phi << 32) | plo);
                const uint32_t stg = ring + (uint32_t)(S * TB + r * C::WSEG);
                if (lane == 0 && !DESC_MUTANT(MUT_SCAN_LC_NO_WAIT))
                    ptx::bulk_wait_group_read<0>();              // last store done reading
                __syncwarp();
#pragma unroll
                for (int h = 0; h < VPT; h += C::HALF) {
                    constexpr int H = C::HALF;
                    uint4 x[H];
#pragma unroll
                    for (int v = 0; v < H; ++v)
                        if (h + v < VPT) x[v] = ptx::tmem_ld4(tm + 4 * (h + v));
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int v = 0; v < H; ++v)
                        asm volatile("" : "+r"(x[v].x), "+r"(x[v].y), "+r"(x[v].z), "+r"(x[v].w));
                    if (h + H >= VPT) {
                        ptx::tmem_fence_before_sync();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&freed[qt]));
                    }
                    Acc vb[H];
#pragma unroll
                    for (int v = 0; v < H; ++v) {
                        vb[v] = run;
                        if (h + v < VPT) run += vec_sum<In, Acc>(x[v]);
                    }
#pragma unroll
                    for (int v = 0; v < H; ++v) {
                        if (h + v >= VPT) break;
                        const int vi = (r * 32 + lane) * VPT + h + v;
                        const int64_t e0 = tbase + (int64_t)vi * V;
                        uint4 o = make_uint4(0, 0, 0, 0);
                        Acc ev = vb[v];
#pragma unroll
                        for (int e = 0; e < V; ++e) {
                            ev += to_acc<Acc>(unpack<In>(x[v], e));
                            set_elem<In>(o, e, (In)ev);
                        }
#if DESC_SCAN_DIAG & 2
                        o = x[v];
#endif
                        if (e0 + V <= n_bulk) {
                            const int sw = DESC_MUTANT(MUT_SCAN_LC_NO_SWIZZLE) ? 0 : (lane & 7);
                            ptx::sts128(stg + (uint32_t)(lane * 128 + (((h + v) ^ sw) << 4)), o);
                        } else {                     // tail beyond the TMA view
#pragma unroll
                            for (int e = 0; e < V; ++e)
                                if (e0 + e < n) out[e0 + e] = unpack<In>(o, e);
                        }
                    }
                }
                if (!DESC_MUTANT(MUT_SCAN_LC_NO_WAIT))
                    ptx::fence_proxy_async_shared(); // staging writes -> async proxy
                __syncwarp();
                if (lane == 0) {
                    const int64_t row0 = (tbase * (int64_t)sizeof(In) + (int64_t)r * C::WSEG) / 128;
                    if (row0 < bulk_rows) {          // rows past the view are clipped by TMA
                        ptx::tma_store_2d(&map_out, stg, 0, (int32_t)row0);
                        ptx::bulk_commit_group();
                    }
                }
            } else {
#pragma unroll
            for (int h = 0; h < VPT; h += C::HALF) {
                constexpr int H = C::HALF;
                uint4 x[H];
#pragma unroll
                for (int v = 0; v < H; ++v)
                    if (h + v < VPT) x[v] = ptx::tmem_ld4(tm + 4 * (h + v));
                ptx::tmem_wait_ld();
#pragma unroll
                for (int v = 0; v < H; ++v)              // registers valid only after the wait
                    asm volatile("" : "+r"(x[v].x), "+r"(x[v].y), "+r"(x[v].z), "+r"(x[v].w));
                if (h + H >= VPT) {                      // last pass: the slot can be reused
                    ptx::tmem_fence_before_sync();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&freed[qt]));
                }
                // the rounds' warp scans are independent: run them level by level together
                Acc wi[H], wex[H], wt[H];
#pragma unroll
                for (int v = 0; v < H; ++v) wi[v] = h + v < VPT ? vec_sum<In, Acc>(x[v]) : Acc(0);
                warp_incl_scan_n<Acc, H>(wi, lane);
#pragma unroll
                for (int v = 0; v < H; ++v) {
                    wex[v] = warp_excl_from_incl(wi[v], lane);
                    wt[v] = __shfl_sync(0xffffffffu, wi[v], 31);
                }
#pragma unroll
                for (int v = 0; v < H; ++v) {
                    if (h + v >= VPT) break;
                    const int vi = (r * VPT + h + v) * 32 + lane;
                    const int64_t e0 = tbase + (int64_t)vi * V;
                    Acc run = rcarry + wex[v];
                    rcarry += wt[v];
                    uint4 o = make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        run += to_acc<Acc>(unpack<In>(x[v], e));
                        set_elem<In>(o, e, (In)run);
                    }
#if DESC_SCAN_DIAG & 2
                    o = x[v];
#endif
                    if (e0 + V <= n) {
                        ptx::stg128_hint(out + e0, o, drop);
                    } else {
#pragma unroll
                        for (int e = 0; e < V; ++e)
                            if (e0 + e < n) out[e0 + e] = unpack<In>(o, e);
                    }
                }
            }
            }   // round layout
        }
    }
    if constexpr (LC) {   // scan warps: their TMA stores have completed before the CTA exits
        if (warp >= NR && warp < 2 * NR && lane == 0) ptx::bulk_wait_group<0>();
    }
    // release TMEM once both warp groups are done with it
    ptx::tmem_fence_before_sync();
    ptx::named_bar_sync(1, 32 * 2 * NR);
    if (warp == 0) {
        ptx::tmem_fence_after_sync();
        ptx::tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace desc
