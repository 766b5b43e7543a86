// reduce_scan.cuh -- the paper's two other memory-bound evaluation kernels (PAPER.md P:1047:
// "block-wide parallel reduction ... scan"), B200-native:
//
//   block reduction   out[b] = sum(in[b*B .. min(n, (b+1)*B)))        (read-bound)
//   inclusive scan    out[i] = sum(in[0 .. i])                          (read + write)
//
// Integers are summed modulo 2^bits (unsigned wrap-around; bit-exact); f32 is accumulated in
// fp64 and rounded once on output; f64 in fp64.
//
// Reduction: a group of G lanes per output block (G = 1, 32 or a 256-thread CTA, chosen by
// B); each group streams its block with 16-byte read-only loads (4 in flight per lane), a
// scalar head/tail around the 16-byte-aligned body, then shuffles (+ shared memory for CTAs).
//
// Scan, short arrays (a few hundred tiles): single pass with decoupled look-back:
// tiles are claimed in order from an atomic counter (so every predecessor is resident),
// each tile scans its 256 x ITEMS elements in registers + shuffles, publishes its aggregate
// (flag A), looks back over predecessors one warp-wide window of 32 at a time (summing
// aggregates until an inclusive prefix, flag P), publishes its own inclusive prefix, and
// writes its outputs.  Flags are released / acquired at gpu scope; aggregate and inclusive
// values live in separate arrays so a reader never mixes them up.  Long arrays: the
// reduce-then-scan route at the end of this file.
#pragma once
#include <cstdint>
#include <cstring>
#include <type_traits>

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
    for (; k + 3 * nl < nv; k += 4 * nl) {
        const uint4 v0 = ld_nc_v4(vp + k), v1 = ld_nc_v4(vp + k + nl),
                    v2 = ld_nc_v4(vp + k + 2 * nl), v3 = ld_nc_v4(vp + k + 3 * nl);
        acc += vec_sum<In, Acc>(v0) + vec_sum<In, Acc>(v1) + vec_sum<In, Acc>(v2) +
               vec_sum<In, Acc>(v3);
    }
    for (; k < nv; k += nl) acc += vec_sum<In, Acc>(ld_nc_v4(vp + k));
    for (int64_t i = a + nv * V + lane; i < hi; i += nl) acc += to_acc<Acc>(in[i]);
    return acc;
}

// G = 1: one thread per output block;  G = 32: one warp per block.
template <typename In, typename Out, int G>
__global__ void __launch_bounds__(256)
block_reduce_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n, int64_t B,
                    int64_t nblocks, bool vec) {
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

// one 256-thread CTA per output block (large B)
template <typename In, typename Out>
__global__ void __launch_bounds__(256)
block_reduce_cta_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n, int64_t B,
                        int64_t nblocks, bool vec) {
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

// ---- scan ---------------------------------------------------------------------------------
template <typename Acc>
struct ScanState {
    uint32_t *counter;   // tile claim counter
    uint32_t *flags;     // 0 = not ready, 1 = aggregate, 2 = inclusive prefix
    Acc *agg;            // per-tile aggregate
    Acc *incl;           // per-tile inclusive prefix (single pass) / exclusive (three-launch)
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Look-back by one warp: exclusive prefix of `tile` = nearest inclusive prefix (flag 2) plus
// the aggregates (flag 1) of the tiles after it.  Each lane inspects LB consecutive
// predecessors per round (a window of 32*LB tiles), so a long run of aggregate-only
// predecessors costs one L2 round trip per 32*LB tiles.  Flags are read relaxed; one gpu-scope
// fence (acquire pattern) orders the value reads after the flags that published them.
template <typename Acc, int LB>
__device__ Acc look_back(const ScanState<Acc> &st, int64_t tile, int lane) {
    constexpr int W = 32 * LB;
    Acc prefix = 0;
    int64_t j = tile - 1;                                   // newest predecessor of the window
    while (true) {
        uint32_t f[LB];
        int dp = W;                                         // distance of the nearest P
#pragma unroll
        for (int m = 0; m < LB; ++m) {
            const int64_t t = j - (lane * LB + m);
            f[m] = t >= 0 ? ld_relaxed(&st.flags[t]) : 2u;
            if (f[m] == 2u && dp == W) dp = lane * LB + m;
        }
        dp = __reduce_min_sync(0xffffffffu, (uint32_t)dp);
        bool missing = false;                               // a needed predecessor unpublished
#pragma unroll
        for (int m = 0; m < LB; ++m)
            if (lane * LB + m <= dp && lane * LB + m < W && f[m] == 0u) missing = true;
        if (__any_sync(0xffffffffu, missing)) continue;
        __threadfence();                                    // acquire: flags -> values
        Acc v = 0;
#pragma unroll
        for (int m = 0; m < LB; ++m) {
            const int d = lane * LB + m;
            const int64_t t = j - d;
            if (d <= dp && t >= 0) v += f[m] == 2u ? __ldcg(&st.incl[t]) : __ldcg(&st.agg[t]);
        }
        prefix += warp_sum(v);
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
template <typename In, typename Out, int ITEMS>
__global__ void __launch_bounds__(256, 4)
scan_kernel(const In *__restrict__ in, Out *__restrict__ out, int64_t n,
            ScanState<typename AccOf<In>::T> st, bool vec) {
    using Acc = typename AccOf<In>::T;
    constexpr int T = 256 * ITEMS;
    constexpr int V = 16 / sizeof(In);
    constexpr int NV = ITEMS / V;
    static_assert(sizeof(In) == sizeof(Out), "scan output has the input's type");
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
    const Acc texcl = wpre + wincl - tsum;                     // exclusive prefix in the tile

    if (warp == 0) {
        Acc prefix = 0;
        if (tile == 0) {
            if (lane == 0) {
                st.incl[0] = agg;
                st_release(&st.flags[0], 2u);
            }
        } else {
            if (lane == 0) {
                st.agg[tile] = agg;
                st_release(&st.flags[tile], 1u);
            }
            prefix = look_back<Acc, 16>(st, tile, lane);
            if (lane == 0) {
                st.incl[tile] = prefix + agg;
                st_release(&st.flags[tile], 2u);
            }
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
        Acc run = carry_s + (warp ? wt[warp - 1] : Acc(0)) + wi - tsum;
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
    Acc wpre = excl[tile];
#pragma unroll
    for (int w = 0; w < 8; ++w)
        if (w < warp) wpre += warp_tot[w];
    Acc rcarry = wpre;                             // prefix before the current round
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e0 = wbase + (int64_t)k * 32 * V + (int64_t)lane * V;
        const Acc ls = vec_sum<In, Acc>(raw[k]);     // recomputed: saves R accumulators
        const Acc wi = warp_incl_scan(ls, lane);
        Acc run = rcarry + wi - ls;
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

}  // namespace desc
