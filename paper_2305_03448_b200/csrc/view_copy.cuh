// view_copy.cuh -- materialise a strided view: out[v] = in[offset + sum_d v_d * stride_d].
//
// Any chain of Descend's basic views (Listing 3: group, transpose, split,
// reverse, map) over a strided root is again a strided view (shape, strides, offset; strides
// may be negative after `reverse`) -- the host compiles the chain (desc_view_compile, the
// analog of "views are compiled into raw indices ... in reversed order", P:509-511,
// P:1039-1042) and the device materialises it.  The dispatcher (desc_transpose.cu) sends
// views whose innermost output dim is a transposition onto the TMA transpose kernels; the
// rest land here.
//
// Work decomposition: after merging, the view is  outer dims x R2 rows x U cells, the cells
// of a row at input stride s1 (+1, -1 or anything), rows at input stride s2.  A work item is
// one (outer index, row chunk, cell chunk): the outer mixed-radix decomposition is paid once
// per item, rows inside the item cost a multiply.  Threads map onto (row, cell) with a
// power-of-two cell width (shift/mask, no division); the output is contiguous, so a warp
// always writes consecutive 16-byte units (or cells).  Cells are 16-byte vectors whenever
// every row is aligned and s1 = +1 (plain) or -1 (vector loaded from the mirrored position
// and its elements reversed in registers), else single elements.
#pragma once
#include <cstdint>

#include "ptx.cuh"
#include <type_traits>

namespace desc {

constexpr int kMaxViewDims = 8;

struct ViewTiles {
    int32_t outer_ndim;
    int64_t outer_shape[kMaxViewDims];
    int64_t outer_stride[kMaxViewDims];  // input strides of the outer dims (elements)
    int64_t R2, s2;                      // rows per outer index and their input stride
    int64_t U;                           // cells per row
    int64_t s1;                          // input stride between cells (elements; +/-1 for vec)
    int64_t offset;                      // input element offset of view element 0
    int64_t outer_count;                 // product of outer_shape
    int64_t rch, uch;                    // row / cell chunk of a work item
    int64_t n_rchunks, n_uchunks, items;
    int32_t ulog;                        // log2 of the thread cell width (pow2 >= min(uch, 256))
};

__device__ __forceinline__ int64_t outer_offset(const ViewTiles &v, int64_t r) {
    int64_t off = v.offset;
    for (int d = v.outer_ndim - 1; d >= 0; --d) {
        const int64_t n = v.outer_shape[d];
        const int64_t q = r / n;
        off += (r - q * n) * v.outer_stride[d];
        r = q;
    }
    return off;
}

__device__ __forceinline__ uint4 reverse_elems(const uint4 &x, int es) {
    if (es == 8) return make_uint4(x.z, x.w, x.x, x.y);
    if (es == 4) return make_uint4(x.w, x.z, x.y, x.x);
    if (es == 2)
        return make_uint4(__byte_perm(x.w, 0, 0x1032), __byte_perm(x.z, 0, 0x1032),
                          __byte_perm(x.y, 0, 0x1032), __byte_perm(x.x, 0, 0x1032));
    return make_uint4(__byte_perm(x.w, 0, 0x0123), __byte_perm(x.z, 0, 0x0123),
                      __byte_perm(x.y, 0, 0x0123), __byte_perm(x.x, 0, 0x0123));
}

template <typename Cell, int MODE>
struct CellIO {
    using T = typename std::conditional<MODE == 0, Cell, uint4>::type;
    static constexpr int CB = MODE == 0 ? (int)sizeof(Cell) : 16;     // bytes per cell
    __device__ static T load(const char *in, int64_t in_row, int64_t u, int64_t s1, int es) {
        if constexpr (MODE == 0) {
            return *reinterpret_cast<const Cell *>(in + (in_row + u * s1) * CB);
        } else if constexpr (MODE == 1) {
            return *reinterpret_cast<const uint4 *>(in + in_row * es + u * 16);
        } else {
            // output cell u holds view elements u*V .. u*V+V-1 = input elements
            // in_row - u*V - (V-1) .. in_row - u*V, in reverse order
            const int V = 16 / es;
            const int64_t first = in_row - u * V - (V - 1);
            return reverse_elems(*reinterpret_cast<const uint4 *>(in + first * es), es);
        }
    }
};

// MODE 0: element cells (Cell), any s1.   MODE 1: 16-byte cells, s1 = +1.
// MODE 2: 16-byte cells, s1 = -1 (mirrored load + in-register element reversal).
// Short rows: up to 4 rows' loads are in flight per thread before their stores.
#ifndef DESC_VIEW_UNR         // rows' loads in flight per thread in the short-row path (A/B)
#define DESC_VIEW_UNR 4
#endif
// MODE 1 keeps 4 CTAs/SM (<= 64 registers) under its persistent grid: residency is what
// keeps its loads in flight (74 registers = 3 CTAs/SM cost the tile view 0.95 -> 0.82).
template <typename Cell, int MODE>
__global__ void __launch_bounds__(256, MODE == 1 ? 4 : 0)
view_tiles_kernel(const char *__restrict__ in, char *__restrict__ out, const ViewTiles v, int es,
                  int pf) {
    using IO = CellIO<Cell, MODE>;
    using T = typename IO::T;
    constexpr int CB = IO::CB;
    if constexpr (MODE == 2) {
        // mirrored rows (reverse views), launched one work item per CTA: L2 prefetch of the
        // item's input rows, one per 128-byte line, before the dependency wait (as TILED,
        // tiled_transpose.cuh: L2 is the point of coherence, a prefetch returns nothing to
        // the SM and cannot fault) -- rot180 of 8192^2 f32 0.955 -> 1.02
        if (pf && (int64_t)blockIdx.x < v.items) {
            int64_t q = blockIdx.x;
            const int64_t uc = q % v.n_uchunks; q /= v.n_uchunks;
            const int64_t rc = q % v.n_rchunks; q /= v.n_rchunks;
            const int64_t obase = outer_offset(v, q);
            const int64_t r0 = rc * v.rch, nr = min(v.R2, r0 + v.rch) - r0;
            const int64_t u0 = uc * v.uch, nu = min(v.U, u0 + v.uch) - u0;
            const int64_t V = 16 / es, lpr = (nu * 16 + 127) / 128;     // lines per row
            for (int64_t i = threadIdx.x; i < nr * lpr; i += blockDim.x) {
                const int64_t rr = r0 + i / lpr, l = i % lpr;
                // first input element of the row segment (walked backwards)
                const int64_t e0 = obase + rr * v.s2 - (u0 + nu) * V + 1;
                ptx::prefetch_l2(in + e0 * es + l * 128);
            }
        }
    }
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    const int uw = 1 << v.ulog;                                    // thread cell width
    const int rpp = blockDim.x >> v.ulog;                          // rows per pass (>= 1)
    const int tu = threadIdx.x & (uw - 1);
    const int tr = threadIdx.x >> v.ulog;
    for (int64_t w = blockIdx.x; w < v.items; w += gridDim.x) {
        int64_t q = w;
        const int64_t uc = q % v.n_uchunks; q /= v.n_uchunks;
        const int64_t rc = q % v.n_rchunks; q /= v.n_rchunks;
        const int64_t obase = outer_offset(v, q);                 // elements
        const int64_t r0 = rc * v.rch, r1 = min(v.R2, r0 + v.rch);
        const int64_t u0 = uc * v.uch, u1 = min(v.U, u0 + v.uch);
        char *oitem = out + (q * v.R2) * v.U * CB;                 // output is contiguous
        if (u1 - u0 <= uw) {                  // one cell per thread per row: unroll rows
            const int64_t u = u0 + tu;
            const bool uok = u < u1;
            for (int64_t r = r0 + tr; r < r1; r += DESC_VIEW_UNR * rpp) {
                T c[DESC_VIEW_UNR];
#pragma unroll
                for (int k = 0; k < DESC_VIEW_UNR; ++k) {
                    const int64_t rr = r + k * rpp;
                    if (uok && rr < r1) c[k] = IO::load(in, obase + rr * v.s2, u, v.s1, es);
                }
#pragma unroll
                for (int k = 0; k < DESC_VIEW_UNR; ++k) {
                    const int64_t rr = r + k * rpp;
                    if (uok && rr < r1) *reinterpret_cast<T *>(oitem + (rr * v.U + u) * CB) = c[k];
                }
            }
        } else {                              // long rows: consecutive cells per warp,
            for (int64_t r = r0 + tr; r < r1; r += rpp) {   // 4 loads in flight per thread
                const int64_t in_row = obase + r * v.s2;
                char *orow = oitem + r * v.U * CB;
                int64_t u = u0 + tu;
                for (; u + 3 * uw < u1; u += 4 * uw) {
                    T c[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) c[k] = IO::load(in, in_row, u + k * uw, v.s1, es);
#pragma unroll
                    for (int k = 0; k < 4; ++k) *reinterpret_cast<T *>(orow + (u + k * uw) * CB) = c[k];
                }
                for (; u < u1; u += uw)
                    *reinterpret_cast<T *>(orow + u * CB) = IO::load(in, in_row, u, v.s1, es);
            }
        }
    }
}

}  // namespace desc
