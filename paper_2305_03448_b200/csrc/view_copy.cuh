// view_copy.cuh -- materialise a strided view: out[v] = in[offset + sum_d v_d * stride_d].
//
// Any chain of Descend's basic views (Listing 3: group, transpose, split,
// reverse, map) over a strided root is again a strided view (shape, strides, offset; strides
// may be negative after `reverse`) -- the host compiles the chain (desc_view_compile, the
// analog of "views are compiled into raw indices ... in reversed order", P:509-511,
// P:1039-1042) and the device materialises it.  The dispatcher (desc_transpose.cu) sends
// views whose innermost output dim is a transposition onto the TMA transpose kernels; the
// rest land here: one CTA per output row (the view's innermost dim), 16-byte vectors when
// every row is contiguous and aligned on both sides, element cells otherwise.
#pragma once
#include <cstdint>

namespace desc {

constexpr int kMaxViewDims = 8;

struct ViewRows {
    int32_t outer_ndim;                  // dims other than the innermost
    int64_t outer_shape[kMaxViewDims];
    int64_t outer_stride[kMaxViewDims];  // input element strides of the outer dims
    int64_t inner;                       // innermost extent (row length, elements)
    int64_t inner_stride;                // input stride of the innermost dim (elements)
    int64_t offset;                      // input element offset of view element 0
    int64_t rows;                        // product of outer_shape
};

// Input element offset of the first element of output row r (mixed-radix decomposition).
__device__ __forceinline__ int64_t view_row_offset(const ViewRows &v, int64_t r) {
    int64_t off = v.offset;
    for (int d = v.outer_ndim - 1; d >= 0; --d) {
        const int64_t n = v.outer_shape[d];
        const int64_t q = r / n;
        off += (r - q * n) * v.outer_stride[d];
        r = q;
    }
    return off;
}

// Cell = element-sized word; inner_stride arbitrary (negative after reverse).
template <typename Cell>
__global__ void __launch_bounds__(256)
view_rows_kernel(const Cell *__restrict__ in, Cell *__restrict__ out, const ViewRows v) {
    for (int64_t r = blockIdx.x; r < v.rows; r += gridDim.x) {
        const Cell *src = in + view_row_offset(v, r);
        Cell *dst = out + r * v.inner;
        int64_t u = threadIdx.x;
        for (; u + 3 * blockDim.x < v.inner; u += 4 * blockDim.x) {
            const Cell c0 = src[u * v.inner_stride];
            const Cell c1 = src[(u + blockDim.x) * v.inner_stride];
            const Cell c2 = src[(u + 2 * blockDim.x) * v.inner_stride];
            const Cell c3 = src[(u + 3 * blockDim.x) * v.inner_stride];
            dst[u] = c0;
            dst[u + blockDim.x] = c1;
            dst[u + 2 * blockDim.x] = c2;
            dst[u + 3 * blockDim.x] = c3;
        }
        for (; u < v.inner; u += blockDim.x) dst[u] = src[u * v.inner_stride];
    }
}

// Contiguous, 16-byte aligned rows on both sides: inner counted in uint4 units.
__global__ void __launch_bounds__(256)
view_rows_vec_kernel(const char *__restrict__ in, char *__restrict__ out, const ViewRows v,
                     int es) {
    const int64_t units = v.inner * es / 16;
    for (int64_t r = blockIdx.x; r < v.rows; r += gridDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(in + view_row_offset(v, r) * es);
        uint4 *dst = reinterpret_cast<uint4 *>(out + r * v.inner * es);
        int64_t u = threadIdx.x;
        for (; u + 3 * blockDim.x < units; u += 4 * blockDim.x) {
            const uint4 a = src[u], b = src[u + blockDim.x], c = src[u + 2 * blockDim.x],
                        d = src[u + 3 * blockDim.x];
            dst[u] = a;
            dst[u + blockDim.x] = b;
            dst[u + 2 * blockDim.x] = c;
            dst[u + 3 * blockDim.x] = d;
        }
        for (; u < units; u += blockDim.x) dst[u] = src[u];
    }
}

}  // namespace desc
