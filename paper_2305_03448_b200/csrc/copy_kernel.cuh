// copy_kernel.cuh -- strided batched block copy  out[b][i][j] = in[b][i][j].
//
// The untransposed "unpack" step of the distributed slab transpose (BASELINE.json
// north_star (4)): the all-to-all delivers P contiguous R x R blocks that
// must land side by side (pitch N) in the output slab.  In the paper's terms it is the
// identity view applied to a `group`-ed place (Listing 3) -- a copy between
// two layouts of the same elements, no transposition.
//
// One CTA per row (a grid of batch*rows CTAs; grid-stride if capped), threads stride over
// 16-byte (or element-sized) units of the row, UNR (4 or 8) units in flight per thread.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace desc {

template <typename V, int UNR = 4>
__global__ void __launch_bounds__(256)
copy_rows_kernel(const char *__restrict__ in, char *__restrict__ out, int64_t rows,
                 int64_t total_rows, int64_t units, int64_t ld_in_b, int64_t ld_out_b,
                 int64_t stride_in_b, int64_t stride_out_b) {
    // The CTA's first row into L2 before the dependency wait (as in the TILED transpose: L2
    // is the point of coherence): 2048^2 f64-sized copies 0.79 -> 1.02 of the copy peak back
    // to back.  Prefetching the NEXT row inside the loop loses (0.96 -> 0.84 at 256 MB): with
    // writes in flight the prefetched lines are evicted before use
    // (profiles/r02_reduce_prefetch.txt).
    if ((int64_t)blockIdx.x < total_rows) {
        const int64_t b = blockIdx.x / rows, i = blockIdx.x - b * rows;
        const char *src = in + b * stride_in_b + i * ld_in_b;
        const int64_t bytes = units * (int64_t)sizeof(V);
        for (int64_t o = (int64_t)threadIdx.x * 128; o < bytes; o += (int64_t)blockDim.x * 128)
            ptx::prefetch_l2(src + o);
    }
    ptx::grid_dependency_wait();       // PDL: previous grid complete before any access
    ptx::grid_launch_dependents();
    for (int64_t r = blockIdx.x; r < total_rows; r += gridDim.x) {
        const int64_t b = r / rows, i = r - b * rows;
        const V *src = reinterpret_cast<const V *>(in + b * stride_in_b + i * ld_in_b);
        V *dst = reinterpret_cast<V *>(out + b * stride_out_b + i * ld_out_b);
        int64_t u = threadIdx.x;
        for (; u + (UNR - 1) * blockDim.x < units; u += UNR * blockDim.x) {
            V v[UNR];
#pragma unroll
            for (int k = 0; k < UNR; ++k) v[k] = src[u + k * blockDim.x];
#pragma unroll
            for (int k = 0; k < UNR; ++k) dst[u + k * blockDim.x] = v[k];
        }
        for (; u < units; u += blockDim.x) dst[u] = src[u];
    }
}

}  // namespace desc
