// sanitizer_controls.cu -- positive controls for the compute-sanitizer gates (NOT product
// code; built into build_variants/libsanitizer_controls.so by scripts/sanitizer_controls.py).
//
// The product kernels run clean under racecheck / synccheck / memcheck
// (profiles/*_sanitizer_*.log).  "Clean" only means something if the tools see the hazard
// archetypes the paper names when they ARE present, on this GPU and toolkit:
//   * rev_per_block (Sec. 2.2 "Data Races"): the paper's own racy kernel.  Its race is
//     on GLOBAL memory, which racecheck does not track -- the control documents that blind
//     spot (expected: no report); the host index-map checker (tests/test_index_maps.py)
//     rejects the same map.  rev_per_block_shared is the same access pattern staged in shared
//     memory, which racecheck must report.
//   * divergent_barrier (Sec. 2.2 "Synchronization"): `if (threadIdx.x < limit)
//     __syncthreads();`.  The paper's own case (limit 32, 64 threads per block: whole warps
//     skip the barrier and exit) is NOT reported by synccheck on B200 -- measured: exited
//     warps count as arrived, the kernel completes -- a second documented blind spot; with
//     the barrier divergent INSIDE a warp (limit 16, 32 threads) synccheck must report it.
// The Listing 1 race and the TILED kernel without its barrier are positive controls
// too; they live in the mutant build of the product library (csrc/mutants.cuh ids 2 and 14).
#include <cuda_runtime.h>

namespace {

__global__ void rev_per_block(double *array) {
    double *block_part = &array[blockIdx.x * blockDim.x];
    block_part[threadIdx.x] = block_part[blockDim.x - 1 - threadIdx.x];
}

__global__ void rev_per_block_shared(double *array) {
    extern __shared__ double part[];
    double *block_part = &array[blockIdx.x * blockDim.x];
    part[threadIdx.x] = block_part[threadIdx.x];
    __syncthreads();
    part[threadIdx.x] = part[blockDim.x - 1 - threadIdx.x];     // read/write race in smem
    __syncthreads();
    block_part[threadIdx.x] = part[threadIdx.x];
}

__global__ void divergent_barrier(int *out, int limit) {
    if ((int)threadIdx.x < limit) { __syncthreads(); }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (int)threadIdx.x;
}

}  // namespace

extern "C" {

int ctl_rev_per_block(double *array, int blocks, int threads, int shared) {
    if (shared)
        rev_per_block_shared<<<blocks, threads, threads * sizeof(double)>>>(array);
    else
        rev_per_block<<<blocks, threads>>>(array);
    return (int)cudaDeviceSynchronize();
}

int ctl_divergent_barrier(int *out, int blocks, int threads, int limit) {
    divergent_barrier<<<blocks, threads>>>(out, limit);
    return (int)cudaDeviceSynchronize();
}

// exact-size device allocations (the caching allocator of torch rounds sizes up, which would
// hide a one-element overrun from memcheck)
void *ctl_malloc(size_t bytes) {
    void *p = nullptr;
    return cudaMalloc(&p, bytes) == cudaSuccess ? p : nullptr;
}

int ctl_free(void *p) { return (int)cudaFree(p); }

}  // extern "C"
