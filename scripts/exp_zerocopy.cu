// exp_zerocopy.cu -- PCIe experiment for the host-buffer (e2e) path: how fast can SM loads /
// stores reach mapped pinned host memory, per direction and both at once, next to the DMA
// engines.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/exp_zerocopy.cu -o /tmp/zc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename V>
__global__ void copy_kernel(const V *__restrict__ in, V *__restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main() {
    const size_t bytes = 256ull << 20;
    char *h_a, *h_b, *d_a, *d_b;
    CK(cudaHostAlloc(&h_a, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_b, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&d_a, bytes));
    CK(cudaMalloc(&d_b, bytes));
    CK(cudaMemset(d_a, 1, bytes));
    for (size_t i = 0; i < bytes; i += 4096) h_a[i] = 1;
    cudaStream_t s0, s1;
    CK(cudaStreamCreate(&s0));
    CK(cudaStreamCreate(&s1));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto time = [&](auto fn, const char *name, double moved) {
        fn();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, s0));
        for (int r = 0; r < 5; ++r) fn();
        CK(cudaEventRecord(e1, s0));
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%-44s %8.1f GB/s\n", name, moved * 5 / (ms / 1e3) / 1e9);
        return 0;
    };
    int grids[] = {148, 296, 592, 1184};
    for (int g : grids) {
        char name[128];
        snprintf(name, sizeof name, "kernel H2D read  (uint4, grid %d)", g);
        time([&] { copy_kernel<uint4><<<g, 256, 0, s0>>>((const uint4 *)h_a, (uint4 *)d_a, bytes / 16); }, name, bytes);
        snprintf(name, sizeof name, "kernel D2H write (uint4, grid %d)", g);
        time([&] { copy_kernel<uint4><<<g, 256, 0, s0>>>((const uint4 *)d_b, (uint4 *)h_b, bytes / 16); }, name, bytes);
        snprintf(name, sizeof name, "kernel H2D read  (u32, grid %d)", g);
        time([&] { copy_kernel<uint32_t><<<g, 256, 0, s0>>>((const uint32_t *)h_a, (uint32_t *)d_a, bytes / 4); }, name, bytes);
        snprintf(name, sizeof name, "kernel D2H write (u32, grid %d)", g);
        time([&] { copy_kernel<uint32_t><<<g, 256, 0, s0>>>((const uint32_t *)d_b, (uint32_t *)h_b, bytes / 4); }, name, bytes);
        snprintf(name, sizeof name, "kernel host->host (uint4, grid %d)", g);
        time([&] { copy_kernel<uint4><<<g, 256, 0, s0>>>((const uint4 *)h_a, (uint4 *)h_b, bytes / 16); }, name, 2.0 * bytes);
    }
    time([&] { cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s0); }, "DMA H2D", bytes);
    time([&] { cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, s0); }, "DMA D2H", bytes);
    time([&] {
        cudaEvent_t f; cudaEventCreateWithFlags(&f, cudaEventDisableTiming);
        cudaEventRecord(f, s0); cudaStreamWaitEvent(s1, f, 0); cudaEventDestroy(f);
        cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s0);
        cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, s1);
        cudaEvent_t x; cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        cudaEventRecord(x, s1); cudaStreamWaitEvent(s0, x, 0); cudaEventDestroy(x);
    }, "DMA H2D || D2H", 2.0 * bytes);
    time([&] {
        cudaEvent_t f; cudaEventCreateWithFlags(&f, cudaEventDisableTiming);
        cudaEventRecord(f, s0); cudaStreamWaitEvent(s1, f, 0); cudaEventDestroy(f);
        copy_kernel<uint4><<<592, 256, 0, s0>>>((const uint4 *)h_a, (uint4 *)d_a, bytes / 16);
        cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, s1);
        cudaEvent_t x; cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        cudaEventRecord(x, s1); cudaStreamWaitEvent(s0, x, 0); cudaEventDestroy(x);
    }, "kernel H2D read || DMA D2H", 2.0 * bytes);
    time([&] {
        cudaEvent_t f; cudaEventCreateWithFlags(&f, cudaEventDisableTiming);
        cudaEventRecord(f, s0); cudaStreamWaitEvent(s1, f, 0); cudaEventDestroy(f);
        cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s1);
        copy_kernel<uint4><<<592, 256, 0, s0>>>((const uint4 *)d_b, (uint4 *)h_b, bytes / 16);
        cudaEvent_t x; cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        cudaEventRecord(x, s1); cudaStreamWaitEvent(s0, x, 0); cudaEventDestroy(x);
    }, "DMA H2D || kernel D2H write", 2.0 * bytes);
    return 0;
}
