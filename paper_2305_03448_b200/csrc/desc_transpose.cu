// desc_transpose.cu -- the C-ABI boundary (include/desc_transpose.h): argument
// validation (ownership, memory space, shape), kernel dispatch, TMA descriptor cache.
//
// Product code.  It shares nothing with oracle/ (task rule ③).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/desc_transpose.h"
#include "smem_transpose.cuh"
#include "tma_transpose.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int g_last_launches = 0;

desc_status fail(desc_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
desc_status fail(desc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

desc_status cuda_fail(cudaError_t e, const char *what) {
    return fail(DESC_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int dtype_size(desc_dtype t) {
    switch (t) {
        case DESC_F32: case DESC_I32: return 4;
        case DESC_F64: case DESC_I64: return 8;
        case DESC_F16: case DESC_BF16: return 2;
        case DESC_U8: return 1;
    }
    return 0;
}

// ---- overflow-checked int64 arithmetic ----------------------------------------
bool mul_ok(int64_t a, int64_t b, int64_t *r) { return !__builtin_mul_overflow(a, b, r); }
bool add_ok(int64_t a, int64_t b, int64_t *r) { return !__builtin_add_overflow(a, b, r); }

// Span in elements of `batch` matrices of `nr` rows x `nc` cols (pitch ld, stride):
// (batch-1)*stride + (nr-1)*ld + nc.
bool span_elems(int64_t batch, int64_t nr, int64_t nc, int64_t ld, int64_t stride, int64_t *out) {
    int64_t a, b, s;
    if (!mul_ok(batch - 1, stride, &a) || !mul_ok(nr - 1, ld, &b)) return false;
    if (!add_ok(a, b, &s) || !add_ok(s, nc, &s)) return false;
    *out = s;
    return true;
}

struct Args {
    const void *in;
    void *out;
    int64_t batch, rows, cols, ld_in, ld_out, stride_in, stride_out;
    int es;
    cudaStream_t stream;
};

// ---- device properties (per device, cached) -------------------------------------
struct DevInfo {
    int sms = 0;
    bool init = false;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];

desc_status device_info(int dev, DevInfo *out) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (dev < 0 || dev >= 64) return fail(DESC_ERR_CUDA, "device ordinal %d out of range", dev);
    if (!g_dev[dev].init) {
        int sms = 0;
        cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
        g_dev[dev].sms = sms;
        g_dev[dev].init = true;
    }
    *out = g_dev[dev];
    return DESC_OK;
}

// ---- cuTensorMapEncodeTiled via the runtime's driver entry point (no -lcuda) ------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

desc_status get_encode(PFN_cuTensorMapEncodeTiled_v12000 *fn) {
    std::call_once(g_encode_once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!g_encode) return fail(DESC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    *fn = g_encode;
    return DESC_OK;
}

struct MapKey {
    uintptr_t ptr;
    int64_t rows, cols, batch, ld, stride;
    int es, box_rows;
    bool operator==(const MapKey &o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && batch == o.batch &&
               ld == o.ld && stride == o.stride && es == o.es && box_rows == o.box_rows;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey &k) const {
        size_t h = std::hash<uintptr_t>()(k.ptr);
        auto mix = [&h](int64_t v) { h ^= std::hash<int64_t>()(v) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2); };
        mix(k.rows); mix(k.cols); mix(k.batch); mix(k.ld); mix(k.stride); mix(k.es); mix(k.box_rows);
        return h;
    }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

desc_status tensor_map(const Args &a, int box_rows, CUtensorMap *out) {
    MapKey key{reinterpret_cast<uintptr_t>(a.in), a.rows, a.cols, a.batch, a.ld_in,
               a.stride_in, a.es, box_rows};
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) { *out = it->second; return DESC_OK; }
    }
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (desc_status s = get_encode(&encode)) return s;
    CUtensorMapDataType dt = a.es == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                           : a.es == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                           : a.es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                       : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const cuuint32_t rank = a.batch > 1 ? 3 : 2;
    cuuint64_t dims[3] = {(cuuint64_t)a.cols, (cuuint64_t)a.rows, (cuuint64_t)a.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(a.ld_in * a.es), (cuuint64_t)(a.stride_in * a.es)};
    cuuint32_t box[3] = {(cuuint32_t)(128 / a.es), (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, dt, rank, const_cast<void *>(a.in), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(DESC_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 256) g_maps.clear();
    g_maps.emplace(key, m);
    *out = m;
    return DESC_OK;
}

// ---- TMA eligibility -------------------------------------------------------------
bool tma_eligible(const Args &a) {
    const uintptr_t pin = reinterpret_cast<uintptr_t>(a.in), pout = reinterpret_cast<uintptr_t>(a.out);
    if (pin % 16 || pout % 16) return false;
    if ((a.ld_in * a.es) % 16 || (a.ld_out * a.es) % 16) return false;
    if (a.batch > 1 && ((a.stride_in * a.es) % 16 || (a.stride_out * a.es) % 16)) return false;
    if (a.batch > 1 && a.stride_in == 0) return false;
    const int64_t lim = (int64_t)1 << 31;
    if (a.rows >= lim || a.cols >= lim || a.batch >= lim) return false;
    if (a.ld_in * a.es >= ((int64_t)1 << 40) || a.stride_in * a.es >= ((int64_t)1 << 40)) return false;
    return true;
}

// ---- launchers -----------------------------------------------------------------------
template <int ES, int TR, int NB, int STAGES>
desc_status launch_tma(const Args &a) {
    using C = desc::TmaConfig<ES, TR, NB, STAGES>;
    auto kern = desc::transpose_tma_kernel<ES, TR, NB, STAGES>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute");

    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    DevInfo di;
    if (desc_status s = device_info(dev, &di)) return s;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM_BYTES);
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (occ < 1) occ = 1;

    CUtensorMap map;
    if (desc_status s = tensor_map(a, TR, &map)) return s;

    desc::TmaParams p;
    p.out = a.out;
    p.ld_out = a.ld_out;
    p.stride_out = a.stride_out;
    p.rows = (int32_t)a.rows;
    p.cols = (int32_t)a.cols;
    p.batch = (int32_t)a.batch;
    p.tiles_r = (int32_t)((a.rows + TR - 1) / TR);
    p.tiles_c = (int32_t)((a.cols + C::TILE_COLS - 1) / C::TILE_COLS);
    p.rank3 = a.batch > 1 ? 1 : 0;
    p.ntiles = (int64_t)p.tiles_r * p.tiles_c * a.batch;
    const int64_t max_grid = (int64_t)di.sms * occ;
    const int grid = (int)(p.ntiles < max_grid ? p.ntiles : max_grid);
    kern<<<grid, C::THREADS, C::SMEM_BYTES, a.stream>>>(map, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

template <typename Cell>
desc_status launch_smem(const Args &a) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    DevInfo di;
    if (desc_status s = device_info(dev, &di)) return s;
    const int64_t tiles_r = (a.rows + 31) / 32, tiles_c = (a.cols + 31) / 32;
    const int64_t ntiles = tiles_r * tiles_c * a.batch;
    const int64_t max_grid = (int64_t)di.sms * 8;    // 8 x 256-thread CTAs per SM
    const int grid = (int)(ntiles < max_grid ? ntiles : max_grid);
    desc::transpose_smem_kernel<Cell><<<grid, dim3(32, 8), 0, a.stream>>>(
        static_cast<const Cell *>(a.in), static_cast<Cell *>(a.out), a.rows, a.cols, a.ld_in,
        a.ld_out, a.stride_in, a.stride_out, tiles_r, tiles_c, ntiles);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_smem_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

desc_status run_tma(const Args &a) {
    switch (a.es) {
        case 4: return launch_tma<4, 128, 1, 4>(a);
        case 8: return launch_tma<8, 128, 1, 4>(a);
        case 2: return launch_tma<2, 128, 1, 4>(a);
        case 1: return launch_tma<1, 128, 1, 4>(a);
    }
    return fail(DESC_ERR_DTYPE, "unsupported element size %d", a.es);
}

desc_status run_smem(const Args &a) {
    switch (a.es) {
        case 4: return launch_smem<uint32_t>(a);
        case 8: return launch_smem<unsigned long long>(a);
        case 2: return launch_smem<uint16_t>(a);
        case 1: return launch_smem<uint8_t>(a);
    }
    return fail(DESC_ERR_DTYPE, "unsupported element size %d", a.es);
}

// ---- validation (P:90-91 ownership, P:641-649 memory spaces, R6-R10) ----------------
desc_status check_memspace(const void *p, int dev, const char *name) {
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear sticky-free error
        return fail(DESC_ERR_MEMSPACE, "%s: cudaPointerGetAttributes failed (%s)", name,
                    cudaGetErrorName(e));
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
        return fail(DESC_ERR_MEMSPACE, "%s is not device memory (cudaMemoryType %d)", name,
                    (int)attr.type);
    if (attr.type == cudaMemoryTypeDevice && attr.device != dev)
        return fail(DESC_ERR_MEMSPACE, "%s lives on device %d, current device is %d", name,
                    attr.device, dev);
    return DESC_OK;
}

desc_status validate(const Args &a, bool *empty) {
    *empty = false;
    if (a.es == 0) return fail(DESC_ERR_DTYPE, "unknown dtype");
    if (a.batch < 0 || a.rows < 0 || a.cols < 0)
        return fail(DESC_ERR_SHAPE, "negative size (batch=%lld rows=%lld cols=%lld)",
                    (long long)a.batch, (long long)a.rows, (long long)a.cols);
    if (a.batch == 0 || a.rows == 0 || a.cols == 0) { *empty = true; return DESC_OK; }
    if (!a.in || !a.out) return fail(DESC_ERR_NULL, "null %s pointer", a.in ? "out" : "in");
    if (a.ld_in < a.cols) return fail(DESC_ERR_SHAPE, "ld_in %lld < cols %lld", (long long)a.ld_in, (long long)a.cols);
    if (a.ld_out < a.rows) return fail(DESC_ERR_SHAPE, "ld_out %lld < rows %lld", (long long)a.ld_out, (long long)a.rows);
    if (a.stride_in < 0 || a.stride_out < 0) return fail(DESC_ERR_SHAPE, "negative batch stride");
    if (a.batch > 1) {
        int64_t need;
        if (!span_elems(1, a.cols, a.rows, a.ld_out, 0, &need))
            return fail(DESC_ERR_SHAPE, "output matrix extent overflows int64");
        if (a.stride_out < need)
            return fail(DESC_ERR_SHAPE,
                        "batched outputs overlap: stride_out %lld < (cols-1)*ld_out+rows = %lld",
                        (long long)a.stride_out, (long long)need);
    }
    int64_t span_in, span_out, bin, bout;
    if (!span_elems(a.batch, a.rows, a.cols, a.ld_in, a.stride_in, &span_in) ||
        !span_elems(a.batch, a.cols, a.rows, a.ld_out, a.stride_out, &span_out) ||
        !mul_ok(span_in, a.es, &bin) || !mul_ok(span_out, a.es, &bout))
        return fail(DESC_ERR_SHAPE, "extent overflows int64");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(a.in), o0 = reinterpret_cast<uintptr_t>(a.out);
    if (i0 < o0 + (uintptr_t)bout && o0 < i0 + (uintptr_t)bin)
        return fail(DESC_ERR_ALIAS, "in [%p, +%lld) and out [%p, +%lld) overlap (&uniq, P:576-579)",
                    a.in, (long long)bin, a.out, (long long)bout);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status s = check_memspace(a.in, dev, "in")) return s;
    if (desc_status s = check_memspace(a.out, dev, "out")) return s;
    return DESC_OK;
}

desc_status run(const Args &a, desc_kernel k) {
    g_last_launches = 0;
    bool empty;
    if (desc_status s = validate(a, &empty)) return s;
    if (empty) return DESC_OK;
    const bool tma_ok = tma_eligible(a);
    if (k == DESC_KERNEL_TMA && !tma_ok)
        return fail(DESC_ERR_KERNEL, "TMA kernel needs 16-byte aligned bases, ld*size and stride*size");
    if (k == DESC_KERNEL_SMEM || (k == DESC_KERNEL_AUTO && !tma_ok)) return run_smem(a);
    if (k == DESC_KERNEL_TMA || k == DESC_KERNEL_AUTO) return run_tma(a);
    return fail(DESC_ERR_KERNEL, "unknown kernel variant %d", (int)k);
}

}  // namespace

extern "C" {

desc_status desc_transpose_ex(const void *in, void *out, int64_t batch, int64_t rows, int64_t cols,
                              int64_t ld_in, int64_t ld_out, int64_t stride_in, int64_t stride_out,
                              desc_dtype dtype, desc_kernel kernel, void *stream) {
    Args a{in, out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out, dtype_size(dtype),
           static_cast<cudaStream_t>(stream)};
    return run(a, kernel);
}

desc_status desc_transpose_batched(const void *in, void *out, int64_t batch, int64_t rows,
                                   int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                                   int64_t stride_out, desc_dtype dtype, void *stream) {
    return desc_transpose_ex(in, out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                             dtype, DESC_KERNEL_AUTO, stream);
}

desc_status desc_transpose(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                           int64_t ld_out, desc_dtype dtype, void *stream) {
    return desc_transpose_ex(in, out, 1, rows, cols, ld_in, ld_out, 0, 0, dtype,
                             DESC_KERNEL_AUTO, stream);
}

desc_kernel desc_select_kernel(const void *in, const void *out, int64_t batch, int64_t rows,
                               int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                               int64_t stride_out, desc_dtype dtype) {
    Args a{in, const_cast<void *>(out), batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
           dtype_size(dtype), nullptr};
    if (a.es == 0) return DESC_KERNEL_SMEM;
    return tma_eligible(a) ? DESC_KERNEL_TMA : DESC_KERNEL_SMEM;
}

int desc_last_launch_count(void) { return g_last_launches; }

const char *desc_status_string(desc_status s) {
    switch (s) {
        case DESC_OK: return "DESC_OK";
        case DESC_ERR_NULL: return "DESC_ERR_NULL";
        case DESC_ERR_SHAPE: return "DESC_ERR_SHAPE";
        case DESC_ERR_DTYPE: return "DESC_ERR_DTYPE";
        case DESC_ERR_ALIAS: return "DESC_ERR_ALIAS";
        case DESC_ERR_MEMSPACE: return "DESC_ERR_MEMSPACE";
        case DESC_ERR_CUDA: return "DESC_ERR_CUDA";
        case DESC_ERR_KERNEL: return "DESC_ERR_KERNEL";
    }
    return "DESC_ERR_UNKNOWN";
}

const char *desc_last_error(void) { return g_last_error.c_str(); }

size_t desc_dtype_size(desc_dtype t) { return (size_t)dtype_size(t); }

int desc_version(void) { return DESC_VERSION; }

}  // extern "C"
