// desc_transpose.cu -- the C-ABI boundary (include/desc_transpose.h): argument
// validation (ownership, memory space, shape), kernel dispatch, TMA descriptor cache.
//
// Product code.  It shares nothing with oracle/ (task rule ③).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/desc_transpose.h"
#include "smem_transpose.cuh"
#include "tiled_transpose.cuh"
#include "tma_transpose.cuh"
#include "tma_store_transpose.cuh"
#include "tma_tile_transpose.cuh"
#include "vtiled_transpose.cuh"
#include "copy_kernel.cuh"
#include "view_copy.cuh"
#include "reduce_scan.cuh"

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

// Are `batch` output matrices of `nr` rows x `nc` cols (pitch ld, batch stride) pairwise
// disjoint?  Two layouts are accepted (the narrowing rule: each batch item
// uniquely owns its part of out): stacked (stride >= (nr-1)*ld + nc) and side by side
// within each row (stride >= nc and (batch-1)*stride + nc <= ld).
bool outputs_disjoint(int64_t batch, int64_t nr, int64_t nc, int64_t ld, int64_t stride) {
    if (batch <= 1) return true;
    int64_t span;
    if (span_elems(1, nr, nc, ld, 0, &span) && stride >= span) return true;
    int64_t last;
    if (stride >= nc && !__builtin_mul_overflow(batch - 1, stride, &last) &&
        !__builtin_add_overflow(last, nc, &last) && last <= ld)
        return true;
    return false;
}

struct Args {
    const void *in;
    void *out;
    int64_t batch, rows, cols, ld_in, ld_out, stride_in, stride_out;
    int es;
    cudaStream_t stream;
    int rev_rows = 0;   // views only: `in` addresses physical row 0, logical row i = rows-1-i
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

// A 2-D (or batched 3-D) row-major matrix seen by TMA: `inner` elements per row (pitch
// ld), `outer` rows, `batch` matrices (pitch stride); box = box_inner x box_outer.
struct MapKey {
    uintptr_t ptr;
    int64_t inner, outer, batch, ld, stride;
    int es, box_inner, box_outer;
    bool operator==(const MapKey &o) const {
        return ptr == o.ptr && inner == o.inner && outer == o.outer && batch == o.batch &&
               ld == o.ld && stride == o.stride && es == o.es && box_inner == o.box_inner &&
               box_outer == o.box_outer;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey &k) const {
        size_t h = std::hash<uintptr_t>()(k.ptr);
        auto mix = [&h](int64_t v) { h ^= std::hash<int64_t>()(v) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2); };
        mix(k.inner); mix(k.outer); mix(k.batch); mix(k.ld); mix(k.stride); mix(k.es);
        mix(k.box_inner); mix(k.box_outer);
        return h;
    }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

CUtensorMapL2promotion promo() {
    static const int v = [] { const char *e = getenv("DESC_TMA_PROMO"); return e ? atoi(e) : 2; }();
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// Encode (or fetch from the cache) a 128-byte-swizzled tiled tensor map.
desc_status tensor_map(const MapKey &key, CUtensorMap *out) {
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) { *out = it->second; return DESC_OK; }
    }
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (desc_status s = get_encode(&encode)) return s;
    CUtensorMapDataType dt = key.es == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                           : key.es == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                           : key.es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                         : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const cuuint32_t rank = key.batch > 1 ? 3 : 2;
    cuuint64_t dims[3] = {(cuuint64_t)key.inner, (cuuint64_t)key.outer, (cuuint64_t)key.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(key.ld * key.es), (cuuint64_t)(key.stride * key.es)};
    cuuint32_t box[3] = {(cuuint32_t)key.box_inner, (cuuint32_t)key.box_outer, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, dt, rank, reinterpret_cast<void *>(key.ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(DESC_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 256) g_maps.clear();
    g_maps.emplace(key, m);
    *out = m;
    return DESC_OK;
}

desc_status in_map(const Args &a, int box_rows, CUtensorMap *m) {
    MapKey k{reinterpret_cast<uintptr_t>(a.in), a.cols, a.rows, a.batch, a.ld_in, a.stride_in,
             a.es, 128 / a.es, box_rows};
    return tensor_map(k, m);
}

desc_status out_map(const Args &a, int box_rows, CUtensorMap *m) {
    const int64_t rows_main = a.rows - a.rows % (16 / a.es);   // 16-byte clipping granule
    MapKey k{reinterpret_cast<uintptr_t>(a.out), rows_main, a.cols, a.batch, a.ld_out, a.stride_out,
             a.es, 128 / a.es, box_rows};
    return tensor_map(k, m);
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
    const int64_t lim40 = (int64_t)1 << 40;
    if (a.ld_in * a.es >= lim40 || a.stride_in * a.es >= lim40) return false;
    if (a.ld_out * a.es >= lim40 || a.stride_out * a.es >= lim40) return false;
    return true;
}

// Development knobs (read once; A/B measurement only).
int dev_knob(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Raster group (tile rows per group).  Default: the whole tile column (tiles walk down
// the input's columns, so the tiles in flight write whole output rows contiguously);
// measured best on 8192^2 f32 (gpurun_out/sweep_group2.txt: 90.6 us vs 92.6 us for
// near-square windows).  DESC_TMA_GROUP=g forces g (A/B only).
int tile_group(int grid, int tr, int tc, int tiles_r) {
    (void)grid; (void)tr; (void)tc;
    static const int forced = dev_knob("DESC_TMA_GROUP", 0);
    int g = forced > 0 ? forced : tiles_r;
    if (g > tiles_r) g = tiles_r;
    return g < 1 ? 1 : g;
}

// The TMA-store kernel takes 4/8-byte cells whose output rows span >= one 16-byte chunk.
bool tma_store_ok(const Args &a) { return (a.es == 4 || a.es == 8) && a.rows * a.es >= 16; }

// ---- launchers -----------------------------------------------------------------------
// Dynamic tile scheduling counters: one zeroed {next, done} pair of 64-bit words per
// (device, stream), allocated on first use (the only device memory the library owns;
// 16 bytes per stream, never freed) and self-reset by the last CTA of every launch.  Launches
// on one stream are ordered, so they can share a counter; different streams get different
// counters, so concurrent launches never share one.  Streams are told apart by
// cudaStreamGetId, not by the handle: the per-thread default stream has the same handle
// (cudaStreamPerThread) in every host thread but a distinct id per thread.  Launches being
// captured into a CUDA graph never use a counter (static schedule): a replay of the graph
// on another stream could otherwise race a live launch on the captured stream's counter.
std::mutex g_sched_mu;
std::unordered_map<uint64_t, unsigned long long *> g_sched;

desc_status sched_counter(int dev, cudaStream_t stream, unsigned long long **out) {
    unsigned long long sid = 0;
    cudaError_t ge = cudaStreamGetId(stream, &sid);
    if (ge != cudaSuccess) return cuda_fail(ge, "cudaStreamGetId");
    const uint64_t key = (uint64_t)sid * 64 + (uint64_t)dev;
    std::lock_guard<std::mutex> lk(g_sched_mu);
    auto it = g_sched.find(key);
    if (it != g_sched.end()) { *out = it->second; return DESC_OK; }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, 2 * sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc (tile counter)");
    e = cudaMemset(p, 0, 2 * sizeof(unsigned long long));   // synchronous: zero before use
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset (tile counter)");
    g_sched.emplace(key, static_cast<unsigned long long *>(p));
    *out = static_cast<unsigned long long *>(p);
    return DESC_OK;
}

// Launch with programmatic stream serialisation (PDL) so that back-to-back transposes
// overlap launch latency and prologue with the previous kernel's tail; the kernels call
// griddepcontrol.wait before touching global memory, so stream order is preserved.
// cluster launch (cluster size `cl`, grid a multiple of it) with programmatic serialisation
template <typename Kern, typename... Args_>
cudaError_t launch_cluster_pdl(Kern kern, int grid, int cl, int threads, int smem,
                               cudaStream_t stream, Args_... args) {
    static const int pdl = dev_knob("DESC_PDL", 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern, typename... Args_>
cudaError_t launch_pdl(Kern kern, int grid, int threads, int smem, cudaStream_t stream,
                       Args_... args);

// Plain launch with programmatic stream serialisation (PDL): for kernels that call
// griddepcontrol.wait before any global access (tiled transpose, row copy, view tiles,
// block reduction).  DESC_PDL=0 turns the attribute off (A/B).
template <typename Kern, typename... Args_>
cudaError_t launch_plain_pdl(Kern kern, int grid, int threads, int smem, cudaStream_t stream,
                             Args_... args);

// 2-CTA cluster launch WITHOUT programmatic serialisation (kernels that do not call
// griddepcontrol.wait, e.g. the scan, whose state is zeroed by a memset just before it).
template <typename Kern, typename... Args_>
cudaError_t launch_cluster2(Kern kern, int grid, int threads, int smem, cudaStream_t stream,
                            Args_... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((grid + 1) / 2 * 2);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern, typename... Args_>
cudaError_t launch_plain_pdl(Kern kern, int grid, int threads, int smem, cudaStream_t stream,
                             Args_... args) {
    static const int pdl = dev_knob("DESC_PDL", 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern, typename... Args_>
cudaError_t launch_pdl(Kern kern, int grid, int threads, int smem, cudaStream_t stream,
                       Args_... args) {
    static const int pdl = dev_knob("DESC_PDL", 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((grid + 1) / 2 * 2);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int n = 0;
    // an explicit cluster launch: st.async (tile ids, TMA-store kernel) is a cluster-scope
    // op, and compute-sanitizer only accepts it in clusters of >= 2 CTAs (the CTAs of a pair
    // do not talk to each other; grid is rounded up to even, a spare CTA finds no tile)
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 2;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
    if (pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Shared launch plumbing of the persistent TMA kernels: dynamic-smem opt-in (once per
// kernel instantiation), grid = min(tiles, SMs x occupancy), tile raster parameters.
template <typename Kern>
desc_status tma_prepare(Kern kern, int threads, int smem, int tr, int tile_cols, const Args &a,
                        desc::TmaParams *p, int *grid, cudaFuncAttributes *) {
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lk(mu);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    DevInfo di;
    if (desc_status s = device_info(dev, &di)) return s;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (occ < 1) occ = 1;
    p->out = a.out;
    p->ld_out = a.ld_out;
    p->stride_out = a.stride_out;
    p->rows = (int32_t)a.rows;
    p->rows_main = (int32_t)(a.rows - a.rows % (16 / a.es));
    p->cols = (int32_t)a.cols;
    p->batch = (int32_t)a.batch;
    p->tiles_r = (int32_t)((a.rows + tr - 1) / tr);
    p->tiles_c = (int32_t)((a.cols + tile_cols - 1) / tile_cols);
    p->rank3 = a.batch > 1 ? 1 : 0;
    p->ntiles = (int64_t)p->tiles_r * p->tiles_c * a.batch;
    const int64_t max_grid = (int64_t)di.sms * occ;
    *grid = (int)(p->ntiles < max_grid ? p->ntiles : max_grid);
    p->group = tile_group(*grid, tr, tile_cols, p->tiles_r);
    p->evict_first = dev_knob("DESC_TMA_EVICT", 0);
    p->sched = nullptr;
    p->rev_rows = a.rev_rows;
    return DESC_OK;
}

template <int ES, int TR, int NB, int STAGES, int CW>
desc_status launch_tma(const Args &a) {
    using C = desc::TmaConfig<ES, TR, NB, STAGES, CW>;
    auto kern = desc::transpose_tma_kernel<ES, TR, NB, STAGES, CW>;
    desc::TmaParams p;
    int grid = 0;
    if (desc_status s = tma_prepare(kern, C::THREADS, C::SMEM_BYTES, TR, C::TILE_COLS, a, &p, &grid, nullptr))
        return s;
    CUtensorMap map;
    if (desc_status s = in_map(a, TR, &map)) return s;
    cudaError_t e = launch_pdl(kern, grid, C::THREADS, C::SMEM_BYTES, a.stream, map, p);
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma_kernel launch");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

template <int ES, int TR, int NB, int STAGES, int CW, int OBUF>
desc_status launch_tma2(const Args &a) {
    using C = desc::Tma2Config<ES, TR, NB, STAGES, CW, OBUF>;
    auto kern = desc::transpose_tma2_kernel<ES, TR, NB, STAGES, CW, OBUF>;
    desc::TmaParams p;
    int grid = 0;
    if (desc_status s = tma_prepare(kern, C::THREADS, C::SMEM_BYTES, TR, C::TILE_COLS, a, &p, &grid, nullptr))
        return s;
    // dynamic scheduling pays when every CTA has many tiles (8192^2 f32: 87.3 -> 85.4 us,
    // 256 x 1024^2: 332 -> 316 us); with a few tiles per CTA the atomics' latency costs more
    // than the balance gains (2048^2 f64: 14.4 -> 16.4 us), so those stay static.
    static const int dyn = dev_knob("DESC_DYN", 1);
    static const int dyn_min = dev_knob("DESC_DYN_MIN", 16);   // tiles per CTA (tests: 1)
    if (dyn && p.ntiles >= (int64_t)dyn_min * grid) {
        int dev = 0;
        cudaGetDevice(&dev);
        // under graph capture: static scheduling (see sched_counter)
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(a.stream, &cap);
        if (cap == cudaStreamCaptureStatusNone)
            if (desc_status s = sched_counter(dev, a.stream, &p.sched)) return s;
    }
    CUtensorMap min, mout;
    if (desc_status s = in_map(a, TR, &min)) return s;
    if (desc_status s = out_map(a, C::TILE_COLS, &mout)) return s;
    cudaError_t e = launch_pdl(kern, grid, C::THREADS, C::SMEM_BYTES, a.stream, min, mout, p);
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma2_kernel launch");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma2_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

// One tile per CTA, hardware-scheduled 1-D grid (tma_tile_transpose.cuh).  Tile order:
// DESC_TMA_TILE_GROUP tile rows per raster group (default 1 = row-major over the tile grid,
// like TILED; 0 = whole tile columns).
template <int ES, int TR, int NB, int CW = 4, int TPC = 1>
desc_status launch_tma_tile(const Args &a) {
    using C = desc::TmaTileConfig<ES, TR, NB, CW, TPC>;
    auto kern = desc::transpose_tma_tile_kernel<ES, TR, NB, CW, TPC>;
    {
        static std::mutex mu;
        static bool opted[64] = {};
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 64 || !opted[dev]) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tma_tile smem)");
            if (dev < 64) opted[dev] = true;
        }
    }
    desc::TmaParams p;
    p.out = a.out;
    p.ld_out = a.ld_out;
    p.stride_out = a.stride_out;
    p.rows = (int32_t)a.rows;
    p.rows_main = (int32_t)(a.rows - a.rows % (16 / a.es));
    p.cols = (int32_t)a.cols;
    p.batch = (int32_t)a.batch;
    p.tiles_r = (int32_t)((a.rows + TR - 1) / TR);
    p.tiles_c = (int32_t)((a.cols + C::TILE_COLS - 1) / C::TILE_COLS);
    p.rank3 = a.batch > 1 ? 1 : 0;
    p.ntiles = (int64_t)p.tiles_r * p.tiles_c * a.batch;
    static const int grp = dev_knob("DESC_TMA_TILE_GROUP", 1);
    p.group = grp <= 0 || grp > p.tiles_r ? p.tiles_r : grp;
    // L2 policy of the loads: normal (evict_first costs 2-3%: with the tensor map's 256-byte
    // L2 promotion a box row's fetch also brings the next box's row, which evict_first can
    // drop before it is read; profiles/r02_tma_tile_sweep.txt)
    static const int evict = dev_knob("DESC_TMA_TILE_EVICT", 0);
    p.evict_first = evict;
    p.sched = nullptr;
    p.rev_rows = 0;
    if (p.ntiles > INT32_MAX) return fail(DESC_ERR_SHAPE, "too many tiles for one launch");
    // extra dynamic shared memory per CTA caps the resident CTAs per SM: 16 KB tiles + 20000
    // bytes -> 6 CTAs/SM (96 KB of loads in flight) measured best; 8 (register-limited) and
    // more lose 1-2%, 12 loses 15% (profiles/r02_tma_tile_sweep.txt)
    static const int pad = dev_knob("DESC_TMA_TILE_SMEM_PAD", TPC == 1 && CW == 4 ? 20000 : 0);
    const int smem = C::SMEM_BYTES + pad;
    if (pad) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tma_tile smem pad)");
    }
    CUtensorMap min, mout;
    if (desc_status s = in_map(a, TR, &min)) return s;
    if (desc_status s = out_map(a, C::TILE_COLS, &mout)) return s;
    cudaError_t e = launch_plain_pdl(kern, (int)((p.ntiles + TPC - 1) / TPC), C::THREADS, smem,
                                     a.stream, min, mout, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tma_tile_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

desc_status run_tma_tile(const Args &a) {
    static const int cfg = dev_knob("DESC_TMA_TILE_CFG", 0);   // A/B of tile shapes
    switch (a.es) {
        case 4:
            switch (cfg) {
                case 1: return launch_tma_tile<4, 128, 2>(a);   // 128 x 64, 32 KB
                case 2: return launch_tma_tile<4, 64, 4>(a);    // 64 x 128, 32 KB
                case 3: return launch_tma_tile<4, 32, 4>(a);    // 32 x 128, 16 KB
                case 4: return launch_tma_tile<4, 64, 2, 8>(a);  // 8 warps
                case 5: return launch_tma_tile<4, 64, 2, 4, 2>(a);  // 2 tiles per CTA
                case 6: return launch_tma_tile<4, 64, 2, 8, 2>(a);
                case 7: return launch_tma_tile<4, 32, 4, 4, 2>(a);
                default: return launch_tma_tile<4, 64, 2>(a);   // 64 x 64 cells, 16 KB
            }
        case 8:
            switch (cfg) {
                case 1: return launch_tma_tile<8, 64, 4>(a);    // 64 x 64, 32 KB
                case 2: return launch_tma_tile<8, 32, 8>(a);    // 32 x 128, 32 KB
                case 3: return launch_tma_tile<8, 64, 2>(a);    // 64 x 32, 16 KB
                case 4: return launch_tma_tile<8, 32, 4, 8>(a);
                case 5: return launch_tma_tile<8, 32, 4, 4, 2>(a);
                case 6: return launch_tma_tile<8, 32, 4, 8, 2>(a);
                case 7: return launch_tma_tile<8, 64, 2, 4, 2>(a);
                default: return launch_tma_tile<8, 32, 4>(a);   // 32 x 64 cells, 16 KB
            }
    }
    return fail(DESC_ERR_KERNEL, "TMA tile kernel supports 4- and 8-byte elements only");
}

// 16-byte-vector tile kernel (vtiled_transpose.cuh): 4/8-byte cells, the TMA alignment rules
// (16-byte bases, ld*size and stride*size multiples of 16) and rows, cols multiples of the
// cells per 16-byte chunk, so edge tiles hold whole chunks and micro-blocks.
bool vtiled_ok(const Args &a) {
    if (a.rev_rows || !tma_eligible(a)) return false;
    const int64_t vec = 16 / a.es;
    return a.rows % vec == 0 && a.cols % vec == 0;
}

// AUTO's kernel for 1/2-byte cells whenever the vector tile kernel's rules hold: its 16 x 16 /
// 8 x 8 byte-permute micro-transposes beat the persistent TMA-load kernel on every measured
// shape (profiles/r02_vtiled_narrow.txt, back to back: 8192^2 u8 0.726 -> 0.933, 16384^2 u8
// 0.690 -> 0.973, 8192^2 bf16 0.761 -> 0.995, 4096^2 bf16 0.613 -> 0.956, 256 x 1024^2 bf16
// 0.960 -> 1.049); 4/8-byte cells keep TILED (tiled_preferred).
bool narrow_vtiled(const Args &a) { return (a.es == 1 || a.es == 2) && vtiled_ok(a); }

template <int ES, int TCH, int NT>
desc_status launch_vtiled(const Args &a) {
    using C = desc::VTiledCfg<ES, TCH, NT>;
    auto kern = desc::transpose_vtiled_kernel<ES, TCH, NT>;
    const int64_t tiles_r = (a.rows + C::TR - 1) / C::TR, tiles_c = (a.cols + C::TC - 1) / C::TC;
    const int64_t ntiles = tiles_r * tiles_c * a.batch;
    const int64_t max_grid = (int64_t)1 << 30;
    const int grid = (int)(ntiles < max_grid ? ntiles : max_grid);
    static_assert(C::SMEM <= 48 * 1024, "vtiled tile fits the default shared-memory window");
    cudaError_t e = launch_plain_pdl(kern, grid, NT, C::SMEM, a.stream,
                                     static_cast<const char *>(a.in), static_cast<char *>(a.out),
                                     a.rows, a.cols, a.ld_in, a.ld_out, a.stride_in, a.stride_out,
                                     tiles_r, tiles_c, ntiles);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_vtiled_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

desc_status run_vtiled(const Args &a) {
    // Tile shapes swept on B200 (profiles/r02_vtiled_ab.txt, back to back, frac of the copy
    // peak): 4-byte cells 64 x 64 with 128 threads (8 copies in flight each; 8192^2 1.023-1.025,
    // 256 threads 0.982), 8-byte cells 32 x 32 with 64 threads (8 copies each; 3000x5000
    // 0.996-0.998, 8192^2 1.033).  DESC_VTILED_CFG=<n> for A/B.
    static const int cfg = dev_knob("DESC_VTILED_CFG", 0);
    switch (a.es) {
        case 4:
            switch (cfg) {
                case 1: return launch_vtiled<4, 16, 256>(a);    // 64 x 64, 4 copies / thread
                case 2: return launch_vtiled<4, 32, 256>(a);    // 64 x 128, 32 KB
                case 3: return launch_vtiled<4, 8, 128>(a);     // 64 x 32, 8 KB
                case 4: return launch_vtiled<4, 16, 64>(a);     // 64 x 64, 16 copies / thread
                case 5: return launch_vtiled<4, 32, 128>(a);    // 64 x 128, 16 copies / thread
                case 6: return launch_vtiled<4, 8, 64>(a);      // 64 x 32, 8 copies / thread
                default: return launch_vtiled<4, 16, 128>(a);   // 64 x 64 cells, 16 KB
            }
        case 8:
            switch (cfg) {
                case 1: return launch_vtiled<8, 16, 256>(a);    // 32 x 32, 2 copies / thread
                case 2: return launch_vtiled<8, 32, 256>(a);    // 32 x 64, 16 KB
                case 3: return launch_vtiled<8, 8, 128>(a);     // 32 x 16, 4 KB
                case 4: return launch_vtiled<8, 16, 128>(a);    // 32 x 32, 4 copies / thread
                case 5: return launch_vtiled<8, 32, 128>(a);    // 32 x 64, 8 copies / thread
                case 6: return launch_vtiled<8, 32, 64>(a);     // 32 x 64, 16 copies / thread
                default: return launch_vtiled<8, 16, 64>(a);    // 32 x 32 cells, 8 KB
            }
        case 2:
            switch (cfg) {
                case 1: return launch_vtiled<2, 16, 256>(a);    // 128 x 128, 8 copies / thread
                case 2: return launch_vtiled<2, 8, 64>(a);      // 128 x 64, 16 copies / thread
                default: return launch_vtiled<2, 8, 128>(a);    // 128 x 64 cells, 16 KB
            }
        case 1:
            switch (cfg) {
                case 1: return launch_vtiled<1, 8, 64>(a);      // 256 x 128, 32 copies / thread
                default: return launch_vtiled<1, 8, 128>(a);    // 256 x 128 cells, 32 KB
            }
    }
    return fail(DESC_ERR_DTYPE, "unsupported element size %d", a.es);
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

template <typename Cell, int TR = 0, int TC = 0, int NT = 256, bool SCATTER = false>
desc_status launch_tiled(const Args &a, const desc::TiledScatter *scatter = nullptr) {
    using C = desc::TiledCfg<Cell, TR, TC, NT>;
    auto kern = desc::transpose_tiled_kernel<Cell, TR, TC, NT, SCATTER>;
    desc::TiledScatter sc;
    memset(&sc, 0, sizeof sc);
    if (scatter) sc = *scatter;
    const int64_t tiles_r = (a.rows + C::TR - 1) / C::TR, tiles_c = (a.cols + C::TC - 1) / C::TC;
    const int64_t ntiles = tiles_r * tiles_c * a.batch;
    // one tile per CTA up to 2^30 tiles (DESC_TILED_TPC=<k>: k tiles per CTA, A/B)
    static const int tpc = dev_knob("DESC_TILED_TPC", 1);
    const int64_t want = tpc > 1 ? (ntiles + tpc - 1) / tpc : ntiles;
    const int64_t max_grid = (int64_t)1 << 30;
    const int grid = (int)(want < max_grid ? want : max_grid);
    if (C::SMEM > 48 * 1024) {
        static std::mutex mu;                              // per device, once
        static bool opted[64] = {};
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 64 || !opted[dev]) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tiled smem)");
            if (dev < 64) opted[dev] = true;
        }
    }
    // L2 prefetch of each CTA's tile before griddepcontrol.wait (tiled_transpose.cuh).  Every
    // CTA prefetches (mode 2, default): same box, back to back (profiles/r02_tiled_prefetch.txt)
    // 8192^2 f32 1.000 -> 1.023, 4096^2 f32 0.933 -> 0.999, 2048^2 f64 0.870 -> 0.980,
    // 3000x5000 f64 0.957 -> 0.997 of the copy peak; only the first wave (mode 1, the CTAs that
    // can be resident while the previous grid runs) recovers the launch ramp but not the
    // extra loads in flight of the later CTAs.  DESC_TILED_PF=0/1/2 for A/B.
    static int64_t pf_slots[64] = {};
    static const int pf_mode = dev_knob("DESC_TILED_PF", 2);   // 0 off, 1 first wave, 2 all
    int64_t pf_ctas = 0;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && pf_slots[dev] == 0) {
            DevInfo di;
            if (desc_status st = device_info(dev, &di)) return st;
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, C::SMEM) != cudaSuccess) {
                cudaGetLastError();
                occ = 1;
            }
            pf_slots[dev] = (int64_t)di.sms * (occ > 0 ? occ : 1);
        }
        pf_ctas = pf_mode == 0 ? 0 : pf_mode == 2 ? ((int64_t)1 << 62) : (dev < 64 ? pf_slots[dev] : 0);
    }
    cudaError_t e = launch_plain_pdl(kern, grid, NT, C::SMEM, a.stream,
                                     static_cast<const Cell *>(a.in), static_cast<Cell *>(a.out),
                                     a.rows, a.cols, a.ld_in, a.ld_out, a.stride_in, a.stride_out,
                                     tiles_r, tiles_c, ntiles, pf_ctas, sc);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "transpose_tiled_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

// Development knob: DESC_TMA_CFG=<n> selects a tile/pipeline configuration for A/B
// measurement (read once).  The default (0) is the tuned configuration.
int tma_cfg() {
    static int cfg = [] {
        const char *e = getenv("DESC_TMA_CFG");
        return e ? atoi(e) : 0;
    }();
    return cfg;
}

desc_status run_tma(const Args &a) {
    const int cfg = tma_cfg();
    switch (a.es) {
        case 4:
            switch (cfg) {
                case 1: return launch_tma<4, 64, 2, 4, 8>(a);
                case 2: return launch_tma<4, 128, 2, 3, 8>(a);
                case 3: return launch_tma<4, 256, 1, 3, 8>(a);
                case 4: return launch_tma<4, 32, 4, 6, 8>(a);
                case 5: return launch_tma<4, 128, 1, 8, 8>(a);
                case 6: return launch_tma<4, 64, 1, 8, 4>(a);
                case 7: return launch_tma<4, 64, 4, 3, 8>(a);
                case 8: return launch_tma<4, 128, 1, 4, 4>(a);
                default: return launch_tma<4, 128, 1, 4, 8>(a);
            }
        case 8:
            switch (cfg) {
                case 1: return launch_tma<8, 64, 2, 4, 8>(a);
                case 2: return launch_tma<8, 128, 2, 3, 16>(a);
                case 3: return launch_tma<8, 256, 1, 3, 16>(a);
                case 4: return launch_tma<8, 32, 4, 6, 8>(a);
                case 5: return launch_tma<8, 128, 1, 8, 16>(a);
                case 6: return launch_tma<8, 64, 1, 8, 4>(a);
                case 7: return launch_tma<8, 64, 4, 3, 16>(a);
                case 8: return launch_tma<8, 128, 1, 4, 8>(a);
                default: return launch_tma<8, 128, 1, 4, 16>(a);
            }
        case 2: return launch_tma<2, 128, 1, 4, 4>(a);
        case 1: return launch_tma<1, 128, 1, 4, 2>(a);
    }
    return fail(DESC_ERR_DTYPE, "unsupported element size %d", a.es);
}

desc_status run_tma2(const Args &a) {
    int cfg = tma_cfg();
    // Small problems (< 64 MB per call): smaller tiles for more CTAs per SM and a
    // finer tail (gpurun_out/sweep_small_tma_st.txt: 2048^2 f64 16.4 -> 14.4 us).
    const bool small = a.batch * a.rows * a.cols * a.es < ((int64_t)64 << 20);
    if (cfg == 0 && small) cfg = 11;
    switch (a.es) {
        case 4:
            switch (cfg) {
                case 1: return launch_tma2<4, 64, 2, 4, 8, 2>(a);
                case 2: return launch_tma2<4, 128, 1, 3, 8, 3>(a);
                case 3: return launch_tma2<4, 128, 1, 4, 4, 2>(a);
                case 4: return launch_tma2<4, 64, 1, 6, 4, 3>(a);
                case 5: return launch_tma2<4, 256, 1, 2, 8, 2>(a);
                case 6: return launch_tma2<4, 256, 1, 3, 8, 2>(a);
                case 7: return launch_tma2<4, 256, 1, 2, 16, 2>(a);
                case 8: return launch_tma2<4, 256, 1, 4, 8, 2>(a);
                case 9: return launch_tma2<4, 128, 2, 2, 8, 2>(a);
                case 10: return launch_tma2<4, 256, 1, 2, 4, 2>(a);
                case 11: return launch_tma2<4, 64, 2, 2, 8, 2>(a);
                case 13: return launch_tma2<4, 128, 1, 2, 8, 2>(a);
                case 12: return launch_tma2<4, 128, 1, 4, 8, 2>(a);
                // tuned (gpurun_out sweeps, profiles/): 128 x 64 tile, 2-stage ring,
                // 2 output buffers, 8 consumer warps, 1 CTA (288 threads, 129 KB) per SM
                default: return launch_tma2<4, 128, 2, 2, 8, 2>(a);
            }
        case 8:
            switch (cfg) {
                case 1: return launch_tma2<8, 64, 2, 4, 8, 2>(a);
                case 2: return launch_tma2<8, 128, 1, 3, 16, 3>(a);
                case 3: return launch_tma2<8, 128, 1, 4, 8, 2>(a);
                case 4: return launch_tma2<8, 64, 1, 6, 8, 3>(a);
                case 5: return launch_tma2<8, 128, 2, 2, 16, 2>(a);
                case 6: return launch_tma2<8, 256, 1, 2, 16, 2>(a);
                case 7: return launch_tma2<8, 256, 1, 3, 16, 2>(a);
                case 8: return launch_tma2<8, 128, 1, 2, 16, 2>(a);
                case 9: return launch_tma2<8, 256, 1, 2, 8, 2>(a);
                case 10: return launch_tma2<8, 128, 2, 3, 16, 2>(a);
                case 11: return launch_tma2<8, 64, 2, 2, 8, 2>(a);
                case 12: return launch_tma2<8, 128, 1, 4, 16, 2>(a);
                // tuned: 128 x 16 tile, 2-stage ring, 2 output buffers, 16 consumer warps
                default: return launch_tma2<8, 128, 1, 2, 16, 2>(a);
            }
    }
    return fail(DESC_ERR_KERNEL, "TMA-store kernel supports 4- and 8-byte elements only");
}

desc_status run_tiled(const Args &a) {
    static const int cfg = dev_knob("DESC_TILED_CFG", 0);     // A/B of tile shapes
    switch (a.es) {
        case 4:
            switch (cfg) {
                case 1: return launch_tiled<uint32_t, 32, 64, 128>(a);
                case 2: return launch_tiled<uint32_t, 32, 128, 256>(a);
                case 3: return launch_tiled<uint32_t, 16, 128, 128>(a);
                case 4: return launch_tiled<uint32_t, 32, 32, 128>(a);
                case 5: return launch_tiled<uint32_t, 64, 32, 128>(a);
                case 6: return launch_tiled<uint32_t, 64, 128, 256>(a);
                default: return launch_tiled<uint32_t>(a);
            }
        case 8:
            // 32 x 32 cells, 128 threads (8 loads of 8 bytes in flight per thread, up to 16
            // CTAs/SM): 2048^2 0.836 -> 0.852, 3000x5000 0.943 -> 0.958 of peak, 4096^2 and
            // 8192^2 unchanged, against 32 x 64 cells with 256 threads
            // (profiles/r02_tiled_shapes.txt)
            switch (cfg) {
                case 1: return launch_tiled<unsigned long long, 16, 64, 128>(a);
                case 2: return launch_tiled<unsigned long long, 16, 128, 256>(a);
                case 3: return launch_tiled<unsigned long long, 32, 64, 256>(a);
                case 4: return launch_tiled<unsigned long long, 64, 32, 128>(a);
                case 5: return launch_tiled<unsigned long long, 32, 64, 128>(a);
                case 6: return launch_tiled<unsigned long long, 64, 64, 256>(a);
                default: return launch_tiled<unsigned long long, 32, 32, 128>(a);
            }
        case 2: return launch_tiled<uint16_t>(a);
        case 1: return launch_tiled<uint8_t>(a);
        default: return fail(DESC_ERR_DTYPE, "unsupported element size %d", a.es);
    }
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
    if (attr.type == cudaMemoryTypeDevice && attr.device != dev) {
        // peer memory (e.g. an IPC-mapped slab of another rank, dist.py): allowed when the
        // current device can access the owning device over NVLink / PCIe
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, dev, attr.device) != cudaSuccess || !can) {
            cudaGetLastError();
            return fail(DESC_ERR_MEMSPACE, "%s lives on device %d, not accessible from device %d",
                        name, attr.device, dev);
        }
    }
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
    if (!outputs_disjoint(a.batch, a.cols, a.rows, a.ld_out, a.stride_out)) {
        int64_t need = 0;
        span_elems(1, a.cols, a.rows, a.ld_out, 0, &need);
        return fail(DESC_ERR_SHAPE,
                        "batched outputs overlap: stride_out %lld is neither >= (cols-1)*ld_out+rows"
                    " = %lld nor a side-by-side layout within ld_out",
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

// AUTO's choice for 4/8-byte cells (scripts/exp_auto.py, profiles/r01_exp_auto.txt): the
// TILED kernel reaches the copy ceiling on every 2-D shape whose sides both hold a whole
// 64-cell tile; TMA keeps the skinny shapes (a side < 64 wastes most of a TILED tile) and
// 1/2-byte cells (TILED's cell-wide accesses move only 32/64 bytes per warp instruction).
bool tiled_preferred(const Args &a) {
    return (a.es == 4 || a.es == 8) && a.rows >= 64 && a.cols >= 64;
}

desc_status dispatch(const Args &a, desc_kernel k) {
    const bool tma_ok = tma_eligible(a);
    if (a.rev_rows) {   // rows read mirrored: TILED (negative pitch) or the TMA-store kernel
        if (k == DESC_KERNEL_TILED || (k == DESC_KERNEL_AUTO && tiled_preferred(a))) {
            Args b = a;     // logical row 0 is the last physical row; walk rows backwards
            b.in = static_cast<const char *>(a.in) + (a.rows - 1) * a.ld_in * a.es;
            b.ld_in = -a.ld_in;
            b.rev_rows = 0;
            return run_tiled(b);
        }
        if (!tma_ok || !tma_store_ok(a) || (k != DESC_KERNEL_AUTO && k != DESC_KERNEL_TMA_ST))
            return fail(DESC_ERR_KERNEL, "reversed rows need the TILED or TMA-store kernel");
        return run_tma2(a);
    }
    if (k == DESC_KERNEL_TMA && !tma_ok)
        return fail(DESC_ERR_KERNEL, "TMA kernel needs 16-byte aligned bases, ld*size and stride*size");
    if (k == DESC_KERNEL_TMA_ST && !tma_ok)
        return fail(DESC_ERR_KERNEL, "TMA kernels need 16-byte aligned bases, ld*size and stride*size");
    if (k == DESC_KERNEL_TMA_ST && !tma_store_ok(a))
        return fail(DESC_ERR_KERNEL, "TMA-store kernel needs 4/8-byte elements and rows*size >= 16");
    if (k == DESC_KERNEL_TMA_ST) return run_tma2(a);
    if (k == DESC_KERNEL_TMA_TILE) {
        if (!tma_ok) return fail(DESC_ERR_KERNEL, "TMA tile kernel needs 16-byte aligned bases, ld*size and stride*size");
        if (!tma_store_ok(a)) return fail(DESC_ERR_KERNEL, "TMA tile kernel needs 4/8-byte elements and rows*size >= 16");
        return run_tma_tile(a);
    }
    if (k == DESC_KERNEL_VTILED) {
        if (!vtiled_ok(a))
            return fail(DESC_ERR_KERNEL, "vector tile kernel needs 16-byte aligned bases, ld*size "
                        "and stride*size, and rows, cols multiples of 16/size");
        return run_vtiled(a);
    }
    if (k == DESC_KERNEL_SMEM) return run_smem(a);
    if (k == DESC_KERNEL_TILED || (k == DESC_KERNEL_AUTO && (!tma_ok || tiled_preferred(a))))
        return run_tiled(a);
    if (k == DESC_KERNEL_AUTO && narrow_vtiled(a)) return run_vtiled(a);
    if (k == DESC_KERNEL_AUTO && tma_store_ok(a)) return run_tma2(a);
    if (k == DESC_KERNEL_TMA || k == DESC_KERNEL_AUTO) return run_tma(a);
    return fail(DESC_ERR_KERNEL, "unknown kernel variant %d", (int)k);
}

// Test-teeth variant (-DDESC_MUTANTS, mutants.cuh): DESC_MUTANT=<id> selects one defect; the
// id is copied to the device once per device.  The product build has no such state.
#ifdef DESC_MUTANTS
int host_mutant() {
    static const int id = [] { const char *e = getenv("DESC_MUTANT"); return e ? atoi(e) : 0; }();
    static bool synced[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev < 64 && !synced[dev]) {
        cudaMemcpyToSymbol(desc::g_desc_mutant, &id, sizeof id);
        synced[dev] = true;
    }
    return id;
}
#else
constexpr int host_mutant() { return 0; }
#endif

desc_status run(const Args &a, desc_kernel k) {
    g_last_launches = 0;
    bool empty;
    if (desc_status s = validate(a, &empty)) return s;
    if (empty) return DESC_OK;
    if (host_mutant() == desc::MUT_SWAP_LD) {
        Args b = a;
        b.ld_in = a.ld_out;
        b.ld_out = a.ld_in;
        return dispatch(b, k);
    }
    return dispatch(a, k);
}

// ---- host-buffer pipeline (desc_transpose_host) ---------------------------------------
// Two internal streams per device alternate over row bands of the input so that the H2D
// copy of band k+1, the transpose of band k and the D2H copy of band k-1 overlap (PCIe is
// full duplex).  The caller's stream is joined at entry and exit with events, so the call
// stays asynchronous and ordered on `stream`.
constexpr int kHostStreams = 3;          // internal streams (2 or 3 used, DESC_HOST_STREAMS)
struct HostPipe {
    bool init = false;
    cudaStream_t s[kHostStreams];
    cudaEvent_t enter, done[kHostStreams];
    // Held for a whole call's enqueue: the join events are shared, and an event wait
    // snapshots the most recent record, so record -> wait must not interleave with another
    // host thread's call on the same device (the internal streams themselves may be shared:
    // each call's work is stream-ordered after its own entry join).
    std::mutex enqueue;
};
std::mutex g_pipe_mu;
HostPipe g_pipe[64];

desc_status host_pipe(int dev, HostPipe **out) {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    HostPipe &hp = g_pipe[dev];
    if (!hp.init) {
        cudaError_t e;
        for (int i = 0; i < kHostStreams; ++i) {
            if ((e = cudaStreamCreateWithFlags(&hp.s[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(e, "cudaStreamCreateWithFlags");
            if ((e = cudaEventCreateWithFlags(&hp.done[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cudaEventCreateWithFlags");
        }
        if ((e = cudaEventCreateWithFlags(&hp.enter, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "cudaEventCreateWithFlags");
        hp.init = true;
    }
    *out = &hp;
    return DESC_OK;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Device bytes one band of `band_rows` input rows needs (input band + output band, both
// with 16-byte padded pitches so the TMA kernels apply), double-buffered.
int64_t band_bytes(int64_t band_rows, int64_t cols, int es) {
    const int64_t v = 16 / es;
    const int64_t in_b = round_up(band_rows * round_up(cols, v) * es, 256);
    const int64_t out_b = round_up(cols * round_up(band_rows, v) * es, 256);
    return 2 * (in_b + out_b);
}

desc_status check_host_ptr(const void *p, const char *name) {
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return DESC_OK;   // unknown to CUDA: plain pageable host memory
    }
    if (attr.type == cudaMemoryTypeDevice)
        return fail(DESC_ERR_MEMSPACE, "%s is device memory; desc_transpose_host takes host buffers", name);
    return DESC_OK;
}

// Page-locked host memory mapped into the device address space: its device pointer.
bool mapped_host(const void *p, void **dptr) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (attr.type != cudaMemoryTypeHost || attr.devicePointer == nullptr) return false;
    *dptr = attr.devicePointer;
    return true;
}

desc_status run_host(const void *h_in, void *h_out, int64_t batch, int64_t rows, int64_t cols,
                     int64_t ld_in, int64_t ld_out, int64_t stride_in, int64_t stride_out, int es,
                     void *d_work, size_t work_bytes, cudaStream_t stream) {
    g_last_launches = 0;
    if (es == 0) return fail(DESC_ERR_DTYPE, "unknown dtype");
    if (batch < 0 || rows < 0 || cols < 0) return fail(DESC_ERR_SHAPE, "negative size");
    if (batch == 0 || rows == 0 || cols == 0) return DESC_OK;
    if (!h_in || !h_out || !d_work) return fail(DESC_ERR_NULL, "null pointer");
    if (ld_in < cols || ld_out < rows) return fail(DESC_ERR_SHAPE, "ld smaller than the row extent");
    if (stride_in < 0 || stride_out < 0) return fail(DESC_ERR_SHAPE, "negative batch stride");
    if (!outputs_disjoint(batch, cols, rows, ld_out, stride_out))
        return fail(DESC_ERR_SHAPE, "batched outputs overlap");
    int64_t span_in, span_out, bin, bout;
    if (!span_elems(batch, rows, cols, ld_in, stride_in, &span_in) ||
        !span_elems(batch, cols, rows, ld_out, stride_out, &span_out) ||
        !mul_ok(span_in, es, &bin) || !mul_ok(span_out, es, &bout))
        return fail(DESC_ERR_SHAPE, "extent overflows int64");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(h_in), o0 = reinterpret_cast<uintptr_t>(h_out);
    if (i0 < o0 + (uintptr_t)bout && o0 < i0 + (uintptr_t)bin)
        return fail(DESC_ERR_ALIAS, "host in and out overlap (&uniq, P:576-579)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status s = check_host_ptr(h_in, "h_in")) return s;
    if (desc_status s = check_host_ptr(h_out, "h_out")) return s;
    if (desc_status s = check_memspace(d_work, dev, "d_work")) return s;
    if ((reinterpret_cast<uintptr_t>(d_work) & 255) != 0)
        return fail(DESC_ERR_SHAPE, "d_work must be 256-byte aligned");

    // Band axis.  Input-row bands make every H2D copy contiguous and every D2H copy 2-D
    // (cols rows of band*size bytes); bands of input COLUMNS (= output rows) make the H2D
    // 2-D and the D2H contiguous.  PCIe Gen5 on B200 reads strided host rows faster than it
    // writes them (scripts/exp_pcie2d.py, profiles/r02_exp_pcie2d.txt, both directions
    // concurrent, 8192^2 f32: 2-KB strided rows 86.2 vs 81.1 GB/s, 4-KB 89.6 vs 86.1), so
    // AUTO bands by columns.  DESC_HOST_AXIS=1 forces row bands, =2 column bands (A/B).
    static const int host_axis = dev_knob("DESC_HOST_AXIS", 0);
    const bool by_cols = host_axis != 1;
    const int64_t span = by_cols ? cols : rows, other = by_cols ? rows : cols;
    // largest band (multiple of 128 when possible) whose double buffers fit d_work, but
    // at most span / DESC_HOST_BANDS (default 8, rounded up to 128): with fewer, larger
    // bands the one-way fill (first H2D) and drain (last D2H) dominate small matrices
    static const int min_bands = dev_knob("DESC_HOST_BANDS", 8);
    // NBUF band buffers on as many internal streams: 2 (double buffering), or 3 with
    // DESC_HOST_STREAMS=3 (A/B; the H2D of band k+2 then never waits for the D2H of band k)
    static const int nbuf_knob = dev_knob("DESC_HOST_STREAMS", 2);
    const int NBUF = nbuf_knob == 3 ? 3 : 2;
    auto fits = [&](int64_t b) { return band_bytes(b, other, es) / 2 * NBUF <= (int64_t)work_bytes; };
    int64_t band = span;
    if (min_bands > 1) {
        const int64_t cap = round_up((span + min_bands - 1) / min_bands, 128);
        if (cap < band) band = cap;
    }
    while (band > 1 && !fits(band))
        band = band > 256 ? (band / 2 + 127) / 128 * 128 : band / 2;
    if (!fits(band))
        return fail(DESC_ERR_SHAPE, "d_work (%zu bytes) too small: need >= %lld", work_bytes,
                    (long long)(band_bytes(1, other, es) / 2 * NBUF));

    // Batch bands: matrices back to back on both sides (stride_in = rows * ld_in; a tight
    // output, ld_out = rows and stride_out = cols * rows, so that no output padding byte is
    // ever written, R8) travel whole -- each band is nb consecutive matrices: ONE contiguous
    // H2D copy, one batched transpose, ONE contiguous D2H copy, no strided rows on either side
    // of PCIe (256 x 1024^2 f32: zero-copy 76.7 GB/s -> see profiles/r02_exp_e2e_batch.txt).
    // At least 8 bands when the batch allows.  DESC_HOST_BATCH=0 turns it off (A/B).
    static const int batch_bands = dev_knob("DESC_HOST_BATCH", 1);
    static const int host_mode = dev_knob("DESC_HOST_MODE", 0);
    if (batch_bands && batch > 1 && host_mode != 2 && stride_in == rows * ld_in &&
        ld_out == rows && stride_out == cols * rows) {
        const int64_t in_m = rows * ld_in * es, out_m = cols * rows * es;   // bytes per matrix
        int64_t nb = (int64_t)work_bytes / (2 * (round_up(in_m, 256) + round_up(out_m, 256)));
        const int64_t cap = (batch + 7) / 8;
        if (nb > cap) nb = cap;
        if (nb >= 1) {
            HostPipe *hp;
            if (desc_status s = host_pipe(dev, &hp)) return s;
            std::lock_guard<std::mutex> lk(hp->enqueue);
            char *w = static_cast<char *>(d_work);
            const int64_t in_b = round_up(nb * in_m, 256), out_b = round_up(nb * out_m, 256);
            char *d_in[2] = {w, w + in_b};
            char *d_out[2] = {w + 2 * in_b, w + 2 * in_b + out_b};
            if ((e = cudaEventRecord(hp->enter, stream)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
            for (int i = 0; i < 2; ++i)
                if ((e = cudaStreamWaitEvent(hp->s[i], hp->enter, 0)) != cudaSuccess)
                    return cuda_fail(e, "cudaStreamWaitEvent");
            int launches = 0;
            int64_t k = 0;
            for (int64_t b0 = 0; b0 < batch; b0 += nb, ++k) {
                const int64_t m = batch - b0 < nb ? batch - b0 : nb;
                const int buf = (int)(k & 1);
                cudaStream_t s = hp->s[buf];
                // the last matrix's last row ends at cols (its pitch padding may lie outside
                // the caller's buffer)
                const int64_t nin = m * in_m - (ld_in - cols) * es;
                e = cudaMemcpyAsync(d_in[buf], static_cast<const char *>(h_in) + b0 * in_m, nin,
                                    cudaMemcpyHostToDevice, s);
                if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
                Args a{d_in[buf], d_out[buf], m, rows, cols, ld_in, rows, rows * ld_in, cols * rows,
                       es, s};
                if (desc_status st = dispatch(a, DESC_KERNEL_AUTO)) return st;
                ++launches;
                e = cudaMemcpyAsync(static_cast<char *>(h_out) + b0 * out_m, d_out[buf], m * out_m,
                                    cudaMemcpyDeviceToHost, s);
                if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
            }
            for (int i = 0; i < 2; ++i) {
                if ((e = cudaEventRecord(hp->done[i], hp->s[i])) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
                if ((e = cudaStreamWaitEvent(stream, hp->done[i], 0)) != cudaSuccess)
                    return cuda_fail(e, "cudaStreamWaitEvent");
            }
            g_last_launches = launches;
            return DESC_OK;
        }
    }

    // Zero-copy mode: when both host buffers are page-locked and mapped, the TILED kernel
    // reads the input and writes the transposed output straight over PCIe in one pass.
    // SM loads / stores reach 51 / 53 GB/s per direction and 80 GB/s both ways at once
    // against the copy engines' 56 / 57 / 99.5 (scripts/exp_zerocopy.cu,
    // profiles/r01_exp_zerocopy.txt), so AUTO keeps the banded copy pipeline unless it
    // would be cut into many small copies (> 64 bands, e.g. 256 x 1024^2: 62 GB/s banded vs
    // 75 GB/s zero-copy).  DESC_HOST_MODE=1 forces bands, =2 forces zero-copy (A/B).
    const int64_t nbands = batch * ((span + band - 1) / band);
    void *dz_in = nullptr, *dz_out = nullptr;
    if ((host_mode == 2 || (host_mode == 0 && nbands > 64)) && mapped_host(h_in, &dz_in) &&
        mapped_host(h_out, &dz_out)) {
        Args a{dz_in, dz_out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out, es, stream};
        if (desc_status st = run_tiled(a)) return st;
        g_last_launches = 1;
        return DESC_OK;
    }

    HostPipe *hp;
    if (desc_status s = host_pipe(dev, &hp)) return s;
    std::lock_guard<std::mutex> lk(hp->enqueue);
    const int64_t v = 16 / es;
    // row bands: band x cols in, cols x band out; column bands: rows x band in, band x rows
    // out (each 16-byte padded; the two together are what band_bytes counts)
    const int64_t wide = round_up(band * round_up(other, v) * es, 256);
    const int64_t narrow = round_up(other * round_up(band, v) * es, 256);
    const int64_t in_b = by_cols ? narrow : wide, out_b = by_cols ? wide : narrow;
    char *w = static_cast<char *>(d_work);
    char *d_in[kHostStreams], *d_out[kHostStreams];
    for (int i = 0; i < NBUF; ++i) {
        d_in[i] = w + i * in_b;
        d_out[i] = w + NBUF * in_b + i * out_b;
    }

    if ((e = cudaEventRecord(hp->enter, stream)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    for (int i = 0; i < NBUF; ++i)
        if ((e = cudaStreamWaitEvent(hp->s[i], hp->enter, 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent");
    int launches = 0;
    int64_t k = 0;
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t p0 = 0; p0 < span; p0 += band, ++k) {
            // fixed bands: measured 81 GB/s vs 77 GB/s with bands ramped at both ends
            // (scripts/exp_e2e_ramp.py; narrow bands make the strided rows short)
            const int64_t np_ = span - p0 < band ? span - p0 : band;
            const int buf = (int)(k % NBUF);
            cudaStream_t s = hp->s[buf];
            // this band's sub-matrix: nr x nc input cells at (r0, c0)
            const int64_t r0 = by_cols ? 0 : p0, c0 = by_cols ? p0 : 0;
            const int64_t nr = by_cols ? rows : np_, nc = by_cols ? np_ : cols;
            const int64_t ldi_d = round_up(nc, v), ldo_d = round_up(nr, v);
            const char *src = static_cast<const char *>(h_in) + (b * stride_in + r0 * ld_in + c0) * es;
            e = cudaMemcpy2DAsync(d_in[buf], ldi_d * es, src, ld_in * es, nc * es, nr,
                                  cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync H2D");
            Args a{d_in[buf], d_out[buf], 1, nr, nc, ldi_d, ldo_d, 0, 0, es, s};
            if (desc_status st = dispatch(a, DESC_KERNEL_AUTO)) return st;
            ++launches;
            // output block: rows c0 .. c0 + nc, columns r0 .. r0 + nr
            char *dst = static_cast<char *>(h_out) + (b * stride_out + c0 * ld_out + r0) * es;
            e = cudaMemcpy2DAsync(dst, ld_out * es, d_out[buf], ldo_d * es, nr * es, nc,
                                  cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync D2H");
        }
    }
    for (int i = 0; i < NBUF; ++i) {
        if ((e = cudaEventRecord(hp->done[i], hp->s[i])) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        if ((e = cudaStreamWaitEvent(stream, hp->done[i], 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent");
    }
    g_last_launches = launches;
    return DESC_OK;
}

// ---- strided batched copy (desc_copy_batched) -----------------------------------------
desc_status run_copy(const void *in, void *out, int64_t batch, int64_t rows, int64_t cols,
                     int64_t ld_in, int64_t ld_out, int64_t stride_in, int64_t stride_out, int es,
                     cudaStream_t stream) {
    g_last_launches = 0;
    if (es == 0) return fail(DESC_ERR_DTYPE, "unknown dtype");
    if (batch < 0 || rows < 0 || cols < 0) return fail(DESC_ERR_SHAPE, "negative size");
    if (batch == 0 || rows == 0 || cols == 0) return DESC_OK;
    if (!in || !out) return fail(DESC_ERR_NULL, "null %s pointer", in ? "out" : "in");
    if (ld_in < cols || ld_out < cols) return fail(DESC_ERR_SHAPE, "ld smaller than cols");
    if (stride_in < 0 || stride_out < 0) return fail(DESC_ERR_SHAPE, "negative batch stride");
    if (!outputs_disjoint(batch, rows, cols, ld_out, stride_out))
        return fail(DESC_ERR_SHAPE, "batched outputs overlap");
    int64_t span_in, span_out, bin, bout;
    if (!span_elems(batch, rows, cols, ld_in, stride_in, &span_in) ||
        !span_elems(batch, rows, cols, ld_out, stride_out, &span_out) ||
        !mul_ok(span_in, es, &bin) || !mul_ok(span_out, es, &bout))
        return fail(DESC_ERR_SHAPE, "extent overflows int64");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
    if (i0 < o0 + (uintptr_t)bout && o0 < i0 + (uintptr_t)bin)
        return fail(DESC_ERR_ALIAS, "in and out overlap (&uniq, P:576-579)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in")) return st;
    if (desc_status st = check_memspace(out, dev, "out")) return st;
    DevInfo di;
    if (desc_status st = device_info(dev, &di)) return st;
    const int64_t total_rows = batch * rows;
    // One row per CTA (the block scheduler balances the SMs and every CTA prefetches its row
    // into L2 before the dependency wait, as TILED) and 8 16-byte loads in flight per thread
    // when rows hold >= 8 per thread, else 4 (scripts/exp_copy.py,
    // profiles/r02_copy_grid_unroll.txt, back to back: 8192^2 f32 0.962 -> 1.049, the slab
    // unpack at P = 2 / 4 / 8 0.90 / 0.92 / 0.94 -> 1.009 / 1.041 / 1.039, 2048^2 f64 0.921 ->
    // 0.981).  A/B knobs: DESC_COPY_GRID=0 the former persistent SMs x 8 grid, DESC_COPY_UNR=4/8.
    static const int copy_grid = dev_knob("DESC_COPY_GRID", 1);
    static const int copy_unr_knob = dev_knob("DESC_COPY_UNR", 0);
    const int copy_unr = copy_unr_knob ? copy_unr_knob : (cols * es / 16 >= 8 * 256 ? 8 : 4);
    // (short rows -- fewer than 256 16-byte units -- keep the persistent grid: a CTA per row
    // would leave most of its threads idle)
    const bool row_per_cta = copy_grid == 1 && cols * es >= 256 * 16;
    const int64_t gcap = row_per_cta ? ((int64_t)1 << 30) : (int64_t)di.sms * 8;
    const int grid = (int)(total_rows < gcap ? total_rows : gcap);
    const bool vec16 = (i0 % 16 == 0) && (o0 % 16 == 0) && (cols * es) % 16 == 0 &&
                       (ld_in * es) % 16 == 0 && (ld_out * es) % 16 == 0 &&
                       (batch == 1 || ((stride_in * es) % 16 == 0 && (stride_out * es) % 16 == 0));
    const char *ci = static_cast<const char *>(in);
    char *co = static_cast<char *>(out);
    const int64_t sib = batch > 1 ? stride_in * es : 0, sob = batch > 1 ? stride_out * es : 0;
    if (vec16 && copy_unr == 8)
        launch_plain_pdl(desc::copy_rows_kernel<uint4, 8>, grid, 256, 0, stream, ci, co, rows, total_rows, cols * es / 16,
                                                                  ld_in * es, ld_out * es, sib, sob);
    else if (vec16)
        launch_plain_pdl(desc::copy_rows_kernel<uint4>, grid, 256, 0, stream, ci, co, rows, total_rows, cols * es / 16,
                                                               ld_in * es, ld_out * es, sib, sob);
    else if (es == 8)
        launch_plain_pdl(desc::copy_rows_kernel<unsigned long long>, grid, 256, 0, stream, ci, co, rows, total_rows, cols,
                                                                            ld_in * es, ld_out * es, sib, sob);
    else if (es == 4)
        launch_plain_pdl(desc::copy_rows_kernel<uint32_t>, grid, 256, 0, stream, ci, co, rows, total_rows, cols,
                                                                  ld_in * es, ld_out * es, sib, sob);
    else if (es == 2)
        launch_plain_pdl(desc::copy_rows_kernel<uint16_t>, grid, 256, 0, stream, ci, co, rows, total_rows, cols,
                                                                  ld_in * es, ld_out * es, sib, sob);
    else
        launch_plain_pdl(desc::copy_rows_kernel<uint8_t>, grid, 256, 0, stream, ci, co, rows, total_rows, cols,
                                                                 ld_in * es, ld_out * es, sib, sob);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "copy_rows_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

// ---- views (desc_view_compile / desc_view_copy) -----------------------------------------
static_assert(DESC_MAX_DIMS == desc::kMaxViewDims, "view rank limits agree");

desc_status view_compile(int32_t ndim, const int64_t *shape, const int64_t *strides,
                         const desc_view_op *ops, int32_t nops, desc_strided_view *out) {
    if (!shape || !out || (nops > 0 && !ops)) return fail(DESC_ERR_NULL, "null pointer");
    if (ndim < 1 || ndim > DESC_MAX_DIMS)
        return fail(DESC_ERR_SHAPE, "root rank %d outside [1, %d]", ndim, DESC_MAX_DIMS);
    desc_strided_view v;
    memset(&v, 0, sizeof v);
    v.ndim = ndim;
    for (int d = 0; d < ndim; ++d) {
        if (shape[d] < 0) return fail(DESC_ERR_SHAPE, "negative extent");
        v.shape[d] = shape[d];
    }
    if (strides) {
        for (int d = 0; d < ndim; ++d) v.stride[d] = strides[d];
    } else {                                          // C-contiguous root
        v.stride[ndim - 1] = 1;
        for (int d = ndim - 2; d >= 0; --d)
            if (!mul_ok(v.stride[d + 1], v.shape[d + 1] > 0 ? v.shape[d + 1] : 1, &v.stride[d]))
                return fail(DESC_ERR_SHAPE, "root extent overflows int64");
    }
    for (int i = 0; i < nops; ++i) {
        const int d = ops[i].depth;
        const int64_t k = ops[i].k;
        if (d < 0 || d >= v.ndim)
            return fail(DESC_ERR_SHAPE, "view %d: map depth %d exceeds the nesting (%d dims)", i, d, v.ndim);
        const int64_t n = v.shape[d];
        switch (ops[i].kind) {
            case DESC_VIEW_GROUP: {                   // [[d;n]] -> [[ [[d;k]]; n/k ]]
                if (k <= 0 || n % k) return fail(DESC_ERR_SHAPE, "view %d: group<%lld> needs k | n = %lld (R12)", i, (long long)k, (long long)n);
                if (v.ndim == DESC_MAX_DIMS) return fail(DESC_ERR_SHAPE, "view %d: more than %d dims", i, DESC_MAX_DIMS);
                for (int e = v.ndim; e > d + 1; --e) { v.shape[e] = v.shape[e - 1]; v.stride[e] = v.stride[e - 1]; }
                v.shape[d + 1] = k;
                v.stride[d + 1] = v.stride[d];
                v.shape[d] = n / k;
                if (!mul_ok(v.stride[d], k, &v.stride[d])) return fail(DESC_ERR_SHAPE, "stride overflow");
                ++v.ndim;
                break;
            }
            case DESC_VIEW_TRANSPOSE: {               // swap the outer two dims
                if (d + 1 >= v.ndim) return fail(DESC_ERR_SHAPE, "view %d: transpose needs a nested array", i);
                int64_t t = v.shape[d]; v.shape[d] = v.shape[d + 1]; v.shape[d + 1] = t;
                t = v.stride[d]; v.stride[d] = v.stride[d + 1]; v.stride[d + 1] = t;
                break;
            }
            case DESC_VIEW_SPLIT_FST:                 // ([[d;k]], [[d;n-k]]).fst
            case DESC_VIEW_SPLIT_SND:
                if (k < 0 || k > n) return fail(DESC_ERR_SHAPE, "view %d: split<%lld> needs n = %lld >= k", i, (long long)k, (long long)n);
                if (ops[i].kind == DESC_VIEW_SPLIT_SND) {
                    v.offset += k * v.stride[d];
                    v.shape[d] = n - k;
                } else {
                    v.shape[d] = k;
                }
                break;
            case DESC_VIEW_REVERSE:
                if (n > 0) v.offset += (n - 1) * v.stride[d];
                v.stride[d] = -v.stride[d];
                break;
            default:
                return fail(DESC_ERR_SHAPE, "view %d: unknown kind %d", i, ops[i].kind);
        }
    }
    *out = v;
    return DESC_OK;
}

desc_status view_copy(const void *in, void *out, const desc_strided_view *view, int es,
                      cudaStream_t stream) {
    g_last_launches = 0;
    if (es == 0) return fail(DESC_ERR_DTYPE, "unknown dtype");
    if (!view) return fail(DESC_ERR_NULL, "null view");
    const desc_strided_view &v = *view;
    if (v.ndim < 1 || v.ndim > DESC_MAX_DIMS) return fail(DESC_ERR_SHAPE, "view rank outside [1, 8]");
    int64_t total = 1, lo = v.offset, hi = v.offset;
    for (int d = 0; d < v.ndim; ++d) {
        if (v.shape[d] < 0) return fail(DESC_ERR_SHAPE, "negative extent");
        if (!mul_ok(total, v.shape[d], &total)) return fail(DESC_ERR_SHAPE, "view size overflows int64");
    }
    if (total == 0) return DESC_OK;
    for (int d = 0; d < v.ndim; ++d) {
        int64_t ext;
        if (!mul_ok(v.shape[d] - 1, v.stride[d], &ext)) return fail(DESC_ERR_SHAPE, "extent overflow");
        if (ext < 0) lo += ext; else hi += ext;
    }
    if (lo < 0) return fail(DESC_ERR_SHAPE, "view reaches before `in` (offset + negative strides < 0)");
    if (!in || !out) return fail(DESC_ERR_NULL, "null %s pointer", in ? "out" : "in");
    int64_t bin_lo, bin_hi, bout;
    if (!mul_ok(lo, es, &bin_lo) || !mul_ok(hi + 1, es, &bin_hi) || !mul_ok(total, es, &bout))
        return fail(DESC_ERR_SHAPE, "extent overflows int64");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
    if (i0 + (uintptr_t)bin_lo < o0 + (uintptr_t)bout && o0 < i0 + (uintptr_t)bin_hi)
        return fail(DESC_ERR_ALIAS, "view of in and out overlap (&uniq, P:576-579)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in")) return st;
    if (desc_status st = check_memspace(out, dev, "out")) return st;

    // normalise: drop unit dims, merge dims that are contiguous in the input (the output is
    // the view's own row-major order, so it merges whenever the input does)
    int nd = 0;
    int64_t sh[DESC_MAX_DIMS], st_in[DESC_MAX_DIMS];
    for (int d = 0; d < v.ndim; ++d)
        if (v.shape[d] != 1) { sh[nd] = v.shape[d]; st_in[nd] = v.stride[d]; ++nd; }
    if (nd == 0) { sh[0] = 1; st_in[0] = 1; nd = 1; }
    int m = 0;
    for (int d = 1; d < nd; ++d) {
        if (st_in[m] == st_in[d] * sh[d]) { sh[m] *= sh[d]; st_in[m] = st_in[d]; }
        else { ++m; sh[m] = sh[d]; st_in[m] = st_in[d]; }
    }
    nd = m + 1;
    int64_t st_out[DESC_MAX_DIMS];
    st_out[nd - 1] = 1;
    for (int d = nd - 2; d >= 0; --d) st_out[d] = st_out[d + 1] * sh[d + 1];
    const int L = nd - 1;
    const char *base = static_cast<const char *>(in) + v.offset * es;

    // transposition of the innermost dim onto an input-contiguous dim: the TMA kernels.
    // A negative innermost stride (rows read bottom-up, e.g. rot90 = transpose.map(reverse))
    // is handled by the TMA-store kernel reading mirrored rows.
    if (st_in[L] > 1 || st_in[L] < -1) {
        int ec = -1, others = 0, b = -1;
        for (int d = 0; d < L; ++d) {
            if (st_in[d] == 1 && ec < 0) ec = d;
            else { ++others; b = d; }
        }
        if (ec >= 0 && others <= 1 && (b < 0 || st_in[b] > 0)) {
            const bool rev = st_in[L] < 0;
            const int64_t ld = rev ? -st_in[L] : st_in[L];
            const char *phys = rev ? base - (sh[L] - 1) * ld * es : base;
            Args a{phys, out, b < 0 ? 1 : sh[b], sh[L], sh[ec], ld, st_out[ec],
                   b < 0 ? 0 : st_in[b], b < 0 ? 0 : st_out[b], es, stream};
            a.rev_rows = rev ? 1 : 0;
            bool empty;
            desc_status s = validate(a, &empty);
            if (s == DESC_OK) {
                s = dispatch(a, DESC_KERNEL_AUTO);
                if (s != DESC_ERR_KERNEL) return s;       // else: not a TMA geometry -> gather
            } else if (s != DESC_ERR_SHAPE) {
                return s;
            }
        }
    }

    // everything else: outer dims x R2 rows x U cells (view_copy.cuh)
    desc::ViewTiles vt;
    memset(&vt, 0, sizeof vt);
    const int64_t U_el = sh[L], s1 = st_in[L];
    vt.R2 = L >= 1 ? sh[L - 1] : 1;
    vt.s2 = L >= 1 ? st_in[L - 1] : 0;
    vt.outer_ndim = L >= 1 ? L - 1 : 0;
    vt.outer_count = 1;
    for (int d = 0; d < vt.outer_ndim; ++d) {
        vt.outer_shape[d] = sh[d];
        vt.outer_stride[d] = st_in[d];
        vt.outer_count *= sh[d];
    }
    vt.offset = v.offset;
    const int V = 16 / es;
    bool aligned = (i0 % 16 == 0) && (o0 % 16 == 0) && (U_el * es) % 16 == 0 &&
                   (vt.R2 == 1 || (vt.s2 * es) % 16 == 0);
    for (int d = 0; d < vt.outer_ndim && aligned; ++d) aligned = (vt.outer_stride[d] * es) % 16 == 0;
    int mode = 0;
    if (aligned && s1 == 1 && (v.offset * es) % 16 == 0) mode = 1;
    else if (aligned && s1 == -1 && ((v.offset - V + 1) * es) % 16 == 0) mode = 2;
    vt.U = mode ? U_el / V : U_el;
    vt.s1 = s1;
    // work items of ~4096 cells (64 KB when vectorised)
    if (vt.U >= 4096) { vt.uch = 4096; vt.rch = 1; }
    else { vt.uch = vt.U; vt.rch = (4096 + vt.U - 1) / vt.U; }
    if (vt.rch > vt.R2) vt.rch = vt.R2;
    vt.n_uchunks = (vt.U + vt.uch - 1) / vt.uch;
    vt.n_rchunks = (vt.R2 + vt.rch - 1) / vt.rch;
    vt.items = vt.outer_count * vt.n_rchunks * vt.n_uchunks;
    int64_t w = vt.uch < 256 ? vt.uch : 256;
    vt.ulog = 0;
    while ((1LL << vt.ulog) < w) ++vt.ulog;
    DevInfo di;
    if (desc_status st = device_info(dev, &di)) return st;
    // Grid: mirrored 16-byte rows (mode 2) launch one work item per CTA and prefetch it into
    // L2 before griddepcontrol.wait (rot180 8192^2 f32 0.955 -> 1.02); the other modes keep
    // the persistent SMs x 8 grid (the tile view: one item per CTA 0.80, with the prefetch
    // 0.64; profiles/r02_view_grid_pf.txt).  DESC_VIEW_GRID=0/1 and DESC_VIEW_PF=0/1 force
    // either choice for every mode (A/B).
    static const int view_grid = dev_knob("DESC_VIEW_GRID", -1);
    static const int view_pf = dev_knob("DESC_VIEW_PF", -1);
    const bool one = view_grid < 0 ? mode == 2 : view_grid == 1;
    const int pf = view_pf < 0 ? (mode == 2 ? 1 : 0) : view_pf;
    const int64_t cap = one ? ((int64_t)1 << 30) : (int64_t)di.sms * 8;
    const int grid = (int)(vt.items < cap ? vt.items : cap);
    const char *ci = static_cast<const char *>(in);
    char *co = static_cast<char *>(out);
    if (mode == 1) launch_plain_pdl(desc::view_tiles_kernel<uint4, 1>, grid, 256, 0, stream, ci, co, vt, es, pf);
    else if (mode == 2) launch_plain_pdl(desc::view_tiles_kernel<uint4, 2>, grid, 256, 0, stream, ci, co, vt, es, pf);
    else if (es == 8) launch_plain_pdl(desc::view_tiles_kernel<unsigned long long, 0>, grid, 256, 0, stream, ci, co, vt, es, pf);
    else if (es == 4) launch_plain_pdl(desc::view_tiles_kernel<uint32_t, 0>, grid, 256, 0, stream, ci, co, vt, es, pf);
    else if (es == 2) launch_plain_pdl(desc::view_tiles_kernel<uint16_t, 0>, grid, 256, 0, stream, ci, co, vt, es, pf);
    else launch_plain_pdl(desc::view_tiles_kernel<uint8_t, 0>, grid, 256, 0, stream, ci, co, vt, es, pf);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "view_tiles_kernel launch");
    g_last_launches = 1;
    return DESC_OK;
}

// ---- block-wide reduction and scan -------------------------------
// element size of the reduce/scan dtypes; 0 for the 2-byte float types (not supported)
int rs_es(desc_dtype t) {
    switch (t) {
        case DESC_U8: return 1;
        case DESC_I32: case DESC_F32: return 4;
        case DESC_I64: case DESC_F64: return 8;
        default: return 0;
    }
}

template <typename In>
desc_status launch_reduce(const void *in, void *out, int64_t n, int64_t B, int64_t nb, bool vec,
                          int sms, cudaStream_t stream) {
    const In *pi = static_cast<const In *>(in);
    In *po = static_cast<In *>(out);
    // grid: one wave of 8 x 256-thread CTAs per SM, grid-striding over the blocks, 8 16-byte
    // loads in flight per lane (2^26 f32, B = 1024: 0.966 of peak; the earlier 16 CTAs/SM
    // with 4 loads in flight 0.89; profiles/r01_reduce_sweep.txt)
#ifndef DESC_REDUCE_CTAS_PER_SM
#define DESC_REDUCE_CTAS_PER_SM 8
#endif
#ifndef DESC_REDUCE_ROWS
#define DESC_REDUCE_ROWS 1
#endif
#ifndef DESC_REDUCE_SEG
#define DESC_REDUCE_SEG 1
#endif
#ifndef DESC_REDUCE_WARP_CTAS         // grid cap (CTAs per SM) of the warp-per-block kernel
#define DESC_REDUCE_WARP_CTAS 16
#endif
#ifndef DESC_REDUCE_ROWS_LOADS        // 16-byte loads in flight per lane in the warp-row kernel
#define DESC_REDUCE_ROWS_LOADS 8
#endif
#ifndef DESC_REDUCE_ROWS_MAX          // largest block (bytes) the warp-row kernel takes
#define DESC_REDUCE_ROWS_MAX 8192     // (4 KB blocks: 0.96 -> 1.05 of peak; profiles/r01_reduce_sweep.txt)
#endif
static_assert(DESC_REDUCE_ROWS_MAX <= 8192, "warp-row kernel: at most 16 rows per block");
    const int64_t cap = (int64_t)sms * DESC_REDUCE_CTAS_PER_SM;
    const int64_t Bb = B * (int64_t)sizeof(In);                    // block bytes
    if (vec && n % B == 0 && Bb % 16 == 0 && Bb <= 256 && DESC_REDUCE_SEG) {
        // 1 … 16 vectors per block: warp-wide coalesced rows, segmented shuffles
        const int64_t g = (nb * (Bb / 16) / 256 + 7) / 8 + 1;
        const int grid = (int)(g < 2 * cap ? g : 2 * cap);
        switch (Bb / 16) {
            case 1: launch_plain_pdl(desc::block_reduce_seg_kernel<In, In, 1>, grid, 256, 0, stream, pi, po, nb); break;
            case 2: launch_plain_pdl(desc::block_reduce_seg_kernel<In, In, 2>, grid, 256, 0, stream, pi, po, nb); break;
            case 4: launch_plain_pdl(desc::block_reduce_seg_kernel<In, In, 4>, grid, 256, 0, stream, pi, po, nb); break;
            case 8: launch_plain_pdl(desc::block_reduce_seg_kernel<In, In, 8>, grid, 256, 0, stream, pi, po, nb); break;
            case 16: launch_plain_pdl(desc::block_reduce_seg_kernel<In, In, 16>, grid, 256, 0, stream, pi, po, nb); break;
            default: {   // 3, 5, 6, 7, 9 … 15 vectors: one thread per block
                const int64_t g1 = (nb + 255) / 256;
                launch_plain_pdl(desc::block_reduce_kernel<In, In, 1>, (int)(g1 < cap ? g1 : cap), 256, 0, stream, pi, po, n, B, nb, vec);
            }
        }
    } else if (vec && n % B == 0 && Bb % 512 == 0 && Bb <= DESC_REDUCE_ROWS_MAX &&
               ((Bb / 512) & (Bb / 512 - 1)) == 0 && DESC_REDUCE_ROWS) {
        // whole blocks of 1, 2, 4, 8 or 16 warp rows (the ragged-tail-free case; other row
        // counts -- 3, 5, 6, 7, 9 ... 15 -- take the warp-per-block kernel below)
        constexpr int L = DESC_REDUCE_ROWS_LOADS;
        const int64_t P = Bb / 512, g = (nb * P / L + 7) / 8 + 1;
        const int grid = (int)(g < 2 * cap ? g : 2 * cap);   // 16 CTAs/SM measured best here
        if (P == 1) launch_plain_pdl(desc::block_reduce_rows_kernel<In, In, 1, L>, grid, 256, 0, stream, pi, po, nb);
        else if (P == 2) launch_plain_pdl(desc::block_reduce_rows_kernel<In, In, 2, L>, grid, 256, 0, stream, pi, po, nb);
        else if (P == 4) launch_plain_pdl(desc::block_reduce_rows_kernel<In, In, 4, L>, grid, 256, 0, stream, pi, po, nb);
        else if (P == 8) launch_plain_pdl(desc::block_reduce_rows_kernel<In, In, 8, (L < 8 ? 8 : L)>, grid, 256, 0, stream, pi, po, nb);
        else launch_plain_pdl(desc::block_reduce_rows_kernel<In, In, 16, (L < 16 ? 16 : L)>, grid, 256, 0, stream, pi, po, nb);
    } else if (B <= 64) {
        const int64_t g = (nb + 255) / 256;                            // thread per block
        launch_plain_pdl(desc::block_reduce_kernel<In, In, 1>, (int)(g < cap ? g : cap), 256, 0, stream, pi, po, n, B, nb, vec);
    } else if (B <= 16384 && (B < 2048 || nb >= (int64_t)sms * 32)) {
        // (long blocks but fewer than 32 per SM: a CTA or a cluster per block, below)
        const int64_t g = (nb + 7) / 8, wcap = (int64_t)sms * DESC_REDUCE_WARP_CTAS;   // warp per block
        launch_plain_pdl(desc::block_reduce_kernel<In, In, 32>, (int)(g < wcap ? g : wcap), 256, 0, stream, pi, po, n, B, nb, vec);
    } else if (nb >= 2 * (int64_t)sms) {
        launch_plain_pdl(desc::block_reduce_cta_kernel<In, In>, (int)(nb < cap ? nb : cap), 256, 0, stream, pi, po, n, B, nb, vec);
    } else {
        // fewer blocks than 2 per SM: a cluster of 8 CTAs per block (one CTA per block left
        // 2^20-element blocks at 0.2 of peak: 64 CTAs on 148 SMs), 16 (non-portable) below
        // SMs / 8 blocks.  CTA size: the largest of 1024 / 512 / 256 threads at which the
        // device can hold all nb clusters at once (cudaOccupancyMaxActiveClusters: registers,
        // GPC shape, MPS/MIG limits), so few blocks still keep enough loads in flight; if none
        // fits in one wave, 256 (the clusters then grid-stride over the blocks).
        static const bool np = cudaFuncSetAttribute(desc::block_reduce_cluster_kernel<In, In, 16>,
                                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
        const bool use16 = nb * 8 < (int64_t)sms && np;
        auto kern = use16 ? desc::block_reduce_cluster_kernel<In, In, 16>
                          : desc::block_reduce_cluster_kernel<In, In, 8>;
        const int CL = use16 ? 16 : 8;
        int threads = 256;
        for (int t : {1024, 512, 256}) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)(nb * CL));
            q.blockDim = dim3(t);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CL;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            q.attrs = at;
            q.numAttrs = 1;
            int active = 0;
            if (cudaOccupancyMaxActiveClusters(&active, kern, &q) != cudaSuccess) {
                cudaGetLastError();
                active = 0;
            }
            if (active >= nb) { threads = t; break; }
        }
#ifdef DESC_REDUCE_CLUSTER_THREADS
        threads = DESC_REDUCE_CLUSTER_THREADS;        // A/B builds only
#endif
        launch_cluster_pdl(kern, (int)(nb * CL), CL, threads, 0, stream, pi, po, n, B, nb, vec);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "block_reduce launch");
    g_last_launches = 1;
    return DESC_OK;
}

desc_status run_reduce(const void *in, void *out, int64_t n, int64_t B, desc_dtype dtype,
                       cudaStream_t stream) {
    g_last_launches = 0;
    host_mutant();
    const int es = rs_es(dtype);
    if (es == 0) return fail(DESC_ERR_DTYPE, "block reduction supports u8, i32, i64, f32, f64");
    if (n < 0 || B <= 0) return fail(DESC_ERR_SHAPE, "need n >= 0 and block > 0");
    if (n == 0) return DESC_OK;
    if (!in || !out) return fail(DESC_ERR_NULL, "null pointer");
    const int64_t nb = (n + B - 1) / B;
    int64_t bin, bout;
    if (!mul_ok(n, es, &bin) || !mul_ok(nb, es, &bout)) return fail(DESC_ERR_SHAPE, "extent overflow");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
    if (i0 < o0 + (uintptr_t)bout && o0 < i0 + (uintptr_t)bin)
        return fail(DESC_ERR_ALIAS, "in and out overlap (&uniq, P:576-579)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in")) return st;
    if (desc_status st = check_memspace(out, dev, "out")) return st;
    DevInfo di;
    if (desc_status st = device_info(dev, &di)) return st;
    const bool vec = i0 % 16 == 0;
    switch (dtype) {
        case DESC_U8: return launch_reduce<uint8_t>(in, out, n, B, nb, vec, di.sms, stream);
        case DESC_I32: return launch_reduce<uint32_t>(in, out, n, B, nb, vec, di.sms, stream);
        case DESC_I64: return launch_reduce<uint64_t>(in, out, n, B, nb, vec, di.sms, stream);
        case DESC_F32: return launch_reduce<float>(in, out, n, B, nb, vec, di.sms, stream);
        case DESC_F64: return launch_reduce<double>(in, out, n, B, nb, vec, di.sms, stream);
        default: return fail(DESC_ERR_DTYPE, "unsupported dtype");
    }
}

// scan tiles: 256 threads x ITEMS elements: 128 bytes per thread for 4/8-byte cells (32 KB
// tiles: few tiles keep the look-back chain short), 64 for bytes (register budget)
int scan_items(int es) { return es == 1 ? 64 : 128 / es; }

int64_t scan_tiles(int64_t n, int es) {
    const int64_t T = 256 * (int64_t)scan_items(es);
    return (n + T - 1) / T;
}

int64_t scan_workspace_bytes(int64_t n, int es) {
    // descriptor words: 8 bytes per tile, twice for 64-bit accumulators (f32 accumulates in
    // f64, i64/f64 in 64 bits; i32/u8 in u32); three-launch arrays: 2 x acc bytes per tile
    const int acc = es == 8 || es == 4 ? 8 : 4;
    const int64_t t = scan_tiles(n, es);
    const int64_t words = es == 1 ? 1 : 2;   // es 4: f32 needs 2 (i32 uses 1)
    const int64_t single = words * round_up(t * 8, 256);
    const int64_t three = 2 * round_up(t * acc, 256);
    return 256 + (single > three ? single : three);
}

// streaming scan: NR reduce + NR scan warps, tiles of NR x 32 lanes x VPT 16-byte vectors,
// an S-stage shared-memory ring, QT tiles parked in TMEM.  Per element type (A/B sweeps in
// profiles/r01_scan_sweeps.txt, fraction of the measured peak):
//   4-byte integers : 8 + 8 warps x 12 vectors (48 KB tiles), 4 stages, 5 slots   i32 0.91
//   f32 (f64 sums)  : 12 + 12 warps x 8 vectors (48 KB), 4 stages, 5 slots       f32 0.843 -> 0.86
//   f64 / 64-bit    : 12 + 12 warps x 10 vectors (60 KB), 3 stages, 4 slots      f64 0.924 -> 0.934
// With 8-byte accumulators every warp-scan level is two shuffles and the adds are f64, so
// the scan warps are the slower side: more warps in flight and shorter per-warp carry
// chains pay there, while the same split costs i32 0.905 -> 0.893.
#ifndef DESC_SCAN_VPT        // compile-time overrides of the 4-byte integer path: A/B builds
#define DESC_SCAN_VPT 12
#endif
#ifndef DESC_SCAN_STAGES
#define DESC_SCAN_STAGES 4
#endif
#ifndef DESC_SCAN_TMEM_SLOTS
#define DESC_SCAN_TMEM_SLOTS 5
#endif
#ifndef DESC_SCAN_LB_WARPS
#define DESC_SCAN_LB_WARPS 1
#endif
#ifndef DESC_SCAN_LC_F32       // f32: lane-contiguous layout + TMA-store staging
#define DESC_SCAN_LC_F32 1
#endif
#ifndef DESC_SCAN_LC_I32       // 4-byte integers: same, NR warps per group
#define DESC_SCAN_LC_I32 1
#endif
#ifndef DESC_SCAN_LC_I32_NR
#define DESC_SCAN_LC_I32_NR 12
#endif
#ifndef DESC_SCAN_LC_F64       // 8-byte values: same
#define DESC_SCAN_LC_F64 1
#endif
template <typename In> struct ScanPick {       // 4-byte integers
    static constexpr int NR = DESC_SCAN_LC_I32 ? DESC_SCAN_LC_I32_NR : 8,
                         VPT = DESC_SCAN_LC_I32 ? 8 : DESC_SCAN_VPT,
                         S = DESC_SCAN_LC_I32 ? 3 : DESC_SCAN_STAGES,
                         QT = DESC_SCAN_TMEM_SLOTS, LC = DESC_SCAN_LC_I32;
};
#ifndef DESC_SCAN_LC_U8        // 1-byte inputs: lane-contiguous layout (2^28 u8: 0.553 -> 0.647)
#define DESC_SCAN_LC_U8 1
#endif
template <> struct ScanPick<uint8_t> {         // 6 vectors per lane (16 elements each), 8 stages
    static constexpr int NR = DESC_SCAN_LC_U8 ? 12 : 8, VPT = DESC_SCAN_LC_U8 ? 8 : 6,
                         S = DESC_SCAN_LC_U8 ? 3 : 8, QT = DESC_SCAN_TMEM_SLOTS,
                         LC = DESC_SCAN_LC_U8;
};
template <> struct ScanPick<float> {           // LC: 48 KB of store staging -> 3 stages
    static constexpr int NR = 12, VPT = 8, S = DESC_SCAN_LC_F32 ? 3 : 4, QT = 5,
                         LC = DESC_SCAN_LC_F32;
};
template <> struct ScanPick<double> {
    static constexpr int NR = 12, VPT = DESC_SCAN_LC_F64 ? 8 : 10, S = 3,
                         QT = DESC_SCAN_LC_F64 ? 5 : 4, LC = DESC_SCAN_LC_F64;
};
template <> struct ScanPick<uint64_t> : ScanPick<double> {};
template <typename In>
using ScanStreamC = desc::ScanStreamCfg<ScanPick<In>::NR, ScanPick<In>::VPT, ScanPick<In>::S,
                                        ScanPick<In>::QT, DESC_SCAN_LB_WARPS, ScanPick<In>::LC>;

// zero `bytes` (a multiple of 16) of scan state in stream order, PDL-chained
desc_status scan_reset(char *work, int64_t bytes, const DevInfo &di, cudaStream_t stream) {
    const int64_t n16 = bytes / 16;
    const int64_t want = (n16 + 255) / 256, cap = (int64_t)di.sms * 4;
    cudaError_t e = launch_plain_pdl(desc::scan_reset_kernel, (int)(want < cap ? want : cap), 256,
                                     0, stream, reinterpret_cast<uint4 *>(work), n16);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "scan_reset launch");
    return DESC_OK;
}

template <typename In, int ITEMS>
desc_status launch_scan(const void *in, void *out, int64_t n, char *work, bool vec,
                        desc_scan_algo algo, cudaStream_t stream) {
    using Acc = typename desc::AccOf<In>::T;
    const int es = (int)sizeof(In);
    const int64_t t = scan_tiles(n, es);
    // workspace: [counter | 256 B] then either the single-pass descriptor words (dlo, and dhi
    // for 64-bit values: 8 bytes per tile each) or the three-launch aggregate and exclusive
    // prefix arrays (sizeof(Acc) per tile each); scan_workspace_bytes covers the larger
    desc::ScanState<Acc> st;
    st.counter = reinterpret_cast<uint32_t *>(work);
    st.dlo = reinterpret_cast<uint64_t *>(work + 256);
    st.dhi = reinterpret_cast<uint64_t *>(work + 256 + round_up(t * 8, 256));
    const int64_t desc_words = sizeof(Acc) == 8 ? 2 : 1;
    char *vals = work + 256;
    st.agg = reinterpret_cast<Acc *>(vals);
    st.incl = reinterpret_cast<Acc *>(vals + round_up(t * (int64_t)sizeof(Acc), 256));
    if (t > INT32_MAX) return fail(DESC_ERR_SHAPE, "scan too long");
    const In *pi = static_cast<const In *>(in);
    In *po = static_cast<In *>(out);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    DevInfo di;
    if (desc_status s = device_info(dev, &di)) return s;
    // streaming tiles (96 KB) are never more than the look-back tiles (<= 32 KB), so the
    // workspace sized by scan_tiles() covers both
    using SP = ScanPick<In>;
    using SC = ScanStreamC<In>;
    constexpr int64_t TBY = SC::TB;
    const int64_t ts = (n * es + TBY - 1) / TBY;
    if (algo == DESC_SCAN_AUTO) {
        static const int single_max = dev_knob("DESC_SCAN_SINGLE_MAX_TILES", 256);
        if (vec && ts >= 2 * (int64_t)di.sms) algo = DESC_SCAN_STREAM;
        else if (t <= single_max) algo = DESC_SCAN_LOOKBACK;
        else algo = DESC_SCAN_THREE_PASS;
    }
    if (algo == DESC_SCAN_STREAM) {
        if (!vec) return fail(DESC_ERR_KERNEL, "streaming scan needs 16-byte aligned in and out");
        auto kern = desc::scan_stream_kernel<In, SP::NR, SP::VPT, SP::S, SP::QT,
                                             DESC_SCAN_LB_WARPS, SP::LC>;
        const int smem = SC::SMEM;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute (scan)");
        st.dhi = reinterpret_cast<uint64_t *>(work + 256 + round_up(ts * 8, 256));
        if (desc_status s = scan_reset(work, 256 + desc_words * round_up(ts * 8, 256), di, stream))
            return s;
        const int64_t grid = ts < di.sms ? ts : di.sms;
        // TMA view of the input: rows of 128 bytes (the < 128-byte tail is read directly)
        const int64_t bulk_rows = n * es / 128;
        CUtensorMap map, map_out;
        memset(&map, 0, sizeof(map));
        memset(&map_out, 0, sizeof(map_out));
        if (bulk_rows > 0) {
            MapKey k{reinterpret_cast<uintptr_t>(in), 128 / es, bulk_rows, 1, 128 / es, 0, es,
                     128 / es, SC::BOX_ROWS};
            if (desc_status s = tensor_map(k, &map)) return s;
            if (SP::LC) {     // the output as the same 128-byte rows, one warp segment per box
                MapKey ko{reinterpret_cast<uintptr_t>(out), 128 / es, bulk_rows, 1, 128 / es, 0,
                          es, 128 / es, 32};
                if (desc_status s = tensor_map(ko, &map_out)) return s;
            }
        }
        e = launch_pdl(kern, (int)grid, SC::THREADS, smem, stream, map, map_out, pi, po, n, ts,
                       bulk_rows, st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "scan_stream launch");
        g_last_launches = 2;
        return DESC_OK;
    }
    if (algo == DESC_SCAN_LOOKBACK) {
        if (desc_status s = scan_reset(work, 256 + desc_words * round_up(t * 8, 256), di, stream))
            return s;
        e = launch_plain_pdl(desc::scan_kernel<In, In, ITEMS>, (int)t, 256, 0, stream, pi, po, n,
                             st, vec);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "scan launch");
        g_last_launches = 2;
        return DESC_OK;
    }
    if (algo != DESC_SCAN_THREE_PASS) return fail(DESC_ERR_KERNEL, "unknown scan algorithm %d", (int)algo);
    const int64_t T = 256 * (int64_t)ITEMS;
    const int64_t g1 = (t + 7) / 8, cap = (int64_t)di.sms * 16;       // one warp per tile
    launch_plain_pdl(desc::block_reduce_kernel<In, Acc, 32>, (int)(g1 < cap ? g1 : cap), 256, 0, stream, 
        pi, st.agg, n, T, t, (reinterpret_cast<uintptr_t>(in) & 15) == 0);
    desc::scan_aggregates_kernel<Acc><<<1, 1024, 0, stream>>>(st.agg, st.incl, t);
    desc::scan_tiles_kernel<In, ITEMS><<<(int)t, 256, 0, stream>>>(pi, po, n, st.incl, vec);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "scan launch");
    g_last_launches = 3;
    return DESC_OK;
}

desc_status run_scan(const void *in, void *out, int64_t n, desc_dtype dtype, void *d_work,
                     size_t work_bytes, desc_scan_algo algo, cudaStream_t stream) {
    g_last_launches = 0;
    host_mutant();
    const int es = rs_es(dtype);
    if (es == 0) return fail(DESC_ERR_DTYPE, "scan supports u8, i32, i64, f32, f64");
    if (n < 0) return fail(DESC_ERR_SHAPE, "negative n");
    if ((int)algo < 0 || (int)algo > 3) return fail(DESC_ERR_KERNEL, "unknown scan algorithm %d", (int)algo);
    if (n == 0) return DESC_OK;
    if (!in || !out || !d_work) return fail(DESC_ERR_NULL, "null pointer");
    int64_t bytes;
    if (!mul_ok(n, es, &bytes)) return fail(DESC_ERR_SHAPE, "extent overflow");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
    if (i0 != o0 && i0 < o0 + (uintptr_t)bytes && o0 < i0 + (uintptr_t)bytes)
        return fail(DESC_ERR_ALIAS, "in and out partially overlap (in == out is allowed)");
    if ((int64_t)work_bytes < scan_workspace_bytes(n, es) || (reinterpret_cast<uintptr_t>(d_work) & 255))
        return fail(DESC_ERR_SHAPE, "d_work must be 256-byte aligned and >= desc_scan_workspace(n)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in")) return st;
    if (desc_status st = check_memspace(out, dev, "out")) return st;
    if (desc_status st = check_memspace(d_work, dev, "d_work")) return st;
    const bool vec = i0 % 16 == 0 && o0 % 16 == 0;
    char *w = static_cast<char *>(d_work);
    switch (dtype) {
        case DESC_U8: return launch_scan<uint8_t, 64>(in, out, n, w, vec, algo, stream);
        case DESC_I32: return launch_scan<uint32_t, 32>(in, out, n, w, vec, algo, stream);
        case DESC_I64: return launch_scan<uint64_t, 16>(in, out, n, w, vec, algo, stream);
        case DESC_F32: return launch_scan<float, 32>(in, out, n, w, vec, algo, stream);
        case DESC_F64: return launch_scan<double, 16>(in, out, n, w, vec, algo, stream);
        default: return fail(DESC_ERR_DTYPE, "unsupported dtype");
    }
}

// ---- fused transpose + exchange: one launch for every destination slab ------------------
desc_status run_slab_peer(const void *in, void *const *outs, int32_t P, int32_t r, int64_t M,
                          int64_t N, int es, cudaStream_t stream) {
    g_last_launches = 0;
    if (es != 4 && es != 8) return fail(DESC_ERR_DTYPE, "peer slab transpose supports 4- and 8-byte cells");
    if (!in || !outs) return fail(DESC_ERR_NULL, "null pointer");
    if (P < 1 || P > desc::kMaxScatter || r < 0 || r >= P)
        return fail(DESC_ERR_SHAPE, "need 1 <= P <= %d and 0 <= r < P (P=%d r=%d)", desc::kMaxScatter, P, r);
    if (M <= 0 || N <= 0 || M % P || N % P)
        return fail(DESC_ERR_SHAPE, "M=%lld and N=%lld must be positive multiples of P=%d (R13)",
                    (long long)M, (long long)N, P);
    const int64_t Rm = M / P, Rn = N / P;
    const int tc = es == 8 ? 32 : 64;                     // TILED tile width (cells)
    if (Rn % tc)
        return fail(DESC_ERR_SHAPE, "N/P = %lld must be a multiple of the %d-cell tile width", (long long)Rn, tc);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in_slab")) return st;
    desc::TiledScatter sc;
    memset(&sc, 0, sizeof sc);
    int64_t in_bytes, out_bytes;
    if (!mul_ok(Rm * N, es, &in_bytes) || !mul_ok(Rn * M, es, &out_bytes))
        return fail(DESC_ERR_SHAPE, "extent overflows int64");
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(in);
    for (int s = 0; s < P; ++s) {
        if (!outs[s]) return fail(DESC_ERR_NULL, "out_slabs[%d] is null", s);
        if (desc_status st = check_memspace(outs[s], dev, "out_slabs[s]")) return st;
        const uintptr_t o0 = reinterpret_cast<uintptr_t>(outs[s]);
        if (i0 < o0 + (uintptr_t)out_bytes && o0 < i0 + (uintptr_t)in_bytes)
            return fail(DESC_ERR_ALIAS, "in_slab and out_slabs[%d] overlap (&uniq, P:576-579)", s);
        sc.dst[s] = outs[s];
    }
    sc.seg = Rn;
    sc.col_off = r * Rm;
    Args a{in, outs[r], 1, Rm, N, N, M, 0, 0, es, stream};
    return es == 8 ? launch_tiled<unsigned long long, 32, 32, 128, true>(a, &sc)
                   : launch_tiled<uint32_t, 64, 64, 256, true>(a, &sc);
}

}  // namespace

extern "C" {

desc_status desc_slab_transpose_peer(const void *in_slab, void *const *out_slabs, int32_t P,
                                     int32_t r, int64_t M, int64_t N, desc_dtype dtype,
                                     void *stream) {
    return run_slab_peer(in_slab, out_slabs, P, r, M, N, dtype_size(dtype),
                         static_cast<cudaStream_t>(stream));
}

size_t desc_read_probe_sink_bytes(void) { return 16 * 8 * 1024; }   // one word per CTA, <= 8192 CTAs

desc_status desc_read_probe(const void *in, size_t bytes, void *sink, void *stream) {
    g_last_launches = 0;
    if (!in || !sink) return fail(DESC_ERR_NULL, "null pointer");
    if (reinterpret_cast<uintptr_t>(in) % 16 || bytes % 16)
        return fail(DESC_ERR_SHAPE, "read probe needs a 16-byte aligned base and size");
    if (bytes == 0) return DESC_OK;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (desc_status st = check_memspace(in, dev, "in")) return st;
    if (desc_status st = check_memspace(sink, dev, "sink")) return st;
    DevInfo di;
    if (desc_status st = device_info(dev, &di)) return st;
    const int grid = di.sms * 16 < 8 * 1024 ? di.sms * 16 : 8 * 1024;  // 16 x 256 threads/SM
                                                                         // (as the reduction)
    e = launch_plain_pdl(desc::read_probe_kernel, grid, 256, 0, static_cast<cudaStream_t>(stream),
                         static_cast<const uint4 *>(in), (int64_t)(bytes / 16),
                         static_cast<uint4 *>(sink));
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "read_probe launch");
    g_last_launches = 1;
    return DESC_OK;
}

desc_status desc_block_reduce(const void *in, void *out, int64_t n, int64_t block,
                              desc_dtype dtype, void *stream) {
    return run_reduce(in, out, n, block, dtype, static_cast<cudaStream_t>(stream));
}

size_t desc_scan_workspace(int64_t n, desc_dtype dtype) {
    const int es = rs_es(dtype);
    if (es == 0 || n <= 0) return 0;
    return (size_t)scan_workspace_bytes(n, es);
}

desc_status desc_scan(const void *in, void *out, int64_t n, desc_dtype dtype, void *d_work,
                      size_t work_bytes, void *stream) {
    return run_scan(in, out, n, dtype, d_work, work_bytes, DESC_SCAN_AUTO,
                    static_cast<cudaStream_t>(stream));
}

#ifdef DESC_SCAN_TRACE
// diagnostics builds only (not in the header): copy the per-tile trace stamps to the host
int desc_scan_trace_copy(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, desc::g_scan_trace, bytes);
}
#endif

desc_status desc_scan_ex(const void *in, void *out, int64_t n, desc_dtype dtype, void *d_work,
                         size_t work_bytes, desc_scan_algo algo, void *stream) {
    return run_scan(in, out, n, dtype, d_work, work_bytes, algo, static_cast<cudaStream_t>(stream));
}

desc_status desc_view_compile(int32_t ndim, const int64_t *shape, const int64_t *strides,
                              const desc_view_op *ops, int32_t nops, desc_strided_view *out) {
    return view_compile(ndim, shape, strides, ops, nops, out);
}

desc_status desc_view_copy(const void *in, void *out, const desc_strided_view *view,
                           desc_dtype dtype, void *stream) {
    return view_copy(in, out, view, dtype_size(dtype), static_cast<cudaStream_t>(stream));
}

desc_status desc_copy_batched(const void *in, void *out, int64_t batch, int64_t rows, int64_t cols,
                              int64_t ld_in, int64_t ld_out, int64_t stride_in,
                              int64_t stride_out, desc_dtype dtype, void *stream) {
    return run_copy(in, out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                    dtype_size(dtype), static_cast<cudaStream_t>(stream));
}

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
    if (a.es == 0 || !tma_eligible(a) || tiled_preferred(a)) return DESC_KERNEL_TILED;
    if (narrow_vtiled(a)) return DESC_KERNEL_VTILED;
    return tma_store_ok(a) ? DESC_KERNEL_TMA_ST : DESC_KERNEL_TMA;
}

desc_status desc_transpose_host(const void *h_in, void *h_out, int64_t batch, int64_t rows,
                                int64_t cols, int64_t ld_in, int64_t ld_out, int64_t stride_in,
                                int64_t stride_out, desc_dtype dtype, void *d_work,
                                size_t work_bytes, void *stream) {
    return run_host(h_in, h_out, batch, rows, cols, ld_in, ld_out, stride_in, stride_out,
                    dtype_size(dtype), d_work, work_bytes, static_cast<cudaStream_t>(stream));
}

size_t desc_transpose_host_workspace(int64_t rows, int64_t cols, desc_dtype dtype) {
    const int es = dtype_size(dtype);
    if (es == 0 || rows <= 0 || cols <= 0) return 0;
    // Bands: the trade-off between pipeline fill/drain and per-copy DMA efficiency on PCIe
    // Gen5, 8192^2 f32 (scripts/exp_e2e.py): column bands (AUTO) 256 -> 85.7, 512 -> 87.3,
    // 1024 -> 88.0, 2048 -> 87.7 GB/s; row bands 256 -> 71.8, 512 -> 82.5, 1024 -> 82.5
    // (profiles/r02_exp_e2e_axis.txt).  Sized for either axis (run_host, DESC_HOST_AXIS).
    const int64_t br = rows < 512 ? rows : 512, bc = cols < 1024 ? cols : 1024;
    const int64_t a = band_bytes(br, cols, es), b = band_bytes(bc, rows, es);
    return (size_t)(a > b ? a : b);
}

desc_status desc_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                        size_t width, size_t height, void *stream) {
    g_last_launches = 0;
    if (width == 0 || height == 0) return DESC_OK;
    if (!dst || !src) return fail(DESC_ERR_NULL, "null %s pointer", dst ? "src" : "dst");
    if (width > spitch || width > dpitch)
        return fail(DESC_ERR_SHAPE, "width %zu exceeds a pitch (%zu, %zu)", width, spitch, dpitch);
    cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                      static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync");
    return DESC_OK;
}

size_t desc_transpose_host_workspace_batched(int64_t batch, int64_t rows, int64_t cols,
                                             desc_dtype dtype) {
    const size_t one = desc_transpose_host_workspace(rows, cols, dtype);
    const int es = dtype_size(dtype);
    if (es == 0 || batch <= 1 || rows <= 0 || cols <= 0) return one;
    // whole-matrix bands (run_host): ~32 MB of input per band and at least 8 bands
    // (scripts/exp_e2e_batch.py, 256 x 1024^2 f32: 4 / 16 / 32 matrices per band 92.5 /
    // 93.1 / 90.0 GB/s against 77 GB/s for one matrix per band or the zero-copy path)
    const int64_t in_m = round_up(rows * cols * es, 256), out_m = in_m;
    int64_t nb = ((int64_t)32 << 20) / in_m;
    if (nb < 1) nb = 1;
    const int64_t cap = (batch + 7) / 8;
    if (nb > cap) nb = cap;
    const size_t want = (size_t)(2 * nb * (in_m + out_m));
    return want > one ? want : one;
}

desc_status desc_ipc_handle(const void *dptr, void *handle_out, uint64_t *offset_out) {
    if (!dptr || !handle_out || !offset_out) return fail(DESC_ERR_NULL, "null pointer");
    // the handle names the whole allocation (a caching allocator sub-allocates), so also
    // report dptr's offset from the allocation base (cuMemGetAddressRange)
    static PFN_cuMemGetAddressRange_v3020 range = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
    });
    if (!range) return fail(DESC_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr));
    if (r != CUDA_SUCCESS) return fail(DESC_ERR_CUDA, "cuMemGetAddressRange failed (CUresult %d)", (int)r);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == DESC_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
    return DESC_OK;
}

desc_status desc_ipc_open(const void *handle, void **dptr_out) {
    if (!handle || !dptr_out) return fail(DESC_ERR_NULL, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    return DESC_OK;
}

desc_status desc_ipc_close(void *dptr) {
    if (!dptr) return fail(DESC_ERR_NULL, "null pointer");
    cudaError_t e = cudaIpcCloseMemHandle(dptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return DESC_OK;
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
