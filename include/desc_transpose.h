/*
 * desc_transpose.h -- C ABI of the B200-native tiled matrix transpose
 * (the running example of "Descend: A Safe GPU Systems Programming Language",
 * arxiv 2305.03448).
 *
 * Operation ("transpose a matrix", P:77 / Listing 2 P:90-105,
 * caption P:108, view type P:539-540; full elementwise transpose per DESIGN.md
 * reading R1):
 *
 *     out[b][j][i] = in[b][i][j]      0 <= b < batch, 0 <= i < rows, 0 <= j < cols
 *
 * Layout.  All counts, leading dimensions and strides are in ELEMENTS (int64).
 *   in  : batch matrices, each rows x cols, row-major, row pitch ld_in >= cols,
 *         matrix b starts at in + b*stride_in.
 *   out : batch matrices, each cols x rows, row-major, row pitch ld_out >= rows,
 *         matrix b starts at out + b*stride_out.
 *   Elements are opaque cells of desc_dtype_size(dtype) bytes: the library never
 *   converts, so every bit pattern (NaN payloads, -0.0, subnormals) is moved
 *   bit-exactly (R4, R11).  Bytes of `out` outside the logical
 *   cols x rows regions (padding columns, gaps between matrices) are never
 *   written (R8).
 *
 * Ownership (P:90-91 `&` / `&uniq`; R9).
 *   `in` is a shared, read-only borrow; `out` is a unique borrow until the
 *   stream reaches the operation.  The byte ranges spanned by in and out must
 *   not overlap (DESC_ERR_ALIAS); in-place transposition is not supported.
 *   For batch > 1 the output matrices must be pairwise disjoint (the narrowing
 *   rule), in one of two layouts: stacked, stride_out >= (cols-1)*ld_out
 *   + rows; or side by side within each output row, stride_out >= rows and
 *   (batch-1)*stride_out + rows <= ld_out.  Otherwise DESC_ERR_SHAPE.  Input matrices may overlap (read-only).  Strides must be >= 0.
 *   The caller owns both buffers; the library allocates no device memory for data
 *   (the one exception: a 16-byte tile counter per (device, stream) for the TMA-store
 *   kernel's dynamic scheduler, created on first use and kept for the process) and
 *   keeps a host-side, thread-safe cache of TMA descriptors.
 *
 * Memory space.
 *   Both pointers must be device (or managed) memory of the CURRENT device, or of a
 *   peer device the current device can access (an IPC-mapped slab of another rank,
 *   desc_ipc_open), checked with cudaPointerGetAttributes, else DESC_ERR_MEMSPACE.
 *   desc_transpose_host is the one entry point that takes host buffers.
 *
 * Launch configuration.  Derived inside the library from the shape
 *   and the device's SM count: the caller passes no grid or block sizes, so the
 *   "shared assumptions" bug of P:278-299 cannot occur.
 *
 * Synchronisation and errors.  Device entry points are ASYNCHRONOUS on `stream`
 *   (a cudaStream_t passed as void*; NULL = legacy default stream).  This
 *   deviates from Descend's implicit host wait.  Argument errors return
 *   before any launch; a failed launch returns DESC_ERR_CUDA.  Nothing is thrown
 *   across the ABI.  desc_last_error() returns a thread-local message for the
 *   last non-OK status of the calling thread.  Empty shapes (batch, rows or
 *   cols == 0) are a successful no-op with no launch (R10).
 */
#ifndef DESC_TRANSPOSE_H
#define DESC_TRANSPOSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DESC_VERSION 100 /* 1.0.0 */

typedef enum desc_status {
    DESC_OK = 0,
    DESC_ERR_NULL = 1,      /* a required pointer is NULL                          */
    DESC_ERR_SHAPE = 2,     /* negative size, ld < extent, overlapping batch outputs,
                               int64 overflow of an extent, unsupported geometry    */
    DESC_ERR_DTYPE = 3,     /* unknown desc_dtype                                   */
    DESC_ERR_ALIAS = 4,     /* in and out byte ranges overlap (&uniq)     */
    DESC_ERR_MEMSPACE = 5,  /* pointer not device memory of the current device       */
    DESC_ERR_CUDA = 6,      /* CUDA runtime/driver error (see desc_last_error)       */
    DESC_ERR_KERNEL = 7     /* requested kernel variant cannot run these arguments   */
} desc_status;

typedef enum desc_dtype {
    DESC_F32 = 0, DESC_F64 = 1, DESC_I32 = 2, DESC_I64 = 3,
    DESC_F16 = 4, DESC_BF16 = 5, DESC_U8 = 6
} desc_dtype;

/* Kernel variants (desc_transpose_ex).  AUTO picks TILED for 4/8-byte cells when rows
 * and cols are both >= 64 (measured fastest there) and whenever the TMA alignment rules
 * below fail; VTILED for 1/2-byte cells when its rules hold (rows, cols multiples of
 * 16/size); otherwise TMA_ST when the element size is 4 or 8 with rows*size >= 16,
 * else TMA.
 *   DESC_KERNEL_SMEM : 32x32 shared-memory tile, padded [32][33], 32x8 threads,
 *                      predicated edges -- the corrected Listing 1 schedule
 *                      (P:49-60 with the P:44 fix).  Any alignment.  Kept as the
 *                      paper's schedule (baseline); AUTO never picks it.
 *   DESC_KERNEL_TILED : any alignment; 64x64 (8-byte cells: 32x64) tiles padded by one
 *                      cell, 256 threads each issuing all of its 16 (8) cell loads
 *                      before staging, one tile per CTA, predicated edge tiles.
 *   DESC_KERNEL_TMA  : persistent, warp-specialised: TMA (cp.async.bulk.tensor)
 *                      loads of 128-byte-swizzled tiles into a multi-stage
 *                      mbarrier ring, conflict-free 16-byte shared reads,
 *                      register micro-transposes, 16-byte coalesced stores.
 *                      Needs 16-byte aligned in/out bases and ld*size,
 *                      stride*size multiples of 16 bytes (when batch > 1);
 *                      element size 1, 2, 4 or 8.
 *   DESC_KERNEL_TMA_ST : as DESC_KERNEL_TMA, but the transposed tile is staged in
 *                      128-byte-swizzled shared memory and written with TMA bulk
 *                      tensor stores (cp.async.bulk.tensor shared->global).  Same
 *                      alignment rules; element size 4 or 8.
 *   DESC_KERNEL_TMA_TILE : one 16 KB tile per 128-thread CTA (64x64 for 4-byte cells,
 *                      32x64 for 8-byte cells), many CTAs per SM: TMA box loads on one
 *                      mbarrier, conflict-free register micro-transposes written back
 *                      into the same (swizzled) buffer, TMA bulk tensor stores.  Same
 *                      alignment rules as DESC_KERNEL_TMA_ST; element size 4 or 8.
 *   DESC_KERNEL_VTILED : one tile per CTA (64x64 cells for 4-byte, 32x32 for 8-byte,
 *                      128x64 for 2-byte, 256x128 for 1-byte cells) staged with 16-byte
 *                      cp.async copies into a 16-byte XOR-swizzled shared tile
 *                      (conflict-free both ways, no padding), VEC x VEC register
 *                      micro-transposes (VEC = 16/size), 16-byte coalesced stores.  Needs
 *                      the TMA alignment rules above plus rows and cols multiples of
 *                      16/size; any element size.  */
typedef enum desc_kernel {
    DESC_KERNEL_AUTO = 0,
    DESC_KERNEL_SMEM = 1,
    DESC_KERNEL_TMA = 2,
    DESC_KERNEL_TMA_ST = 3,
    DESC_KERNEL_TILED = 4,
    DESC_KERNEL_TMA_TILE = 5,
    DESC_KERNEL_VTILED = 6
} desc_kernel;

/* Single transpose: in (rows x cols, pitch ld_in) -> out (cols x rows, pitch ld_out). */
desc_status desc_transpose(const void *in, void *out, int64_t rows, int64_t cols,
                           int64_t ld_in, int64_t ld_out, desc_dtype dtype,
                           void *stream);

/* Batched: `batch` independent transposes (layout above). */
desc_status desc_transpose_batched(const void *in, void *out, int64_t batch,
                                   int64_t rows, int64_t cols, int64_t ld_in,
                                   int64_t ld_out, int64_t stride_in,
                                   int64_t stride_out, desc_dtype dtype,
                                   void *stream);

/* Batched with an explicit kernel variant (tests / A-B measurement).  Returns
 * DESC_ERR_KERNEL if the variant's alignment rules do not hold. */
desc_status desc_transpose_ex(const void *in, void *out, int64_t batch,
                              int64_t rows, int64_t cols, int64_t ld_in,
                              int64_t ld_out, int64_t stride_in,
                              int64_t stride_out, desc_dtype dtype,
                              desc_kernel kernel, void *stream);

/* The variant AUTO would run for these arguments (no launch, no pointer
 * checks beyond alignment).  Returns DESC_KERNEL_TILED, _VTILED, _TMA or _TMA_ST. */
desc_kernel desc_select_kernel(const void *in, const void *out, int64_t batch,
                               int64_t rows, int64_t cols, int64_t ld_in,
                               int64_t ld_out, int64_t stride_in,
                               int64_t stride_out, desc_dtype dtype);

/* Host-buffer transpose (same operation and layout rules as desc_transpose_batched,
 * but h_in / h_out are HOST memory -- pinned for full PCIe overlap, pageable works).
 * The library streams column bands of the input (= row bands of the output: 2-D H2D
 * copies, contiguous D2H copies -- PCIe reads strided host rows faster than it writes
 * them) through the caller-provided device workspace d_work (256-byte aligned,
 * work_bytes >= desc_transpose_host_workspace recommended; smaller works down to one
 * column): H2D copy of band k+1, transpose of band k and D2H copy of band k-1 overlap on
 * two internal streams.  When that would
 * take more than 64 bands (e.g. many small batched matrices) and both host buffers are
 * page-locked and mapped, one TILED kernel instead reads and writes the host buffers
 * directly over PCIe (zero-copy; d_work is then unused).  Asynchronous on
 * `stream` like the device entry points: the host buffers must stay valid and
 * untouched until the stream reaches the end of the operation.  h_in/h_out that are
 * device memory give DESC_ERR_MEMSPACE; a too-small workspace gives DESC_ERR_SHAPE. */
desc_status desc_transpose_host(const void *h_in, void *h_out, int64_t batch,
                                int64_t rows, int64_t cols, int64_t ld_in,
                                int64_t ld_out, int64_t stride_in,
                                int64_t stride_out, desc_dtype dtype, void *d_work,
                                size_t work_bytes, void *stream);

/* 2-D copy of `height` rows of `width` bytes between any two memory spaces (host <-> device,
 * device <-> device; direction inferred through unified addressing), asynchronous on
 * `stream`: the host-buffer slab pipeline's (paper_2305_03448_b200/dist.py
 * slab_transpose_host) H2D of input column stripes.  Plumbing, no method arithmetic.
 * width > spitch or width > dpitch gives DESC_ERR_SHAPE; null pointers DESC_ERR_NULL; a zero
 * width or height is a no-op. */
desc_status desc_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                        size_t width, size_t height, void *stream);

/* Strided batched copy, NO transposition:  out[b][i][j] = in[b][i][j]
 * (in: rows x cols, pitch ld_in >= cols; out: rows x cols, pitch ld_out >= cols; batch
 * strides as above).  The unpack step of the distributed slab transpose
 * (paper_2305_03448_b200/dist.py): P received R x R blocks placed side by side in the
 * output slab.  Same ownership / memory-space / error rules as desc_transpose_batched
 * (output matrices pairwise disjoint: stacked, stride_out >= (rows-1)*ld_out + cols,
 * or side by side, stride_out >= cols and (batch-1)*stride_out + cols <= ld_out). */
desc_status desc_copy_batched(const void *in, void *out, int64_t batch, int64_t rows,
                              int64_t cols, int64_t ld_in, int64_t ld_out,
                              int64_t stride_in, int64_t stride_out, desc_dtype dtype,
                              void *stream);

/* CUDA IPC plumbing for the fused peer-to-peer distributed transpose (dist.py):
 * desc_ipc_handle exports the allocation containing dptr as a DESC_IPC_HANDLE_BYTES-byte
 * handle plus dptr's byte offset inside that allocation; desc_ipc_open maps a peer's
 * handle into this process (peer access enabled lazily) and returns the allocation BASE
 * (add the exported offset); desc_ipc_close unmaps it.  Errors: DESC_ERR_NULL,
 * DESC_ERR_CUDA. */
#define DESC_IPC_HANDLE_BYTES 64
desc_status desc_ipc_handle(const void *dptr, void *handle_out, uint64_t *offset_out);
desc_status desc_ipc_open(const void *handle, void **dptr_out);
desc_status desc_ipc_close(void *dptr);

/* ---- view-composed copies (Listing 3) ----
 * Descend's basic views on a (nested) array: group<k>, transpose (outer two dims), split<k>
 * (.fst / .snd), reverse; map(v) is encoded as v applied at `depth` = number of enclosing
 * maps.  A chain of views over a strided root compiles (on the host, no GPU needed) to a
 * strided view: element v of the view lives at in[offset + sum_d v_d * stride[d]] (strides
 * in elements, negative after reverse) -- "views are compiled into raw indices"
 * (P:509-511).  desc_view_copy materialises it: out (contiguous, the view's
 * row-major order, prod(shape) elements) = the view of `in`.  Views whose innermost dim
 * transposes onto an input-contiguous dim run on the TMA transpose kernels; the rest on a
 * row-gather kernel (16-byte vectors when rows are contiguous).  Errors: DESC_ERR_SHAPE for
 * a view the types of Listing 3 reject (group with k not dividing n -- reading R12; split
 * with k > n; transpose of a flat array; map deeper than the nesting; > DESC_MAX_DIMS
 * dims; a view reaching before `in`), plus the usual NULL / DTYPE / ALIAS / MEMSPACE /
 * CUDA rules.  The caller guarantees the compiled view lies inside the `in` allocation. */
#define DESC_MAX_DIMS 8
typedef enum desc_view_kind {
    DESC_VIEW_GROUP = 0, DESC_VIEW_TRANSPOSE = 1, DESC_VIEW_SPLIT_FST = 2,
    DESC_VIEW_SPLIT_SND = 3, DESC_VIEW_REVERSE = 4
} desc_view_kind;
typedef struct desc_view_op {
    int32_t kind;   /* desc_view_kind                                  */
    int32_t depth;  /* number of enclosing map(...) (0 = outermost dim) */
    int64_t k;      /* nat argument of group / split (ignored otherwise) */
} desc_view_op;
typedef struct desc_strided_view {
    int32_t ndim;
    int32_t reserved;
    int64_t offset;                 /* elements                           */
    int64_t shape[DESC_MAX_DIMS];
    int64_t stride[DESC_MAX_DIMS];  /* elements, may be negative          */
} desc_strided_view;

/* Compile a view chain over a root of rank ndim (shape; strides in elements, NULL =
 * C-contiguous) into *out.  Host only. */
desc_status desc_view_compile(int32_t ndim, const int64_t *shape, const int64_t *strides,
                              const desc_view_op *ops, int32_t nops,
                              desc_strided_view *out);

/* out[0 .. prod(view->shape)) = the view of in, in the view's row-major order. */
desc_status desc_view_copy(const void *in, void *out, const desc_strided_view *view,
                           desc_dtype dtype, void *stream);

/* ---- the paper's other memory-bound benchmarks ----
 * Block-wide reduction: out[b] = sum(in[b*block .. min(n, (b+1)*block))), b < ceil(n/block),
 * out has the input's dtype.  Integers (DESC_U8, DESC_I32, DESC_I64) sum modulo 2^bits
 * (bit-exact); DESC_F32 accumulates in fp64 and rounds once; DESC_F64 in fp64 (float results
 * depend on the summation order only within the usual gamma_B * sum|x| bound; the order is
 * fixed for a given n, block, dtype, input alignment and device (its SM count and occupancy
 * pick the summing group -- warp, CTA or cluster -- and the CTA size, so f32/f64 sums may
 * differ in the last bits between devices or MIG slices): no atomics, runs on one device
 * repeat bit for bit;
 * the launch configuration is derived inside).  DESC_F16 /
 * DESC_BF16 give DESC_ERR_DTYPE; block <= 0 or n < 0 give DESC_ERR_SHAPE; in/out overlap
 * gives DESC_ERR_ALIAS.  Asynchronous on `stream`. */
desc_status desc_block_reduce(const void *in, void *out, int64_t n, int64_t block,
                              desc_dtype dtype, void *stream);

/* Inclusive scan: out[i] = sum(in[0..i]), same dtypes and arithmetic as desc_block_reduce.
 * Needs a device workspace of desc_scan_workspace(n, dtype) bytes, 256-byte aligned (tile
 * status; zeroed by the call with a reset kernel on `stream`), else DESC_ERR_SHAPE.  in ==
 * out (in place) is allowed; partial overlap gives DESC_ERR_ALIAS.
 * Algorithms (desc_scan_ex; desc_scan = AUTO):
 *   DESC_SCAN_LOOKBACK  : state reset + one launch, one 8-32 KB tile per CTA, decoupled look-back.
 *   DESC_SCAN_THREE_PASS: tile aggregates -> aggregate scan -> tile scans (3 launches,
 *                         3 n bytes of traffic; the paper's multi-kernel shape).
 *   DESC_SCAN_STREAM    : state reset + one launch, persistent CTAs stream 32-48 KB tiles
 *                         through a shared-memory ring (TMA loads) with a coalesced
 *                         look-back; results of 4/8-byte types leave through swizzled
 *                         staging and TMA tensor stores; 2 n bytes.  Needs 16-byte
 *                         aligned in and out.
 * AUTO takes STREAM for aligned arrays of >= 2 tiles per SM, LOOKBACK for shorter ones,
 * THREE_PASS for unaligned long ones.  An explicit algorithm whose rule does not hold
 * gives DESC_ERR_KERNEL. */
typedef enum desc_scan_algo {
    DESC_SCAN_AUTO = 0,
    DESC_SCAN_LOOKBACK = 1,
    DESC_SCAN_THREE_PASS = 2,
    DESC_SCAN_STREAM = 3
} desc_scan_algo;
size_t desc_scan_workspace(int64_t n, desc_dtype dtype);
desc_status desc_scan(const void *in, void *out, int64_t n, desc_dtype dtype, void *d_work,
                      size_t work_bytes, void *stream);
desc_status desc_scan_ex(const void *in, void *out, int64_t n, desc_dtype dtype, void *d_work,
                         size_t work_bytes, desc_scan_algo algo, void *stream);

/* Fused transpose + exchange of the distributed slab transpose (BASELINE north_star (4);
 * SURVEY.md 8(f) NEXT #1; reading R13) in ONE launch.  The global M x N matrix is
 * held as row slabs: this rank r of P owns input rows [r*Rm, (r+1)*Rm), Rm = M/P, as in_slab
 * (Rm x N, row pitch N); rank s owns output rows [s*Rn, (s+1)*Rn) of the N x M transpose,
 * Rn = N/P, as out_slabs[s] (Rn x M, pitch M) -- this rank's own slab, or another rank's slab
 * mapped into this process (desc_ipc_open; same device or a peer device this one can access).
 * Writes block (r, s)^T = (in_slab[:, s*Rn : (s+1)*Rn])^T into columns [r*Rm, (r+1)*Rm) of
 * out_slabs[s] for every s: one TILED launch whose tiles pick their destination slab, so the
 * local transpose and every rank's NVLink stores run in the same kernel (2S HBM per rank, no
 * pack / unpack, no NCCL kernels).  Only this rank's column blocks are written.
 * 1 <= P <= 8, 0 <= r < P, P | M, P | N, Rn a multiple of the tile width (64 cells for 4-byte,
 * 32 for 8-byte types), else DESC_ERR_SHAPE; 4/8-byte dtypes only (DESC_ERR_DTYPE); in_slab
 * overlapping an out slab gives DESC_ERR_ALIAS.  Asynchronous on `stream`; it does NOT order
 * the ranks: the caller completes every rank's call (e.g. a group barrier after the stream)
 * before any rank reads its slab. */
desc_status desc_slab_transpose_peer(const void *in_slab, void *const *out_slabs, int32_t P,
                                     int32_t r, int64_t M, int64_t N, desc_dtype dtype,
                                     void *stream);

/* Measurement helper (not part of the method): the HBM READ-only roofline of the block-wide
 * reduction (the reduction reads n elements and writes n/block).  Reads `bytes` bytes
 * of device memory at `in` (16-byte aligned, bytes a multiple of 16) with 16-byte
 * ld.global.nc loads, 8 in flight per lane, one wave of CTAs grid-striding, XOR-folds them and
 * writes one 16-byte word per CTA to `sink` (device memory of >= desc_read_probe_sink_bytes()
 * bytes).  Asynchronous on `stream`.  DESC_ERR_SHAPE for a misaligned base or size,
 * DESC_ERR_NULL / DESC_ERR_MEMSPACE as elsewhere. */
desc_status desc_read_probe(const void *in, size_t bytes, void *sink, void *stream);
size_t desc_read_probe_sink_bytes(void);

/* Recommended workspace bytes for desc_transpose_host (double-buffered 1024-column bands,
 * or 512-row bands if larger). */
size_t desc_transpose_host_workspace(int64_t rows, int64_t cols, desc_dtype dtype);

/* Recommended workspace bytes for a BATCHED desc_transpose_host call whose matrices are
 * stored back to back with a tight output (stride_in = rows*ld_in, ld_out = rows, stride_out
 * = cols*rows): room for whole-matrix bands of ~32 MB of input (at least 8 bands), which move
 * each band with one contiguous H2D and one contiguous D2H copy.  Never less than
 * desc_transpose_host_workspace(rows, cols, dtype). */
size_t desc_transpose_host_workspace_batched(int64_t batch, int64_t rows, int64_t cols,
                                             desc_dtype dtype);

/* Number of kernel launches the last successful call of this thread issued (0 for an
 * empty shape, 1 per device call, one per band for desc_transpose_host). */
int desc_last_launch_count(void);

const char *desc_status_string(desc_status s);
const char *desc_last_error(void);
size_t desc_dtype_size(desc_dtype t);
int desc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DESC_TRANSPOSE_H */
