/*
 * oracle/transpose_ref.c -- the CPU ORACLE for the matrix transpose.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link,
 * load or call this file.  It is used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg, nothing else.  It shares no
 * code, header, table or helper with paper_2305_03448_b200/ (the CUDA path).
 *
 * What it computes (PAPER.md, Descend arxiv 2305.03448):
 *   P:40   "a CUDA kernel function ... to transpose a matrix"
 *   P:77   "the matrix transposition function in Descend"  (Listing 2)
 *   P:108  caption "A Descend function performing matrix transposition."
 *   P:539-540  view `transpose : [[ [[d;n]]; m]] -> [[ [[d;m]]; n]]`
 * i.e. the plain definition   out[j][i] = in[i][j],  0 <= i < rows, 0 <= j < cols,
 * where `in` is rows x cols and `out` is cols x rows (reading R7).
 *
 * Generalisations (readings R6-R8, R10, R11):
 *   - leading dimensions ld_in >= cols, ld_out >= rows, counted in ELEMENTS;
 *   - a batch of independent transposes with element strides stride_in/out;
 *   - elements are opaque `es`-byte cells copied with memcpy: a transpose moves
 *     bits and performs no arithmetic, so f32/i32 (es=4) and f64 (es=8) are
 *     the same operation (R4, R11).  No floating-point conversion happens
 *     (this is exactly the P:51 `float tmp` bug the reading R4 forbids);
 *   - bytes of `out` outside the logical region (padding, guard bands) are
 *     never touched (R8);
 *   - an empty shape is a no-op (R10).
 *
 * It is deliberately a naive loop in the definition's order (b, then i, then
 * j): no blocking, no tiling, no reordering, no threads, no intrinsics.
 *
 * Parity pins: see tests/test_oracle.py (numpy .T copy, self-describing
 * decode, involution, block identity, 1xN memcpy, the paper's corrected
 * Listing 1 schedule simulated from P:49-60 with the P:44 fix).
 *
 * Build: gcc -O2 -shared -fPIC -o oracle/liboracle_transpose.so oracle/transpose_ref.c
 */
#include <stdint.h>
#include <string.h>

/* Returns 0 on success, -1 on an argument the definition does not cover. */
int oracle_transpose_batched(const void *in, void *out,
                             int64_t batch, int64_t rows, int64_t cols,
                             int64_t ld_in, int64_t ld_out,
                             int64_t stride_in, int64_t stride_out,
                             int64_t es)
{
    if (batch < 0 || rows < 0 || cols < 0 || es <= 0) return -1;
    if (batch == 0 || rows == 0 || cols == 0) return 0;       /* R10: no-op */
    if (!in || !out) return -1;
    if (ld_in < cols || ld_out < rows) return -1;
    if (stride_in < 0 || stride_out < 0) return -1;

    const unsigned char *src = (const unsigned char *)in;
    unsigned char *dst = (unsigned char *)out;
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t i = 0; i < rows; ++i) {
            for (int64_t j = 0; j < cols; ++j) {
                /* out[b][j][i] = in[b][i][j] */
                const int64_t s = b * stride_in + i * ld_in + j;
                const int64_t d = b * stride_out + j * ld_out + i;
                memcpy(dst + d * es, src + s * es, (size_t)es);
            }
        }
    }
    return 0;
}

int oracle_transpose(const void *in, void *out, int64_t rows, int64_t cols,
                     int64_t ld_in, int64_t ld_out, int64_t es)
{
    return oracle_transpose_batched(in, out, 1, rows, cols, ld_in, ld_out,
                                    0, 0, es);
}
