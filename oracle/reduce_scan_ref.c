/*
 * oracle/reduce_scan_ref.c -- CPU ORACLE for the paper's two other memory-bound evaluation
 * kernels.  TEST INFRASTRUCTURE ONLY (see transpose_ref.c).
 *
 * PAPER.md P:1047 "block-wide parallel reduction, matrix transposition, scan and matrix
 * multiplication"; "The scan benchmark uses two different kernels".  The paper gives
 * no code for either, so the oracle is the plain definition of each (R18, R19):
 *
 *   block reduction:  out[b] = sum_{i = b*B}^{min(n, (b+1)*B) - 1} in[i],  b < ceil(n / B)
 *   inclusive scan:   out[i] = sum_{j <= i} in[j]
 *
 * Integers (es = 1, 2, 4, 8 bytes, two's complement) are summed modulo 2^(8 es) -- unsigned
 * wrap-around, the result every correct order of additions produces.  Floats (f32: es = 4,
 * f64: es = 8) are summed sequentially, left to right, in fp64, and returned as fp64.
 * Naive loops in the definition's order; nothing else.
 */
#include <stdint.h>
#include <string.h>

static uint64_t load_u(const unsigned char *p, int64_t i, int64_t es) {
    uint64_t v = 0;
    memcpy(&v, p + i * es, (size_t)es);    /* little-endian: low es bytes */
    return v;
}

static void store_u(unsigned char *p, int64_t i, int64_t es, uint64_t v) {
    memcpy(p + i * es, &v, (size_t)es);
}

static double load_f(const unsigned char *p, int64_t i, int64_t es) {
    if (es == 4) {
        float f;
        memcpy(&f, p + i * 4, 4);
        return (double)f;
    }
    double d;
    memcpy(&d, p + i * 8, 8);
    return d;
}

/* Integer block reduction: out has ceil(n/B) cells of es bytes. */
int oracle_block_reduce_int(const void *in, void *out, int64_t n, int64_t block, int64_t es) {
    if (n < 0 || block <= 0 || (es != 1 && es != 2 && es != 4 && es != 8)) return -1;
    const unsigned char *src = (const unsigned char *)in;
    unsigned char *dst = (unsigned char *)out;
    for (int64_t b = 0; b * block < n; ++b) {
        uint64_t s = 0;
        for (int64_t i = b * block; i < n && i < (b + 1) * block; ++i) s += load_u(src, i, es);
        store_u(dst, b, es, s);             /* keeps the low 8*es bits: sum mod 2^(8 es) */
    }
    return 0;
}

/* Float block reduction: out has ceil(n/B) doubles (sequential fp64 sums). */
int oracle_block_reduce_float(const void *in, double *out, int64_t n, int64_t block, int64_t es) {
    if (n < 0 || block <= 0 || (es != 4 && es != 8)) return -1;
    const unsigned char *src = (const unsigned char *)in;
    for (int64_t b = 0; b * block < n; ++b) {
        double s = 0.0;
        for (int64_t i = b * block; i < n && i < (b + 1) * block; ++i) s += load_f(src, i, es);
        out[b] = s;
    }
    return 0;
}

/* Integer inclusive scan, wrapping. */
int oracle_scan_int(const void *in, void *out, int64_t n, int64_t es) {
    if (n < 0 || (es != 1 && es != 2 && es != 4 && es != 8)) return -1;
    const unsigned char *src = (const unsigned char *)in;
    unsigned char *dst = (unsigned char *)out;
    uint64_t s = 0;
    for (int64_t i = 0; i < n; ++i) {
        s += load_u(src, i, es);
        store_u(dst, i, es, s);
    }
    return 0;
}

/* Float inclusive scan: out[i] = fp64 sequential prefix sum of in[0..i]. */
int oracle_scan_float(const void *in, double *out, int64_t n, int64_t es) {
    if (n < 0 || (es != 4 && es != 8)) return -1;
    const unsigned char *src = (const unsigned char *)in;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        s += load_f(src, i, es);
        out[i] = s;
    }
    return 0;
}
