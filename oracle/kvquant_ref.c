/* Scalar C restatement of the reference KV quantizer — TEST INFRASTRUCTURE ONLY.
 *
 * Follows /root/reference/pkg/src/servesim/kvmanager.py:
 *   quantize   :108-149   dequantize :152-154
 * Built with -ffp-contract=off (see oracle/Makefile): the reference is numpy
 * float64, which never fuses multiply-add; with contraction the snap loop's
 * s*(qmax-z) - s*(0-z) fuses and ~11% of INT8 row scales differ.
 * rint() runs in the default round-to-nearest-even mode.
 *
 * Used by tests as a second, independent restatement (cross-checked against
 * oracle/kv_oracle.py and the golden vectors) and as a fast checker at sizes
 * numpy would take minutes on.  Never linked into the product library.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* status: 0 ok, 1 bad args, 2 non-finite input */
int oracle_quantize_f64(const double *x, int64_t rows, int64_t len, int bits,
                        uint8_t *codes, double *scale, double *zero) {
    if ((bits != 4 && bits != 8) || rows <= 0 || len <= 0) return 1;
    const double qmax = (double)((1 << bits) - 1);
    for (int64_t r = 0; r < rows; ++r) {
        const double *row = x + r * len;
        double lo = row[0], hi = row[0];
        for (int64_t i = 0; i < len; ++i) {
            double v = row[i];
            if (!isfinite(v)) return 2;
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
        double s, z;
        if (hi == lo) {
            s = 1.0; z = -lo;
        } else {
            s = (hi - lo) / qmax;
            z = rint(-lo / s);
            for (int it = 0; it < 32; ++it) {
                double a = s * (qmax - z);
                double b = s * (0.0 - z);
                double nxt = (a - b) / qmax;
                if (nxt == s) break;
                s = nxt;
            }
        }
        scale[r] = s; zero[r] = z;
        uint8_t *q = codes + r * len;
        for (int64_t i = 0; i < len; ++i) {
            double t = rint(row[i] / s + z);
            if (t < 0.0) t = 0.0;
            if (t > qmax) t = qmax;
            q[i] = (uint8_t)t;
        }
    }
    return 0;
}

/* fp16 bit patterns in, same semantics (fp16 -> f64 is exact). */
static double half_to_double(uint16_t h) {
    int sign = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m | 1024), e - 25);
    return sign ? -v : v;
}

int oracle_quantize_f16(const uint16_t *x, int64_t rows, int64_t len, int bits,
                        uint8_t *codes, double *scale, double *zero, double *scratch) {
    /* scratch: len doubles */
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t i = 0; i < len; ++i) scratch[i] = half_to_double(x[r * len + i]);
        int st = oracle_quantize_f64(scratch, 1, len, bits, codes + r * len, scale + r, zero + r);
        if (st) return st;
    }
    return 0;
}

void oracle_dequantize(const uint8_t *codes, const double *scale, const double *zero,
                       int64_t rows, int64_t len, double *out) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t i = 0; i < len; ++i)
            out[r * len + i] = scale[r] * ((double)codes[r * len + i] - zero[r]);
}
