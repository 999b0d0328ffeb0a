/*
 * approx8_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference codec (approx8/codecs.py:131-288) used as a fast checker for
 * large parity cases.  It is never linked into or called by the product.
 *
 * Algorithm, following the reference line by line:
 *   payload values        codecs.py:136-158   (float64 formulas)
 *   decode table          codecs.py:189-192   (float32, -0 folded to +0)
 *   distinct sorted set   codecs.py:194-200   (lowest code per value)
 *   scale                 codecs.py:232-241   (absmax | 10^d | 1 -> float32)
 *   encode                codecs.py:260-268   (float64 y = |x|/s, left binary
 *                         search clipped to [1, D-1], ties to the smaller
 *                         value, sign bit only for non-zero values)
 *   decode                codecs.py:281       (table[c] * scale, float32)
 *
 * Built by oracle/Makefile into oracle/_build/liba8oracle.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    float table[256];
    double values[128];
    uint8_t codes[128];
    int D;
} book_t;

static double centre(int k, int t) { return 0.1 + (k + 0.5) * 0.9 / (double)(1 << t); }

static void payload(int kind, double* v) {
    for (int p = 0; p < 128; ++p) {
        double x = 0.0;
        if (kind == 0 && p) { /* dynamic-tree */
            int bl = 0;
            for (int q = p; q; q >>= 1) ++bl;
            int z = 7 - bl, t = 6 - z;
            x = centre(p - (1 << t), t) * pow(10.0, -z);
        } else if (kind == 1 && p) { /* static-tree */
            x = centre(p & 15, 4) * pow(10.0, -(p >> 4));
        } else if (kind == 3) { /* mantissa */
            x = (double)(p & 15) * pow(10.0, -(p >> 4));
        } else if (kind == 2) { /* linear */
            x = p / 127.0;
        }
        v[p] = x;
    }
}

static void make_book(int kind, book_t* b) {
    double v[128];
    payload(kind, v);
    for (int p = 0; p < 128; ++p) {
        float f = (float)v[p], g = -f;
        b->table[p] = f == 0.0f ? 0.0f : f;
        b->table[128 + p] = g == 0.0f ? 0.0f : g;
    }
    /* insertion sort of (value, code) keeps the lowest code first */
    double sv[128];
    uint8_t sc[128];
    for (int p = 0; p < 128; ++p) {
        double x = (double)b->table[p];
        int i = p;
        while (i > 0 && sv[i - 1] > x) {
            sv[i] = sv[i - 1];
            sc[i] = sc[i - 1];
            --i;
        }
        sv[i] = x;
        sc[i] = (uint8_t)p;
    }
    int d = 0;
    for (int i = 0; i < 128; ++i) {
        if (d && b->values[d - 1] == sv[i]) continue;
        b->values[d] = sv[i];
        b->codes[d] = sc[i];
        ++d;
    }
    b->D = d;
}

/* returns 0 ok, 1 non-finite input (reference InputError), 2 bad spec */
int a8o_encode(const float* x, int64_t n, int kind, int norm, int decades, uint8_t* codes, float* scale_out) {
    if (kind < 0 || kind > 3) return 2;
    book_t b;
    make_book(kind, &b);
    double peak = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(x[i])) return 1;
        double a = fabs((double)x[i]);
        if (a > peak) peak = a;
    }
    double s = 1.0;
    if (norm == 1) s = peak > 0.0 ? peak : 1.0;
    if (norm == 2) s = pow(10.0, decades);
    float sf = (float)s;
    *scale_out = sf;
    s = (double)sf;
    const int D = b.D;
    for (int64_t i = 0; i < n; ++i) {
        const double xv = (double)x[i];
        const double y = fabs(xv) / s;
        int lo = 0, hi = D; /* first index with values[idx] >= y */
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (b.values[mid] < y)
                lo = mid + 1;
            else
                hi = mid;
        }
        int idx = lo < 1 ? 1 : (lo > D - 1 ? D - 1 : lo);
        int pick = ((y - b.values[idx - 1]) <= (b.values[idx] - y)) ? idx - 1 : idx;
        uint8_t c = b.codes[pick];
        if (xv < 0 && b.values[pick] != 0.0) c |= 0x80;
        codes[i] = c;
    }
    return 0;
}

int a8o_decode(const uint8_t* codes, int64_t n, int kind, float scale, float* out) {
    if (kind < 0 || kind > 3) return 2;
    book_t b;
    make_book(kind, &b);
    for (int64_t i = 0; i < n; ++i) out[i] = b.table[codes[i]] * scale;
    return 0;
}
