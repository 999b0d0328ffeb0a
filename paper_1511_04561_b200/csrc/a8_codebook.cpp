// Host side of the C ABI: codebooks (K0), fixed scales, host decision tables.
//
// Codebook formulas follow approx8/codecs.py:131-204 and are evaluated in the
// same float64 operation order, then rounded to float32, so the tables are
// bit-identical to the reference (pinned by the sha256 digests in
// tests/golden/golden.json).
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "a8_core.cuh"
#include "approx8_b200.h"

namespace a8 {
thread_local std::string g_last_error;

int fail(int code, const char* msg) {
    g_last_error = msg;
    return code;
}
}  // namespace a8

using a8::fail;

extern "C" int a8_abi_version(void) { return A8_ABI_VERSION; }

extern "C" const char* a8_last_error(void) { return a8::g_last_error.c_str(); }

// Centre of slice k of [0.1, 1.0) cut into 2^t parts (codecs.py:131-133).
static double tree_centre(int k, int t) { return 0.1 + (k + 0.5) * 0.9 / (double)(1 << t); }

// codecs.py:136-158 -- 7-bit payload magnitudes, float64.
static void payload_values(int kind, double* v) {
    for (int p = 0; p < 128; ++p) v[p] = 0.0;
    switch (kind) {
        case A8_DYNAMIC_TREE:
            for (int p = 1; p < 128; ++p) {
                int bitlen = 0;
                for (int q = p; q; q >>= 1) ++bitlen;
                const int z = 7 - bitlen;  // leading zeros before the flag bit
                const int t = 6 - z;
                const int k = p - (1 << t);
                v[p] = tree_centre(k, t) * pow(10.0, (double)(-z));
            }
            break;
        case A8_STATIC_TREE:
            for (int p = 1; p < 128; ++p) v[p] = tree_centre(p & 15, 4) * pow(10.0, (double)(-(p >> 4)));
            break;
        case A8_MANTISSA:
            for (int p = 0; p < 128; ++p) v[p] = (double)(p & 15) * pow(10.0, (double)(-(p >> 4)));
            break;
        case A8_LINEAR:
            for (int p = 0; p < 128; ++p) v[p] = (double)p / 127.0;
            break;
    }
}

extern "C" int a8_codebook(int kind, a8_book_t* out) {
    if (!out) return fail(A8_ERR_USAGE, "a8_codebook: null output");
    if (kind < 0 || kind > 3) return fail(A8_ERR_CONFIG, "a8_codebook: unknown data type kind");
    memset(out, 0, sizeof(*out));
    double pay[128];
    payload_values(kind, pay);
    for (int p = 0; p < 128; ++p) {
        float f = (float)pay[p];
        float g = -f;
        if (f == 0.0f) f = 0.0f;  // fold -0 into +0 (codecs.py:192)
        if (g == 0.0f) g = 0.0f;
        out->table[p] = f;
        out->table[128 + p] = g;
    }
    // distinct non-negative values ascending, each with its first (lowest)
    // payload index (np.unique(..., return_index=True), codecs.py:194-200)
    int order[128];
    for (int p = 0; p < 128; ++p) order[p] = p;
    std::stable_sort(order, order + 128, [&](int a, int b) {
        return (double)out->table[a] < (double)out->table[b];
    });
    int d = 0;
    for (int i = 0; i < 128; ++i) {
        const double v = (double)out->table[order[i]];
        if (d > 0 && out->values[d - 1] == v) continue;  // stable: first index kept
        out->values[d] = v;
        out->codes[d] = (uint8_t)order[i];
        ++d;
    }
    for (int i = d; i < 128; ++i) {  // padding for the branch-free search
        out->values[i] = out->values[d - 1];
        out->codes[i] = out->codes[d - 1];
    }
    out->ndistinct = d;
    out->kind = kind;
    return A8_OK;
}

extern "C" int a8_fixed_scale(int norm, int decades, float* scale_out) {
    if (!scale_out) return fail(A8_ERR_USAGE, "a8_fixed_scale: null output");
    if (norm == A8_NORM_NONE) {
        if (decades != 0) return fail(A8_ERR_CONFIG, "decades is only meaningful with decade normalization");
        *scale_out = 1.0f;
    } else if (norm == A8_NORM_DECADE) {
        if (decades < -7 || decades > 7) return fail(A8_ERR_CONFIG, "decade offset must lie in [-7, 7]");
        *scale_out = (float)pow(10.0, (double)decades);  // codecs.py:237,241
    } else {
        return fail(A8_ERR_USAGE, "a8_fixed_scale: absmax scale is data dependent");
    }
    return A8_OK;
}

extern "C" int a8_build_lut_host(const a8_book_t* book, float scale, a8_lut_t* out) {
    if (!book || !out) return fail(A8_ERR_USAGE, "a8_build_lut_host: null argument");
    memset(out, 0, sizeof(*out));
    out->scale = scale;
    for (int i = 0; i < 128; ++i) out->T[i] = a8::kInfBits;
    uint32_t F = 0;
    if (a8::scale_ok(scale)) {
        const double s = (double)scale;
        for (int i = 0; i + 1 < book->ndistinct; ++i)
            out->T[i] = a8::threshold(s, book->values[i], book->values[i + 1]);
        while (F < 127 && out->T[F] < a8::kInfBits) ++F;
    }
    out->nfinite = F;
    int32_t kbase;
    uint32_t len;
    a8::lut_geometry(out->T, F, &kbase, &len);
    out->kbase = kbase;
    out->len = len;
    out->valid = 0;
    if (len <= (uint32_t)a8::kLutMax) {
        bool ok = true;
        for (uint32_t j = 0; j < len; ++j) ok &= a8::lut_entry(out->T, F, book->codes, kbase, j, &out->e[j]);
        out->valid = ok ? 1u : 0u;
    }
    return A8_OK;
}
