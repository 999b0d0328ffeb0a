// Host+device core of the approx8 B200 codec: decision thresholds and the
// bucketed decision table.  Compiled into the device kernels AND the host
// builder, so the CPU tests exercise the same arithmetic the GPU runs.
//
// The reference decision (approx8/codecs.py:260-265), for sorted distinct
// values v_0 = 0 < ... < v_{D-1} and y = fl64(|x| / s):
//     idx  = clip(searchsorted_left(v, y), 1, D-1)
//     pick = (fl64(y - v[idx-1]) <= fl64(v[idx] - y)) ? idx-1 : idx
// pick is monotone in |x|, so pick(|x|) = #{ i : T_i <= bits(|x|) } where T_i
// is the smallest float32 bit pattern for which the pair (v_i, v_{i+1})
// resolves upward.  T_i is found by a bracketed bisection using the same
// float64 operations (IEEE round-to-nearest divide and subtract).
#pragma once

#include <stdint.h>
#include <string.h>

#include "approx8_b200.h"

#if defined(__CUDACC__)
#define A8_HD __host__ __device__ __forceinline__
#else
#define A8_HD inline
#endif

namespace a8 {

constexpr uint32_t kInfBits = 0x7f800000u;
constexpr int kLutMax = A8_LUT_MAX;
constexpr int kKeyShift = 16;  // bucket key = top 15 bits of |x| (8 exp + 7 mantissa)

A8_HD double f32bits_to_f64(uint32_t a) {
    if (a < 0x00800000u) return (double)a * 0x1p-149;  // zero and subnormals, exact
#if defined(__CUDA_ARCH__)
    return (double)__uint_as_float(a);
#else
    float f;
    memcpy(&f, &a, 4);
    return (double)f;
#endif
}

A8_HD uint32_t f32_bits(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}

A8_HD double div_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}

A8_HD double sub_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}

// true iff the reference rounds |x| (bit pattern a) above v_lo (codecs.py:263-265)
A8_HD bool picks_upper(uint32_t a, double s, double v_lo, double v_hi) {
    const double y = div_rn(f32bits_to_f64(a), s);
    return !(sub_rn(y, v_lo) <= sub_rn(v_hi, y));
}

// T_i for the pair (v_lo, v_hi) at scale s (s finite, > 0).
A8_HD uint32_t threshold(double s, double v_lo, double v_hi) {
    // guess: the real midpoint times s, as float32; the true threshold is a
    // few ulps away unless the scale is extreme -> verify the bracket
    const double m = 0.5 * (v_lo + v_hi) * s;
    uint32_t g;
    if (!(m < 3.4028234663852886e38)) {
        g = kInfBits;
    } else {
        g = f32_bits((float)m);
    }
    // the rounded midpoint is almost always within a step or two of the
    // threshold: walk from it (2-3 predicate evaluations), and fall back to
    // a full bisection if the walk does not settle quickly
    uint32_t lo = 0u, hi = kInfBits;
    if (g > 0u && g < kInfBits) {
        if (picks_upper(g, s, v_lo, v_hi)) {
            uint32_t a = g;
            int steps = 0;
            while (a > 0u && steps < 4 && picks_upper(a - 1u, s, v_lo, v_hi)) {
                --a;
                ++steps;
            }
            if (a == 0u || steps < 4) return a;  // pred(a) true, pred(a-1) false
            hi = a;
        } else {
            uint32_t a = g + 1u;
            int steps = 0;
            while (a < kInfBits && steps < 4 && !picks_upper(a, s, v_lo, v_hi)) {
                ++a;
                ++steps;
            }
            if (a == kInfBits || steps < 4) return a;  // pred(a-1) false, pred(a) true
            lo = a - 1u;                                // pred(a-1) false is known
        }
    }
    while (hi - lo > 1u) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (picks_upper(mid, s, v_lo, v_hi))
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

// threshold() with one predicate evaluation.  g = RN32(m) is within half a
// float32 ulp of the real midpoint; the float64 decision resolves the
// neighbours g-1 (half an ulp or more below) and g+1 (above) correctly
// because its own rounding error is ~2^-29 of a float32 ulp.  Hence
// T is g or g+1 and pred(g) tells which.  Near the ends of the float32
// range (g < 8 or g within 8 of Inf) the walk + bisection is used.
// tests/cpp/threshold_window.cpp checks it against threshold() over
// millions of normal, tiny and huge scales for all four codebooks.
A8_HD uint32_t threshold_fast(double s, double v_lo, double v_hi) {
    const double m = 0.5 * (v_lo + v_hi) * s;
    const uint32_t g = m < 3.4028234663852886e38 ? f32_bits((float)m) : kInfBits;
    if (g < 8u || g >= kInfBits - 8u) return threshold(s, v_lo, v_hi);
    return picks_upper(g, s, v_lo, v_hi) ? g : g + 1u;
}

A8_HD bool scale_ok(float s) {
    const uint32_t b = f32_bits(s);
    return b != 0u && b < kInfBits;  // positive, finite, non-zero
}

// Bucket table entry encoding: t_low << 16 | code_hi << 8 | code_lo, where
// t_low is the low half of the bucket's threshold: an element of the bucket
// takes code_hi iff lo16(bits) >= t_low, which is exactly
// ((bits << 16) | 0xffff) >= entry because codes never exceed 0x7f7f.
// A bucket without a threshold stores t_low = 0 and code_hi = code_lo.

// #{i < F : T[i] < key}, branch-free over a 128-entry array (F <= 127).
A8_HD uint32_t count_below(const uint32_t* T, uint32_t F, uint32_t key) {
    uint32_t p = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (uint32_t step = 64; step; step >>= 1)
        if (p + step <= F && T[p + step - 1] < key) p += step;
    return p;
}

// One entry of the bucket table (same encoding as lut_fill), computed
// independently of its neighbours.  Returns false if the bucket holds two
// distinct thresholds.
A8_HD bool lut_entry(const uint32_t* T, uint32_t F, const uint8_t* canon, int32_t kbase, uint32_t j,
                     uint32_t* out) {
    const int64_t k = (int64_t)kbase + j;
    const uint32_t start = k <= 0 ? 0u : (uint32_t)(k << kKeyShift);
    const uint32_t end = (uint32_t)((k + 1) << kKeyShift);  // k+1 <= 0x7f81
    const uint32_t lo = count_below(T, F, start);
    const uint32_t hi = count_below(T, F, end);
    if (hi == lo) {
        *out = (uint32_t)canon[lo] | ((uint32_t)canon[lo] << 8);
        return true;
    }
    *out = (uint32_t)canon[lo] | ((uint32_t)canon[hi] << 8) | ((T[lo] & 0xffffu) << 16);
    return T[lo] == T[hi - 1];
}

// Table geometry from the thresholds: keys [kmin-1, kmax+1].
A8_HD void lut_geometry(const uint32_t* T, uint32_t F, int32_t* kbase, uint32_t* len) {
    if (F == 0) {
        *kbase = 0;
        *len = 1;
        return;
    }
    const int32_t kmin = (int32_t)(T[0] >> kKeyShift);
    const int32_t kmax = (int32_t)(T[F - 1] >> kKeyShift);
    *kbase = kmin - 1;
    *len = (uint32_t)(kmax - kmin + 3);
}

// One element: bits(x) -> code via the bucket table (codecs.py:262-268).
A8_HD uint32_t encode_lut(uint32_t b, const uint32_t* e, int32_t kbase, int32_t lenm1) {
    int32_t j = (int32_t)((b & 0x7fffffffu) >> kKeyShift) - kbase;
    j = j < 0 ? 0 : (j > lenm1 ? lenm1 : j);
    const uint32_t v = e[j];
    uint32_t c = (((b << 16) | 0xffffu) >= v) ? (v >> 8) : v;
    c &= 0xffu;
    // sign bit only for non-zero values (codecs.py:267-268); code 0 is the
    // only zero code, and c + 127 carries into bit 7 iff c != 0
    return c | ((c + 0x7fu) & (b >> 24) & 0x80u);
}

#if defined(__CUDACC__)
// Canonical code (no sign) in the low byte of the result, garbage above.
// Key and operand arithmetic use IMAD (FMA pipe); the ALU pipe does the
// clamp, compare and select.
// `ebase` is the 32-bit shared-memory address of the table pre-offset by
// -kbase entries: one IMAD forms the entry's address from the clamped key.
__device__ __forceinline__ uint32_t lut_code_lo(uint32_t b, uint32_t ebase, int32_t kmin, int32_t kmax) {
    const int32_t key = (int32_t)__umulhi(b * 2u, 1u << (31 - kKeyShift));  // (b & 0x7fffffff) >> 16
    const int32_t k = min(max(key, kmin), kmax);
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ebase + (uint32_t)k * 4u));
    return (b * 65536u + 0xffffu >= v) ? (v >> 8) : v;
}

// Sign attachment for 4 packed canonical codes (each <= 127): bit 7 of a
// byte is set iff the input is negative and the code is non-zero
// (codecs.py:267-268).  c + 0x7f carries into bit 7 iff c != 0; no byte
// overflows into its neighbour.
__device__ __forceinline__ uint32_t attach_signs4(uint32_t packed, uint32_t b0, uint32_t b1, uint32_t b2,
                                                  uint32_t b3) {
    const uint32_t s = __byte_perm(__byte_perm(b0, b1, 0x0073), __byte_perm(b2, b3, 0x0073), 0x5410);
    return packed | ((packed + 0x7f7f7f7fu) & s & 0x80808080u);
}

// One element as lut_code_lo, also returning the unclamped key (>= 0x7f80
// iff |x| is Inf or NaN: the fixed-scale specs' non-finite check).
__device__ __forceinline__ uint32_t lut_code_lo_k(uint32_t b, uint32_t ebase, int32_t kmin, int32_t kmax,
                                                  int32_t& key) {
    key = (int32_t)__umulhi(b * 2u, 1u << (31 - kKeyShift));  // (b & 0x7fffffff) >> 16
    const int32_t k = min(max(key, kmin), kmax);
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ebase + (uint32_t)k * 4u));
    return (b * 65536u + 0xffffu >= v) ? (v >> 8) : v;
}

// encode4_lut that also folds the four keys into `kacc` (running max).
__device__ __forceinline__ uint32_t encode4_lut_k(uint4 v, uint32_t ebase, int32_t kmin, int32_t kmax,
                                                  int32_t& kacc) {
    int32_t k0, k1, k2, k3;
    const uint32_t c0 = lut_code_lo_k(v.x, ebase, kmin, kmax, k0);
    const uint32_t c1 = lut_code_lo_k(v.y, ebase, kmin, kmax, k1);
    const uint32_t c2 = lut_code_lo_k(v.z, ebase, kmin, kmax, k2);
    const uint32_t c3 = lut_code_lo_k(v.w, ebase, kmin, kmax, k3);
    kacc = max(max(kacc, k0), max(k1, max(k2, k3)));
    const uint32_t packed = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
    return attach_signs4(packed, v.x, v.y, v.z, v.w);
}

// Four elements -> four codes packed little-endian (bucket table).
__device__ __forceinline__ uint32_t encode4_lut(uint4 v, uint32_t ebase, int32_t kmin, int32_t kmax) {
    const uint32_t c0 = lut_code_lo(v.x, ebase, kmin, kmax);
    const uint32_t c1 = lut_code_lo(v.y, ebase, kmin, kmax);
    const uint32_t c2 = lut_code_lo(v.z, ebase, kmin, kmax);
    const uint32_t c3 = lut_code_lo(v.w, ebase, kmin, kmax);
    const uint32_t packed = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
    return attach_signs4(packed, v.x, v.y, v.z, v.w);
}
#endif

// ---------------------------------------------------------------------------
// "Carry" bucket table, for codebooks whose canonical code of sorted value i
// is i itself (dynamic-tree and linear: exactly the kinds that allow absmax,
// codecs.py:89-94).  Entry of the bucket with key k:
//     lo << 16  +  (bucket holds threshold T_lo ? 0x10000 - lo16(T_lo) : 0)
// where lo = #thresholds below the bucket.  For an element with bits b in the
// bucket, entry + (b & 0x8000ffff) has the code in byte 2 (lo, plus the carry
// out of the low half iff lo16(b) >= lo16(T_lo), i.e. iff b >= T_lo) and the
// sign bit of x alone in byte 3 (the sum stays below 2^23).  A bucket can
// hold at most one threshold (else the table is invalid and the caller
// searches the thresholds).  Keys below the table clamp to entry 0, which is
// 0 (code 0, no threshold); absmax tables extend up to the key of the scale
// itself, the largest |x| of the segment, so no upper clamp is needed.
A8_HD uint32_t carry_entry(uint32_t lo, uint32_t count, uint32_t t_lo) {
    return (lo << 16) + (count ? 0x10000u - (t_lo & 0xffffu) : 0u);
}

// Scalar form with both clamps (any key; slow paths and host checks).
A8_HD uint32_t encode_carry(uint32_t b, const uint32_t* e, int32_t kbase, int32_t lenm1) {
    int32_t j = (int32_t)((b & 0x7fffffffu) >> kKeyShift) - kbase;
    j = j < 0 ? 0 : (j > lenm1 ? lenm1 : j);
    const uint32_t c = ((e[j] + (b & 0xffffu)) >> 16) & 0xffu;
    return c | ((c + 0x7fu) & (b >> 24) & 0x80u);
}

#if defined(__CUDACC__)
// One element: the table sum (code in byte 2, sign in byte 3).  `ebase` is
// the shared address of the table minus kbase entries, `emin` the table's
// own address (signed max: ebase may wrap below zero).  5 instructions:
// LOP3, IMAD.HI (key * 4 + ebase), VIMNMX, LDS, IADD3.
__device__ __forceinline__ uint32_t carry_sum(uint32_t b, uint32_t ebase, int32_t emin) {
    const uint32_t m = b & 0x7fff0000u;
    const int32_t a = max((int32_t)(__umulhi(m, 1u << 18) + ebase), emin);
    uint32_t e, r;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(a));
    // e + b - m in one IADD3 (the compiler otherwise forms b & 0x8000ffff first)
    asm("{\n\t.reg .u32 t;\n\tsub.u32 t, %1, %2;\n\tadd.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(b), "r"(m), "r"(e));
    return r;
}

// Four table sums -> four final code bytes, little-endian: code | sign for
// non-zero codes (codecs.py:267-268; c + 0x7f carries into bit 7 iff c != 0).
__device__ __forceinline__ uint32_t pack4_carry(uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3) {
    const uint32_t w01 = __byte_perm(s0, s1, 0x7632);  // c0 g0 c1 g1
    const uint32_t w23 = __byte_perm(s2, s3, 0x7632);  // c2 g2 c3 g3
    const uint32_t codes = __byte_perm(w01, w23, 0x6420);
    const uint32_t signs = __byte_perm(w01, w23, 0x7531);
    return codes | (signs & (codes + 0x7f7f7f7fu));
}

__device__ __forceinline__ uint32_t encode4_carry(uint4 v, uint32_t ebase, int32_t emin) {
    return pack4_carry(carry_sum(v.x, ebase, emin), carry_sum(v.y, ebase, emin), carry_sum(v.z, ebase, emin),
                       carry_sum(v.w, ebase, emin));
}

// carry_sum with the upper clamp too (`emax`: address of the table's last
// entry), for tables whose top key comes from a caller-supplied max that
// may be wrong (a8_encode_premax): any |x| stays inside the table.
__device__ __forceinline__ uint32_t carry_sum_clamp(uint32_t b, uint32_t ebase, int32_t emin, int32_t emax) {
    const uint32_t m = b & 0x7fff0000u;
    const int32_t a = min(max((int32_t)(__umulhi(m, 1u << 18) + ebase), emin), emax);
    uint32_t e, r;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(a));
    asm("{\n\t.reg .u32 t;\n\tsub.u32 t, %1, %2;\n\tadd.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(b), "r"(m), "r"(e));
    return r;
}

__device__ __forceinline__ uint32_t encode4_carry_clamp(uint4 v, uint32_t ebase, int32_t emin, int32_t emax) {
    return pack4_carry(carry_sum_clamp(v.x, ebase, emin, emax), carry_sum_clamp(v.y, ebase, emin, emax),
                       carry_sum_clamp(v.z, ebase, emin, emax), carry_sum_clamp(v.w, ebase, emin, emax));
}

// Running max of |x| over raw float32 bits without masking the sign: the
// unsigned max over the raw bits is the largest negative magnitude (when
// any x has its sign bit set), the signed max is the largest positive
// magnitude (when any x has it clear).  abs_of_maxes folds the two.
__device__ __forceinline__ void absmax_raw4(uint4 v, uint32_t& u, int32_t& s) {
    u = __vimax3_u32(u, v.x, v.y);
    u = __vimax3_u32(u, v.z, v.w);
    s = __vimax3_s32(s, (int32_t)v.x, (int32_t)v.y);
    s = __vimax3_s32(s, (int32_t)v.z, (int32_t)v.w);
}
__device__ __forceinline__ uint32_t abs_of_maxes(uint32_t u, int32_t s) {
    return max(u >= 0x80000000u ? u & 0x7fffffffu : 0u, s >= 0 ? (uint32_t)s : 0u);
}
#endif

// ---------------------------------------------------------------------------
// Guess-and-verify encode for an absmax scale s (dynamic-tree / linear):
//   guess  c = G[key(fl32(|x| * fl32(1/s)))]   (G: scale-independent, per codebook)
//   verify p = c + (bits|x| >= T_c(s))          (T: the scale's exact thresholds)
// G[k] counts the midpoints surely below bucket k, so c <= p <= c + 1 as
// long as every bucket (widened by the rounding of the normalised value)
// holds at most one midpoint -- true for both absmax codebooks
// (tests/test_blocked.py checks it).  Valid for 2^-100 <= s <= 2^100.
inline constexpr int kGKey0 = 0x3400;                 // key (bits >> 16) of 2^-23: every midpoint lies above
inline constexpr int kGLen = 0x3f80 - kGKey0 + 1;      // keys up to that of 1.0 (|x|/s <= 1 up to rounding)
inline constexpr double kGMargin = 0x1p-18;            // > rounding of fl32(|x| * fl32(1/s)) and of T_i / s

#if defined(__CUDACC__)
// One element: guess + verify.  `gaddr` = shared address of G minus kGKey0,
// `gmin` = shared address of G (keys below the table clamp to entry 0),
// `taddr` = shared address of the block's thresholds.  About 10 instructions:
// FMUL, SHF, VIADDMNMX, LDS.U8, IMAD, LDS, LOP3, IADD3, LEA.HI (+ packing).
__device__ __forceinline__ uint32_t guess_verify(uint32_t b, float r, uint32_t gaddr, uint32_t gmin, uint32_t taddr) {
    const float y = fabsf(__uint_as_float(b)) * r;
    // signed: gaddr may wrap below zero (shared addresses are < 2^31)
    const uint32_t ga = (uint32_t)max((int32_t)((__float_as_uint(y) >> 16) + gaddr), (int32_t)gmin);
    uint32_t c, t;
    asm("ld.shared.u8 %0, [%1];" : "=r"(c) : "r"(ga));
    asm("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(taddr + 4u * c));
    // c + (|x| bits >= T_c): T_c - 1 - |x| is negative exactly then
    return c + ((t + ~(b & 0x7fffffffu)) >> 31);
}

// G (one byte per key of the normalised value, kGKey0 .. 0x3f80): the
// number of codebook midpoints surely below the bucket.  Built once per
// codebook by a one-CTA kernel and cached on the device (a8_encode_blocked).
static __global__ void guess_table_kernel(const a8_book_t* book, uint8_t* G) {
    __shared__ double sMid[128];
    const int D = book->ndistinct;
    const int tid = threadIdx.x;
    if (tid < 128) sMid[tid] = tid + 1 < D ? 0.5 * (book->values[tid] + book->values[tid + 1]) : 1e300;
    __syncthreads();
    for (int j = tid; j < kGLen; j += blockDim.x) {
        const double yk = (double)__uint_as_float((uint32_t)(kGKey0 + j) << 16);
        int p = 0;
        for (int step = 64; step; step >>= 1)
            if (p + step <= D - 1 && sMid[p + step - 1] * (1.0 + kGMargin) < yk) p += step;
        G[j] = (uint8_t)p;
    }
}

#endif

// One element by binary search over the padded thresholds (paper's method).
A8_HD uint32_t encode_search(uint32_t b, const uint32_t* T128, const uint8_t* canon128) {
    const uint32_t a = b & 0x7fffffffu;
    uint32_t p = 0;
#pragma unroll
    for (uint32_t step = 64; step; step >>= 1)
        if (T128[p + step - 1] <= a) p += step;
    const uint32_t c = canon128[p];
    return c | ((c + 0x7fu) & (b >> 24) & 0x80u);
}

#ifdef __CUDACC__
// Four elements by encode_search, packed little-endian into one word.
__device__ __forceinline__ uint32_t encode4_search(uint4 v, const uint32_t* T128, const uint8_t* canon128) {
    return encode_search(v.x, T128, canon128) | (encode_search(v.y, T128, canon128) << 8) |
           (encode_search(v.z, T128, canon128) << 16) | (encode_search(v.w, T128, canon128) << 24);
}
#endif

}  // namespace a8
