// Host check of the resident kernel's parallel threshold search
// (threshold_parallel in csrc/a8_kernels.cu): the first of the 8 float32
// patterns g-3 .. g+4 around the rounded midpoint g that resolves upward must
// equal threshold() (the sequential walk + bisection), or the window must
// report "not inside" (all 8 predicates equal) so the kernel falls back.
// Also: threshold_fast() (one predicate evaluation, used by the encode
// kernels) must equal threshold() for normal, tiny and huge scales.
// Built and run by tests/test_host_lib.py::test_parallel_threshold_window.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "a8_core.cuh"

using namespace a8;
int a8_codebook(int kind, a8_book_t* out);

int main(int argc, char** argv) {
    const int scales = argc > 1 ? atoi(argv[1]) : 2000;
    std::mt19937_64 rng(1);
    long bad = 0, fallback = 0, total = 0, bad_fast = 0;
    for (int kind = 0; kind < 4; ++kind) {
        a8_book_t bk;
        a8_codebook(kind, &bk);
        for (int it = 0; it < scales; ++it) {
            uint32_t sb;
            if (it % 3 == 0)
                sb = 0x00800000u + (uint32_t)(rng() % (0x7f800000u - 0x00800000u));  // any normal scale
            else if (it % 3 == 1)
                sb = 0x00800000u + (uint32_t)(rng() % 0x08000000u);  // tiny scales
            else
                sb = 0x77000000u + (uint32_t)(rng() % 0x08800000u);  // huge scales
            float scale;
            memcpy(&scale, &sb, 4);
            for (int i = 0; i + 1 < bk.ndistinct; ++i) {
                const double s = scale, vlo = bk.values[i], vhi = bk.values[i + 1];
                const uint32_t ref = threshold(s, vlo, vhi);
                const double m = 0.5 * (vlo + vhi) * s;
                const uint32_t g = m < 3.4028234663852886e38 ? f32_bits((float)m) : kInfBits;
                uint32_t t = 0;
                bool fb = g < 8u || g >= kInfBits - 8u;
                if (!fb) {
                    unsigned bits = 0;
                    for (int q = 0; q < 8; ++q) bits |= (picks_upper(g - 3 + q, s, vlo, vhi) ? 1u : 0u) << q;
                    if (bits == 0u || bits == 0xffu)
                        fb = true;
                    else
                        t = g - 3 + (uint32_t)__builtin_popcount(~bits & 0xffu);
                }
                if (fb) {
                    ++fallback;
                    t = threshold(s, vlo, vhi);
                }
                ++total;
                if (t != ref) ++bad;
                if (threshold_fast(s, vlo, vhi) != ref) ++bad_fast;
            }
        }
    }
    printf("%ld %ld %ld %ld\n", total, bad, fallback, bad_fast);
    return bad || bad_fast ? 1 : 0;
}
