// Round-trip error aggregates on sm_100a: the GPU error bench
// (approx8/errorbench.py:79-99, measure_error) and the hook statistics
// (approx8/mlp.py:146-153, _HookStats.record).
//
// Per element, in float64 exactly as the reference computes it:
//   d    = float32(table[c] * scale)            (the decode, codecs.py:281)
//          or a given float32 `after` value      (a decoded tensor)
//   err  = |float64(x) - float64(d)|             (errorbench.py:89-91)
//   rel  = err / |float64(x)|  for x != 0        (errorbench.py:92-97)
// and the sums  sum(err), sum(rel over x != 0), #(x != 0).
//
// One launch: a grid-stride pass with 16-byte loads (4 B of x + 1 B of code
// per element, nothing written), per-CTA float64 partials in a fixed order,
// and the last CTA reduces the partials in CTA order -- deterministic for a
// given grid.  The per-element values are identical to NumPy's; the sums are
// a fixed-order tree instead of NumPy's pairwise sum (differences are at the
// float64 rounding level, ~1e-16 relative).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);
}  // namespace a8

using a8::fail;

namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 1184;  // 8 CTAs x 148 SMs

struct Partial {
    double sum_abs, sum_rel;
    unsigned long long nnz;
    unsigned long long pad;
};

struct Ws {
    unsigned int done;
    unsigned int pad[15];
    Partial part[kMaxGrid];
};

__device__ __forceinline__ void accum(double xd, float d, double& sa, double& sr, unsigned long long& nz) {
    const double e = fabs(__dsub_rn(xd, (double)d));
    sa = __dadd_rn(sa, e);
    if (xd != 0.0) {
        sr = __dadd_rn(sr, __ddiv_rn(e, fabs(xd)));
        ++nz;
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fixed-order block reduction of three values; result valid in thread 0
__device__ void block_reduce(double& a, double& r, unsigned long long& z) {
    __shared__ double sa[kThreads / 32], sr[kThreads / 32];
    __shared__ unsigned long long sz[kThreads / 32];
    a = warp_sum(a);
    r = warp_sum(r);
    z = warp_sum(z);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sa[w] = a;
        sr[w] = r;
        sz[w] = z;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = 0.0;
        r = 0.0;
        z = 0;
        for (int i = 0; i < kThreads / 32; ++i) {
            a += sa[i];
            r += sr[i];
            z += sz[i];
        }
    }
}

template <bool kF64>
__global__ void __launch_bounds__(kThreads) error_stats_kernel(const void* xv, int64_t n, const uint8_t* codes,
                                                               const float* scale, const a8_book_t* book,
                                                               const float* after, double* out, int accumulate,
                                                               Ws* ws) {
    __shared__ float sTab[256];
    __shared__ int sLast;
    const int tid = threadIdx.x;
    if (codes) sTab[tid] = __fmul_rn(book->table[tid], __ldg(scale));  // codecs.py:281
    __syncthreads();
    double sa = 0.0, sr = 0.0;
    unsigned long long nz = 0;
    const int64_t gstride = (int64_t)gridDim.x * kThreads;
    const int64_t g0 = (int64_t)blockIdx.x * kThreads + tid;
    int64_t done = 0;
    // 4 elements per step (one 16-byte load of x, and 4 codes or 4 decoded
    // values).  Both forms visit the elements in the same order, so the
    // codes and the decoded-tensor forms give identical sums.
    const bool vec = !kF64 && (reinterpret_cast<uintptr_t>(xv) % 16) == 0 &&
                     (codes ? (reinterpret_cast<uintptr_t>(codes) % 4) == 0 : (reinterpret_cast<uintptr_t>(after) % 16) == 0);
    if (vec) {
        const float4* x4 = reinterpret_cast<const float4*>(xv);
        const int64_t n4 = n >> 2;
        // kU groups per thread per round, all loads issued before the math
        // (bytes in flight); the accumulation order is the same either way
        constexpr int kU = 4;
        int64_t i = g0;
        if (codes) {
            const uint32_t* c4 = reinterpret_cast<const uint32_t*>(codes);
            for (; i + (kU - 1) * gstride < n4; i += kU * gstride) {
                float4 v[kU];
                uint32_t c[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    v[u] = __ldcs(x4 + i + u * gstride);
                    c[u] = __ldcs(c4 + i + u * gstride);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    accum((double)v[u].x, sTab[c[u] & 255u], sa, sr, nz);
                    accum((double)v[u].y, sTab[(c[u] >> 8) & 255u], sa, sr, nz);
                    accum((double)v[u].z, sTab[(c[u] >> 16) & 255u], sa, sr, nz);
                    accum((double)v[u].w, sTab[c[u] >> 24], sa, sr, nz);
                }
            }
            for (; i < n4; i += gstride) {
                const float4 v = __ldcs(x4 + i);
                const uint32_t c = __ldcs(c4 + i);
                accum((double)v.x, sTab[c & 255u], sa, sr, nz);
                accum((double)v.y, sTab[(c >> 8) & 255u], sa, sr, nz);
                accum((double)v.z, sTab[(c >> 16) & 255u], sa, sr, nz);
                accum((double)v.w, sTab[c >> 24], sa, sr, nz);
            }
        } else {
            const float4* a4 = reinterpret_cast<const float4*>(after);
            for (; i + (kU - 1) * gstride < n4; i += kU * gstride) {
                float4 v[kU], d[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    v[u] = __ldcs(x4 + i + u * gstride);
                    d[u] = __ldcs(a4 + i + u * gstride);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    accum((double)v[u].x, d[u].x, sa, sr, nz);
                    accum((double)v[u].y, d[u].y, sa, sr, nz);
                    accum((double)v[u].z, d[u].z, sa, sr, nz);
                    accum((double)v[u].w, d[u].w, sa, sr, nz);
                }
            }
            for (; i < n4; i += gstride) {
                const float4 v = __ldcs(x4 + i);
                const float4 d = __ldcs(a4 + i);
                accum((double)v.x, d.x, sa, sr, nz);
                accum((double)v.y, d.y, sa, sr, nz);
                accum((double)v.z, d.z, sa, sr, nz);
                accum((double)v.w, d.w, sa, sr, nz);
            }
        }
        done = n4 << 2;
    }
    for (int64_t i = done + g0; i < n; i += gstride) {
        const double xd = kF64 ? reinterpret_cast<const double*>(xv)[i] : (double)reinterpret_cast<const float*>(xv)[i];
        const float d = codes ? sTab[codes[i]] : after[i];
        accum(xd, d, sa, sr, nz);
    }
    block_reduce(sa, sr, nz);
    if (tid == 0) {
        ws->part[blockIdx.x] = Partial{sa, sr, nz, 0ull};
        __threadfence();
        sLast = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!sLast) return;
    __threadfence();
    // last CTA: partials in CTA order (strided per thread, then the fixed block tree)
    double a = 0.0, r = 0.0;
    unsigned long long z = 0;
    for (int i = tid; i < (int)gridDim.x; i += kThreads) {
        const Partial p = ws->part[i];
        a += p.sum_abs;
        r += p.sum_rel;
        z += p.nnz;
    }
    block_reduce(a, r, z);
    if (tid == 0) {
        if (accumulate) {
            out[0] = __dadd_rn(out[0], a);
            out[1] = __dadd_rn(out[1], r);
            out[2] = __dadd_rn(out[2], (double)z);
        } else {
            out[0] = a;
            out[1] = r;
            out[2] = (double)z;
        }
        ws->done = 0u;  // left zeroed for the next call
    }
}

}  // namespace

extern "C" size_t a8_error_workspace_bytes(void) { return sizeof(Ws); }

extern "C" int a8_error_stats(const void* x, int x_is_f64, int64_t n, const uint8_t* codes, const float* scale_dev,
                              const void* book_dev, const float* after, double* out_dev, int accumulate,
                              void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0) return fail(A8_ERR_USAGE, "a8_error_stats: negative length");
    if (!out_dev || !workspace) return fail(A8_ERR_USAGE, "a8_error_stats: null argument");
    if (workspace_bytes < sizeof(Ws)) return fail(A8_ERR_USAGE, "a8_error_stats: workspace too small");
    if (n > 0 && !x) return fail(A8_ERR_USAGE, "a8_error_stats: null input");
    if (n > 0 && !codes && !after) return fail(A8_ERR_USAGE, "a8_error_stats: need codes or decoded values");
    if (codes && (!scale_dev || !book_dev)) return fail(A8_ERR_USAGE, "a8_error_stats: codes need a scale and a codebook");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + kThreads * 16 - 1) / (kThreads * 16);  // >= 16 elements per thread
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(kMaxGrid, 8 * std::max(sms, 1)), want));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const a8_book_t* book = static_cast<const a8_book_t*>(book_dev);
    Ws* ws = static_cast<Ws*>(workspace);
    if (x_is_f64)
        error_stats_kernel<true><<<grid, kThreads, 0, st>>>(x, n, codes, scale_dev, book, after, out_dev, accumulate, ws);
    else
        error_stats_kernel<false><<<grid, kThreads, 0, st>>>(x, n, codes, scale_dev, book, after, out_dev, accumulate, ws);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
    return A8_OK;
}
