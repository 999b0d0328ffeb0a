// Producer passes with the per-tensor max |y| fused in (a8_produce_absmax),
// so the encode that follows needs no max pass of its own
// (a8_encode_premax).
//
//   A8_PRODUCE_SCALE      y = fl(alpha * x): the pre-scaling a data-parallel
//                         step applies to its gradients (1/N averaging, loss
//                         scale); alpha == 1 with y == x is the max alone
//   A8_PRODUCE_RELU       y = np.maximum(x, 0)   (mlp.py:205: NaN propagates,
//                         -0 becomes +0)
//   A8_PRODUCE_RELU_MASK  y = fl(relu(x) * mask)  (mlp.py:205-207, the
//                         dropout-masked activation shipped by the
//                         model-parallel forward hook, mlp.py:208-209)
//
// The pass is HBM-bound streaming: 8 B per element (12 B with a mask, 4 B
// for the max alone).  Each CTA takes a contiguous range of 4096-element
// tiles (ranges cross few segment boundaries, so each warp publishes one
// atomic max per segment it touched); every thread has its 4 float4 loads
// of a tile in flight before it computes.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <string>

#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);
}  // namespace a8

using a8::fail;

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 4096;  // elements: 4 float4 per thread
constexpr int kSegs = 32;

struct PSeg {
    const float* x;
    float* y;
    const float* mask;
    int64_t n;
    int64_t t0;   // first tile of the segment in the launch's tile space
    int32_t vec;  // x, y (and mask) 16-byte aligned
    int32_t store;  // 0: y == x unchanged (alpha == 1), nothing to write
};

struct PParams {
    PSeg segs[kSegs + 1];  // segs[nseg].t0 = total tiles
    int nseg;
    int op;
    float alpha;
    unsigned int* amax;
    int64_t tiles;
};

template <int kOp>
__device__ __forceinline__ float produce(float x, float m, float alpha) {
    if (kOp == A8_PRODUCE_SCALE) return alpha == 1.0f ? x : __fmul_rn(alpha, x);  // 1 * x keeps a NaN's bits
    // np.maximum(x, 0.0) on the bits: x if x > 0 or NaN (its payload kept,
    // as NumPy does; a float max instruction would return the canonical NaN)
    const uint32_t b = __float_as_uint(x);
    const float r = ((int32_t)b > 0 || (b & 0x7fffffffu) > 0x7f800000u) ? x : 0.0f;
    return kOp == A8_PRODUCE_RELU_MASK ? __fmul_rn(r, m) : r;
}

// max |y| over raw bits, sign not masked (see a8_core.cuh absmax_raw4)
__device__ __forceinline__ void track(float v, unsigned int& u, int& s) {
    const unsigned int b = __float_as_uint(v);
    u = max(u, b);
    s = max(s, (int)b);
}

template <int kOp>
__global__ void __launch_bounds__(kThreads, 4) produce_kernel(const __grid_constant__ PParams p) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t t_lo = p.tiles * blockIdx.x / gridDim.x, t_hi = p.tiles * (blockIdx.x + 1) / gridDim.x;
    int s = 0;
    while (s + 1 < p.nseg && p.segs[s + 1].t0 <= t_lo) ++s;
    unsigned int u = 0u;
    int sm = INT_MIN;
    auto publish = [&](int seg) {
        const unsigned int wu = __reduce_max_sync(0xffffffffu, u);
        const int ws = __reduce_max_sync(0xffffffffu, sm);
        const unsigned int a = max(wu >= 0x80000000u ? wu & 0x7fffffffu : 0u, ws >= 0 ? (unsigned int)ws : 0u);
        if (lane == 0 && a) atomicMax(p.amax + seg, a);
        u = 0u;
        sm = INT_MIN;
    };
    for (int64_t t = t_lo; t < t_hi; ++t) {
        if (t >= p.segs[s + 1].t0) {
            publish(s);
            do ++s;
            while (t >= p.segs[s + 1].t0);
        }
        const PSeg& g = p.segs[s];
        const int64_t base = (t - g.t0) * kTile;
        const int64_t cnt = min((int64_t)kTile, g.n - base);
        if (g.vec && cnt == kTile) {
            const float4* x4 = reinterpret_cast<const float4*>(g.x + base);
            float4 v[4], mk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(x4 + k * kThreads + tid);
            if (kOp == A8_PRODUCE_RELU_MASK) {
                const float4* m4 = reinterpret_cast<const float4*>(g.mask + base);
#pragma unroll
                for (int k = 0; k < 4; ++k) mk[k] = __ldg(m4 + k * kThreads + tid);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 m = kOp == A8_PRODUCE_RELU_MASK ? mk[k] : make_float4(1.f, 1.f, 1.f, 1.f);
                const float4 r = make_float4(produce<kOp>(v[k].x, m.x, p.alpha), produce<kOp>(v[k].y, m.y, p.alpha),
                                             produce<kOp>(v[k].z, m.z, p.alpha), produce<kOp>(v[k].w, m.w, p.alpha));
                track(r.x, u, sm);
                track(r.y, u, sm);
                track(r.z, u, sm);
                track(r.w, u, sm);
                if (g.store) reinterpret_cast<float4*>(g.y + base)[k * kThreads + tid] = r;
            }
        } else {
            for (int64_t i = base + tid; i < base + cnt; i += kThreads) {
                const float r = produce<kOp>(g.x[i], kOp == A8_PRODUCE_RELU_MASK ? g.mask[i] : 1.f, p.alpha);
                track(r, u, sm);
                if (g.store) g.y[i] = r;
            }
        }
    }
    if (t_hi > t_lo) publish(s);
}

}  // namespace

extern "C" int a8_produce_absmax(const a8_prod_seg_t* segs, int nseg, int op, float alpha, uint32_t* amax_out,
                                 void* stream) {
    if (nseg < 0 || (nseg > 0 && (!segs || !amax_out))) return fail(A8_ERR_USAGE, "a8_produce_absmax: bad argument");
    if (op != A8_PRODUCE_SCALE && op != A8_PRODUCE_RELU && op != A8_PRODUCE_RELU_MASK)
        return fail(A8_ERR_USAGE, "a8_produce_absmax: unknown op");
    for (int i = 0; i < nseg; ++i) {
        const a8_prod_seg_t& g = segs[i];
        if (g.n < 0 || (g.n > 0 && (!g.x || !g.y || (op == A8_PRODUCE_RELU_MASK && !g.mask))))
            return fail(A8_ERR_USAGE, "a8_produce_absmax: bad segment");
    }
    if (nseg == 0) return A8_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(amax_out, 0, sizeof(uint32_t) * (size_t)nseg, st);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int c0 = 0; c0 < nseg; c0 += kSegs) {
        PParams p;
        p.nseg = std::min(kSegs, nseg - c0);
        p.op = op;
        p.alpha = alpha;
        p.amax = amax_out + c0;
        int64_t t = 0;
        for (int i = 0; i < p.nseg; ++i) {
            const a8_prod_seg_t& g = segs[c0 + i];
            PSeg& d = p.segs[i];
            d.x = g.x;
            d.y = g.y;
            d.mask = g.mask;
            d.n = g.n;
            d.t0 = t;
            const uintptr_t a = reinterpret_cast<uintptr_t>(g.x) | reinterpret_cast<uintptr_t>(g.y) |
                                (op == A8_PRODUCE_RELU_MASK ? reinterpret_cast<uintptr_t>(g.mask) : 0);
            d.vec = (a % 16) == 0;
            d.store = !(op == A8_PRODUCE_SCALE && alpha == 1.0f && g.x == g.y);
            t += (g.n + kTile - 1) / kTile;
        }
        p.segs[p.nseg] = PSeg{nullptr, nullptr, nullptr, 0, t, 0, 0};
        p.tiles = t;
        if (t == 0) continue;
        const unsigned grid = (unsigned)std::min<int64_t>(t, (int64_t)sms * 4);
        if (op == A8_PRODUCE_SCALE)
            produce_kernel<A8_PRODUCE_SCALE><<<grid, kThreads, 0, st>>>(p);
        else if (op == A8_PRODUCE_RELU)
            produce_kernel<A8_PRODUCE_RELU><<<grid, kThreads, 0, st>>>(p);
        else
            produce_kernel<A8_PRODUCE_RELU_MASK><<<grid, kThreads, 0, st>>>(p);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
