// 1-bit error-feedback quantizer (approx8/codecs.py:291-348) on sm_100a.
//
//   corrected = float64(g) + residual
//   positive  = corrected >= 0
//   pos_level = float32(mean(corrected[positive]))   (0 if none), same for neg
//   residual  = corrected - (positive ? pos_level : neg_level)     (float64)
//   bits      = packbits(positive), first element in the MSB (np.packbits)
//
// Two launches: stats (per-CTA float64 sums and counts per sign, non-finite
// flag) and apply (every CTA reduces the partials in the same fixed order,
// so all CTAs see identical levels; then the residual update and the bit
// packing, 8 elements -> 1 byte per thread).  The float64 sums are exact
// to float64 rounding; the summation order differs from NumPy's pairwise
// sum, which can only change a level when the float64 mean lies within a
// float64 ulp of a float32 rounding boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);
extern thread_local std::string g_last_error;
}  // namespace a8

using a8::fail;

namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 480;

struct Partial {
    double sum_pos, sum_neg;
    unsigned long long cnt_pos, cnt_neg;
    unsigned int bad;
    unsigned int pad[3];
};

__device__ __forceinline__ double load_g(const void* g, int f64, int64_t i) {
    return f64 ? reinterpret_cast<const double*>(g)[i] : (double)reinterpret_cast<const float*>(g)[i];
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    T s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kThreads / 32; ++i) s += red[i];  // fixed order
    return s;  // valid in thread 0
}

// One tensor's stats as block j of a G-block grid (the single-tensor launch
// has j = blockIdx.x, G = gridDim.x; the multi-tensor launch gives each
// tensor its own range of blocks with the same G, so the sums match).
__device__ __forceinline__ void stats_body(const void* g, int f64, const double* res, int64_t n, int j, int G,
                                           Partial* out) {
    __shared__ double rd[kThreads / 32];
    __shared__ unsigned long long ru[kThreads / 32];
    double sp = 0.0, sn = 0.0;
    unsigned long long cp = 0, cn = 0;
    unsigned int bad = 0;
    // the same per-thread element order (i, i+S, i+2S, ...) as a plain
    // grid-stride loop -- so the sums are bit-identical to it -- with the
    // loads of 4 elements issued before any of them is accumulated
    #ifndef A8_OB_STATS_U
#define A8_OB_STATS_U 4  // 4 loads in flight: 138 us for the C3 stats; 2: 227, 6: 161, 8: 160, 16: 227
#endif
    constexpr int U = A8_OB_STATS_U;
    const int64_t S = (int64_t)G * kThreads;
    for (int64_t i0 = (int64_t)j * kThreads + threadIdx.x; i0 < n; i0 += U * S) {
        double gv[U], rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * S;
            gv[u] = i < n ? load_g(g, f64, i) : 0.0;
            rv[u] = i < n ? res[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (i0 + u * S >= n) break;
            if (!isfinite(gv[u])) bad = 1;
            const double c = __dadd_rn(gv[u], rv[u]);
            if (c >= 0.0) {
                sp = __dadd_rn(sp, c);
                ++cp;
            } else {
                sn = __dadd_rn(sn, c);
                ++cn;
            }
        }
    }
    const double SP = block_sum(sp, rd);
    const double SN = block_sum(sn, rd);
    const unsigned long long CP = block_sum(cp, ru);
    const unsigned long long CN = block_sum(cn, ru);
    const int B = __syncthreads_or(bad);
    if (threadIdx.x == 0) *out = Partial{SP, SN, CP, CN, (unsigned)B, {0, 0, 0}};
}

__global__ void __launch_bounds__(kThreads) onebit_stats(const void* g, int f64, const double* res, int64_t n,
                                                          Partial* part) {
    stats_body(g, f64, res, n, blockIdx.x, gridDim.x, part + blockIdx.x);
}

// One tensor's apply as block j of a G-block grid; part = its G partials.
__device__ __forceinline__ void apply_body(const void* g, int f64, double* res, int64_t n, const Partial* part,
                                           int nparts, uint8_t* bits, float* levels, uint32_t* status, int j,
                                           int G) {
    __shared__ double rd[kThreads / 32];
    __shared__ unsigned long long ru[kThreads / 32];
    __shared__ float sLv[2];
    double sp = 0.0, sn = 0.0;
    unsigned long long cp = 0, cn = 0;
    unsigned int bad = 0;
    for (int i = threadIdx.x; i < nparts; i += kThreads) {
        sp += part[i].sum_pos;
        sn += part[i].sum_neg;
        cp += part[i].cnt_pos;
        cn += part[i].cnt_neg;
        bad |= part[i].bad;
    }
    const double SP = block_sum(sp, rd);
    const double SN = block_sum(sn, rd);
    const unsigned long long CP = block_sum(cp, ru);
    const unsigned long long CN = block_sum(cn, ru);
    const int B = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        // codecs.py:327-328: float32 of the float64 mean, 0.0 for an empty side
        sLv[0] = CP ? __double2float_rn(__ddiv_rn(SP, (double)CP)) : 0.0f;
        sLv[1] = CN ? __double2float_rn(__ddiv_rn(SN, (double)CN)) : 0.0f;
        if (j == 0) {
            levels[0] = sLv[0];
            levels[1] = sLv[1];
            *status = B ? A8_STATUS_NONFINITE : 0u;
        }
    }
    __syncthreads();
    // codecs.py:317-318 raises before touching the state: non-finite input
    // leaves the residual (and the bits) as they were
    if (B) return;
    const double pl = (double)sLv[0], nl = (double)sLv[1];
    // warp chunks of 1024 consecutive elements: in step k the lanes take
    // elements 32k + lane (coalesced loads and stores of g and the residual),
    // the ballot gives those 32 sign bits, and lane k keeps them; at the end
    // every lane stores its 4 bytes (128 coalesced bytes of bits per warp)
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)G * (kThreads / 32);
    const int64_t nbytes = (n + 7) / 8;
    for (int64_t wc = (int64_t)j * (kThreads / 32) + (threadIdx.x >> 5); wc * 1024 < n; wc += warps) {
        const int64_t base = wc * 1024;
        uint32_t mine = 0;
        constexpr int U = 8;  // steps whose loads are issued together
        for (int k0 = 0; k0 < 32; k0 += U) {
            double gv[U], rv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = base + 32 * (k0 + u) + lane;
                gv[u] = i < n ? load_g(g, f64, i) : 0.0;
                rv[u] = i < n ? res[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = base + 32 * (k0 + u) + lane;
                const double c = __dadd_rn(gv[u], rv[u]);
                const bool pos = i < n && c >= 0.0;
                if (i < n) res[i] = __dsub_rn(c, pos ? pl : nl);
                const uint32_t bal = __ballot_sync(0xffffffffu, pos);
                if (lane == k0 + u) mine = bal;
            }
        }
        // np.packbits order: element 8j + t is bit 7 - t of byte j
        const uint32_t w = __byte_perm(__brev(mine), 0, 0x0123);
        const int64_t b0 = base / 8 + 4 * lane;
        if (b0 + 4 <= nbytes && (reinterpret_cast<uintptr_t>(bits) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(bits + b0) = w;
        } else {
            for (int t = 0; t < 4; ++t)
                if (b0 + t < nbytes) bits[b0 + t] = (uint8_t)(w >> (8 * t));
        }
    }
}

__global__ void __launch_bounds__(kThreads) onebit_apply(const void* g, int f64, double* res, int64_t n,
                                                          const Partial* part, int nparts, uint8_t* bits,
                                                          float* levels, uint32_t* status) {
    apply_body(g, f64, res, n, part, nparts, bits, levels, status, blockIdx.x, gridDim.x);
}

// The multi-tensor launches: tensor s owns blocks [p0[s], p0[s+1]).
constexpr int kQSegs = 32;
struct QParams {
    a8_ob_q_seg_t segs[kQSegs];
    int p0[kQSegs + 1];
    int nseg, f64;
    Partial* part;
};

__device__ __forceinline__ int qseg_of(const QParams& p, int b) {
    int s = 0;
    while (s + 1 < p.nseg && p.p0[s + 1] <= b) ++s;
    return s;
}

__global__ void __launch_bounds__(kThreads) onebit_stats_multi(const __grid_constant__ QParams p) {
    const int s = qseg_of(p, blockIdx.x);
    const a8_ob_q_seg_t& q = p.segs[s];
    stats_body(q.g, p.f64, q.residual, q.n, blockIdx.x - p.p0[s], p.p0[s + 1] - p.p0[s], p.part + blockIdx.x);
}

__global__ void __launch_bounds__(kThreads) onebit_apply_multi(const __grid_constant__ QParams p) {
    const int s = qseg_of(p, blockIdx.x);
    const a8_ob_q_seg_t& q = p.segs[s];
    const int G = p.p0[s + 1] - p.p0[s];
    apply_body(q.g, p.f64, q.residual, q.n, p.part + p.p0[s], G, q.bits, q.levels, q.status, blockIdx.x - p.p0[s], G);
}

__global__ void __launch_bounds__(kThreads) onebit_decode_k(const uint8_t* bits, int64_t n, const float* levels,
                                                             float* out) {
    const float pl = levels[0], nl = levels[1];
    // lane l of a warp writes float4 number l of each 128-element group: its
    // 4 elements are one nibble (high nibble first, np.packbits order)
    const int64_t nq = n / 4;  // full float4 groups
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const int64_t S = (int64_t)gridDim.x * kThreads;
    if (vec) {
        constexpr int U = 8;  // float4 groups per thread per step, loads first
        for (int64_t q0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; q0 < nq; q0 += U * S) {
            uint32_t nib[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = q0 + u * S;
                nib[u] = q < nq ? (__ldg(bits + (q >> 1)) >> ((q & 1) ? 0 : 4)) & 15u : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = q0 + u * S;
                if (q < nq)
                    __stcs(reinterpret_cast<float4*>(out) + q, make_float4(nib[u] & 8u ? pl : nl, nib[u] & 4u ? pl : nl,
                                                                         nib[u] & 2u ? pl : nl, nib[u] & 1u ? pl : nl));
            }
        }
    }
    for (int64_t i = (vec ? nq * 4 : 0) + (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += S)
        out[i] = (bits[i >> 3] >> (7 - (i & 7))) & 1u ? pl : nl;
}

// The 1-bit exchange's decode-sum(-average) over N gathered slabs (the DP
// seam of mlp.py:313-321 across ranks): out[i] = sum_r (bit_r(i) ? pos_r :
// neg_r), rank order, float32, then / N.  One thread per byte of bits (8
// elements); segments are located by a search over the byte prefix sums.
constexpr int kObSegs = 32;
struct ObParams {
    a8_ob_seg_t segs[kObSegs];
    int64_t unit_start[kObSegs + 1];  // prefix sums of ceil(n / 1024): one warp per 1024 elements
    const uint8_t* slabs;
    int64_t rank_stride, levels_off, status_off;
    int nseg, nranks, op, nstatus;
    uint32_t* status_out;
};

// One warp per 1024 elements (128 bytes of bits): lane l loads bit word l
// of each rank (128 coalesced bytes), then for store q in 0..7 takes, by a
// shuffle, the word holding float4 number 32 q + l and writes that float4 --
// every store instruction covers 512 contiguous bytes.
__global__ void __launch_bounds__(kThreads) onebit_reduce_k(const __grid_constant__ ObParams p) {
    if (p.status_out && blockIdx.x == 0) {
        __shared__ unsigned int sSt;
        if (threadIdx.x == 0) sSt = 0u;
        __syncthreads();
        for (int i = threadIdx.x; i < p.nranks * p.nstatus; i += kThreads) {
            const int r = i / p.nstatus, sg = i % p.nstatus;
            atomicOr(&sSt, *reinterpret_cast<const uint32_t*>(p.slabs + r * p.rank_stride + p.status_off + 4 * sg));
        }
        __syncthreads();
        if (threadIdx.x == 0) *p.status_out = sSt;
    }
    const int lane = threadIdx.x & 31;
    const int64_t total = p.unit_start[p.nseg];
    const float invn = 1.0f / (float)p.nranks;
    const bool pow2 = (p.nranks & (p.nranks - 1)) == 0;
    const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t u = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); u < total; u += warps) {
        int lo = 0, hi = p.nseg;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (p.unit_start[mid] <= u) lo = mid; else hi = mid;
        }
        const a8_ob_seg_t sg = p.segs[lo];
        const int64_t e_unit = (u - p.unit_start[lo]) * 1024;  // first element of this unit
        const int64_t nwords = ((sg.n + 7) / 8 + 3) / 4;
        const int64_t wj = e_unit / 32 + lane;                 // this lane's bit word
        float acc[8][4];
        for (int r = 0; r < p.nranks; ++r) {
            const uint8_t* slab = p.slabs + r * p.rank_stride;
            const uint32_t w = wj < nwords ? __ldg(reinterpret_cast<const uint32_t*>(slab + sg.bit_off) + wj) : 0u;
            const float* lv = reinterpret_cast<const float*>(slab + p.levels_off) + 2 * lo;
            const float pl = lv[0], nl = lv[1];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                // float4 number 32 q + lane = elements 4 (32 q + lane) .. +3: byte (lane & 7) >> 1 of
                // word 4 q + (lane >> 3), high nibble for even lanes (np.packbits: first element in the MSB)
                const uint32_t ww = __shfl_sync(0xffffffffu, w, 4 * q + (lane >> 3));
                const uint32_t nib = (ww >> (8 * ((lane & 7) >> 1) + ((lane & 1) ? 0 : 4))) & 15u;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float d = (nib >> (3 - t)) & 1u ? pl : nl;
                    acc[q][t] = r == 0 ? d : __fadd_rn(acc[q][t], d);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (p.op == 1) {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    acc[q][t] = pow2 ? __fmul_rn(acc[q][t], invn) : __fdiv_rn(acc[q][t], (float)p.nranks);
            }
            const int64_t e = e_unit + 4 * (32 * q + lane);
            if (e + 4 <= sg.n && (reinterpret_cast<uintptr_t>(sg.out) & 15) == 0) {
                *reinterpret_cast<float4*>(sg.out + e) = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (e + t < sg.n) sg.out[e + t] = acc[q][t];
            }
        }
    }
}

int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + kThreads * 8 - 1) / (kThreads * 8);
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min(kMaxGrid, sms * 3)));
}

int check(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        a8::g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return A8_ERR_CUDA;
    }
    return A8_OK;
}

}  // namespace

extern "C" size_t a8_onebit_workspace_bytes(void) { return sizeof(Partial) * kMaxGrid; }

extern "C" int a8_onebit_quantize(const void* g, int g_is_f64, double* residual, int64_t n, uint8_t* bits,
                                  float* levels, uint32_t* status_out, void* workspace, size_t workspace_bytes,
                                  void* stream) {
    if (n < 0 || (n > 0 && (!g || !residual || !bits)) || !levels || !status_out || !workspace)
        return fail(A8_ERR_USAGE, "a8_onebit_quantize: bad argument");
    if (workspace_bytes < sizeof(Partial) * kMaxGrid)
        return fail(A8_ERR_USAGE, "a8_onebit_quantize: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Partial* part = static_cast<Partial*>(workspace);
    const int grid = grid_for(n);
    // stats -> apply share the partials in `workspace`: another host thread's
    // pair on the same stream and workspace must not interleave between them
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    onebit_stats<<<grid, kThreads, 0, st>>>(g, g_is_f64, residual, n, part);
    if (int rc = check("a8_onebit_quantize(stats)")) return rc;
    onebit_apply<<<grid, kThreads, 0, st>>>(g, g_is_f64, residual, n, part, grid, bits, levels, status_out);
    return check("a8_onebit_quantize(apply)");
}

extern "C" size_t a8_onebit_multi_workspace_bytes(int nseg) {
    return sizeof(Partial) * (size_t)kMaxGrid * (size_t)std::max(1, std::min(nseg, kQSegs));
}

extern "C" int a8_onebit_quantize_multi(const a8_ob_q_seg_t* segs, int nseg, int g_is_f64, void* workspace,
                                        size_t workspace_bytes, void* stream) {
    if (nseg < 0 || nseg > kQSegs || (nseg > 0 && !segs) || !workspace)
        return fail(A8_ERR_USAGE, "a8_onebit_quantize_multi: bad argument (at most 32 segments per call)");
    QParams p{};
    int b = 0;
    for (int i = 0; i < nseg; ++i) {
        const a8_ob_q_seg_t& q = segs[i];
        if (q.n < 0 || (q.n > 0 && (!q.g || !q.residual || !q.bits)) || !q.levels || !q.status)
            return fail(A8_ERR_USAGE, "a8_onebit_quantize_multi: bad segment");
        p.segs[i] = q;
        p.p0[i] = b;
        b += grid_for(q.n);  // the single-tensor grid: identical partials and sums
    }
    p.p0[nseg] = b;
    p.nseg = nseg;
    p.f64 = g_is_f64 ? 1 : 0;
    p.part = static_cast<Partial*>(workspace);
    if (nseg == 0) return A8_OK;
    if (workspace_bytes < sizeof(Partial) * (size_t)b)
        return fail(A8_ERR_USAGE, "a8_onebit_quantize_multi: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static std::mutex mu;  // stats -> apply share the partials (see a8_onebit_quantize)
    std::lock_guard<std::mutex> lk(mu);
    onebit_stats_multi<<<b, kThreads, 0, st>>>(p);
    if (int rc = check("a8_onebit_quantize_multi(stats)")) return rc;
    onebit_apply_multi<<<b, kThreads, 0, st>>>(p);
    return check("a8_onebit_quantize_multi(apply)");
}

extern "C" int a8_onebit_decode(const uint8_t* bits, int64_t n, const float* levels, float* out, void* stream) {
    if (n < 0 || (n > 0 && (!bits || !out)) || !levels) return fail(A8_ERR_USAGE, "a8_onebit_decode: bad argument");
    if (n == 0) return A8_OK;
    onebit_decode_k<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(bits, n, levels, out);
    return check("a8_onebit_decode");
}

extern "C" int a8_onebit_reduce(const a8_ob_seg_t* segs, int nseg, const uint8_t* slabs, int64_t rank_stride,
                                int64_t levels_off, int64_t status_off, int nstatus, int nranks, int op,
                                uint32_t* status_out, void* stream) {
    if (nseg < 0 || nseg > kObSegs || (nseg > 0 && !segs) || !slabs || nranks < 1 || nranks > 1024 || op < 0 ||
        op > 1 || nstatus < 0)
        return fail(A8_ERR_USAGE, "a8_onebit_reduce: bad argument (at most 32 segments per call)");
    ObParams p{};
    int64_t acc = 0;
    for (int i = 0; i < nseg; ++i) {
        if (segs[i].n < 0 || (segs[i].n > 0 && !segs[i].out)) return fail(A8_ERR_USAGE, "a8_onebit_reduce: bad segment");
        if (segs[i].bit_off % 16) return fail(A8_ERR_USAGE, "a8_onebit_reduce: bit_off must be a multiple of 16");
        p.segs[i] = segs[i];
        p.unit_start[i] = acc;
        acc += (segs[i].n + 1023) / 1024;
    }
    p.unit_start[nseg] = acc;
    p.slabs = slabs;
    p.rank_stride = rank_stride;
    p.levels_off = levels_off;
    p.status_off = status_off;
    p.nseg = nseg;
    p.nranks = nranks;
    p.op = op;
    p.nstatus = nstatus;
    p.status_out = status_out;
    if (acc == 0 && !status_out) return A8_OK;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((acc + kThreads / 32 - 1) / (kThreads / 32), 148 * 8));
    onebit_reduce_k<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return check("a8_onebit_reduce");
}
