// Per-block max-abs codec (the north star's "optional per-block max-abs"):
// every block of B consecutive elements (B = 1024, 2048 or 4096) gets its own
// absmax scale, computed exactly as the reference computes a tensor's
// (codecs.py:232-241), and is encoded with the reference decision
// (codecs.py:254-268) -- i.e. the result equals encode_buffer applied to
// each block separately.  Not a reference feature: it has its own oracle
// (oracle.encode_blocked) and tests.
//
// Because a block fits in one CTA's registers, the encode is a single pass:
// 4 B read + 1 B written per element (+4 B per block), no cross-CTA
// dependency, no second read of the data.  Per block: a CTA loads B floats
// (float4 per thread), reduces the max (warp shuffles + shared memory), 127
// threads evaluate the decision thresholds for that scale (threshold(), the
// reference's float64 decision), and every thread encodes its elements by a
// branch-free 7-step search over the thresholds (the paper's method).  The
// decode is table[c] * s_block (one RN multiply, codecs.py:281).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "a8_core.cuh"
#include "a8_ptx.cuh"
#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);

// G for the codebook `book_dev` (device pointer), built once per (device,
// book) by a one-CTA kernel on `stream` and cached for the process.
const uint8_t* guess_table_dev(const void* book_dev, cudaStream_t stream) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, uint8_t*> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, book_dev});
    if (it != cache.end()) return it->second;
    uint8_t* G = nullptr;
    if (cudaMalloc(&G, (kGLen + 15) & ~15) != cudaSuccess) return nullptr;
    guess_table_kernel<<<1, 256, 0, stream>>>(static_cast<const a8_book_t*>(book_dev), G);
    cache[{dev, book_dev}] = G;
    return G;
}
}  // namespace a8

using namespace a8;

namespace {

constexpr int kThreads = 256;


__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Blocks are streamed global -> shared by the TMA bulk engine, two stages per
// CTA: block k+1 is in flight while block k is reduced, its thresholds
// evaluated and its codes written.  Full blocks only; the ragged last block
// (and unaligned inputs) take plain loads.
template <int V>  // float4 groups per thread: B = 1024 * V
__global__ void __launch_bounds__(kThreads, 4) blocked_encode_kernel(const float* __restrict__ x, int64_t n,
                                                                    const a8_book_t* book, uint8_t* codes,
                                                                    float* scales, unsigned int* status) {
    constexpr int B = kThreads * 4 * V;
    extern __shared__ __align__(128) float sBuf[];  // [2][B]
    __shared__ __align__(8) uint64_t sBar[2];
    __shared__ double sV[128];
    __shared__ uint32_t sT[128];
    __shared__ uint8_t sCanon[128];
    __shared__ unsigned int sRed[kThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid < 128) {
        sV[tid] = book->values[tid];
        sCanon[tid] = book->codes[tid];
    }
    const int D = book->ndistinct;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const int64_t nblk = (n + B - 1) / B;
    const int64_t nfull = aligned ? n / B : 0;  // blocks taken by bulk copies
    if (tid == 0) {
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sBar[i])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t blk, int st) {  // thread 0: bulk copy of a full block into stage st
        const uint32_t bar = smem_u32(&sBar[st]);
        asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}" ::"r"(bar),
                     "r"((uint32_t)(B * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sBuf + st * B)),
            "l"(x + blk * B), "r"((uint32_t)(B * 4)), "r"(bar)
            : "memory");
    };
    unsigned int bad = 0;
    int it = 0;
    if (tid == 0 && blockIdx.x < nfull) issue(blockIdx.x, 0);
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int st = it & 1;
        const int64_t base = blk * B;
        const int cnt = (int)min((int64_t)B, n - base);
        const bool full = blk < nfull;
        // prefetch this CTA's next block into the other stage (its previous
        // contents were consumed in iteration it-1, closed by a barrier)
        if (tid == 0 && blk + gridDim.x < nfull) issue(blk + gridDim.x, st ^ 1);
        uint4 v[V];
        unsigned int mx = 0;  // bits * 2 (drops the sign)
        if (full) {
            const uint32_t bar = smem_u32(&sBar[st]);
            const uint32_t par = (uint32_t)(it >> 1) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                    bar),
                "r"(par)
                : "memory");
#pragma unroll
            for (int q = 0; q < V; ++q) {
                v[q] = reinterpret_cast<const uint4*>(sBuf + st * B)[q * kThreads + tid];
                mx = __vimax3_u32(mx, v[q].x * 2u, v[q].y * 2u);
                mx = __vimax3_u32(mx, v[q].z * 2u, v[q].w * 2u);
            }
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const int e = (q * kThreads + tid) * 4;
                uint32_t b[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) b[k] = e + k < cnt ? __float_as_uint(x[base + e + k]) : 0u;
                v[q] = make_uint4(b[0], b[1], b[2], b[3]);
                mx = __vimax3_u32(mx, b[0] * 2u, b[1] * 2u);
                mx = __vimax3_u32(mx, b[2] * 2u, b[3] * 2u);
            }
        }
        mx = __reduce_max_sync(0xffffffffu, mx);
        __syncthreads();  // the previous block's sT / sRed are no longer read
        if (lane == 0) sRed[w] = mx;
        __syncthreads();
        unsigned int amax = 0;
#pragma unroll
        for (int i = 0; i < kThreads / 32; ++i) amax = max(amax, sRed[i]);
        amax >>= 1;
        const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);  // codecs.py:237-241
        if (amax >= kInfBits) bad = 1u;
        if (tid < 128) {
            uint32_t t = kInfBits;
            if (scale_ok(scale) && tid + 1 < D) t = threshold_fast((double)scale, sV[tid], sV[tid + 1]);
            sT[tid] = t;
        }
        if (tid == 0) scales[blk] = scale;
        __syncthreads();
        if (cnt == B && aligned) {
            uint32_t* out = reinterpret_cast<uint32_t*>(codes + base);
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const uint32_t c0 = encode_search(v[q].x, sT, sCanon), c1 = encode_search(v[q].y, sT, sCanon);
                const uint32_t c2 = encode_search(v[q].z, sT, sCanon), c3 = encode_search(v[q].w, sT, sCanon);
                __stcs(out + q * kThreads + tid, c0 | (c1 << 8) | (c2 << 16) | (c3 << 24));
            }
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const int e = (q * kThreads + tid) * 4;
                const uint32_t b[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (e + k < cnt) codes[base + e + k] = (uint8_t)encode_search(b[k], sT, sCanon);
            }
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, A8_STATUS_NONFINITE);
}

// ---------------------------------------------------------------------------
// Per-block encode, streaming form (full 4096-element chunks of 16-byte
// aligned input).  Warp 0 streams chunks global -> shared with bulk copies
// into a kBStages ring; 8 consumer warps process chunk k in two halves
// that are software-pipelined across iterations:
//   iteration k: block maxes of chunk k -> barrier -> thresholds of chunk
//   k's blocks (float64, the reference decision) AND the encode of chunk
//   k-1 (whose thresholds the previous iteration computed) -> barrier
// so the float64 latency of the thresholds overlaps the encode work.
// Encode per element, exactly the reference decision (codecs.py:254-268):
//   guess  c = G[key(fl32(|x| * fl32(1/s)))]   (G: scale-independent, per codebook)
//   verify p = c + (bits|x| >= T_c(s))          (T: the block's exact thresholds)
// G[k] counts the midpoints surely below bucket k, so c <= p <= c + 1 as
// long as every bucket (widened by the rounding of the normalised value)
// holds at most one midpoint -- true for the two absmax codebooks
// (dynamic-tree, linear; tests/test_blocked.py checks it).  Scales outside
// [2^-100, 2^100] and non-finite blocks take the 7-step threshold search.
constexpr int kBStages = 6;
constexpr int kBChunk = 4096;
constexpr int kBWarps = 8;
constexpr int kBCons = kBWarps * 32;
constexpr size_t kBDynSmem = (size_t)kBStages * kBChunk * sizeof(float);

template <int V>  // B = 1024 * V; NB = 4 / V blocks per chunk
__global__ void __launch_bounds__(kBCons + 32, 2) blocked_encode_stream(const float* __restrict__ x, int64_t nchunks,
                                                                       const a8_book_t* book, const uint8_t* Gdev,
                                                                       uint8_t* codes, float* scales,
                                                                       unsigned int* status) {
    constexpr int NB = 4 / V;
    extern __shared__ __align__(128) float sStage[];  // [kBStages][kBChunk]
    __shared__ __align__(16) uint8_t sG[(kGLen + 15) & ~15];
    __shared__ uint32_t sT[2][NB][128];
    __shared__ float sR[2][NB];
    __shared__ int sFast[2];
    __shared__ unsigned int sRed[kBWarps][NB];
    __shared__ double sV[128];
    __shared__ uint8_t sCanon[128];
    __shared__ __align__(8) uint64_t sFull[kBStages];
    __shared__ __align__(8) uint64_t sEmpty[kBStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int D = book->ndistinct;
    if (tid < 128) {
        sV[tid] = book->values[tid];
        sCanon[tid] = book->codes[tid];
    }
    for (int j = tid; j < (kGLen + 15) / 16; j += blockDim.x)
        reinterpret_cast<uint4*>(sG)[j] = reinterpret_cast<const uint4*>(Gdev)[j];
    if (tid == 0) {
        for (int i = 0; i < kBStages; ++i) {
            mbar_init(&sFull[i], 1);
            mbar_init(&sEmpty[i], kBWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t nmy = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t full0 = smem_addr(&sFull[0]), empty0 = smem_addr(&sEmpty[0]);
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t drop = policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            const float* src = x + (int64_t)blockIdx.x * kBChunk;
            const int64_t step = (int64_t)gridDim.x * kBChunk;
            for (int64_t it = 0; it < nmy; ++it, src += step) {
                mbar_wait_a(empty0 + 8u * st, ph ^ 1u);
                mbar_arrive_expect_tx(&sFull[st], kBChunk * 4);
                bulk_g2s(sStage + (size_t)st * kBChunk, src, kBChunk * 4, &sFull[st], drop);
                if (++st == kBStages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int ct = tid - 32, cw = warp - 1;
    const uint32_t gmin = smem_addr(sG), gaddr = gmin - (uint32_t)kGKey0;
    unsigned int bad = 0;
    int st = 0, pst = 0;  // stage of chunk it / it-1
    uint32_t ph = 0;
    for (int64_t it = 0; it <= nmy; ++it) {
        const int slot = (int)(it & 1);
        const int64_t chunk = blockIdx.x + it * gridDim.x;
        // sFast[slot]: cleared below by any non-fast block of chunk it; its
        // last readers (iteration it-1's encode of chunk it-2) passed the barrier
        if (ct == 0) sFast[slot] = 1;
        if (it < nmy) {  // ---- block maxes of chunk it
            mbar_wait_a(full0 + 8u * st, ph);
            const uint4* in = reinterpret_cast<const uint4*>(sStage + (size_t)st * kBChunk) + ct;
            unsigned int mx[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) mx[j] = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = in[q * kBCons];
                mx[q / V] = __vimax3_u32(mx[q / V], v.x * 2u, v.y * 2u);
                mx[q / V] = __vimax3_u32(mx[q / V], v.z * 2u, v.w * 2u);
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const unsigned int w = __reduce_max_sync(0xffffffffu, mx[j]) >> 1;
                if (lane == 0) sRed[cw][j] = w;
            }
        }
        nbar_sync(1, kBCons);
        if (it < nmy) {  // ---- thresholds of chunk it's blocks (codecs.py:237-241, 260-265)
            bool fast = true;
            for (int k = ct; k < 128 * NB; k += kBCons) {
                const int j = k >> 7, i = k & 127;
                unsigned int amax = 0;
#pragma unroll
                for (int w = 0; w < kBWarps; ++w) amax = max(amax, sRed[w][j]);
                const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
                uint32_t t = kInfBits;
                if (scale_ok(scale) && i + 1 < D) t = threshold_fast((double)scale, sV[i], sV[i + 1]);
                sT[slot][j][i] = t;
                fast &= amax >= 0x0d800000u && amax <= 0x71800000u;  // 2^-100 <= s <= 2^100
                if (i == 0) {
                    scales[chunk * NB + j] = scale;
                    sR[slot][j] = __frcp_rn(scale);
                    if (amax >= kInfBits) bad = 1u;
                }
            }
            if (!fast) sFast[slot] = 0;
        }
        if (it > 0) {  // ---- encode chunk it-1 with the previous iteration's thresholds
            const int ps = slot ^ 1;
            const uint4* in = reinterpret_cast<const uint4*>(sStage + (size_t)pst * kBChunk) + ct;
            uint32_t* out = reinterpret_cast<uint32_t*>(codes + (chunk - gridDim.x) * (int64_t)kBChunk) + ct;
            if (sFast[ps]) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = q / V;
                    const uint4 v = in[q * kBCons];
                    const float r = sR[ps][j];
                    const uint32_t ta = smem_addr(sT[ps][j]);
                    const uint32_t c0 = guess_verify(v.x, r, gaddr, gmin, ta), c1 = guess_verify(v.y, r, gaddr, gmin, ta);
                    const uint32_t c2 = guess_verify(v.z, r, gaddr, gmin, ta), c3 = guess_verify(v.w, r, gaddr, gmin, ta);
                    const uint32_t packed = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
                    __stcs(out + q * kBCons, attach_signs4(packed, v.x, v.y, v.z, v.w));
                }
            } else {  // tiny / huge scales or non-finite blocks: 7-step threshold search
#pragma unroll 1
                for (int q = 0; q < 4; ++q) {
                    const uint32_t* T = sT[ps][q / V];
                    const uint4 v = in[q * kBCons];
                    const uint32_t c0 = encode_search(v.x & 0x7fffffffu, T, sCanon), c1 = encode_search(v.y & 0x7fffffffu, T, sCanon);
                    const uint32_t c2 = encode_search(v.z & 0x7fffffffu, T, sCanon), c3 = encode_search(v.w & 0x7fffffffu, T, sCanon);
                    const uint32_t packed = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
                    __stcs(out + q * kBCons, attach_signs4(packed, v.x, v.y, v.z, v.w));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_a(empty0 + 8u * pst);
        }
        nbar_sync(1, kBCons);  // sT[slot] / sFast[slot] complete; sRed free
        pst = st;
        if (++st == kBStages) {
            st = 0;
            ph ^= 1u;
        }
    }
    if (bad) atomicOr(status, A8_STATUS_NONFINITE);
}

template <int V>
__global__ void __launch_bounds__(kThreads) blocked_decode_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                                 const float* __restrict__ scales,
                                                                 const a8_book_t* book, float* __restrict__ out) {
    constexpr int B = kThreads * 4 * V;
    __shared__ float sTab[256];
    sTab[threadIdx.x] = book->table[threadIdx.x];
    __syncthreads();
    const int tid = threadIdx.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const int64_t nblk = (n + B - 1) / B;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t base = blk * B;
        const int cnt = (int)min((int64_t)B, n - base);
        const float s = __ldg(scales + blk);
        if (cnt == B && aligned) {
            uint32_t wd[V];
#pragma unroll
            for (int q = 0; q < V; ++q) wd[q] = __ldcs(reinterpret_cast<const uint32_t*>(codes + base) + q * kThreads + tid);
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const float4 d = make_float4(__fmul_rn(sTab[wd[q] & 255u], s), __fmul_rn(sTab[(wd[q] >> 8) & 255u], s),
                                             __fmul_rn(sTab[(wd[q] >> 16) & 255u], s), __fmul_rn(sTab[wd[q] >> 24], s));
                __stcs(reinterpret_cast<float4*>(out + base) + q * kThreads + tid, d);  // codecs.py:281
            }
        } else {
            for (int i = tid; i < cnt; i += kThreads) out[base + i] = __fmul_rn(sTab[codes[base + i]], s);
        }
    }
}

// Per-block decode of full 4096-element chunks, staged like the exchange's
// decode_tma_kernel: a producer lane bulk-copies each chunk's 4 KB of codes
// into a 3-stage ring; 8 consumer warps decode (the 256-entry table
// replicated per lane, one scale per block of the chunk) into a 16 KB
// output buffer that one thread bulk-stores (3 buffers in flight).
constexpr int kDbStages = 3, kDbOut = 3;
constexpr size_t kDbDynSmem = 256u * 32u * sizeof(float) + (size_t)kDbStages * kBChunk +
                              (size_t)kDbOut * kBChunk * sizeof(float);

template <int V>  // B = 1024 * V; NB = 4 / V blocks per chunk
__global__ void __launch_bounds__(kBCons + 32, 2) blocked_decode_stream(const uint8_t* __restrict__ codes,
                                                                       int64_t nchunks,
                                                                       const float* __restrict__ scales,
                                                                       const a8_book_t* book, float* out) {
    constexpr int NB = 4 / V;
    extern __shared__ __align__(128) float sDyn[];
    float* const sTab = sDyn;                                                       // [256][32]
    uint8_t* const sCodes = reinterpret_cast<uint8_t*>(sDyn + 256 * 32);           // [stage][4096]
    float* const sOut = reinterpret_cast<float*>(sCodes + (size_t)kDbStages * kBChunk);  // [3][4096]
    __shared__ __align__(8) uint64_t sFull[kDbStages];
    __shared__ __align__(8) uint64_t sEmpty[kDbStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < kDbStages; ++i) {
            mbar_init(&sFull[i], 1);
            mbar_init(&sEmpty[i], kBWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t nmy = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t full0 = smem_addr(&sFull[0]), empty0 = smem_addr(&sEmpty[0]);
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t drop = policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < nmy; ++k) {
                const int64_t c = blockIdx.x + k * gridDim.x;
                mbar_wait_a(empty0 + 8u * st, ph ^ 1u);
                mbar_arrive_expect_tx(&sFull[st], kBChunk);
                bulk_g2s(sCodes + (size_t)st * kBChunk, codes + c * kBChunk, kBChunk, &sFull[st], drop);
                if (++st == kDbStages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int ct = tid - 32;
    {
        const float v = book->table[ct];
        float4* d = reinterpret_cast<float4*>(sTab + ct * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = make_float4(v, v, v, v);
    }
    nbar_sync(2, kBCons);
    const float* tl = sTab + lane;
    const uint64_t wpol = policy_evict_first();
    int st = 0, ob = 0;
    uint32_t ph = 0;
    for (int64_t k = 0; k < nmy; ++k) {
        const int64_t c = blockIdx.x + k * gridDim.x;
        float sc[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) sc[j] = __ldg(scales + c * NB + j);  // issued before the wait
        mbar_wait_a(full0 + 8u * st, ph);
        const uint8_t* cs = sCodes + (size_t)st * kBChunk;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint32_t*>(cs + q * 1024 + ct * 4);
        __syncwarp();
        if (lane == 0) mbar_arrive_a(empty0 + 8u * st);  // this warp is done with the codes
        float* o = sOut + (size_t)ob * kBChunk;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float s = sc[q / V];  // element q * 1024 + 4 ct + t lies in block q / V (codecs.py:281)
            reinterpret_cast<float4*>(o)[q * kBCons + ct] =
                make_float4(__fmul_rn(tl[(w[q] & 255u) * 32u], s), __fmul_rn(tl[((w[q] >> 8) & 255u) * 32u], s),
                            __fmul_rn(tl[((w[q] >> 16) & 255u) * 32u], s), __fmul_rn(tl[(w[q] >> 24) * 32u], s));
        }
        fence_proxy_async_smem();
        nbar_sync(1, kBCons);
        if (ct == 0) {
            bulk_s2g(out + c * kBChunk, o, kBChunk * 4u, wpol);
            bulk_commit();
            bulk_wait_read<kDbOut - 2>();  // the buffer of the next chunk (used 2 stores ago) is free
        }
        if (++st == kDbStages) {
            st = 0;
            ph ^= 1u;
        }
        if (++ob == kDbOut) ob = 0;
    }
    if (ct == 0) bulk_wait_all();
}

int grid_for(int64_t nblk, int per_sm) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>(nblk, (int64_t)std::max(sms, 1) * per_sm));
}

}  // namespace

extern "C" int a8_encode_blocked(const float* x, int64_t n, int64_t block, const void* book_dev, uint8_t* codes,
                                 float* scales, uint32_t* status_out, void* stream) {
    if (n < 0 || (n > 0 && (!x || !codes || !scales)) || !book_dev || !status_out)
        return fail(A8_ERR_USAGE, "a8_encode_blocked: bad argument");
    if (block != 1024 && block != 2048 && block != 4096)
        return fail(A8_ERR_USAGE, "a8_encode_blocked: block must be 1024, 2048 or 4096");
    if (reinterpret_cast<uintptr_t>(codes) & 3) return fail(A8_ERR_USAGE, "a8_encode_blocked: codes must be 4-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(status_out, 0, sizeof(uint32_t), st);
    // full 4096-element chunks of aligned input: the streaming kernel; the
    // ragged tail (and unaligned input) below
    const int64_t nchunks = (reinterpret_cast<uintptr_t>(x) & 15) ? 0 : n / kBChunk;
    if (nchunks > 0) {
        const uint8_t* G = guess_table_dev(book_dev, st);
        if (!G) return fail(A8_ERR_CUDA, "a8_encode_blocked: guess table");
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaFuncSetAttribute(blocked_encode_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBDynSmem);
            cudaFuncSetAttribute(blocked_encode_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBDynSmem);
            cudaFuncSetAttribute(blocked_encode_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBDynSmem);
        }
        const int g = (int)std::min<int64_t>(nchunks, (int64_t)sms * 2);
        const a8_book_t* book = static_cast<const a8_book_t*>(book_dev);
        unsigned int* stt = reinterpret_cast<unsigned int*>(status_out);
        if (block == 1024)
            blocked_encode_stream<1><<<g, kBCons + 32, kBDynSmem, st>>>(x, nchunks, book, G, codes, scales, stt);
        else if (block == 2048)
            blocked_encode_stream<2><<<g, kBCons + 32, kBDynSmem, st>>>(x, nchunks, book, G, codes, scales, stt);
        else
            blocked_encode_stream<4><<<g, kBCons + 32, kBDynSmem, st>>>(x, nchunks, book, G, codes, scales, stt);
        const int64_t done = nchunks * kBChunk;
        x += done;
        n -= done;
        codes += done;
        scales += done / block;
    }
    const int64_t nblk = (n + block - 1) / block;
    if (nblk > 0) {
        const a8_book_t* book = static_cast<const a8_book_t*>(book_dev);
        const int g = grid_for(nblk, 8);
        unsigned int* stt = reinterpret_cast<unsigned int*>(status_out);
        if (block == 1024)
            blocked_encode_kernel<1><<<g, kThreads, 2 * 1024 * sizeof(float), st>>>(x, n, book, codes, scales, stt);
        else if (block == 2048)
            blocked_encode_kernel<2><<<g, kThreads, 2 * 2048 * sizeof(float), st>>>(x, n, book, codes, scales, stt);
        else
            blocked_encode_kernel<4><<<g, kThreads, 2 * 4096 * sizeof(float), st>>>(x, n, book, codes, scales, stt);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int a8_decode_blocked(const uint8_t* codes, int64_t n, int64_t block, const float* scales,
                                 const void* book_dev, float* out, void* stream) {
    if (n < 0 || (n > 0 && (!codes || !scales || !out)) || !book_dev) return fail(A8_ERR_USAGE, "a8_decode_blocked: bad argument");
    if (block != 1024 && block != 2048 && block != 4096)
        return fail(A8_ERR_USAGE, "a8_decode_blocked: block must be 1024, 2048 or 4096");
    if (reinterpret_cast<uintptr_t>(codes) & 3) return fail(A8_ERR_USAGE, "a8_decode_blocked: codes must be 4-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const a8_book_t* book = static_cast<const a8_book_t*>(book_dev);
    // full chunks of 16-byte aligned codes and output, B >= 2048: the staged
    // kernel (2^30: B = 4096 1026 -> 907 us, 2048 1012 -> 920 us; for
    // B = 1024 the register kernel stays ahead, 985 vs 1022 us)
    static const bool tma = [] {
        const char* e = getenv("A8_BLK_DEC_TMA");
        return !(e && e[0] == '0');
    }();
    const int64_t nchunks = (!tma || block < 2048 ||
                             ((reinterpret_cast<uintptr_t>(codes) | reinterpret_cast<uintptr_t>(out)) & 15))
                                ? 0 : n / kBChunk;
    if (nchunks > 0) {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaFuncSetAttribute(blocked_decode_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDbDynSmem);
            cudaFuncSetAttribute(blocked_decode_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDbDynSmem);
            cudaFuncSetAttribute(blocked_decode_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDbDynSmem);
        }
        const int g = (int)std::min<int64_t>(nchunks, (int64_t)sms * 2);
        if (block == 1024)
            blocked_decode_stream<1><<<g, kBCons + 32, kDbDynSmem, st>>>(codes, nchunks, scales, book, out);
        else if (block == 2048)
            blocked_decode_stream<2><<<g, kBCons + 32, kDbDynSmem, st>>>(codes, nchunks, scales, book, out);
        else
            blocked_decode_stream<4><<<g, kBCons + 32, kDbDynSmem, st>>>(codes, nchunks, scales, book, out);
        const int64_t done = nchunks * kBChunk;
        codes += done;
        n -= done;
        out += done;
        scales += done / block;
    }
    const int64_t nblk = (n + block - 1) / block;
    if (nblk > 0) {
        const int g = grid_for(nblk, 8);
        if (block == 1024)
            blocked_decode_kernel<1><<<g, kThreads, 0, st>>>(codes, n, scales, book, out);
        else if (block == 2048)
            blocked_decode_kernel<2><<<g, kThreads, 0, st>>>(codes, n, scales, book, out);
        else
            blocked_decode_kernel<4><<<g, kThreads, 0, st>>>(codes, n, scales, book, out);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
