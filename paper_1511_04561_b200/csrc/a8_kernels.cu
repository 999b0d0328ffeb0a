// approx8 B200 kernels (sm_100a) and their C-ABI launchers.
//
//   a8_encode  -- K1+K2+K3 fused into one persistent kernel:
//                 segmented max-abs (+ non-finite detection), per-scale
//                 decision thresholds and bucket table, then the encode.
//                 Replaces encode_buffer (approx8/codecs.py:244-269).
//   a8_decode  -- K4/K5: table lookup x scale, fused with the rank-ordered
//                 float32 sum and 1/N average of N gathered code slabs.
//                 Replaces decode_buffer (codecs.py:272-282) and the
//                 cross-GPU average of the data-parallel seam (mlp.py:367-369).
//
// Both are HBM-bandwidth bound (4 B read + 1 B written per element, and the
// reverse); no tensor cores are involved.  Design notes: DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "a8_core.cuh"
#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);
extern thread_local std::string g_last_error;

constexpr int kEncThreads = 256;
constexpr int kDecThreads = 256;
constexpr int kGroups = 4;                          // float4 groups per thread per chunk
constexpr int kChunk = kEncThreads * kGroups * 4;   // 4096 elements
constexpr int kDecChunk = kDecThreads * kGroups * 4;
constexpr int kInlineSegs = 48;
constexpr int kLag = 2;        // E(s) is scheduled after A(s + kLag)
constexpr int kDecRep = 4;     // replicated decode tables (bank-conflict relief)
constexpr int kMaxRanks = 16;

// ---------------------------------------------------------------------------
// device-side plan / workspace

struct EncSegD {
    const float* x;
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t nA;       // absmax chunks (0 for fixed scales)
    int32_t nE;       // encode chunks
    int32_t aligned;  // x is 16-byte aligned
};

struct DecSegD {
    float* out;
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t aligned;
    int64_t cstart;  // first chunk id of this segment
};

struct WsHead {
    unsigned int ticket;
    unsigned int ctas_done;
    unsigned int status;
    unsigned int pad[13];
};

struct SegCtl {
    unsigned int amax;
    unsigned int a_done;
    unsigned int ready;
    unsigned int pad;
};

struct EncParams {
    a8_layout_t lay;
    const a8_book_t* book;
    const a8_lut_t* static_lut;
    WsHead* head;
    SegCtl* ctl;
    a8_lut_t* luts;
    const unsigned int* status_in;
    unsigned int* status_out;
    const EncSegD* segs_dev;
    const int64_t* bstart_dev;
    int nseg;
    int nblk;
    int lag;
    int absmax;
    int64_t total;
    EncSegD segs[kInlineSegs];
    int64_t bstart[kInlineSegs + kLag + 1];
};

struct DecParams {
    a8_layout_t lay;
    const a8_book_t* book;
    const DecSegD* segs_dev;
    int nseg;
    int nranks;
    int op;
    int status_idx;
    int status_blocks;
    unsigned int* status_out;
    int64_t total;
    DecSegD segs[kInlineSegs];
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static size_t ctl_off() { return sizeof(WsHead); }
static size_t lut_off(int nseg) { return align_up(ctl_off() + sizeof(SegCtl) * (size_t)nseg, 256); }
static size_t plan_off(int nseg) { return align_up(lut_off(nseg) + sizeof(a8_lut_t) * (size_t)nseg, 256); }
static size_t plan_bytes(int nseg) {
    const size_t enc = sizeof(EncSegD) * (size_t)nseg + sizeof(int64_t) * (size_t)(nseg + kLag + 1);
    const size_t dec = sizeof(DecSegD) * (size_t)nseg;
    return align_up(std::max(enc, dec), 256);
}

// ---------------------------------------------------------------------------
// memory helpers

__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned int ld_stream_u32(const uint8_t* p) {
    unsigned int v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// K2: thresholds + bucket table for one scale, built by one whole CTA into
// global memory (`dst`), staged through shared memory.

__device__ void build_lut_cta(const a8_book_t* book, float scale, a8_lut_t* dst, uint32_t* sT,
                              uint8_t* sCanon) {
    const int tid = threadIdx.x;
    const int D = book->ndistinct;
    if (tid < 128) {
        sCanon[tid] = book->codes[tid];
        uint32_t t = kInfBits;
        if (scale_ok(scale) && tid + 1 < D)
            t = threshold((double)scale, book->values[tid], book->values[tid + 1]);
        sT[tid] = t;
    }
    const int F = __syncthreads_count(tid < 127 && sT[tid < 128 ? tid : 0] < kInfBits);
    int32_t kbase;
    uint32_t len;
    lut_geometry(sT, (uint32_t)F, &kbase, &len);
    bool ok = true;
    if (len <= (uint32_t)kLutMax) {
        const uint32_t per = (len + blockDim.x - 1) / blockDim.x;
        const uint32_t j0 = min(len, per * tid), j1 = min(len, j0 + per);
        ok = lut_fill(sT, (uint32_t)F, sCanon, kbase, j0, j1, dst->e + j0);
    }
    const int valid = __syncthreads_and(ok) && len <= (uint32_t)kLutMax;
    if (tid < 128) dst->T[tid] = sT[tid];
    if (tid == 0) {
        dst->len = len;
        dst->kbase = kbase;
        dst->valid = valid;
        dst->nfinite = F;
        dst->scale = scale;
    }
}

// Copy a table into shared memory (readers bypass L1: the table may have
// been written by another CTA of this launch).
__device__ void load_lut_smem(const a8_lut_t* src, uint32_t* sE, uint32_t* sT, uint8_t* sCanon,
                              const a8_book_t* book, int* sHdr) {
    const int tid = threadIdx.x;
    const uint32_t len = __ldcg(&src->len);
    const uint32_t valid = __ldcg(&src->valid);
    if (valid) {
        for (uint32_t j = tid; j < len; j += blockDim.x) sE[j] = __ldcg(&src->e[j]);
    } else if (tid < 128) {
        sT[tid] = __ldcg(&src->T[tid]);
        sCanon[tid] = book->codes[tid];
    }
    if (tid == 0) {
        sHdr[0] = (int)valid;
        sHdr[1] = __ldcg(&src->kbase);
        sHdr[2] = (int)len - 1;
    }
}

// ---------------------------------------------------------------------------
// K1+K2+K3: persistent encode.  Work items ("tickets") are handed out in a
// fixed order by an atomic counter:  block b = [A-chunks of segment b]
// followed by [E-chunks of segment b - lag].  A-chunks reduce max|x| into the
// segment; the CTA finishing the last A-chunk builds that segment's table and
// publishes it; E-chunks wait for the table (it is always produced by a
// lower ticket, so the wait cannot deadlock) and encode.  E-chunks of a
// segment run in reverse order so the most recently read data (still in L2)
// is re-read first.

__global__ void __launch_bounds__(kEncThreads) encode_kernel(const __grid_constant__ EncParams p) {
    __shared__ uint32_t sE[kLutMax];
    __shared__ uint32_t sT[128];
    __shared__ uint8_t sCanon[128];
    __shared__ int sHdr[4];
    __shared__ int64_t sTicket;
    __shared__ unsigned int sRed[kEncThreads / 32];
    __shared__ int sLast;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const EncSegD* segs = p.segs_dev ? p.segs_dev : p.segs;
    const int64_t* bstart = p.bstart_dev ? p.bstart_dev : p.bstart;
    int cur = -1;  // segment whose table is in shared memory

    const uint8_t* codes_base = p.lay.codes;
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;

    if (!p.absmax) {  // fixed scale: one table for every segment
        load_lut_smem(p.static_lut, sE, sT, sCanon, p.book, sHdr);
        __syncthreads();
    }

    for (;;) {
        if (tid == 0) sTicket = (int64_t)atomicAdd(&p.head->ticket, 1u);
        __syncthreads();
        const int64_t t = sTicket;
        __syncthreads();
        if (t >= p.total) break;

        // locate the block holding ticket t (uniform across the CTA)
        int lo = 0, hi = p.nblk;  // bstart[lo] <= t < bstart[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (bstart[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        const int b = lo;
        int64_t k = t - bstart[b];
        const int nA_b = b < p.nseg ? segs[b].nA : 0;

        if (k < nA_b) {
            // ---------------- A: max-abs over one chunk --------------------
            const EncSegD sg = segs[b];
            const int64_t base = k * kChunk;
            const int64_t cnt = min((int64_t)kChunk, sg.n - base);
            unsigned int m = 0;
            if (cnt == kChunk && sg.aligned) {
                float4 v[kGroups];
#pragma unroll
                for (int q = 0; q < kGroups; ++q)
                    v[q] = ld_stream(sg.x + base + q * (kEncThreads * 4) + tid * 4);
#pragma unroll
                for (int q = 0; q < kGroups; ++q) {
                    m = max(m, __float_as_uint(v[q].x) & 0x7fffffffu);
                    m = max(m, __float_as_uint(v[q].y) & 0x7fffffffu);
                    m = max(m, __float_as_uint(v[q].z) & 0x7fffffffu);
                    m = max(m, __float_as_uint(v[q].w) & 0x7fffffffu);
                }
            } else {
                for (int64_t i = tid; i < cnt; i += kEncThreads)
                    m = max(m, __float_as_uint(sg.x[base + i]) & 0x7fffffffu);
            }
            m = __reduce_max_sync(0xffffffffu, m);
            if (lane == 0) sRed[tid >> 5] = m;
            __syncthreads();
            if (tid == 0) {
                unsigned int mm = 0;
#pragma unroll
                for (int w = 0; w < kEncThreads / 32; ++w) mm = max(mm, sRed[w]);
                SegCtl* c = p.ctl + b;
                if (mm) atomicMax(&c->amax, mm);
                __threadfence();
                const unsigned int done = atomicAdd(&c->a_done, 1u);
                sLast = (done == (unsigned int)sg.nA - 1u);
                if (sLast) {
                    __threadfence();
                    sHdr[3] = (int)atomicAdd(&c->amax, 0u);
                }
            }
            __syncthreads();
            if (sLast) {
                // K2 for this segment: scale, thresholds, bucket table
                const unsigned int amax = (unsigned int)sHdr[3];
                const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
                if (amax >= kInfBits && tid == 0) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
                build_lut_cta(p.book, scale, p.luts + b, sT, sCanon);
                if (tid < p.lay.scale_reps)
                    p.lay.scales[tid * p.lay.scale_block_stride + sg.scale_idx] = scale;
                __threadfence();
                __syncthreads();
                if (tid == 0) st_release(&p.ctl[b].ready, 1u);
                cur = -1;  // sT/sCanon were used as scratch
            }
            continue;
        }

        // ---------------- E: encode one chunk ------------------------------
        const int s = b - p.lag;
        k -= nA_b;
        const EncSegD sg = segs[s];
        const int64_t chunk = (int64_t)sg.nE - 1 - k;
        if (p.absmax) {
            if (cur != s) {
                if (tid == 0) {
                    unsigned int ns = 32;
                    while (ld_acquire(&p.ctl[s].ready) == 0u) {
                        __nanosleep(ns);
                        ns = min(ns * 2u, 1024u);
                    }
                }
                __syncthreads();
                load_lut_smem(p.luts + s, sE, sT, sCanon, p.book, sHdr);
                __syncthreads();
                cur = s;
            }
        } else if (chunk == 0 && tid < p.lay.scale_reps) {
            p.lay.scales[tid * p.lay.scale_block_stride + sg.scale_idx] = p.static_lut->scale;
        }
        const int valid = sHdr[0];
        const int32_t kbase = sHdr[1];
        const int32_t lenm1 = sHdr[2];
        const int64_t base = chunk * kChunk;
        const int64_t cnt = min((int64_t)kChunk, sg.n - base);
        unsigned int bad = 0;  // max |x| bits seen (fixed-scale specs detect NaN/Inf here)

        // flat position of this chunk and its block
        const int64_t f0 = sg.flat_off + base;
        int64_t j = f0 / L;
        int64_t bnd = (j + 1) * L;

        if (cnt == kChunk && sg.aligned) {
            float4 v[kGroups];
#pragma unroll
            for (int q = 0; q < kGroups; ++q) v[q] = ld_stream(sg.x + base + q * (kEncThreads * 4) + tid * 4);
#pragma unroll
            for (int q = 0; q < kGroups; ++q) {
                const uint32_t b0 = __float_as_uint(v[q].x), b1 = __float_as_uint(v[q].y);
                const uint32_t b2 = __float_as_uint(v[q].z), b3 = __float_as_uint(v[q].w);
                uint32_t c0, c1, c2, c3;
                if (valid) {
                    c0 = encode_lut(b0, sE, kbase, lenm1);
                    c1 = encode_lut(b1, sE, kbase, lenm1);
                    c2 = encode_lut(b2, sE, kbase, lenm1);
                    c3 = encode_lut(b3, sE, kbase, lenm1);
                } else {
                    c0 = encode_search(b0, sT, sCanon);
                    c1 = encode_search(b1, sT, sCanon);
                    c2 = encode_search(b2, sT, sCanon);
                    c3 = encode_search(b3, sT, sCanon);
                }
                bad = max(bad, max(max(b0 & 0x7fffffffu, b1 & 0x7fffffffu), max(b2 & 0x7fffffffu, b3 & 0x7fffffffu)));
                const int64_t f = f0 + q * (kEncThreads * 4) + tid * 4;
                while (f >= bnd) {
                    ++j;
                    bnd += L;
                }
                *reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(codes_base) + f + j * gap) =
                    c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
            }
        } else {
            for (int64_t i = tid; i < cnt; i += kEncThreads) {
                const uint32_t bb = __float_as_uint(sg.x[base + i]);
                const uint32_t c = valid ? encode_lut(bb, sE, kbase, lenm1) : encode_search(bb, sT, sCanon);
                bad = max(bad, bb & 0x7fffffffu);
                const int64_t f = f0 + i;
                const int64_t jj = f / L;
                const_cast<uint8_t*>(codes_base)[f + jj * gap] = (uint8_t)c;
            }
        }
        if (!p.absmax) {
            if (__syncthreads_or(bad >= kInfBits) && tid == 0) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
        }
    }

    // last CTA out leaves the workspace zeroed for the next call
    __shared__ int sFinal;
    if (tid == 0) {
        __threadfence();
        sFinal = atomicAdd(&p.head->ctas_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sFinal) {
        __threadfence();
        for (int i = tid; i < p.nseg; i += kEncThreads) {
            p.ctl[i].amax = 0u;
            p.ctl[i].a_done = 0u;
            p.ctl[i].ready = 0u;
        }
        if (tid < p.lay.scale_reps) {
            const unsigned int st = atomicAdd(&p.head->status, 0u) | (p.status_in ? *p.status_in : 0u);
            p.status_out[(int64_t)tid * p.lay.scale_block_stride] = st;
        }
        __syncthreads();
        if (tid == 0) {
            p.head->ticket = 0u;
            p.head->ctas_done = 0u;
            p.head->status = 0u;
        }
        __threadfence();
    }
}

// ---------------------------------------------------------------------------
// K4/K5: decode (+ rank-ordered sum, + 1/N average).

__global__ void __launch_bounds__(kDecThreads) decode_kernel(const __grid_constant__ DecParams p) {
    extern __shared__ float sTab[];  // [nranks][256][kDecRep]
    const int tid = threadIdx.x;
    const int rep = tid & (kDecRep - 1);
    const DecSegD* segs = p.segs_dev ? p.segs_dev : p.segs;
    const int R = p.nranks;
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;
    const float invN = 1.0f / (float)R;                  // exact when R is a power of two
    const bool pow2 = (R & (R - 1)) == 0;
    int cur = -1;
    int64_t cbase = 0;
    const uint8_t* src = nullptr;  // codes of rank 0 for this segment, flat-indexed

    if (p.status_out && blockIdx.x == 0) {
        __shared__ unsigned int sSt;
        if (tid == 0) sSt = 0u;
        __syncthreads();
        for (int i = tid; i < R * p.status_blocks; i += kDecThreads) {
            const int r = i / p.status_blocks, j = i % p.status_blocks;
            const unsigned int* w = reinterpret_cast<const unsigned int*>(
                reinterpret_cast<const uint8_t*>(p.lay.scales) + (int64_t)r * p.lay.rank_stride) +
                (int64_t)j * p.lay.scale_block_stride + p.status_idx;
            atomicOr(&sSt, __ldcg(w));
        }
        __syncthreads();
        if (tid == 0) *p.status_out = sSt;
    }

    for (int64_t c = blockIdx.x; c < p.total; c += gridDim.x) {
        int lo = 0, hi = p.nseg;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (segs[mid].cstart <= c)
                lo = mid;
            else
                hi = mid;
        }
        const DecSegD sg = segs[lo];
        if (lo != cur) {
            __syncthreads();
            const int64_t j = sg.flat_off / L;
            for (int i = tid; i < R * 256; i += kDecThreads) {
                const int r = i >> 8, code = i & 255;
                const float* sc = reinterpret_cast<const float*>(
                                      reinterpret_cast<const uint8_t*>(p.lay.scales) + (int64_t)r * p.lay.rank_stride) +
                                  j * p.lay.scale_block_stride + sg.scale_idx;
                const float v = __fmul_rn(p.book->table[code], __ldg(sc));  // codecs.py:281
#pragma unroll
                for (int q = 0; q < kDecRep; ++q) sTab[(i << 2) + q] = v;
            }
            __syncthreads();
            cur = lo;
            cbase = sg.cstart;
            src = p.lay.codes + j * gap;
        }
        const int64_t base = (c - cbase) * kDecChunk;
        const int64_t cnt = min((int64_t)kDecChunk, sg.n - base);
        const int64_t f0 = sg.flat_off + base;

        if (cnt == kDecChunk && sg.aligned) {
#pragma unroll
            for (int q = 0; q < kGroups; ++q) {
                const int64_t e = q * (kDecThreads * 4) + tid * 4;
                float a0, a1, a2, a3;
                {
                    const uint32_t w = ld_stream_u32(src + f0 + e);
                    a0 = sTab[((w & 255u) << 2) + rep];
                    a1 = sTab[(((w >> 8) & 255u) << 2) + rep];
                    a2 = sTab[(((w >> 16) & 255u) << 2) + rep];
                    a3 = sTab[((w >> 24) << 2) + rep];
                }
                for (int r = 1; r < R; ++r) {
                    const uint32_t w = ld_stream_u32(src + (int64_t)r * p.lay.rank_stride + f0 + e);
                    const float* T = sTab + r * 1024;
                    a0 = __fadd_rn(a0, T[((w & 255u) << 2) + rep]);
                    a1 = __fadd_rn(a1, T[(((w >> 8) & 255u) << 2) + rep]);
                    a2 = __fadd_rn(a2, T[(((w >> 16) & 255u) << 2) + rep]);
                    a3 = __fadd_rn(a3, T[((w >> 24) << 2) + rep]);
                }
                if (p.op == 1 && R > 1) {
                    if (pow2) {
                        a0 = __fmul_rn(a0, invN); a1 = __fmul_rn(a1, invN);
                        a2 = __fmul_rn(a2, invN); a3 = __fmul_rn(a3, invN);
                    } else {
                        const float fn = (float)R;
                        a0 = __fdiv_rn(a0, fn); a1 = __fdiv_rn(a1, fn);
                        a2 = __fdiv_rn(a2, fn); a3 = __fdiv_rn(a3, fn);
                    }
                }
                __stcs(reinterpret_cast<float4*>(sg.out + base + e), make_float4(a0, a1, a2, a3));
            }
        } else {
            for (int64_t i = tid; i < cnt; i += kDecThreads) {
                float a = sTab[((uint32_t)src[f0 + i] << 2) + rep];
                for (int r = 1; r < R; ++r)
                    a = __fadd_rn(a, sTab[r * 1024 + ((uint32_t)src[(int64_t)r * p.lay.rank_stride + f0 + i] << 2) + rep]);
                if (p.op == 1 && R > 1) a = pow2 ? __fmul_rn(a, invN) : __fdiv_rn(a, (float)R);
                sg.out[base + i] = a;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host launchers

struct DevInfo {
    int sms = 0;
    int enc_occ = 0;
    int dec_occ = 0;
};

static std::mutex g_mu;
static DevInfo g_dev[64];

static int dev_info(int device, DevInfo* out) {
    if (device < 0 || device >= 64) return fail(A8_ERR_USAGE, "device index out of range");
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo& d = g_dev[device];
    if (d.sms == 0) {
        cudaError_t e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.enc_occ, encode_kernel, kEncThreads, 0);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        const size_t dsm = (size_t)8 * 256 * kDecRep * sizeof(float);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.dec_occ, decode_kernel, kDecThreads, dsm);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        d.enc_occ = std::max(1, d.enc_occ);
        d.dec_occ = std::max(1, d.dec_occ);
    }
    *out = d;
    return A8_OK;
}

static int check_layout(const a8_layout_t& lay) {
    if (!lay.codes || !lay.scales) return fail(A8_ERR_USAGE, "layout: null codes or scales");
    if (lay.block_len <= 0 || lay.block_len % 16) return fail(A8_ERR_USAGE, "layout: block_len must be a positive multiple of 16");
    if (lay.block_stride < lay.block_len || lay.block_stride % 16)
        return fail(A8_ERR_USAGE, "layout: block_stride must be >= block_len and a multiple of 16");
    if (reinterpret_cast<uintptr_t>(lay.codes) % 16) return fail(A8_ERR_USAGE, "layout: codes must be 16-byte aligned");
    if (lay.rank_stride % 16) return fail(A8_ERR_USAGE, "layout: rank_stride must be a multiple of 16");
    if (lay.rank_stride % 4 || lay.scale_block_stride < 0) return fail(A8_ERR_USAGE, "layout: bad scale strides");
    return A8_OK;
}

static int cuda_check(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return A8_ERR_CUDA;
    }
    return A8_OK;
}

}  // namespace a8

using namespace a8;

extern "C" size_t a8_workspace_bytes(int nseg) {
    if (nseg < 1) nseg = 1;
    return plan_off(nseg) + plan_bytes(nseg);
}

extern "C" int a8_device_info(int device, int* num_sms, int* enc_ctas_per_sm, int* dec_ctas_per_sm) {
    DevInfo d;
    const int rc = dev_info(device, &d);
    if (rc) return rc;
    if (num_sms) *num_sms = d.sms;
    if (enc_ctas_per_sm) *enc_ctas_per_sm = d.enc_occ;
    if (dec_ctas_per_sm) *dec_ctas_per_sm = d.dec_occ;
    return A8_OK;
}

extern "C" int a8_encode(const a8_enc_seg_t* segs, int nseg, const void* book_dev, int norm,
                         const void* static_lut_dev, a8_layout_t layout, void* workspace,
                         const uint32_t* status_in, uint32_t* status_out, void* stream) {
    if (nseg <= 0) return fail(A8_ERR_USAGE, "a8_encode: need at least one segment");
    if (!segs || !book_dev || !workspace || !status_out) return fail(A8_ERR_USAGE, "a8_encode: null argument");
    if (norm != A8_NORM_ABSMAX && !static_lut_dev) return fail(A8_ERR_USAGE, "a8_encode: fixed-scale spec needs a static table");
    if (int rc = check_layout(layout)) return rc;
    if (layout.scale_reps < 1 || layout.scale_reps > kEncThreads) return fail(A8_ERR_USAGE, "a8_encode: scale_reps out of range");
    int device = 0;
    cudaGetDevice(&device);
    DevInfo di;
    if (int rc = dev_info(device, &di)) return rc;

    const bool absmax = norm == A8_NORM_ABSMAX;
    // scheduling order: ascending size, so that the E-chunks of the big
    // segments trail at the end and cover the last table builds
    std::vector<int> order(nseg);
    for (int i = 0; i < nseg; ++i) order[i] = i;
    if (absmax)
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return segs[a].n < segs[b].n; });

    std::vector<EncSegD> d(nseg);
    for (int i = 0; i < nseg; ++i) {
        const a8_enc_seg_t& s = segs[order[i]];
        if (s.n < 0 || (s.n > 0 && !s.x)) return fail(A8_ERR_USAGE, "a8_encode: bad segment");
        if (s.flat_off % 16) return fail(A8_ERR_USAGE, "a8_encode: flat_off must be a multiple of 16");
        const int64_t nch = (s.n + kChunk - 1) / kChunk;
        if (nch > INT32_MAX / 2) return fail(A8_ERR_USAGE, "a8_encode: segment too large");
        d[i].x = s.x;
        d[i].n = s.n;
        d[i].flat_off = s.flat_off;
        d[i].scale_idx = s.scale_idx;
        d[i].nA = absmax ? (int32_t)std::max<int64_t>(1, nch) : 0;
        d[i].nE = absmax ? (int32_t)nch : (int32_t)std::max<int64_t>(1, nch);
        d[i].aligned = (reinterpret_cast<uintptr_t>(s.x) % 16) == 0;
    }
    const int lag = absmax ? std::min(kLag, nseg) : 0;
    const int nblk = nseg + lag;
    std::vector<int64_t> bstart(nblk + 1);
    bstart[0] = 0;
    for (int b = 0; b < nblk; ++b)
        bstart[b + 1] = bstart[b] + (b < nseg ? d[b].nA : 0) + (b >= lag ? d[b - lag].nE : 0);

    uint8_t* ws = static_cast<uint8_t*>(workspace);
    EncParams p;
    memset(&p, 0, sizeof(p));
    p.lay = layout;
    p.book = static_cast<const a8_book_t*>(book_dev);
    p.static_lut = static_cast<const a8_lut_t*>(static_lut_dev);
    p.head = reinterpret_cast<WsHead*>(ws);
    p.ctl = reinterpret_cast<SegCtl*>(ws + ctl_off());
    p.luts = reinterpret_cast<a8_lut_t*>(ws + lut_off(nseg));
    p.status_in = status_in;
    p.status_out = status_out;
    p.nseg = nseg;
    p.nblk = nblk;
    p.lag = lag;
    p.absmax = absmax ? 1 : 0;
    p.total = bstart[nblk];
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nseg <= kInlineSegs) {
        std::copy(d.begin(), d.end(), p.segs);
        std::copy(bstart.begin(), bstart.end(), p.bstart);
    } else {
        uint8_t* plan = ws + plan_off(nseg);
        const size_t sb = sizeof(EncSegD) * nseg;
        cudaMemcpyAsync(plan, d.data(), sb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(plan + sb, bstart.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, st);
        p.segs_dev = reinterpret_cast<const EncSegD*>(plan);
        p.bstart_dev = reinterpret_cast<const int64_t*>(plan + sb);
    }
    const int64_t grid = std::min<int64_t>((int64_t)di.sms * di.enc_occ, std::max<int64_t>(1, p.total));
    encode_kernel<<<(unsigned)grid, kEncThreads, 0, st>>>(p);
    return cuda_check("a8_encode");
}

extern "C" int a8_decode(const a8_dec_seg_t* segs, int nseg, const void* book_dev, a8_layout_t layout,
                         int nranks, int op, int status_idx, int status_blocks, uint32_t* status_out,
                         void* workspace, void* stream) {
    if (nseg <= 0 && !status_out) return A8_OK;
    if (nseg < 0) return fail(A8_ERR_USAGE, "a8_decode: negative segment count");
    if (status_out && (status_idx < 0 || status_blocks < 1)) return fail(A8_ERR_USAGE, "a8_decode: bad status request");
    if ((nseg > 0 && !segs) || !book_dev || !workspace) return fail(A8_ERR_USAGE, "a8_decode: null argument");
    if (nranks < 1 || nranks > kMaxRanks) return fail(A8_ERR_USAGE, "a8_decode: nranks out of range");
    if (op != 0 && op != 1) return fail(A8_ERR_USAGE, "a8_decode: op must be 0 (sum) or 1 (avg)");
    if (int rc = check_layout(layout)) return rc;
    int device = 0;
    cudaGetDevice(&device);
    DevInfo di;
    if (int rc = dev_info(device, &di)) return rc;

    std::vector<DecSegD> d(nseg);
    int64_t chunks = 0;
    for (int i = 0; i < nseg; ++i) {
        const a8_dec_seg_t& s = segs[i];
        if (s.n < 0 || (s.n > 0 && !s.out)) return fail(A8_ERR_USAGE, "a8_decode: bad segment");
        if (s.flat_off % 16) return fail(A8_ERR_USAGE, "a8_decode: flat_off must be a multiple of 16");
        if (s.n > 0 && (s.flat_off / layout.block_len) != ((s.flat_off + s.n - 1) / layout.block_len))
            return fail(A8_ERR_USAGE, "a8_decode: a segment may not straddle blocks");
        d[i].out = s.out;
        d[i].n = s.n;
        d[i].flat_off = s.flat_off;
        d[i].scale_idx = s.scale_idx;
        d[i].aligned = (reinterpret_cast<uintptr_t>(s.out) % 16) == 0;
        d[i].cstart = chunks;
        chunks += (s.n + kDecChunk - 1) / kDecChunk;
    }
    if (chunks == 0 && !status_out) return A8_OK;
    DecParams p;
    memset(&p, 0, sizeof(p));
    p.lay = layout;
    p.book = static_cast<const a8_book_t*>(book_dev);
    p.nseg = nseg;
    p.nranks = nranks;
    p.op = op;
    p.status_idx = status_idx;
    p.status_blocks = status_blocks;
    p.status_out = status_out;
    p.total = chunks;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nseg <= kInlineSegs) {
        std::copy(d.begin(), d.end(), p.segs);
    } else {
        uint8_t* plan = static_cast<uint8_t*>(workspace) + plan_off(nseg);
        cudaMemcpyAsync(plan, d.data(), sizeof(DecSegD) * nseg, cudaMemcpyHostToDevice, st);
        p.segs_dev = reinterpret_cast<const DecSegD*>(plan);
    }
    const size_t smem = (size_t)nranks * 256 * kDecRep * sizeof(float);
    if (smem > 48 * 1024) {
        static thread_local bool attr_set[64] = {false};
        if (!attr_set[device]) {
            cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            attr_set[device] = true;
        }
    }
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)di.sms * di.dec_occ, chunks));
    decode_kernel<<<(unsigned)grid, kDecThreads, smem, st>>>(p);
    return cuda_check("a8_decode");
}
