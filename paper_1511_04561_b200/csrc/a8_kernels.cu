// approx8 B200 kernels (sm_100a) and their C-ABI launchers.
//
//   a8_encode  -- K1+K2+K3 fused into one persistent, warp-specialised kernel:
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
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "a8_core.cuh"
#include "a8_ptx.cuh"
#include "approx8_b200.h"

namespace a8 {
int fail(int code, const char* msg);
extern thread_local std::string g_last_error;

// ---- encode geometry ---------------------------------------------------------
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;  // threads doing reduce / encode
constexpr int kEncThreads = kConsumers + 32;     // + one producer warp
#ifndef A8_STAGES
#define A8_STAGES 4
#endif
constexpr int kStages = A8_STAGES;               // bulk-copy ring depth per CTA
constexpr int kChunk = 4096;                     // elements per stage (16 KB)
constexpr int kBarC = 1;                         // named barrier of the consumer warps
constexpr size_t kEncDynSmem = (size_t)kStages * kChunk * sizeof(float) + 2 * sizeof(a8_lut_t);  // ring + 2 table slots

// ---- decode geometry ---------------------------------------------------------
constexpr int kDecThreads = 256;
constexpr int kMaxRanks = 16;

constexpr int kInlineSegs = 32;
constexpr int kInlineBlks = 3 * kInlineSegs + 2;
static int max_blocks(int nseg) { return 7 * nseg + 8; }

// ---------------------------------------------------------------------------
// device-side plan / workspace

struct EncSegD {
    const float* x;
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t nA;       // absmax chunks (0 for fixed scales)
    int32_t nE;       // encode chunks
    int32_t aligned;  // x is 16-byte aligned (bulk copies allowed)
    int32_t src;      // index of the segment in the caller's array (a8_encode_premax maxima)
    int32_t pad;
};

// Ticket kinds.  A: max-abs of a chunk; E: encode a chunk with the segment's
// table; F: a whole single-chunk segment (max, thresholds and encode in one
// CTA, no cross-CTA dependency); END: no more work.
// B ("build") tickets: the CTA that takes one waits for the segment's A
// pass and builds + publishes its table ahead of the E pass.  The producer
// treats a B ticket like any other (it streams the segment's chunk 0, which
// the consumers ignore), so the per-ticket producer path is unchanged.
constexpr int kA = 0, kE = 1, kB = 2, kF = 3, kEnd = 4;  // kEnd: stage metadata only
#ifndef A8_BUILD_TICKETS
#define A8_BUILD_TICKETS 1
#endif

// A contiguous run of tickets over one segment: chunks c0, c0+1, ... (A, F)
// or c0, c0-1, ... (E).  c0k = c0 << 2 | kind.
struct EncBlk {
    int64_t tstart;
    int32_t seg;
    int32_t c0k;
};

struct DecSegD {
    float* out;
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t aligned;
    int64_t cstart;  // first chunk id of this segment
    const float* local;  // local-gradient variant: this rank's float32 input for the piece
};

struct WsHead {
    unsigned int ticket;
    unsigned int ctas_done;
    unsigned int status;
    unsigned int waits;  // table waits (trace)
    unsigned long long t_start_inv;  // ~min(CTA start time), trace
    unsigned long long wait_ns;      // total CTA time spent waiting for tables, trace
    // copies of the last call's trace (kept across the reset)
    unsigned long long tr_start, tr_end, tr_wait_ns;
    unsigned int tr_waits;
    unsigned int pad;
};
static_assert(sizeof(WsHead) == 64, "workspace head");

struct SegCtl {
    unsigned int amax;
    unsigned int a_done;
    unsigned int ready;  // 8-byte aligned with len: the producer reads both in one acquire load
    unsigned int len;    // published table length
    unsigned long long t_b0, t_b1;  // table build start / end (globaltimer ns), trace
    unsigned long long t_thr, t_fill;  // thresholds done / table filled, trace
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

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
    const EncBlk* blks_dev;
    int nseg;
    int nblk;
    int absmax;
    int code_hint;  // L2 policy of the code stores: 0 default, 1 evict_first, 2 evict_last (A8_CODE_HINT)
    int64_t total;
    const unsigned int* amax_in;  // a8_encode_premax: bits of max|x| per caller segment (else null)
    int64_t keep_tail;            // A8_KEEP_TAIL (tuning): < 0 keeps every A read in L2
    int pol_a, pol_e;             // L2 policies of the A / E reads (A8_POL_A / A8_POL_E)
    int pre_tables;               // a8_encode_premax: tables published by premax_tables_kernel
    EncSegD segs[kInlineSegs];
    EncBlk blks[kInlineBlks];
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
    int local_rank;  // >= 0: rank whose term is the local float32 input (decode_kernel<true>)
    int64_t rank_off[kMaxRanks];  // bytes from rank 0's codes/scales to rank r's: r * rank_stride, or
                                  // the distance between peers' slabs (a8_decode_peers, UVA)
    int rpol, wpol;               // decode_tma_kernel L2 policies (A8_DEC_RPOL / A8_DEC_WPOL tuning)
    DecSegD segs[kInlineSegs];
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Workspace layout for a capacity of `cap` segments:
//   [head][ctl x cap][tables x cap][plan for cap segments]
// The layout depends only on the capacity (derived from the workspace size),
// never on a call's segment count, so the control slots that kernels leave
// zeroed are never overlapped by another call's tables or plan.
static size_t ctl_off() { return sizeof(WsHead); }
static size_t lut_off(int cap) { return align_up(ctl_off() + sizeof(SegCtl) * (size_t)cap, 256); }
static size_t plan_off(int cap) { return align_up(lut_off(cap) + sizeof(a8_lut_t) * (size_t)cap, 256); }
static size_t plan_bytes(int nseg) {
    const size_t enc = sizeof(EncSegD) * (size_t)nseg + sizeof(EncBlk) * (size_t)max_blocks(nseg);
    const size_t dec = sizeof(DecSegD) * (size_t)nseg;
    return align_up(std::max(enc, dec), 256);
}

// ---------------------------------------------------------------------------
// K2: the decision table of one scale.  Every CTA that encodes a segment
// builds its own copy in shared memory once the segment's max is final: 128
// threads evaluate the thresholds (threshold(), two predicate evaluations
// each), then fill_lut_local expands them into the bucket table.  No table
// travels between CTAs.

__device__ __forceinline__ unsigned long long gtime();

// Expand thresholds into the bucket table in shared memory (kConsumers
// threads, 16 consecutive buckets each): count thresholds per bucket with
// shared atomics, exclusive-scan the counts (lo = #(key < k), hi = lo +
// count), then write the entries in place.  Entry-for-entry equal to
// lut_entry(); returns false (for this thread) if one of its buckets holds
// two distinct thresholds.  Needs len <= kLutMax = 16 * kConsumers.
// Carry = true: the carry format of a8_core.cuh (carry_entry; monotone
// codebooks), where a bucket may hold at most one threshold.
static_assert(kLutMax == 16 * kConsumers, "one thread per 16 buckets");
template <bool Carry = false>
__device__ bool fill_lut_local(const uint32_t* T, uint32_t F, const uint8_t* canon, int32_t kbase, uint32_t* e,
                               unsigned int* sWarp, int ctid) {
    const int lane = ctid & 31, w = ctid >> 5;
    uint4* e4 = reinterpret_cast<uint4*>(e) + 4 * ctid;
#pragma unroll
    for (int q = 0; q < 4; ++q) e4[q] = make_uint4(0u, 0u, 0u, 0u);
    nbar_sync(kBarC, kConsumers);
    if ((uint32_t)ctid < F) atomicAdd(&e[(int32_t)(T[ctid] >> kKeyShift) - kbase], 1u);
    nbar_sync(kBarC, kConsumers);
    uint32_t c[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 v = e4[q];
        c[4 * q] = v.x;
        c[4 * q + 1] = v.y;
        c[4 * q + 2] = v.z;
        c[4 * q + 3] = v.w;
    }
    uint32_t tot = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) tot += c[i];
    uint32_t inc = tot;  // inclusive warp scan of the per-thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sWarp[w] = inc;
    nbar_sync(kBarC, kConsumers);
    uint32_t lo = inc - tot;
    for (int i = 0; i < w; ++i) lo += sWarp[i];
    bool ok = true;
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const uint32_t hi = lo + c[i];
        if (Carry) {
            v[i] = carry_entry(lo, c[i], c[i] ? T[lo] : 0u);
            ok &= c[i] <= 1u;
        } else {
            v[i] = (uint32_t)canon[lo] | ((uint32_t)canon[hi] << 8);
            if (c[i]) {
                v[i] |= (T[lo] & 0xffffu) << 16;
                ok &= T[lo] == T[hi - 1];
            }
        }
        lo = hi;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) e4[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return ok;
}

// The carry-format table (a8_core.cuh carry_entry) without atomics, zero
// fill or scans: thread ctid owns buckets [16 ctid, 16 ctid + 16); two
// independent branch-free searches give the thresholds below and inside its
// range, then it walks its 16 buckets.  No barrier inside (T[] must be
// complete before the call).  Returns false (for this thread) if one of its
// buckets holds two thresholds.
__device__ __forceinline__ bool fill_lut_carry(const uint32_t* T, uint32_t F, int32_t kbase, uint32_t len,
                                               uint32_t* e, int ctid) {
    const int32_t j0 = 16 * ctid;
    if ((uint32_t)j0 >= len) return true;
    const int32_t k0 = kbase + j0;
    uint32_t p = k0 <= 0 ? 0u : count_below(T, F, (uint32_t)k0 << kKeyShift);
    const uint32_t hi = count_below(T, F, (uint32_t)(k0 + 16) << kKeyShift);
    uint32_t tp = p < hi ? T[p] : 0xffffffffu;  // next threshold inside the range
    bool ok = true;
    uint32_t v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const bool has = (int32_t)(tp >> kKeyShift) == k0 + q;
        v[q] = carry_entry(p, has ? 1u : 0u, tp);
        if (has) {
            ++p;
            tp = p < hi ? T[p] : 0xffffffffu;
            ok &= (int32_t)(tp >> kKeyShift) != k0 + q;  // a second threshold in this bucket
        }
    }
    uint4* e4 = reinterpret_cast<uint4*>(e) + 4 * ctid;
#pragma unroll
    for (int q = 0; q < 4; ++q) e4[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return ok;
}

// Copy a table into shared memory.  Readers bypass L1: the table may have
// been written by another CTA of this launch.
__device__ void load_lut_smem(const a8_lut_t* src, uint32_t* sE, uint32_t* sT, uint8_t* sCanon,
                              const a8_book_t* book, int* sHdr, int ctid, int nthreads) {
    const uint32_t len = __ldcg(&src->len);
    const uint32_t valid = __ldcg(&src->valid);
    if (valid) {  // 16-byte loads, several in flight per thread (e[] is 4096 entries)
        const uint4* s4 = reinterpret_cast<const uint4*>(src->e);
        uint4* d4 = reinterpret_cast<uint4*>(sE);
        const uint32_t n4 = (len + 3) >> 2;
#pragma unroll 4
        for (uint32_t j = ctid; j < n4; j += nthreads) d4[j] = __ldcg(&s4[j]);
    } else if (ctid < 128) {
        sT[ctid] = __ldcg(&src->T[ctid]);
        sCanon[ctid] = book->codes[ctid];
    }
    if (ctid == 0) {
        sHdr[0] = (int)valid;
        sHdr[1] = __ldcg(&src->kbase);
        sHdr[2] = (int)len - 1;
    }
}

// a8_encode_premax: a supplied max that is not max|x|.  Two non-finite
// values agree (NaN payloads differ between producers; the encode reports
// A8_STATUS_NONFINITE for them either way).
__device__ __forceinline__ bool amax_differs(unsigned int a, unsigned int b) {
    return a != b && (a < kInfBits || b < kInfBits);
}

struct StageMeta {
    int64_t base;      // first element of the chunk inside its segment
    int64_t code_off;  // byte offset of the chunk's first code (valid if simple)
    int32_t cnt;       // elements in the chunk
    int32_t bulk;      // leading elements delivered to shared memory by the bulk copy
    int32_t seg;
    int32_t kind;      // 0 A, 1 E, 2 end
    int32_t simple;    // full chunk inside one block of the code layout
    int32_t last;      // the producer's next ticket is not in this run: flush after this A-chunk
    int32_t tkt;       // A8_TICKET_TRACE builds: the ticket
    int32_t tslot;     // E: table slot of this run (when the segment changes)
    int32_t tpre;      // 1: the producer bulk-copied the published table into tslot; 2: consumers fill it
    int32_t tpar;      // tpre 1: parity of that slot's fill barrier
    int32_t pad;
};

#ifdef A8_TICKET_TRACE
// Debug builds only (build.py --ticket-trace): per-ticket issue / done times.
constexpr int kTraceTickets = 1 << 17;
__device__ unsigned long long g_ticket_trace[kTraceTickets][5];  // issue, done, kind|seg|cta, t known, stage free
__device__ unsigned long long g_flush_trace[32][512][4];  // per (seg, cta): flush start, atom back, amax back, chunks
// table switches / B builds: ticket, cta | kind << 16 | tpre << 20 | mode << 24, seg, t0 (stage ready),
// t1 (max final), t2 (thresholds), t3 (table complete), t4 (published / switch done)
constexpr int kTraceSw = 1 << 14;
__device__ unsigned long long g_switch_trace[kTraceSw][8];
__device__ unsigned int g_switch_n;
#define SW_STAMP(k) do { if (ctid == 0) sw[k] = gtime(); } while (0)
#else
#define SW_STAMP(k) do { } while (0)
#endif

#ifndef A8_TICKET_BATCH
#define A8_TICKET_BATCH 2
#endif
constexpr unsigned int kTicketBatch = A8_TICKET_BATCH;  // tickets per atomic (two batches prefetched)
constexpr int kSmemSegs = 64;
constexpr int kSmemBlks = 6 * kSmemSegs + 8;  // larger plans are read from global memory

// ---------------------------------------------------------------------------
// K1+K2+K3: persistent encode.
//
// Work items ("tickets", one 4096-element chunk each) are taken in a fixed
// global order by an atomic counter.  The host builds the order as blocks of
// A-chunks (max-abs) and E-chunks (encode) per segment.  Warp 0 (producer)
// takes tickets and streams each chunk global->shared with a bulk async copy
// into a kStages-deep ring guarded by mbarriers; warps 1..8 (consumers)
// reduce or encode from shared memory.  The CTA finishing a segment's last
// A-chunk builds that segment's threshold table and publishes it; E-chunks
// wait for the table.  Every wait is on a strictly lower ticket, so the
// schedule cannot deadlock; the producer keeps prefetching while consumers
// wait, so HBM stays busy.  E-chunks run in reverse order so the data most
// recently read by the A pass (still in L2) is re-read first.

// kPremax: a8_encode_premax (maxima supplied; a separate instance so the
// two-pass kernel's code is unchanged by the check)
// Programmatic dependent launch: wait until the preceding grid (the premax
// table prologue) has completed and its writes are visible; a no-op when the
// kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// a8_encode_premax prologue: with the maxima supplied, every multi-chunk
// segment's thresholds and carry table are built and published (ready = 2)
// by one CTA each before the encode starts, so the encode's producers
// prefetch published tables from its first E ticket on (no ramp of local
// builds).  CTA b builds segment nseg-1-b (plans are sorted by size).
__global__ void __launch_bounds__(kConsumers) premax_tables_kernel(const __grid_constant__ EncParams p) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the encode may start streaming now
    __shared__ uint32_t sT[128];
    __shared__ __align__(16) uint32_t sE[kLutMax];
    const int ctid = threadIdx.x;
    const int seg = p.nseg - 1 - (int)blockIdx.x;
    const EncSegD* segs = p.segs_dev ? p.segs_dev : p.segs;
    const unsigned int amax = __ldg(p.amax_in + segs[seg].src);
    const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
    uint32_t t = kInfBits;
    if (ctid < 128) {
        if (scale_ok(scale) && ctid + 1 < p.book->ndistinct)
            t = threshold_fast((double)scale, p.book->values[ctid], p.book->values[ctid + 1]);
        sT[ctid] = t;
    }
    const int nf = __syncthreads_count(ctid < 127 && t < kInfBits);
    int32_t kb;
    uint32_t len;
    lut_geometry(sT, (uint32_t)nf, &kb, &len);
    len = max((int32_t)len, (int32_t)(amax >> kKeyShift) - kb + 1);
    const bool ok = len <= (uint32_t)kLutMax && fill_lut_carry(sT, (uint32_t)nf, kb, len, sE, ctid);
    const int valid = __syncthreads_and(ok);
    a8_lut_t* G = p.luts + seg;
    if (ctid < 128) G->T[ctid] = sT[ctid];
    if (valid) {
        uint4* d4 = reinterpret_cast<uint4*>(G->e);
        const uint4* s4 = reinterpret_cast<const uint4*>(sE);
        for (uint32_t j = ctid; j < (len + 3) >> 2; j += kConsumers) d4[j] = s4[j];
    }
    if (ctid == 0) {
        G->len = len;
        G->kbase = kb;
        G->valid = (uint32_t)valid;
        G->nfinite = (uint32_t)nf;
        G->scale = scale;
        p.ctl[seg].len = valid ? len : 0u;  // the producers copy header + e[len]: none when invalid
        p.ctl[seg].ready = 1u;  // claimed: no encode CTA builds and publishes it again
    }
    __syncthreads();
    if (ctid == 0) {
        __threadfence();
        st_release(&p.ctl[seg].ready, 2u);
    }
}

template <bool kPremax>
__global__ void __launch_bounds__(kEncThreads, 2) encode_kernel(const __grid_constant__ EncParams p) {
    extern __shared__ __align__(128) float sStage[];  // [kStages][kChunk], then a8_lut_t[2] (table slots)
    a8_lut_t* const sLut = reinterpret_cast<a8_lut_t*>(sStage + (size_t)kStages * kChunk);
    __shared__ uint32_t sT[128];  // F tickets: thresholds of a single-chunk segment
    __shared__ uint8_t sCanon[128];
    __shared__ double sV[128];
    __shared__ __align__(8) uint64_t sFull[kStages];
    __shared__ __align__(8) uint64_t sEmpty[kStages];
    __shared__ __align__(8) uint64_t sTFull[2];  // table slot s filled by the producer's bulk copy
    __shared__ unsigned int sRel[2];             // warps that left table slot s (monotone count)
    __shared__ StageMeta sMeta[kStages];
    __shared__ int sHdr[4];
    __shared__ unsigned int sRed[kConsumerWarps];
    __shared__ unsigned int sRed2[2][kConsumerWarps];  // A-run flushes
    __shared__ int sMode;                              // E switch: build / copy / build + publish
    __shared__ int sFinal;
    // the plan, staged in shared memory when it fits: the producer reads it
    // on every ticket, and kernel-parameter / global reads cost it latency
    __shared__ EncSegD sSeg[kSmemSegs];
    __shared__ EncBlk sBlk[kSmemBlks];
    __shared__ unsigned int sPmax[kPremax ? kSmemSegs : 1];  // supplied maxima, by (sorted) segment

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const EncSegD* segs = p.segs_dev ? p.segs_dev : p.segs;
    const EncBlk* blks = p.blks_dev ? p.blks_dev : p.blks;
    if (p.nseg <= kSmemSegs && p.nblk + 1 <= kSmemBlks) {
        for (int i = tid; i < p.nseg; i += kEncThreads) sSeg[i] = segs[i];
        for (int i = tid; i <= p.nblk; i += kEncThreads) sBlk[i] = blks[i];
        segs = sSeg;
        blks = sBlk;
    }

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sFull[s], 1);
            mbar_init(&sEmpty[s], kConsumerWarps);
        }
        mbar_init(&sTFull[0], 1);
        mbar_init(&sTFull[1], 1);
        sRel[0] = sRel[1] = 0u;
        mbar_fence_init();
    }
    if (tid == 0) atomicMax(&p.head->t_start_inv, ~gtime());
    if (tid >= 32 && tid < 32 + 128) {  // codebook in shared memory (table builds)
        sV[tid - 32] = p.book->values[tid - 32];
        sCanon[tid - 32] = p.book->codes[tid - 32];
    }
    if (!p.absmax && tid >= 32)  // fixed scale: one table (slot 0) for every segment
        load_lut_smem(p.static_lut, sLut[0].e, sLut[0].T, sCanon, p.book, sHdr, tid - 32, kConsumers);
    if (kPremax) {
        const EncSegD* gs = p.segs_dev ? p.segs_dev : p.segs;
        for (int i = tid; i < min(p.nseg, kSmemSegs); i += kEncThreads) sPmax[i] = __ldg(p.amax_in + gs[i].src);
    }
    __syncthreads();
    const uint32_t full0 = smem_addr(&sFull[0]), empty0 = smem_addr(&sEmpty[0]);  // ring barriers

    if (warp == 0) {
        // ===================== producer =====================
        if (lane == 0) {
            // L2 policies (A8_POL_A / A8_POL_E tuning: 0 evict_first, 1 normal, 2 evict_last).
            // Both evict_first: the A pass's lines are not worth keeping (the E
            // re-read comes a fill distance later, ~100 MB of traffic away), and
            // keeping them evicts what is reused: C3 encode 105.0 -> 96.8 us,
            // bench step 171.7 -> 161.6 us (the decode gains too).
            auto pol = [](int k) { return k == 2 ? policy_evict_last() : k == 1 ? policy_evict_normal() : policy_evict_first(); };
            const uint64_t keep = pol(p.pol_a);  // A reads
            const uint64_t drop = pol(p.pol_e);  // E reads: last use
            const int64_t L = p.lay.block_len;
            const int64_t gap = p.lay.block_stride - p.lay.block_len;
            // tickets come in batches, requested two batches ahead so the
            // atomic's round trip (1-3 us under full HBM load) never stalls
            int64_t tb = (int64_t)atomicAdd(&p.head->ticket, kTicketBatch);
            int64_t tq1 = (int64_t)atomicAdd(&p.head->ticket, kTicketBatch);
            int64_t tq2 = 0;
            int lo = 0;       // block of the current ticket (tickets only increase)
            unsigned int g = 0;
            // table slots: every change of the E segment in this CTA's ticket
            // stream moves to the other slot; the producer fills it with a
            // bulk copy of the published table when it can (tpre = 1), else
            // the consumers copy or build it (tpre = 2)
            int pseg = -1, pslot = 1;
            unsigned int uses0 = 0u, uses1 = 0u, fills0 = 0u, fills1 = 0u;  // per slot (scalars: no local memory)
            for (int it = 0;; ++it) {
                const int st = it % kStages;
                if (g == 0) tq2 = (int64_t)atomicAdd(&p.head->ticket, kTicketBatch);
                const int64_t t = tb + g;
                if (++g == kTicketBatch) {
                    g = 0;
                    tb = tq1;
                    tq1 = tq2;
                }
#ifdef A8_TICKET_TRACE
                asm volatile("" ::"l"(t));
                const unsigned long long tr_known = gtime();
#endif
                mbar_wait_a(empty0 + 8u * st, ((it / kStages) & 1) ^ 1);
#ifdef A8_TICKET_TRACE
                const unsigned long long tr_free = gtime();
#endif
                StageMeta m;
                if (t >= p.total) {
                    m.kind = kEnd;
                    sMeta[st] = m;
                    mbar_arrive(&sFull[st]);
                    break;
                }
                while (blks[lo + 1].tstart <= t) ++lo;  // blks[lo].tstart <= t < blks[lo+1].tstart
                const EncBlk bk = blks[lo];
                const EncSegD& sg = segs[bk.seg];
                const int64_t k = t - bk.tstart;
                const int kind = bk.c0k & 3;
                const int64_t c0 = bk.c0k >> 2;
                const int64_t chunk = kind == kE ? c0 - k : c0 + k;
                m.base = chunk * kChunk;
                m.cnt = (int32_t)min((int64_t)kChunk, sg.n - m.base);
                m.bulk = (sg.aligned && kind != kB) ? (m.cnt & ~3) : 0;  // B: the stage is build scratch
                m.seg = bk.seg;
                m.kind = kind;
                m.tpre = 0;
                {
                    const int64_t f0 = sg.flat_off + m.base;
                    if (f0 < L) {  // one block (the common layout): no 64-bit divide or multiply
                        m.code_off = f0;
                        m.simple = m.bulk == kChunk && f0 + kChunk <= L;
                    } else {
                        const int64_t j = f0 / L;
                        m.code_off = f0 + j * gap;
                        m.simple = m.bulk == kChunk && f0 + kChunk <= (j + 1) * L;
                    }
                }
                {   // peek at this CTA's next ticket (tb + g after the advance above): an
                    // A run's partial max is published as soon as its last chunk is
                    // reduced, not when the next chunk's data arrives
                    const int64_t tn = tb + g;
                    m.last = !(tn < blks[lo + 1].tstart);
                }
                if (p.absmax && kind == kE && bk.seg != pseg) {
                    if (kPremax && p.pre_tables && pseg < 0) pdl_wait();  // tables of the prologue launch
                    pseg = bk.seg;
                    pslot ^= 1;
                    const unsigned int u = pslot ? uses1++ : uses0++;
                    m.tslot = pslot;
                    m.tpre = 2;
                    // the slot is free once all consumer warps left its previous table
                    if (u == 0u || *(volatile unsigned int*)&sRel[pslot] >= kConsumerWarps * u) {
                        const uint2 rl = ld_acquire_v2(&p.ctl[bk.seg].ready);  // {ready, len}
                        if (rl.x == 2u) {
                            fence_proxy_async();  // the acquired table, seen by the bulk copy
                            const uint32_t bytes = (uint32_t)(offsetof(a8_lut_t, e) + ((rl.y * 4u + 15u) & ~15u));
                            mbar_arrive_expect_tx(&sTFull[pslot], bytes);
                            bulk_g2s(&sLut[pslot], p.luts + bk.seg, bytes, &sTFull[pslot], keep);
                            m.tpre = 1;
                            m.tpar = (int32_t)((pslot ? fills1++ : fills0++) & 1u);
                        }
                    }
                }
#ifdef A8_TICKET_TRACE
                m.tkt = (int32_t)t;
                if (t < kTraceTickets) {
                    g_ticket_trace[t][0] = gtime();
                    g_ticket_trace[t][2] = ((uint64_t)kind << 40) | ((uint64_t)bk.seg << 20) | blockIdx.x;
                    g_ticket_trace[t][3] = tr_known;
                    g_ticket_trace[t][4] = tr_free;
                }
#endif
                sMeta[st] = m;
                const uint32_t tx = (uint32_t)m.bulk * 4u;
                if (tx > 0) {
                    mbar_arrive_expect_tx(&sFull[st], tx);
                    // A reads take the `keep` policy; with keep_tail set (A8_KEEP_TAIL,
                    // tuning) only the largest segment's last keep_tail chunks do
                    const bool kp = kind == kA && (p.keep_tail < 0 || (bk.seg == p.nseg - 1 && chunk >= sg.nA - p.keep_tail));
                    bulk_g2s(sStage + (size_t)st * kChunk, sg.x + m.base, tx, &sFull[st], kp ? keep : drop);
                } else {
                    mbar_arrive(&sFull[st]);
                }
            }
        }
    } else {
        // ===================== consumers =====================
        const int ctid = tid - 32;
        const int cw = warp - 1;
        int cur = p.absmax ? -1 : -2;  // segment whose table is in slot `cslot` (-2: static)
        int cslot = 0;
        const a8_lut_t* tab = &sLut[0];
        int tvalid = sHdr[0], tkbase = sHdr[1], tlenm1 = sHdr[2];  // that table's geometry
        unsigned int tamax = 0;  // that table's max |x| bits
        uint8_t* const codes_base = p.lay.codes;
        const int64_t L = p.lay.block_len;
        const int64_t gap = p.lay.block_stride - p.lay.block_len;

        // A-chunks of one segment are reduced in registers; the CTA publishes
        // its partial max and chunk count once per run (when the next stage
        // is not an A-chunk of the same segment), so the global atomics and
        // barriers are off the per-chunk path.
#ifdef A8_TICKET_TRACE
        int sw_tkt = 0;  // ticket of the stage being processed (switch trace)
#endif
        // a8_encode_premax: max |x| of the E chunks this thread encoded since
        // the segment changed (raw-bit maxima, see absmax_raw4; chk_a from the
        // slow paths), published to ctl[seg].amax and compared at the end
        uint32_t chk_u = 0u, chk_a = 0u;
        int32_t chk_s = INT32_MIN;
        int chk_seg = -1;
        auto chk_flush = [&]() {
            const uint32_t u = __reduce_max_sync(0xffffffffu, chk_u);
            const int32_t sm = __reduce_max_sync(0xffffffffu, chk_s);
            const uint32_t a = max(__reduce_max_sync(0xffffffffu, chk_a), abs_of_maxes(u, sm));
            if (lane == 0 && a) red_max_u32(&p.ctl[chk_seg].amax, a);
            chk_u = chk_a = 0u;
            chk_s = INT32_MIN;
            chk_seg = -1;
        };
        int aseg = -1;          // segment of the pending A run
        unsigned int amx = 0;   // per-thread max of bits(|x|) * 2
        unsigned int acnt = 0;  // A-chunks in the pending run

        // A-run flush: the CTA's partial max and chunk count go out as
        // fire-and-forget reductions (the count with release semantics, so
        // the max is visible before it); nobody waits for a round trip here.
        int fpar = 0;  // sRed2 buffer of this flush (double-buffered: no trailing barrier)
        auto flush = [&]() {
            const unsigned int wmx = __reduce_max_sync(0xffffffffu, amx) >> 1;
            if (lane == 0) sRed2[fpar][cw] = wmx;
            nbar_sync(kBarC, kConsumers);
            if (ctid == 0) {
                unsigned int mm = 0;
#pragma unroll
                for (int w = 0; w < kConsumerWarps; ++w) mm = max(mm, sRed2[fpar][w]);
                SegCtl* c = p.ctl + aseg;
                if (mm) red_max_u32(&c->amax, mm);
                red_add_release(&c->a_done, acnt);
            }
            fpar ^= 1;
            aseg = -1;
            amx = 0;
            acnt = 0;
        };

        // K2 for segment `seg` into table `L` (shared memory): wait for the
        // segment's A pass, then copy its published table, or build it
        // (thresholds, 2 predicate evaluations each; carry-format buckets)
        // and, as the first CTA there, publish it.  All consumer threads.
        // kind B: only the claimant builds (T into sT, the buckets into the
        // B ticket's own 16 KB stage; Lt = null) and publishes.
        auto table_switch = [&](int seg, uint32_t* T, uint32_t* E, a8_lut_t* Lt, bool btk) {
#ifdef A8_TICKET_TRACE
            unsigned long long sw[5] = {gtime(), 0, 0, 0, 0};
#endif
            if (kPremax && p.pre_tables) {
                // published by premax_tables_kernel before this launch: copy
                if (btk) return;
                pdl_wait();
                load_lut_smem(p.luts + seg, E, T, sCanon, p.book, sHdr, ctid, kConsumers);
                nbar_sync(kBarC, kConsumers);
                if (ctid == 0) {
                    Lt->valid = (uint32_t)sHdr[0];
                    Lt->kbase = sHdr[1];
                    Lt->len = (uint32_t)sHdr[2] + 1u;
                    Lt->scale = __ldcg(&p.luts[seg].scale);
                }
                nbar_sync(kBarC, kConsumers);
                return;
            }
            if (kPremax) {
                // The max is known (shared memory): build at once, no global
                // round trip on the critical path.  The CAS that elects the
                // segment's publisher is issued now and read after the build.
                unsigned int claim = 1u;
                if (ctid == 128) claim = atomicCAS(&p.ctl[seg].ready, 0u, 1u);
                const unsigned int amax = seg < kSmemSegs ? sPmax[seg] : __ldg(p.amax_in + segs[seg].src);
                const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
                uint32_t t = kInfBits;
                if (ctid < 128) {
                    if (scale_ok(scale) && ctid + 1 < p.book->ndistinct) t = threshold_fast((double)scale, sV[ctid], sV[ctid + 1]);
                    T[ctid] = t;
                }
                const int nf = nbar_popc(kBarC, kConsumers, ctid < 127 && t < kInfBits);
                SW_STAMP(2);
                int32_t kb;
                uint32_t len;
                lut_geometry(T, (uint32_t)nf, &kb, &len);
                len = max((int32_t)len, (int32_t)(amax >> kKeyShift) - kb + 1);
                const bool ok = len <= (uint32_t)kLutMax && fill_lut_carry(T, (uint32_t)nf, kb, len, E, ctid);
                const int valid = nbar_and(kBarC, kConsumers, ok);
                SW_STAMP(3);
                if (Lt && ctid == 0) {
                    Lt->len = len;
                    Lt->kbase = kb;
                    Lt->valid = (uint32_t)valid;
                    Lt->nfinite = (uint32_t)nf;
                    Lt->scale = scale;
                }
                if (ctid == 128) sMode = claim == 0u ? 3 : 1;
                nbar_sync(kBarC, kConsumers);
                const int mode = sMode;
                if (mode == 3) {
                    a8_lut_t* G = p.luts + seg;
                    if (ctid < 128) G->T[ctid] = T[ctid];
                    if (valid) {
                        uint4* d4 = reinterpret_cast<uint4*>(G->e);
                        const uint4* s4 = reinterpret_cast<const uint4*>(E);
                        for (uint32_t j = ctid; j < (len + 3) >> 2; j += kConsumers) d4[j] = s4[j];
                    }
                    if (ctid == 0) {
                        G->len = len;
                        G->kbase = kb;
                        G->valid = (uint32_t)valid;
                        G->nfinite = (uint32_t)nf;
                        G->scale = scale;
                        p.ctl[seg].len = valid ? len : 0u;  // the producers copy header + e[len]: none when invalid
                    }
                    nbar_sync(kBarC, kConsumers);
                    if (ctid == 0) {
                        __threadfence();
                        st_release(&p.ctl[seg].ready, 2u);
                    }
                }
                nbar_sync(kBarC, kConsumers);  // sMode read by all before the next switch rewrites it
#ifdef A8_TICKET_TRACE
                if (ctid == 0) {
                    sw[4] = gtime();
                    const unsigned int i = atomicAdd(&g_switch_n, 1u);
                    if (i < kTraceSw) {
                        g_switch_trace[i][0] = (unsigned long long)sw_tkt;
                        g_switch_trace[i][1] = blockIdx.x | ((unsigned long long)btk << 16) | ((unsigned long long)mode << 24);
                        g_switch_trace[i][2] = seg;
                        for (int q = 0; q < 5; ++q) g_switch_trace[i][3 + q] = sw[q];
                    }
                }
#endif
                return;
            }
            if (ctid == 0) {
                // every A-chunk of the segment reduced -> its max is final
                const SegCtl* c = p.ctl + seg;
                const unsigned int nA = (unsigned int)segs[seg].nA;
                if (ld_acquire(&c->a_done) != nA) {
                    const unsigned long long w0 = gtime();
                    unsigned int ns = 32;
                    while (ld_acquire(&c->a_done) != nA) {
                        __nanosleep(ns);
                        ns = min(ns * 2u, 256u);
                    }
                    atomicAdd(&p.head->wait_ns, gtime() - w0);  // trace
                    atomicAdd(&p.head->waits, 1u);
                }
                // the producer's max (a8_encode_premax: no A pass) or the A pass's
                sHdr[3] = (int)(kPremax ? __ldg(p.amax_in + segs[seg].src) : __ldcg(&c->amax));
                // ready: 0 none, 1 being built, 2 published
                const unsigned int r = ld_acquire(&p.ctl[seg].ready);
                int mode = 1;  // 1 build locally, 2 copy, 3 build + publish
                if (r == 2u)
                    mode = 2;
                else if (r == 0u && atomicCAS(&p.ctl[seg].ready, 0u, 1u) == 0u)
                    mode = 3;
                if (btk && mode != 3) mode = 0;  // B: someone else has it
                sMode = mode;
            }
            SW_STAMP(1);
            nbar_sync(kBarC, kConsumers);
            const unsigned int amax = (unsigned int)sHdr[3];
            const int mode = sMode;
#ifdef A8_TICKET_TRACE
            auto sw_log = [&](int md) {
                if (ctid == 0) {
                    sw[4] = gtime();
                    const unsigned int i = atomicAdd(&g_switch_n, 1u);
                    if (i < kTraceSw) {
                        g_switch_trace[i][0] = (unsigned long long)sw_tkt;
                        g_switch_trace[i][1] = blockIdx.x | ((unsigned long long)btk << 16) | ((unsigned long long)md << 24);
                        g_switch_trace[i][2] = seg;
                        for (int q = 0; q < 5; ++q) g_switch_trace[i][3 + q] = sw[q];
                    }
                }
            };
#else
            auto sw_log = [&](int) {};
#endif
            if (mode == 0) {
                sw_log(0);
                return;
            }
            if (mode == 2) {
                load_lut_smem(p.luts + seg, E, T, sCanon, p.book, sHdr, ctid, kConsumers);
                nbar_sync(kBarC, kConsumers);
                if (ctid == 0) {
                    Lt->valid = (uint32_t)sHdr[0];
                    Lt->kbase = sHdr[1];
                    Lt->len = (uint32_t)sHdr[2] + 1u;
                    Lt->scale = __ldcg(&p.luts[seg].scale);
                }
                nbar_sync(kBarC, kConsumers);
                sw_log(2);
                return;
            }
            const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
            uint32_t t = kInfBits;
            if (ctid < 128) {
                if (scale_ok(scale) && ctid + 1 < p.book->ndistinct) t = threshold_fast((double)scale, sV[ctid], sV[ctid + 1]);
                T[ctid] = t;
            }
            const int nf = nbar_popc(kBarC, kConsumers, ctid < 127 && t < kInfBits);
            SW_STAMP(2);
            int32_t kb;
            uint32_t len;
            lut_geometry(T, (uint32_t)nf, &kb, &len);
            // carry tables reach the key of the max itself: no upper clamp
            len = max((int32_t)len, (int32_t)(amax >> kKeyShift) - kb + 1);
            const bool ok = len <= (uint32_t)kLutMax && fill_lut_carry(T, (uint32_t)nf, kb, len, E, ctid);
            const int valid = nbar_and(kBarC, kConsumers, ok);  // also: e[] complete
            SW_STAMP(3);
            if (Lt && ctid == 0) {
                Lt->len = len;
                Lt->kbase = kb;
                Lt->valid = (uint32_t)valid;
                Lt->nfinite = (uint32_t)nf;
                Lt->scale = scale;
            }
            if (mode == 3) {  // publish for the CTAs that come later
                a8_lut_t* G = p.luts + seg;
                if (ctid < 128) G->T[ctid] = T[ctid];
                if (valid) {
                    uint4* d4 = reinterpret_cast<uint4*>(G->e);
                    const uint4* s4 = reinterpret_cast<const uint4*>(E);
                    for (uint32_t j = ctid; j < (len + 3) >> 2; j += kConsumers) d4[j] = s4[j];
                }
                if (ctid == 0) {
                    G->len = len;
                    G->kbase = kb;
                    G->valid = (uint32_t)valid;
                    G->nfinite = (uint32_t)nf;
                    G->scale = scale;
                    p.ctl[seg].len = valid ? len : 0u;  // the producers copy header + e[len]: none when invalid
                }
                nbar_sync(kBarC, kConsumers);
                if (ctid == 0) {
                    __threadfence();
                    st_release(&p.ctl[seg].ready, 2u);
                }
            }
            nbar_sync(kBarC, kConsumers);  // the table in Lt is complete
            sw_log(mode);
        };

        for (int it = 0;; ++it) {
            const int st = it % kStages;
            mbar_wait_a(full0 + 8u * st, (it / kStages) & 1);
            const StageMeta m = sMeta[st];
#ifdef A8_TICKET_TRACE
            sw_tkt = m.tkt | (m.tpre << 28);
#endif
            if (aseg >= 0 && (m.kind != kA || m.seg != aseg)) flush();
            if (kPremax && chk_seg >= 0 && (m.kind == kEnd || (m.kind == kE && m.seg != chk_seg))) chk_flush();
            if (m.kind == kEnd) break;
            const EncSegD& sg = segs[m.seg];
            const float* stage = sStage + (size_t)st * kChunk;

            // per-thread max of bits(x) * 2 over the chunk (the doubling drops
            // the sign on the FMA pipe; 3-way integer max)
            auto part_max = [&]() -> unsigned int {
                unsigned int mx = 0;
                if (m.bulk == kChunk) {
                    const uint4* in = reinterpret_cast<const uint4*>(stage) + ctid;
#pragma unroll
                    for (int q = 0; q < kChunk / (kConsumers * 4); ++q) {
                        const uint4 v = in[q * kConsumers];
                        mx = __vimax3_u32(mx, v.x * 2u, v.y * 2u);
                        mx = __vimax3_u32(mx, v.z * 2u, v.w * 2u);
                    }
                } else {
                    for (int i = ctid * 4; i + 4 <= m.bulk; i += kConsumers * 4) {
                        const uint4 v = *reinterpret_cast<const uint4*>(stage + i);
                        mx = __vimax3_u32(mx, v.x * 2u, v.y * 2u);
                        mx = __vimax3_u32(mx, v.z * 2u, v.w * 2u);
                    }
                    for (int i = m.bulk + ctid; i < m.cnt; i += kConsumers)
                        mx = max(mx, __float_as_uint(sg.x[m.base + i]) * 2u);
                }
                return mx;
            };

            if (m.kind == kA) {
                // ---------------- A: max |x| over the chunk ----------------
                amx = max(amx, part_max());
                __syncwarp();
                if (lane == 0) mbar_arrive_a(empty0 + 8u * st);  // stage consumed
#ifdef A8_TICKET_TRACE
                if (ctid == 0 && m.tkt < kTraceTickets) g_ticket_trace[m.tkt][1] = gtime();
#endif
                aseg = m.seg;
                ++acnt;
                if (m.last) flush();
                continue;
            }
            if (m.kind == kB) {
                // ---------------- B: build + publish the segment's table ---------
                // (if nobody has claimed it); the stage is the scratch table
                nbar_sync(kBarC, kConsumers);  // every warp is at this stage
                table_switch(m.seg, sT, reinterpret_cast<uint32_t*>(sStage + (size_t)st * kChunk), nullptr, true);
                __syncwarp();
                if (lane == 0) mbar_arrive_a(empty0 + 8u * st);
                continue;
            }

            int valid;
            int32_t kbase, lenm1;
            const uint32_t* Tsrch = sT;  // thresholds for the search fallback
            if (m.kind == kF) {
                // -------- F: a single-chunk segment, entirely in this CTA ------
                const unsigned int wmx = __reduce_max_sync(0xffffffffu, part_max()) >> 1;
                if (lane == 0) sRed[cw] = wmx;
                nbar_sync(kBarC, kConsumers);
                unsigned int amax = 0;
#pragma unroll
                for (int w = 0; w < kConsumerWarps; ++w) amax = max(amax, sRed[w]);
                const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
                if (ctid < 128) {
                    uint32_t t = kInfBits;
                    if (scale_ok(scale) && ctid + 1 < p.book->ndistinct)
                        t = threshold_fast((double)scale, sV[ctid], sV[ctid + 1]);
                    sT[ctid] = t;
                }
                if (amax >= kInfBits && ctid == 0) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
                if (kPremax && ctid == 0 && amax_differs(amax, __ldg(p.amax_in + sg.src)))
                    atomicOr(&p.head->status, A8_STATUS_AMAX_MISMATCH);
                if (ctid < p.lay.scale_reps) p.lay.scales[ctid * p.lay.scale_block_stride + sg.scale_idx] = scale;
                nbar_sync(kBarC, kConsumers);  // thresholds ready; sRed fully read
                valid = 0;  // encode by branch-free search over sT
                kbase = 0;
                lenm1 = 0;
            } else {
            // ---------------- E: encode the chunk -----------
            if (cur != m.seg && cur != -2) {
                // switch to the table slot the producer chose for this run
                const int ns = m.tslot;
                a8_lut_t* Lt = &sLut[ns];
                if (m.tpre == 1) {
#ifdef A8_TICKET_TRACE
                    const unsigned long long w0 = gtime();
#endif
                    mbar_wait(&sTFull[ns], (uint32_t)m.tpar);  // the producer's bulk copy landed
#ifdef A8_TICKET_TRACE
                    if (ctid == 0) {
                        const unsigned int i = atomicAdd(&g_switch_n, 1u);
                        if (i < kTraceSw) {
                            g_switch_trace[i][0] = (unsigned long long)sw_tkt;
                            g_switch_trace[i][1] = blockIdx.x | (4ull << 24);
                            g_switch_trace[i][2] = m.seg;
                            g_switch_trace[i][3] = w0;
                            g_switch_trace[i][4] = g_switch_trace[i][5] = g_switch_trace[i][6] = 0;
                            g_switch_trace[i][7] = gtime();
                        }
                    }
#endif
                } else {
                    nbar_sync(kBarC, kConsumers);  // every warp is at this stage (left the old slot's table)
                    table_switch(m.seg, Lt->T, Lt->e, Lt, false);
                }
                if (cur >= 0) {  // this warp has left the previous slot
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        atomicAdd(&sRel[cslot], 1u);
                    }
                }
                cur = m.seg;
                cslot = ns;
                tab = Lt;
                tvalid = (int)Lt->valid;
                tkbase = Lt->kbase;
                tlenm1 = (int)Lt->len - 1;
                tamax = __float_as_uint(Lt->scale);  // scale bits (1.0 for an all-zero segment)
            }
            if (cur != -2 && m.base == 0) {  // the CTA encoding chunk 0 publishes scale and status
                if (ctid < p.lay.scale_reps) p.lay.scales[ctid * p.lay.scale_block_stride + sg.scale_idx] = tab->scale;
                if (ctid == 0 && tamax >= kInfBits) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
            }
            if (cur == -2 && m.base == 0 && ctid < p.lay.scale_reps)
                p.lay.scales[ctid * p.lay.scale_block_stride + sg.scale_idx] = p.static_lut->scale;
            valid = tvalid;
            kbase = tkbase;
            lenm1 = tlenm1;
            Tsrch = tab->T;
            }
            const uint32_t* sEt = tab->e;
            unsigned int big = 0;  // max |x| bits (fixed-scale specs detect NaN/Inf here)
            if (m.simple && valid && m.kind == kE) {
                // fast path: a full chunk inside one block, bucket table
                uint32_t* out = reinterpret_cast<uint32_t*>(codes_base + m.code_off) + ctid;
                const uint4* in = reinterpret_cast<const uint4*>(stage) + ctid;
                const uint32_t eb = smem_addr(sEt) - (uint32_t)kbase * 4u;  // indexed by the clamped key
                const int32_t kmax = kbase + lenm1;
                if (p.absmax) {  // carry table (a8_core.cuh), 5 instructions per element
                    const int32_t emin = (int32_t)smem_addr(sEt);
                    if (kPremax) {  // supplied max: clamp the top too, and check the max
                        const int32_t emax = emin + 4 * lenm1;
#pragma unroll
                        for (int q = 0; q < kChunk / (kConsumers * 4); ++q) {
                            const uint4 v = in[q * kConsumers];
                            out[q * kConsumers] = encode4_carry_clamp(v, eb, emin, emax);
                            absmax_raw4(v, chk_u, chk_s);
                        }
                        chk_seg = m.seg;
                    } else if (p.code_hint) {
                        const uint64_t pol = p.code_hint == 1 ? policy_evict_first() : policy_evict_last();
#pragma unroll
                        for (int q = 0; q < kChunk / (kConsumers * 4); ++q)
                            st_hint_u32(out + q * kConsumers, encode4_carry(in[q * kConsumers], eb, emin), pol);
                    } else {
#pragma unroll
                        for (int q = 0; q < kChunk / (kConsumers * 4); ++q)
                            out[q * kConsumers] = encode4_carry(in[q * kConsumers], eb, emin);
                    }
                } else {
                    int32_t kacc = 0;  // max key: >= 0x7f80 iff some |x| is Inf/NaN
#pragma unroll
                    for (int q = 0; q < kChunk / (kConsumers * 4); ++q)
                        out[q * kConsumers] = encode4_lut_k(in[q * kConsumers], eb, kbase, kmax, kacc);
                    big = (uint32_t)kacc << kKeyShift;
                }
            } else {
            const int64_t f0 = sg.flat_off + m.base;
            int64_t j = f0 / L;
            int64_t bnd = (j + 1) * L;
#pragma unroll 1
            for (int q = 0; q < kChunk / (kConsumers * 4); ++q) {
                const int i = q * (kConsumers * 4) + ctid * 4;
                if (i >= m.cnt) break;
                const int64_t f = f0 + i;
                while (f >= bnd) {
                    ++j;
                    bnd += L;
                }
                if (i + 4 <= m.bulk) {
                    const uint4 v = *reinterpret_cast<const uint4*>(stage + i);
                    uint32_t c0, c1, c2, c3;
                    if (valid && p.absmax) {
                        c0 = encode_carry(v.x, sEt, kbase, lenm1);
                        c1 = encode_carry(v.y, sEt, kbase, lenm1);
                        c2 = encode_carry(v.z, sEt, kbase, lenm1);
                        c3 = encode_carry(v.w, sEt, kbase, lenm1);
                    } else if (valid) {
                        c0 = encode_lut(v.x, sEt, kbase, lenm1);
                        c1 = encode_lut(v.y, sEt, kbase, lenm1);
                        c2 = encode_lut(v.z, sEt, kbase, lenm1);
                        c3 = encode_lut(v.w, sEt, kbase, lenm1);
                    } else {
                        c0 = encode_search(v.x, Tsrch, sCanon);
                        c1 = encode_search(v.y, Tsrch, sCanon);
                        c2 = encode_search(v.z, Tsrch, sCanon);
                        c3 = encode_search(v.w, Tsrch, sCanon);
                    }
                    big = max(big, max(max(v.x & 0x7fffffffu, v.y & 0x7fffffffu), max(v.z & 0x7fffffffu, v.w & 0x7fffffffu)));
                    *reinterpret_cast<uint32_t*>(codes_base + f + j * gap) = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
                } else {
                    const int e_end = min(i + 4, m.cnt);
                    for (int e = i; e < e_end; ++e) {
                        const uint32_t b = e < m.bulk ? __float_as_uint(stage[e]) : __float_as_uint(sg.x[m.base + e]);
                        const uint32_t c = !valid ? encode_search(b, Tsrch, sCanon)
                                           : p.absmax ? encode_carry(b, sEt, kbase, lenm1)
                                                      : encode_lut(b, sEt, kbase, lenm1);
                        big = max(big, b & 0x7fffffffu);
                        const int64_t fe = f0 + e;
                        const int64_t je = fe / L;
                        codes_base[fe + je * gap] = (uint8_t)c;
                    }
                }
            }
            }
            if (!p.absmax && __any_sync(0xffffffffu, big >= kInfBits) && lane == 0)
                atomicOr(&p.head->status, A8_STATUS_NONFINITE);
            if (kPremax && m.kind == kE && !(m.simple && valid)) {  // slow path: big is max |x|
                chk_a = max(chk_a, big);
                chk_seg = m.seg;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_a(empty0 + 8u * st);
#ifdef A8_TICKET_TRACE
            if (ctid == 0 && m.tkt < kTraceTickets) g_ticket_trace[m.tkt][1] = gtime();
#endif
        }
    }

    // last CTA out publishes the status and leaves the workspace zeroed
    if (kPremax && p.pre_tables) pdl_wait();  // (it resets the prologue's table flags)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        sFinal = atomicAdd(&p.head->ctas_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sFinal) {
        __threadfence();
        for (int i = tid; i < p.nseg; i += kEncThreads) {
            // a8_encode_premax: the E pass's max of each multi-chunk segment
            // must be the supplied one (F segments checked their own)
            if (kPremax && segs[i].nE > 0 && amax_differs(__ldcg(&p.ctl[i].amax), __ldg(p.amax_in + segs[i].src)))
                atomicOr(&p.head->status, A8_STATUS_AMAX_MISMATCH);
            p.ctl[i].amax = 0u;
            p.ctl[i].a_done = 0u;
            p.ctl[i].ready = 0u;
            p.ctl[i].len = 0u;
        }
        __syncthreads();
        if (tid < p.lay.scale_reps) {
            const unsigned int stt = atomicAdd(&p.head->status, 0u) | (p.status_in ? *p.status_in : 0u);
            p.status_out[(int64_t)tid * p.lay.scale_block_stride] = stt;
        }
        __syncthreads();
        if (tid == 0) {
            WsHead* h = p.head;
            h->tr_start = ~h->t_start_inv;
            h->tr_end = gtime();
            h->tr_wait_ns = h->wait_ns;
            h->tr_waits = h->waits;
            h->ticket = 0u;
            h->ctas_done = 0u;
            h->status = 0u;
            h->waits = 0u;
            h->t_start_inv = 0ull;
            h->wait_ns = 0ull;
        }
        __threadfence();
    }
}

// ---------------------------------------------------------------------------
// K1+K2+K3 resident: absmax calls whose data fits in the shared memory of the
// whole GPU (148 SMs x ~200 KB ~ 30 MB: small models, DDP-sized buckets).
//
// One CTA per SM, cooperative launch.  Each CTA owns one contiguous slice of
// the concatenated elements and streams it global->shared ONCE with bulk
// async copies (the 16-byte aligned middle of every segment piece; scalar
// loads for the ragged ends).  Per-piece max-abs from shared memory ->
// atomicMax per segment -> one grid barrier -> every CTA builds the
// thresholds and bucket table of the segments it holds and encodes them
// from shared memory.  DRAM traffic is the 5 B/element floor (4 read + 1
// written) instead of 9, and there is one global synchronisation instead of
// per-segment ticket dependencies.

#ifdef A8_TICKET_TRACE
__device__ unsigned long long g_res_trace[2][8];  // CTA 0 and the last CTA: phase stamps (debug builds)
#define RES_STAMP(i)                                                                       \
    do {                                                                                   \
        if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))                  \
            g_res_trace[blockIdx.x == 0 ? 0 : 1][i] = gtime();                             \
    } while (0)
#else
#define RES_STAMP(i) \
    do {             \
    } while (0)
#endif

// The 127 decision thresholds of one scale with 4 threads per threshold
// (threads 0..511): the 8 float32 patterns around the rounded midpoint are
// tested in parallel and the first one resolving upward is T_i -- the same
// result as threshold() (the reference decision is monotone), in one
// predicate evaluation instead of a sequential walk.  If the transition is
// outside the window, lane 0 of the group falls back to threshold().
__device__ void threshold_parallel(float scale, const a8_book_t* book, uint32_t* sT, int tid) {
    const int i = tid >> 2, j = tid & 3;
    uint32_t t = kInfBits;
    bool fallback = false;
    const bool active = i < 128 && scale_ok(scale) && i + 1 < book->ndistinct;
    double s = scale, vlo = 0.0, vhi = 0.0;
    uint32_t g = 0;
    if (active) {
        vlo = book->values[i];
        vhi = book->values[i + 1];
        const double m = 0.5 * (vlo + vhi) * s;
        g = m < 3.4028234663852886e38 ? f32_bits((float)m) : kInfBits;
        fallback = g < 8u || g >= kInfBits - 8u;
    }
    bool p0 = false, p1 = false;
    if (active && !fallback) {
        const uint32_t c0 = g - 3u + 2u * (uint32_t)j;
        p0 = picks_upper(c0, s, vlo, vhi);
        p1 = picks_upper(c0 + 1u, s, vlo, vhi);
    }
    // the group's 8 predicates, candidate order g-3 .. g+4
    const unsigned int b = __ballot_sync(0xffffffffu, p0) , c = __ballot_sync(0xffffffffu, p1);
    const int base = (tid & 31) & ~3;
    unsigned int bits = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) bits |= (((b >> (base + q)) & 1u) << (2 * q)) | (((c >> (base + q)) & 1u) << (2 * q + 1));
    if (active && !fallback) {
        if (bits == 0u || bits == 0xffu)
            fallback = true;  // transition not inside the window
        else
            t = g - 3u + (uint32_t)__popc(~bits & 0xffu);  // predicates are false...false true...true
    }
    if (j == 0 && i < 128) sT[i] = (active && fallback) ? threshold(s, vlo, vhi) : t;
}

constexpr int kRThreads = 512;
constexpr size_t kRDynSmem = 200u * 1024u;
constexpr int kRCap = (int)(kRDynSmem / sizeof(float));  // floats per CTA
#ifndef A8_RES_SEARCH_MAX
#define A8_RES_SEARCH_MAX 4096
#endif
constexpr int64_t kRSearchMax = A8_RES_SEARCH_MAX;  // pieces up to this size skip the bucket table

struct RSeg {
    const float* x;
    float* out;  // fused round trip: decoded values (codecs.py:285-288), or null
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t aligned;  // x (and out) 16-byte aligned
    int32_t cta0;     // first CTA of the segment; its CTAs are [cta0, next segment's cta0)
    int32_t pad;
};

struct RParams {
    a8_layout_t lay;
    const a8_book_t* book;
    const a8_lut_t* static_lut;  // fixed-scale specs: the one table (no max pass, no barrier)
    WsHead* head;
    SegCtl* ctl;
    const unsigned int* status_in;
    unsigned int* status_out;
    int nseg;
    int write_codes;  // 0: fused round trip only (no codes in memory)
    const unsigned int* amax_in;  // a8_encode_premax: checked against the computed maxima
    RSeg segs[kInlineSegs + 1];  // segs[nseg].cta0 = grid
};

// Encode elements [lo, hi) of segment g from shared memory (dst[i]) with the
// table in sE (valid) or the thresholds in sT; codes through the layout.
// With g.out set, the decoded values fl(table[c] * scale) (sDec) are written
// too: the fused round trip of codecs.py:285-288.
__device__ void resident_encode_piece(const RParams& p, const RSeg& g, const float* dst, int64_t lo, int64_t hi,
                                      int64_t a0, int64_t a1, int valid, int32_t kb, uint32_t len, const uint32_t* sE,
                                      const uint32_t* sT, const uint8_t* sCanon, const float* sDec, int tid) {
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;
    const bool wc = p.write_codes != 0;
    float* const out = g.out;
    if (hi > lo) {
        const int64_t f_lo = g.flat_off + lo, f_hi = g.flat_off + hi - 1;
        const int32_t kmax = kb + (int32_t)len - 1;
        auto one = [&](int64_t i) {  // element i alone
            const uint32_t b = __float_as_uint(dst[i]);
            const uint32_t cc = valid ? encode_lut(b, sE, kb, (int32_t)len - 1) : encode_search(b, sT, sCanon);
            if (wc) {
                const int64_t f = g.flat_off + i;
                p.lay.codes[f + (f / L) * gap] = (uint8_t)cc;
            }
            if (out) out[i] = sDec[cc & 255u];
        };
        if ((f_lo / L) == (f_hi / L)) {
            uint8_t* cb = wc ? p.lay.codes + (f_lo / L) * gap + g.flat_off : nullptr;  // code of element i at cb[i]
            const uint32_t eb = smem_addr(sE) - (uint32_t)kb * 4u;
            auto group = [&](int64_t i, uint32_t w) {
                if (wc) *reinterpret_cast<uint32_t*>(cb + i) = w;
                if (out)
                    *reinterpret_cast<float4*>(out + i) =
                        make_float4(sDec[w & 255u], sDec[(w >> 8) & 255u], sDec[(w >> 16) & 255u], sDec[w >> 24]);
            };
            if (valid) {  // separate loops: the table loop stays as tight as before the search mode
                for (int64_t i = a0 + 4 * (int64_t)tid; i < a1; i += 4 * kRThreads)
                    group(i, encode4_lut(*reinterpret_cast<const uint4*>(dst + i), eb, kb, kmax));
            } else {
                for (int64_t i = a0 + 4 * (int64_t)tid; i < a1; i += 4 * kRThreads)
                    group(i, encode4_search(*reinterpret_cast<const uint4*>(dst + i), sT, sCanon));
            }
            if (tid < a0 - lo) one(lo + tid);
            if (tid < hi - a1) one(a1 + tid);
        } else {
            for (int64_t i = lo + tid; i < hi; i += kRThreads) one(i);
        }
    }
}

// Phase 4: the last CTA out publishes the status and re-zeroes the workspace.
__device__ void resident_finish(const RParams& p, int tid) {
    __shared__ int sFinal;
    __syncthreads();
    RES_STAMP(5);
    if (tid == 0) {
        __threadfence();
        sFinal = atomicAdd(&p.head->ctas_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sFinal) {
        __threadfence();
        for (int i = tid; i < p.nseg; i += kRThreads) p.ctl[i].amax = 0u;
        if (tid < p.lay.scale_reps) {
            const unsigned int stt = atomicAdd(&p.head->status, 0u) | (p.status_in ? *p.status_in : 0u);
            p.status_out[(int64_t)tid * p.lay.scale_block_stride] = stt;
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

__global__ void __launch_bounds__(kRThreads, 1) resident_encode_kernel(const __grid_constant__ RParams p) {
    extern __shared__ __align__(128) float sData[];
    __shared__ __align__(16) uint32_t sE[kLutMax];
    __shared__ uint32_t sT[128];
    __shared__ uint8_t sCanon[128];
    __shared__ unsigned int sWarp[kRThreads / 32];
    __shared__ int sHdr[4];
    __shared__ unsigned int sAmax;
    __shared__ float sDec[256];  // fused round trip: fl(table[c] * scale)
    __shared__ __align__(8) uint64_t sBar;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    // this CTA's piece: part q of c of segment s, elements [lo, hi); shared
    // offset off = lo (mod 4) keeps 16-byte groups aligned in both spaces
    int s = 0;
    while (s + 1 < p.nseg && p.segs[s + 1].cta0 <= (int)blockIdx.x) ++s;
    const RSeg& g = p.segs[s];
    const int c = p.segs[s + 1].cta0 - g.cta0, q = (int)blockIdx.x - g.cta0;
    const int64_t lo = g.n * q / c, hi = g.n * (q + 1) / c;
    const int off = (int)(lo & 3);
    float* const dst = sData + off - lo;  // dst[i], i in [lo, hi)
    const int64_t a0 = min(hi, (int64_t)((lo + 3) & ~3ll)), a1 = max(a0, (int64_t)(hi & ~3ll));
    if (tid == 0) {
        mbar_init(&sBar, 1);
        mbar_fence_init();
    }
    if (tid < 128) sCanon[tid] = p.book->codes[tid];
    RES_STAMP(0);
    __syncthreads();

    // ---- phase 1: global -> shared, once; max |x| of the piece ----------------
    if (tid == 0) {
        const bool bulk = g.aligned && a1 > a0;
        mbar_arrive_expect_tx(&sBar, bulk ? (uint32_t)(a1 - a0) * 4u : 0u);
        if (bulk) bulk_g2s(dst + a0, g.x + a0, (uint32_t)(a1 - a0) * 4u, &sBar, policy_evict_first());
    }
    if (g.aligned) {  // ragged ends by plain loads
        if (tid < a0 - lo) dst[lo + tid] = g.x[lo + tid];
        if (tid < hi - a1) dst[a1 + tid] = g.x[a1 + tid];
    } else {
        for (int64_t i = lo + tid; i < hi; i += kRThreads) dst[i] = g.x[i];
    }
    mbar_wait(&sBar, 0);
    __syncthreads();
    RES_STAMP(1);
    {
        unsigned int mx = 0;  // bits * 2 (drops the sign)
        const uint32_t* src = reinterpret_cast<const uint32_t*>(dst);
        for (int64_t i = a0 + 4 * (int64_t)tid; i < a1; i += 4 * kRThreads) {
            const uint4 v = *reinterpret_cast<const uint4*>(src + i);
            mx = __vimax3_u32(mx, v.x * 2u, v.y * 2u);
            mx = __vimax3_u32(mx, v.z * 2u, v.w * 2u);
        }
        if (tid < a0 - lo) mx = max(mx, src[lo + tid] * 2u);
        if (tid < hi - a1) mx = max(mx, src[a1 + tid] * 2u);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) sWarp[w] = mx;
        __syncthreads();
        if (tid == 0) {
            unsigned int m = 0;
            for (int i = 0; i < kRThreads / 32; ++i) m = max(m, sWarp[i]);
            if (p.static_lut) {
                sAmax = m >> 1;  // fixed scale: only the non-finite check needs the max
            } else if (m) {
                atomicMax(&p.ctl[s].amax, m >> 1);
            }
        }
    }

    if (p.static_lut) {  // fixed-scale spec: one shared table, no cross-CTA dependency
        if (tid == 0 && sAmax >= kInfBits) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
        int* hdr = sHdr;  // [valid, kbase, len-1]
        load_lut_smem(p.static_lut, sE, sT, sCanon, p.book, hdr, tid, kRThreads);
        __syncthreads();
        const float scale = p.static_lut->scale;
        if (g.out && tid < 256) sDec[tid] = __fmul_rn(p.book->table[tid], scale);  // codecs.py:281
        __syncthreads();
        if (q == 0 && tid < p.lay.scale_reps) p.lay.scales[tid * p.lay.scale_block_stride + g.scale_idx] = scale;
        if (blockIdx.x == 0)
            for (int e = 0; e < p.nseg; ++e)
                if (p.segs[e].n == 0 && tid < p.lay.scale_reps)
                    p.lay.scales[tid * p.lay.scale_block_stride + p.segs[e].scale_idx] = scale;
        resident_encode_piece(p, g, dst, lo, hi, a0, a1, hdr[0], hdr[1], (uint32_t)hdr[2] + 1u, sE, sT, sCanon, sDec,
                              tid);
        resident_finish(p, tid);
        return;
    }

    // ---- phase 2: grid barrier (cooperative launch: all CTAs are resident) ----
    RES_STAMP(2);
    if (tid == 0) {
        __threadfence();
        atomicAdd(&p.head->ticket, 1u);
        unsigned int ns = 32;
        while (ld_acquire(&p.head->ticket) < gridDim.x) {
            __nanosleep(ns);
            ns = min(ns * 2u, 256u);
        }
        sAmax = __ldcg(&p.ctl[s].amax);
    }
    __syncthreads();
    RES_STAMP(3);

    // ---- phase 3: this CTA's own table (no cross-CTA dependency), encode ------
    const unsigned int amax = sAmax;
    const float scale = amax == 0u ? 1.0f : __uint_as_float(amax);
    threshold_parallel(scale, p.book, sT, tid);
    if (g.out && tid < 256) sDec[tid] = __fmul_rn(p.book->table[tid], scale);  // codecs.py:281
    __syncthreads();  // sT[i] is written by thread 4i; the count below reads sT[tid]
    const int F = __syncthreads_count(tid < 127 && sT[tid] < kInfBits);
    int32_t kb;
    uint32_t len;
    lut_geometry(sT, (uint32_t)F, &kb, &len);
    // small pieces search the 127 thresholds directly: filling the bucket
    // table costs more than the extra shared-memory steps it saves
    bool ok = len <= (uint32_t)kLutMax && hi - lo > kRSearchMax;
    if (ok && tid < kConsumers) ok = fill_lut_local(sT, (uint32_t)F, sCanon, kb, sE, sWarp, tid);
    const int valid = __syncthreads_and(ok);
    RES_STAMP(4);
    if (q == 0) {  // the segment's first CTA publishes its scale
        if (tid < p.lay.scale_reps) p.lay.scales[tid * p.lay.scale_block_stride + g.scale_idx] = scale;
        if (tid == 0 && amax >= kInfBits) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
        if (tid == 0 && p.amax_in && amax_differs(amax, p.amax_in[s])) atomicOr(&p.head->status, A8_STATUS_AMAX_MISMATCH);
    }
    if (blockIdx.x == 0) {  // empty segments own no CTA: scale of an empty buffer (codecs.py:257-258)
        for (int e = 0; e < p.nseg; ++e) {
            if (p.segs[e].n == 0 && tid < p.lay.scale_reps)
                p.lay.scales[tid * p.lay.scale_block_stride + p.segs[e].scale_idx] = 1.0f;
            if (p.segs[e].n == 0 && tid == 0 && p.amax_in && p.amax_in[e] != 0u)
                atomicOr(&p.head->status, A8_STATUS_AMAX_MISMATCH);
        }
    }
    resident_encode_piece(p, g, dst, lo, hi, a0, a1, valid, kb, len, sE, sT, sCanon, sDec, tid);
    resident_finish(p, tid);
}

// ---------------------------------------------------------------------------
// K4/K5: decode (+ rank-ordered sum, + 1/N average).
//
// Per segment, each CTA keeps pre-scaled tables fl(table[c] * s_r) for every
// rank in shared memory, replicated 4 times.  Each thread decodes 4 groups
// of 4 elements of a chunk with all code words loaded before any store.

#ifndef A8_DEC_GROUPS
#define A8_DEC_GROUPS 4
#endif
constexpr int kDecGroups = A8_DEC_GROUPS;
constexpr int kDecChunkD = kDecThreads * kDecGroups * 4;  // 4096 elements



// 4 CTAs/SM (64 registers).  Measured: 2 CTAs (96 registers, the default
// when min-blocks is 1) 30% slower, 5-8 CTAs (48-32 registers) slower at 2^30.
//
// kLocal: the paper's "8-bit for incoming GPUs, 32-bit for the local GPU"
// (SURVEY 8(e)): rank p.local_rank's term is its own float32 input, read
// from seg.local (which may alias seg.out: each thread reads its elements
// before it stores them), instead of the decoded codes.
template <bool kLocal>
__global__ void __launch_bounds__(kDecThreads, 4) decode_kernel(const __grid_constant__ DecParams p) {
    // One UNSCALED decode table, one copy per lane ([256][32]: lane j reads
    // column j, so table lookups never conflict on a bank), built once per
    // CTA; the per-rank scale is applied in registers: fl(table[c] * s_r) is
    // exactly the pre-scaled entry of codecs.py:281.  No per-segment table
    // rebuild, and the table size does not grow with the rank count.
    extern __shared__ float sTab[];  // [256][32]
    __shared__ float sScale[kInlineSegs * kMaxRanks];  // [segment][rank] (inline plans), else [rank]
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const DecSegD* segs = p.segs_dev ? p.segs_dev : p.segs;
    const int R = p.nranks;
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;
    const float invN = 1.0f / (float)R;  // exact when R is a power of two
    const bool pow2 = (R & (R - 1)) == 0;
    int cur = -1;
    int64_t cbase = 0;
    const uint8_t* src = nullptr;  // codes of rank 0 for this segment, flat-indexed

    {
        static_assert(kDecThreads == 256, "one code per thread");
        const float v = p.book->table[tid];
        float4* d = reinterpret_cast<float4*>(sTab + tid * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = make_float4(v, v, v, v);
    }
    const float* tl = sTab + lane;  // this lane's column: entry c at tl[c * 32]
    // inline plans: every (segment, rank) scale is loaded once, up front, in
    // parallel (one round trip instead of one per segment switch)
    const bool preload = p.nseg <= kInlineSegs;
    if (preload) {
        for (int i = tid; i < R * p.nseg; i += kDecThreads) {
            const int sgi = i / R, r = i % R;
            const DecSegD& d = segs[sgi];
            sScale[i] = __ldcg(reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(p.lay.scales) +
                                                              p.rank_off[r]) +
                               (d.flat_off / L) * p.lay.scale_block_stride + d.scale_idx);
        }
    }
    const float* scl = sScale;  // the current segment's per-rank scales

    if (p.status_out && blockIdx.x == 0) {
        __shared__ unsigned int sSt;
        if (tid == 0) sSt = 0u;
        __syncthreads();
        for (int i = tid; i < R * p.status_blocks; i += kDecThreads) {
            const int r = i / p.status_blocks, j = i % p.status_blocks;
            const unsigned int* w = reinterpret_cast<const unsigned int*>(
                                        reinterpret_cast<const uint8_t*>(p.lay.scales) + p.rank_off[r]) +
                                    (int64_t)j * p.lay.scale_block_stride + p.status_idx;
            atomicOr(&sSt, __ldcg(w));
        }
        __syncthreads();
        if (tid == 0) {
            if (p.lay.flags & A8_LAYOUT_STATUS_COUNT) {
                volatile unsigned int* w = p.status_out;  // may be host-mapped: stream order makes this safe
                if (sSt) *w = *w + 1u;
            } else {
                *p.status_out = sSt;
            }
        }
    }

    auto seg_of = [&](int64_t c) {
        int lo = 0, hi = p.nseg;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (segs[mid].cstart <= c)
                lo = mid;
            else
                hi = mid;
        }
        return lo;
    };
    auto dec = [&](uint32_t code, float s) { return __fmul_rn(tl[code * 32u], s); };  // codecs.py:281

    for (int64_t c = blockIdx.x; c < p.total; c += gridDim.x) {
        const int lo = seg_of(c);
        const DecSegD sg = segs[lo];
        if (lo != cur) {
            const int64_t j = sg.flat_off / L;
            if (preload) {
                if (cur < 0) __syncthreads();  // table + scales complete before the first lookups
                scl = sScale + lo * R;
            } else {
                __syncthreads();  // (also orders the table build before the first lookups)
                if (tid < R)
                    sScale[tid] = __ldcg(reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(p.lay.scales) +
                                                                        p.rank_off[tid]) +
                                         j * p.lay.scale_block_stride + sg.scale_idx);
                __syncthreads();
            }
            cur = lo;
            cbase = sg.cstart;
            src = p.lay.codes + j * gap;
        }
        const int64_t base = (c - cbase) * kDecChunkD;
        const int64_t cnt = min((int64_t)kDecChunkD, sg.n - base);
        const int64_t f0 = sg.flat_off + base;

        if (cnt == kDecChunkD && sg.aligned) {
            float acc[kDecGroups][4];
            {
                uint32_t w[kDecGroups];
#pragma unroll
                for (int q = 0; q < kDecGroups; ++q) w[q] = ld_stream_u32(src + f0 + q * (kDecThreads * 4) + tid * 4);
                const float s0 = scl[0];
                if (kLocal && p.local_rank == 0) {
#pragma unroll
                    for (int q = 0; q < kDecGroups; ++q) {
                        const float4 v = __ldcs(reinterpret_cast<const float4*>(sg.local + base + q * (kDecThreads * 4) + tid * 4));
                        acc[q][0] = v.x;
                        acc[q][1] = v.y;
                        acc[q][2] = v.z;
                        acc[q][3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < kDecGroups; ++q) {
                        acc[q][0] = dec(w[q] & 255u, s0);
                        acc[q][1] = dec((w[q] >> 8) & 255u, s0);
                        acc[q][2] = dec((w[q] >> 16) & 255u, s0);
                        acc[q][3] = dec(w[q] >> 24, s0);
                    }
                }
            }
            // rank r+1's code words are loaded before rank r's are decoded
            uint32_t wn[kDecGroups];
            if (R > 1) {
                const uint8_t* s1 = src + p.rank_off[1] + f0 + tid * 4;
#pragma unroll
                for (int q = 0; q < kDecGroups; ++q) wn[q] = ld_stream_u32(s1 + q * (kDecThreads * 4));
            }
            for (int r = 1; r < R; ++r) {
                const float sc = scl[r];
                uint32_t w[kDecGroups];
#pragma unroll
                for (int q = 0; q < kDecGroups; ++q) w[q] = wn[q];
                if (r + 1 < R) {
                    const uint8_t* sn = src + p.rank_off[r + 1] + f0 + tid * 4;
#pragma unroll
                    for (int q = 0; q < kDecGroups; ++q) wn[q] = ld_stream_u32(sn + q * (kDecThreads * 4));
                }
                if (kLocal && r == p.local_rank) {
#pragma unroll
                    for (int q = 0; q < kDecGroups; ++q) {
                        const float4 v = __ldcs(reinterpret_cast<const float4*>(sg.local + base + q * (kDecThreads * 4) + tid * 4));
                        acc[q][0] = __fadd_rn(acc[q][0], v.x);
                        acc[q][1] = __fadd_rn(acc[q][1], v.y);
                        acc[q][2] = __fadd_rn(acc[q][2], v.z);
                        acc[q][3] = __fadd_rn(acc[q][3], v.w);
                    }
                    continue;
                }
#pragma unroll
                for (int q = 0; q < kDecGroups; ++q) {
                    acc[q][0] = __fadd_rn(acc[q][0], dec(w[q] & 255u, sc));
                    acc[q][1] = __fadd_rn(acc[q][1], dec((w[q] >> 8) & 255u, sc));
                    acc[q][2] = __fadd_rn(acc[q][2], dec((w[q] >> 16) & 255u, sc));
                    acc[q][3] = __fadd_rn(acc[q][3], dec(w[q] >> 24, sc));
                }
            }
#pragma unroll
            for (int q = 0; q < kDecGroups; ++q) {
                const int64_t e = q * (kDecThreads * 4) + tid * 4;
                float a0 = acc[q][0], a1 = acc[q][1], a2 = acc[q][2], a3 = acc[q][3];
                if (p.op == 1 && R > 1) {
                    if (pow2) {
                        a0 = __fmul_rn(a0, invN);
                        a1 = __fmul_rn(a1, invN);
                        a2 = __fmul_rn(a2, invN);
                        a3 = __fmul_rn(a3, invN);
                    } else {
                        const float fn = (float)R;
                        a0 = __fdiv_rn(a0, fn);
                        a1 = __fdiv_rn(a1, fn);
                        a2 = __fdiv_rn(a2, fn);
                        a3 = __fdiv_rn(a3, fn);
                    }
                }
                __stcs(reinterpret_cast<float4*>(sg.out + base + e), make_float4(a0, a1, a2, a3));
            }
        } else {
            for (int64_t i = tid; i < cnt; i += kDecThreads) {
                auto term = [&](int r) {
                    return (kLocal && r == p.local_rank) ? sg.local[base + i]
                                                         : dec(src[p.rank_off[r] + f0 + i], scl[r]);
                };
                float a = term(0);
                for (int r = 1; r < R; ++r) a = __fadd_rn(a, term(r));
                if (p.op == 1 && R > 1) a = pow2 ? __fmul_rn(a, invN) : __fdiv_rn(a, (float)R);
                sg.out[base + i] = a;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K4/K5 streaming form for 1-2 ranks (the N = 1 round trip, N = 2
// all-gather): codes come in by bulk copies (TMA) into a 3-stage ring, each
// chunk is decoded (+ rank sum, + 1/N) into one of 3 shared-memory output
// buffers, and the decoded chunk leaves by ONE bulk store (full lines, no
// per-thread global stores) -- the decode writes 4 of every 5 bytes it moves.
// Warp 0 is the producer; 8 consumer warps decode.  One consumer barrier per
// chunk: the bulk store of chunk k is issued after it, and the wait for the
// store of chunk k-1 to finish reading its buffer happens before the next
// barrier, so with 3 buffers no chunk overwrites a buffer still being read.
constexpr int kDtWarps = 8;
constexpr int kDtCons = kDtWarps * 32;
#ifndef A8_DT_STAGES
#define A8_DT_STAGES 3
#endif
#ifndef A8_DT_OUT
#define A8_DT_OUT 3
#endif
#ifndef A8_DT_REP
#define A8_DT_REP 32
#endif
#ifndef A8_DT_CTAS
#define A8_DT_CTAS 2
#endif
constexpr int kDtStages = A8_DT_STAGES;
constexpr int kDtRep = A8_DT_REP;    // copies of the decode table (lane-private at 32)
constexpr int kDtCtas = A8_DT_CTAS;  // CTAs per SM
constexpr int kDtOut = A8_DT_OUT;
constexpr int kDtMaxRanks = 2;
constexpr int kDtChunk = 4096;  // elements (16 KB out)
static size_t dt_smem(int R) {
    return 256u * kDtRep * sizeof(float) + (size_t)kDtStages * R * kDtChunk + (size_t)kDtOut * kDtChunk * sizeof(float);
}

struct DtMeta {
    int32_t seg;
    int32_t pad;
    int64_t base;  // first element of the chunk inside its segment
    int32_t cnt;
    int32_t pad2;
};

__global__ void __launch_bounds__(kDtCons + 32, kDtCtas) decode_tma_kernel(const __grid_constant__ DecParams p) {
    extern __shared__ __align__(128) float sDyn[];
    float* const sTab = sDyn;                                                              // [256][kDtRep]
    uint8_t* const sCodes = reinterpret_cast<uint8_t*>(sDyn + 256 * kDtRep);                  // [stage][rank][4096]
    float* const sOut = reinterpret_cast<float*>(sCodes + (size_t)kDtStages * p.nranks * kDtChunk);  // [3][4096]
    __shared__ float sScale[kInlineSegs * kDtMaxRanks];
    __shared__ __align__(8) uint64_t sFull[kDtStages];
    __shared__ __align__(8) uint64_t sEmpty[kDtStages];
    __shared__ DtMeta sMeta[kDtStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const DecSegD* segs = p.segs;  // inline plans only
    const int R = p.nranks;
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;
    if (tid == 0) {
        for (int i = 0; i < kDtStages; ++i) {
            mbar_init(&sFull[i], 1);
            mbar_init(&sEmpty[i], kDtWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();  // the ring barriers are initialised: the producer starts at once, the
                      // consumers' prologue (tables, scales, status) overlaps its first loads
    auto seg_of = [&](int64_t c) {
        int lo = 0, hi = p.nseg;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (segs[mid].cstart <= c) lo = mid; else hi = mid;
        }
        return lo;
    };
    const uint32_t full0 = smem_addr(&sFull[0]), empty0 = smem_addr(&sEmpty[0]);
    const int64_t nmy = p.total > blockIdx.x ? (p.total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t drop = p.rpol == 2 ? policy_evict_last() : p.rpol == 1 ? policy_evict_normal() : policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < nmy; ++k) {
                const int64_t c = blockIdx.x + k * gridDim.x;
                const int lo = seg_of(c);
                const DecSegD& sg = segs[lo];
                DtMeta m;
                m.seg = lo;
                m.base = (c - sg.cstart) * kDtChunk;
                m.cnt = (int32_t)min((int64_t)kDtChunk, sg.n - m.base);
                mbar_wait_a(empty0 + 8u * st, ph ^ 1u);
                sMeta[st] = m;
                const uint32_t bytes = ((uint32_t)m.cnt + 15u) & ~15u;  // segments are padded to 16 codes
                mbar_arrive_expect_tx(&sFull[st], bytes * (uint32_t)R);
                const int64_t f0 = sg.flat_off + m.base;
                const uint8_t* src = p.lay.codes + (f0 / L) * p.lay.block_stride + f0 % L;
                for (int r = 0; r < R; ++r)
                    bulk_g2s(sCodes + ((size_t)st * R + r) * kDtChunk, src + p.rank_off[r], bytes, &sFull[st], drop);
                if (++st == kDtStages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int ct = tid - 32;
    {
        const float v = p.book->table[ct];
        float4* d = reinterpret_cast<float4*>(sTab + ct * kDtRep);
#pragma unroll
        for (int q = 0; q < kDtRep / 4; ++q) d[q] = make_float4(v, v, v, v);
    }
    for (int i = ct; i < R * p.nseg; i += kDtCons) {
        const int sgi = i / R, r = i % R;
        const DecSegD& d = segs[sgi];
        sScale[i] = __ldcg(reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(p.lay.scales) + p.rank_off[r]) +
                           (d.flat_off / L) * p.lay.scale_block_stride + d.scale_idx);
    }
    if (p.status_out && blockIdx.x == 0) {
        __shared__ unsigned int sSt;
        if (ct == 0) sSt = 0u;
        nbar_sync(2, kDtCons);
        for (int i = ct; i < R * p.status_blocks; i += kDtCons) {
            const int r = i / p.status_blocks, j = i % p.status_blocks;
            const unsigned int* w = reinterpret_cast<const unsigned int*>(
                                        reinterpret_cast<const uint8_t*>(p.lay.scales) + p.rank_off[r]) +
                                    (int64_t)j * p.lay.scale_block_stride + p.status_idx;
            atomicOr(&sSt, __ldcg(w));
        }
        nbar_sync(2, kDtCons);
        if (ct == 0) {
            if (p.lay.flags & A8_LAYOUT_STATUS_COUNT) {
                volatile unsigned int* w = p.status_out;
                if (sSt) *w = *w + 1u;
            } else {
                *p.status_out = sSt;
            }
        }
    }
    nbar_sync(2, kDtCons);  // tables and scales complete
    const float* tl = sTab + (lane & (kDtRep - 1));
    const float invN = 1.0f / (float)R;
    const bool pow2 = (R & (R - 1)) == 0;
    const uint64_t wpol = p.wpol == 2 ? policy_evict_last() : p.wpol == 1 ? policy_evict_normal() : policy_evict_first();
    int st = 0, ob = 0;
    uint32_t ph = 0;
    for (int64_t k = 0; k < nmy; ++k) {
        mbar_wait_a(full0 + 8u * st, ph);
        const DtMeta m = sMeta[st];
        const DecSegD& sg = segs[m.seg];
        const float* scl = sScale + m.seg * R;
        float* out = sOut + (size_t)ob * kDtChunk;
        float acc[4][4];
#pragma unroll
        for (int r = 0; r < kDtMaxRanks; ++r) {
            if (r >= R) break;
            const uint8_t* cs = sCodes + ((size_t)st * R + r) * kDtChunk;
            const float s = scl[r];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(cs + q * 1024 + ct * 4);
                const float d0 = __fmul_rn(tl[(w & 255u) * kDtRep], s), d1 = __fmul_rn(tl[((w >> 8) & 255u) * kDtRep], s);
                const float d2 = __fmul_rn(tl[((w >> 16) & 255u) * kDtRep], s), d3 = __fmul_rn(tl[(w >> 24) * kDtRep], s);
                if (r == 0) {
                    acc[q][0] = d0; acc[q][1] = d1; acc[q][2] = d2; acc[q][3] = d3;
                } else {
                    acc[q][0] = __fadd_rn(acc[q][0], d0); acc[q][1] = __fadd_rn(acc[q][1], d1);
                    acc[q][2] = __fadd_rn(acc[q][2], d2); acc[q][3] = __fadd_rn(acc[q][3], d3);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(empty0 + 8u * st);  // this warp is done with the codes
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float a0 = acc[q][0], a1 = acc[q][1], a2 = acc[q][2], a3 = acc[q][3];
            if (p.op == 1) {
                if (pow2) {
                    a0 = __fmul_rn(a0, invN); a1 = __fmul_rn(a1, invN); a2 = __fmul_rn(a2, invN); a3 = __fmul_rn(a3, invN);
                } else {
                    a0 = __fdiv_rn(a0, (float)R); a1 = __fdiv_rn(a1, (float)R); a2 = __fdiv_rn(a2, (float)R); a3 = __fdiv_rn(a3, (float)R);
                }
            }
            const int e = q * 1024 + ct * 4;
            reinterpret_cast<float4*>(out)[e >> 2] = make_float4(a0, a1, a2, a3);
            // the ragged end of a segment: the elements past the last full 4 go out directly
            if (e + 4 > (m.cnt & ~3) && e < m.cnt) {
                const float a[4] = {a0, a1, a2, a3};
                for (int t = max(e, m.cnt & ~3); t < min(e + 4, m.cnt); ++t) sg.out[m.base + t] = a[t - e];
            }
        }
        fence_proxy_async_smem();
        nbar_sync(1, kDtCons);
        if (ct == 0) {
            const uint32_t bytes = (uint32_t)(m.cnt & ~3) * 4u;
            if (bytes) bulk_s2g(sg.out + m.base, out, bytes, wpol);
            bulk_commit();
            bulk_wait_read<kDtOut - 2>();  // the buffer of the next chunk (used 2 stores ago) is free
        }
        if (++st == kDtStages) {
            st = 0;
            ph ^= 1u;
        }
        if (++ob == kDtOut) ob = 0;
    }
    if (ct == 0) bulk_wait_all();
}

static size_t dec_smem(int) { return 256u * 32u * sizeof(float); }  // lane-private table copies

// ---------------------------------------------------------------------------
// host launchers

struct DevInfo {
    int sms = 0;
    int enc_occ = 0;
    int dec_occ = 0;
    int res_occ = 0;  // resident encode: CTAs per SM (1, or 0 if it cannot run)
};

static std::mutex g_mu;
static std::mutex g_plan_mu;  // serialises workspace plan upload + launch pairs
static DevInfo g_dev[64];

static int dev_info(int device, DevInfo* out) {
    if (device < 0 || device >= 64) return fail(A8_ERR_USAGE, "device index out of range");
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo& d = g_dev[device];
    if (d.sms == 0) {
        cudaError_t e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaFuncSetAttribute(encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEncDynSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEncDynSmem);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaFuncSetAttribute(decode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dec_smem(kMaxRanks));
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaFuncSetAttribute(decode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dec_smem(kMaxRanks));
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.enc_occ, encode_kernel<false>, kEncThreads, kEncDynSmem);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        const size_t dsm = dec_smem(1);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.dec_occ, decode_kernel<false>, kDecThreads, dsm);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaFuncSetAttribute(resident_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRDynSmem);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.res_occ, resident_encode_kernel, kRThreads, kRDynSmem);
        if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
        d.enc_occ = std::max(1, d.enc_occ);
        d.dec_occ = std::max(1, d.dec_occ);
    }
    *out = d;
    return A8_OK;
}

static int check_layout(const a8_layout_t& lay) {
    if (!lay.codes || !lay.scales) return fail(A8_ERR_USAGE, "layout: null codes or scales");
    if (lay.block_len <= 0 || lay.block_len % 16)
        return fail(A8_ERR_USAGE, "layout: block_len must be a positive multiple of 16");
    if (lay.block_stride < lay.block_len || lay.block_stride % 16)
        return fail(A8_ERR_USAGE, "layout: block_stride must be >= block_len and a multiple of 16");
    if (reinterpret_cast<uintptr_t>(lay.codes) % 16) return fail(A8_ERR_USAGE, "layout: codes must be 16-byte aligned");
    if (lay.rank_stride % 16) return fail(A8_ERR_USAGE, "layout: rank_stride must be a multiple of 16");
    if (lay.scale_block_stride < 0) return fail(A8_ERR_USAGE, "layout: bad scale strides");
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

// Ticket order (host).
//  * Fixed-scale specs: E-chunks only.
//  * absmax: single-chunk segments become one F ticket each (no dependency),
//    issued first.  Then the A-chunks of the multi-chunk segments, largest
//    first.  A segment's E-chunks (reverse chunk order, so the data its A
//    pass read last -- still in L2 -- comes first) are issued `wf` tickets
//    after its last A-chunk, interrupting the A stream: `wf` covers the
//    tickets the CTAs hold reserved in their rings plus the table build, so
//    by the time a CTA reaches an E-chunk its table is normally published.
//    When no A work is left to fill that distance, the filler is a
//    held-back part of the largest segment's E pass (its L2-cold head,
//    whose table is long done); what remains of it ends the launch, so the
//    launch tail is dependency-free streaming.
static void schedule(const std::vector<EncSegD>& d, bool absmax, int64_t wf, std::vector<EncBlk>* blks) {
    struct Run {
        int s;
        int kind;
        int64_t c0;  // first chunk
        int64_t cnt;
    };
    int64_t t = 0;
    auto emit = [&](const Run& r) {
        if (r.cnt <= 0) return;
        blks->push_back(EncBlk{t, r.s, (int32_t)((r.c0 << 2) | r.kind)});
        t += r.cnt;
    };
    const int nseg = (int)d.size();
    if (!absmax) {
        for (int s = 0; s < nseg; ++s) emit(Run{s, kE, d[s].nE - 1, d[s].nE});
        blks->push_back(EncBlk{t, -1, 0});  // sentinel: total tickets
        return;
    }
    for (int s = 0; s < nseg; ++s)
        if (d[s].n <= kChunk) emit(Run{s, kF, 0, 1});
    std::deque<Run> aq;  // A runs, largest segment first (d is ascending)
    for (int s = nseg - 1; s >= 0 && d[s].n > kChunk; --s) aq.push_back(Run{s, kA, 0, d[s].nA});
    struct Pending {
        int64_t ready;
        int s;
    };
    std::deque<Pending> pend;  // E passes waiting for their fill distance, in A order
    Run pool{-1, kE, 0, 0};    // held-back E chunks (one segment's cold head)
    const bool hold = aq.size() > 1;
    auto emit_e = [&](int s) {
        Run e{s, kE, d[s].nE - 1, d[s].nE};
        if (hold && pool.s < 0) {  // first E pass: keep its cold head as filler
            static const int pool_div = [] {  // A8_SCHED_POOL: held-back share 1/div (tuning)
                const char* v = getenv("A8_SCHED_POOL");
                return v ? std::max(1, atoi(v)) : 2;
            }();
            const int64_t h = std::min<int64_t>(e.cnt / pool_div, 2 * wf);
            pool = Run{s, kE, h - 1, h};
            e.cnt -= h;
        }
        emit(e);
    };
    while (!aq.empty() || !pend.empty()) {
        if (!pend.empty() && pend.front().ready <= t) {
            emit_e(pend.front().s);
            pend.pop_front();
            continue;
        }
        const int64_t until = pend.empty() ? INT64_MAX : pend.front().ready;
        if (!aq.empty()) {
            Run& r = aq.front();
            const int64_t now = std::min(r.cnt, until - t);
            emit(Run{r.s, kA, r.c0, now});
            r.c0 += now;
            r.cnt -= now;
            if (r.cnt == 0) {
                // B ticket right after the A pass: its table is built and
                // published while the fill distance runs
                // (only when other work can fill the distance: a lone segment's
                // E pass follows at once, measured 1.5% slower with a B ticket)
                if (A8_BUILD_TICKETS && hold) emit(Run{r.s, kB, 0, 1});
                pend.push_back(Pending{t + wf, r.s});
                aq.pop_front();
            }
            continue;
        }
        if (pool.cnt > 0) {  // no A work left: fill from the pool
            const int64_t now = std::min(pool.cnt, until - t);
            emit(Run{pool.s, kE, pool.c0, now});
            pool.c0 -= now;
            pool.cnt -= now;
            continue;
        }
        emit_e(pend.front().s);  // nothing independent left: the wait is unavoidable
        pend.pop_front();
    }
    emit(pool);
    blks->push_back(EncBlk{t, -1, 0});  // sentinel: total tickets
}

// a8_encode_premax: the maxima are known, so there is no A pass and no
// dependency to hide.  F tickets (single-chunk segments) first, then one B
// ticket per multi-chunk segment (its table is built and published at once;
// CTAs that reach the segment's E-chunks before that build their own copy),
// then the E passes, largest segment first -- except that the last `hold`
// chunks of the largest segment end the launch: every CTA finishes on a
// long run whose table is published (no table switches in the tail).
static void schedule_premax(const std::vector<EncSegD>& d, int64_t ctas, bool build_tickets, std::vector<EncBlk>* blks) {
    int64_t t = 0;
    auto emit = [&](int s, int kind, int64_t c0, int64_t cnt) {
        if (cnt <= 0) return;
        blks->push_back(EncBlk{t, s, (int32_t)((c0 << 2) | kind)});
        t += cnt;
    };
    const int nseg = (int)d.size();
    for (int s = 0; s < nseg; ++s)
        if (d[s].n <= kChunk) emit(s, kF, 0, 1);
    if (build_tickets)
        for (int s = nseg - 1; s >= 0 && d[s].n > kChunk; --s) emit(s, kB, 0, 1);
    const int big = nseg - 1;
    const bool several = nseg >= 2 && d[nseg - 2].n > kChunk;
    static const int64_t hold_per_cta = [] {  // A8_PREMAX_HOLD: tail chunks per CTA (tuning)
        const char* v = getenv("A8_PREMAX_HOLD");
        return v ? std::max(0ll, atoll(v)) : 32ll;
    }();
    const int64_t hold = several && d[big].n > kChunk ? std::min<int64_t>(d[big].nE / 2, hold_per_cta * ctas) : 0;
    for (int s = nseg - 1; s >= 0 && d[s].n > kChunk; --s)
        emit(s, kE, d[s].nE - 1, s == big ? d[s].nE - hold : d[s].nE);
    emit(big, kE, hold - 1, hold);  // chunks hold-1 .. 0 of the largest segment
    blks->push_back(EncBlk{t, -1, 0});  // sentinel: total tickets
}

// Fill distance in tickets: what the CTAs hold reserved (ring + ticket
// batches) plus enough throughput for the B ticket's wait and build to end
// before the E pass is reached.  Measured (C3, with B tickets): 2880 -> 115.0
// us, 6400 -> 113.0 us, flat up to 12000.  A8_SCHED_FILL overrides it.
static int64_t fill_distance(int64_t ctas) {
    static const int64_t env = [] {
        const char* e = getenv("A8_SCHED_FILL");
        return e ? atoll(e) : -1ll;
    }();
    return env >= 0 ? env : ctas * 20 + 512;
}

}  // namespace a8

using namespace a8;

static size_t ws_bytes_for(int cap) { return plan_off(cap) + plan_bytes(cap); }

// Largest capacity whose layout fits in `bytes` (0 if none).
static int ws_capacity(size_t bytes) {
    int lo = 0, hi = 1;
    while (ws_bytes_for(hi) <= bytes) {
        lo = hi;
        hi *= 2;
        if (hi > (1 << 24)) break;
    }
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (ws_bytes_for(mid) <= bytes)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

extern "C" int a8_encode_trace(const void* workspace, int nseg, uint64_t* out) {
    if (!workspace || !out || nseg < 1) return fail(A8_ERR_USAGE, "a8_encode_trace: bad argument");
    WsHead h;
    std::vector<SegCtl> c(nseg);
    const uint8_t* ws = static_cast<const uint8_t*>(workspace);
    cudaError_t e = cudaMemcpy(&h, ws, sizeof(h), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(c.data(), ws + ctl_off(), sizeof(SegCtl) * nseg, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(A8_ERR_CUDA, cudaGetErrorString(e));
    out[0] = h.tr_start;
    out[1] = h.tr_end;
    out[2] = h.tr_wait_ns;
    out[3] = h.tr_waits;
    for (int i = 0; i < nseg; ++i) {
        out[4 + 4 * i] = c[i].t_b0;
        out[5 + 4 * i] = c[i].t_thr;
        out[6 + 4 * i] = c[i].t_fill;
        out[7 + 4 * i] = c[i].t_b1;
    }
    return A8_OK;
}

#ifdef A8_TICKET_TRACE
extern "C" int a8_debug_ticket_trace(uint64_t* out, int64_t n) {
    if (n > a8::kTraceTickets) n = a8::kTraceTickets;
    cudaError_t e = cudaMemcpyFromSymbol(out, a8::g_ticket_trace, sizeof(uint64_t) * 5 * n);
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
extern "C" int a8_debug_res_trace(uint64_t* out) {  // [2][8]
    cudaError_t e = cudaMemcpyFromSymbol(out, a8::g_res_trace, sizeof(a8::g_res_trace));
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
extern "C" int a8_debug_switch_trace(uint64_t* out, int64_t n, int reset) {  // [n][8]; returns the count
    unsigned int cnt = 0;
    cudaMemcpyFromSymbol(&cnt, a8::g_switch_n, sizeof(cnt));
    if (n > a8::kTraceSw) n = a8::kTraceSw;
    cudaError_t e = cudaMemcpyFromSymbol(out, a8::g_switch_trace, sizeof(uint64_t) * 8 * n);
    if (reset) {
        const unsigned int z = 0;
        cudaMemcpyToSymbol(a8::g_switch_n, &z, sizeof(z));
    }
    return e == cudaSuccess ? (int)cnt : -fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
extern "C" int a8_debug_flush_trace(uint64_t* out) {  // [32][512][4]
    cudaError_t e = cudaMemcpyFromSymbol(out, a8::g_flush_trace, sizeof(a8::g_flush_trace));
    return e == cudaSuccess ? A8_OK : fail(A8_ERR_CUDA, cudaGetErrorString(e));
}
#endif

extern "C" size_t a8_workspace_bytes(int nseg) {
    if (nseg < 1) nseg = 1;
    return ws_bytes_for(nseg);
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

// Resident encode (calls that fit in shared memory, any spec).  A8_RESIDENT=0
// disables it (A/B measurements).
static bool resident_enabled() {
    static const bool on = [] {
        const char* e = getenv("A8_RESIDENT");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Launches the resident kernel if the call fits; *done = false otherwise.
// Every non-empty segment gets its own CTAs (at least enough for its data to
// fit, then a share of the remaining SMs proportional to its size), so each
// CTA holds one piece of one segment and builds one table.
static int encode_resident(const a8_enc_seg_t* segs, int nseg, const void* book_dev, const void* static_lut_dev,
                           const a8_layout_t& layout, void* workspace, const uint32_t* status_in,
                           uint32_t* status_out, const DevInfo& di, cudaStream_t st, bool* done,
                           float* const* outs = nullptr, const uint32_t* amax_in = nullptr) {
    *done = false;
    if (!resident_enabled() || di.res_occ < 1 || nseg > kInlineSegs) return A8_OK;
    const int64_t per = kRCap - 4;  // elements per CTA (+ up to 3 of alignment offset)
    int64_t total = 0, need = 0;
    std::vector<int64_t> c(nseg, 0);
    for (int i = 0; i < nseg; ++i) {
        total += segs[i].n;
        c[i] = (segs[i].n + per - 1) / per;
        need += c[i];
    }
    if (total == 0 || need > di.sms) return A8_OK;
    // spread the rest of the SMs (about 2048 elements per CTA at least)
    const int64_t target = std::min<int64_t>(di.sms, std::max<int64_t>(need, (total + 2047) / 2048));
    int64_t extra = target - need;
    for (int i = 0; i < nseg && extra > 0; ++i) {
        const int64_t add = std::min<int64_t>(extra * segs[i].n / total, std::max<int64_t>(0, segs[i].n - c[i]));
        c[i] += add;
    }
    RParams p;
    memset(&p, 0, sizeof(p));
    p.lay = layout;
    p.book = static_cast<const a8_book_t*>(book_dev);
    p.static_lut = static_cast<const a8_lut_t*>(static_lut_dev);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    p.head = reinterpret_cast<WsHead*>(ws);
    p.ctl = reinterpret_cast<SegCtl*>(ws + ctl_off());
    p.status_in = status_in;
    p.status_out = status_out;
    p.nseg = nseg;
    p.write_codes = outs ? 0 : 1;
    p.amax_in = amax_in;
    int64_t grid = 0;
    for (int i = 0; i < nseg; ++i) {
        p.segs[i].x = segs[i].x;
        p.segs[i].out = outs ? outs[i] : nullptr;
        p.segs[i].n = segs[i].n;
        p.segs[i].flat_off = segs[i].flat_off;
        p.segs[i].scale_idx = segs[i].scale_idx;
        p.segs[i].aligned = (reinterpret_cast<uintptr_t>(segs[i].x) % 16) == 0 &&
                            (!outs || (reinterpret_cast<uintptr_t>(outs[i]) % 16) == 0);
        p.segs[i].cta0 = (int32_t)grid;
        grid += c[i];
    }
    p.segs[nseg].cta0 = (int32_t)grid;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kRThreads);
    cfg.dynamicSmemBytes = kRDynSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = static_lut_dev ? 0 : 1;  // fixed scales: no barrier
    cudaLaunchKernelEx(&cfg, resident_encode_kernel, p);
    *done = true;
    return cuda_check("a8_encode (resident)");
}

extern "C" int a8_roundtrip(const a8_enc_seg_t* segs, float* const* outs, int nseg, const void* book_dev, int norm,
                            const void* static_lut_dev, float* scales_out, uint32_t* status_out, void* workspace,
                            size_t workspace_bytes, void* stream) {
    if (nseg <= 0 || !segs || !outs || !book_dev || !scales_out || !status_out || !workspace)
        return fail(A8_ERR_USAGE, "a8_roundtrip: bad argument");
    if (norm != A8_NORM_ABSMAX && !static_lut_dev) return fail(A8_ERR_USAGE, "a8_roundtrip: fixed-scale spec needs a static table");
    for (int i = 0; i < nseg; ++i) {
        if (segs[i].n < 0 || (segs[i].n > 0 && (!segs[i].x || !outs[i]))) return fail(A8_ERR_USAGE, "a8_roundtrip: bad segment");
        if (segs[i].flat_off % 16 || segs[i].flat_off < 0) return fail(A8_ERR_USAGE, "a8_roundtrip: flat_off must be a multiple of 16");
    }
    if (ws_capacity(workspace_bytes) < nseg) return fail(A8_ERR_USAGE, "a8_roundtrip: workspace too small");
    int device = 0;
    cudaGetDevice(&device);
    DevInfo di;
    if (int rc = dev_info(device, &di)) return rc;
    a8_layout_t lay;
    memset(&lay, 0, sizeof(lay));
    lay.scales = scales_out;
    lay.block_len = (int64_t)1 << 40;  // one block: no code layout (codes are not written)
    lay.block_stride = lay.block_len;
    lay.scale_reps = 1;
    bool done = false;
    const int rc = encode_resident(segs, nseg, book_dev, norm == A8_NORM_ABSMAX ? nullptr : static_lut_dev, lay, workspace,
                                   nullptr, status_out, di, static_cast<cudaStream_t>(stream), &done, outs);
    if (rc) return rc;
    return done ? A8_OK : fail(A8_ERR_USAGE, "a8_roundtrip: call does not fit the fused path (use a8_encode + a8_decode)");
}

// encode_kernel<true>; after the table prologue it is launched as a
// programmatic dependent (PDL): its CTAs start streaming while the prologue
// runs and wait for it (griddepcontrol.wait) only before reading a table.
static void launch_premax(const EncParams& p, unsigned grid, bool pre, cudaStream_t st) {
    static const bool pdl = [] {
        const char* v = getenv("A8_PREMAX_PDL");
        return !(v && v[0] == '0');
    }();
    if (!pre || !pdl) {
        encode_kernel<true><<<grid, kEncThreads, kEncDynSmem, st>>>(p);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kEncThreads);
    cfg.dynamicSmemBytes = kEncDynSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, encode_kernel<true>, p);
}

static int encode_impl(const a8_enc_seg_t* segs, int nseg, const void* book_dev, int norm,
                       const void* static_lut_dev, a8_layout_t layout, void* workspace,
                       size_t workspace_bytes, const uint32_t* status_in, uint32_t* status_out,
                       void* stream, const uint32_t* amax_in) {
    if (nseg <= 0) return fail(A8_ERR_USAGE, "a8_encode: need at least one segment");
    if (!segs || !book_dev || !workspace || !status_out) return fail(A8_ERR_USAGE, "a8_encode: null argument");
    if (norm != A8_NORM_ABSMAX && !static_lut_dev)
        return fail(A8_ERR_USAGE, "a8_encode: fixed-scale spec needs a static table");
    if (int rc = check_layout(layout)) return rc;
    if (layout.scale_reps < 1 || layout.scale_reps > kConsumers)
        return fail(A8_ERR_USAGE, "a8_encode: scale_reps out of range");
    int device = 0;
    cudaGetDevice(&device);
    DevInfo di;
    if (int rc = dev_info(device, &di)) return rc;

    const bool absmax = norm == A8_NORM_ABSMAX;
    {
        for (int i = 0; i < nseg; ++i) {
            const a8_enc_seg_t& s = segs[i];
            if (s.n < 0 || (s.n > 0 && !s.x)) return fail(A8_ERR_USAGE, "a8_encode: bad segment");
            if (s.flat_off % 16 || s.flat_off < 0) return fail(A8_ERR_USAGE, "a8_encode: flat_off must be a multiple of 16");
        }
        if (ws_capacity(workspace_bytes) < nseg) return fail(A8_ERR_USAGE, "a8_encode: workspace too small for the segment count");
        bool done = false;
        const int rc = encode_resident(segs, nseg, book_dev, absmax ? nullptr : static_lut_dev, layout, workspace,
                                       status_in, status_out, di, static_cast<cudaStream_t>(stream), &done,
                                       nullptr, amax_in);
        if (rc || done) return rc;
    }

    std::vector<int> order(nseg);
    for (int i = 0; i < nseg; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return segs[a].n < segs[b].n; });

    std::vector<EncSegD> d(nseg);
    for (int i = 0; i < nseg; ++i) {
        const a8_enc_seg_t& s = segs[order[i]];
        if (s.n < 0 || (s.n > 0 && !s.x)) return fail(A8_ERR_USAGE, "a8_encode: bad segment");
        if (s.flat_off % 16 || s.flat_off < 0) return fail(A8_ERR_USAGE, "a8_encode: flat_off must be a multiple of 16");
        const int64_t nch = (s.n + kChunk - 1) / kChunk;
        if (nch > INT32_MAX / 2) return fail(A8_ERR_USAGE, "a8_encode: segment too large");
        d[i].x = s.x;
        d[i].n = s.n;
        d[i].flat_off = s.flat_off;
        d[i].scale_idx = s.scale_idx;
        // absmax: multi-chunk segments take A- and E-chunks; single-chunk
        // (and empty) segments are one F ticket.  Fixed scale: E-chunks.
        const bool fused = absmax && s.n <= kChunk;
        d[i].nA = absmax && !fused && !amax_in ? (int32_t)nch : 0;  // premax: no A pass
        d[i].nE = fused ? 0 : absmax ? (int32_t)nch : (int32_t)std::max<int64_t>(1, nch);
        d[i].aligned = (reinterpret_cast<uintptr_t>(s.x) % 16) == 0;
        d[i].src = order[i];
        d[i].pad = 0;
    }
    // a8_encode_premax: the tables are built by a prologue launch (A8_PREMAX_TABLES=0:
    // by B tickets inside the encode, the round-2 form)
    static const bool pre_tables = [] {
        const char* v = getenv("A8_PREMAX_TABLES");
        return !(v && v[0] == '0');
    }();
    int nbig = 0;
    for (int i = 0; i < nseg; ++i) nbig += d[i].n > kChunk;
    const bool pre = amax_in && pre_tables && nbig > 0;
    std::vector<EncBlk> blks;
    if (amax_in)
        schedule_premax(d, (int64_t)di.sms * di.enc_occ, !pre, &blks);
    else
        schedule(d, absmax, fill_distance((int64_t)di.sms * di.enc_occ), &blks);
    const int nblk = (int)blks.size() - 1;

    uint8_t* ws = static_cast<uint8_t*>(workspace);
    EncParams p;
    memset(&p, 0, sizeof(p));
    p.lay = layout;
    p.book = static_cast<const a8_book_t*>(book_dev);
    p.static_lut = static_cast<const a8_lut_t*>(static_lut_dev);
    p.head = reinterpret_cast<WsHead*>(ws);
    const int cap = ws_capacity(workspace_bytes);
    if (cap < nseg) return fail(A8_ERR_USAGE, "a8_encode: workspace too small for the segment count");
    p.ctl = reinterpret_cast<SegCtl*>(ws + ctl_off());
    p.luts = reinterpret_cast<a8_lut_t*>(ws + lut_off(cap));
    p.status_in = status_in;
    p.status_out = status_out;
    p.nseg = nseg;
    p.nblk = nblk;
    p.absmax = absmax ? 1 : 0;
    {
        static const int hint = [] {
            const char* v = getenv("A8_CODE_HINT");
            return v ? atoi(v) : 0;
        }();
        p.code_hint = hint;
    }
    p.total = blks[nblk].tstart;
    p.amax_in = reinterpret_cast<const unsigned int*>(amax_in);
    {
        static const int64_t kt = [] {
            const char* v = getenv("A8_KEEP_TAIL");
            return v ? atoll(v) : -1ll;
        }();
        p.keep_tail = kt;
        static const int pa = [] {
            const char* v = getenv("A8_POL_A");
            return v ? atoi(v) : 0;
        }();
        static const int pe = [] {
            const char* v = getenv("A8_POL_E");
            return v ? atoi(v) : 0;
        }();
        p.pol_a = pa;
        p.pol_e = pe;
        p.pre_tables = pre ? 1 : 0;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if ((int)blks.size() > max_blocks(nseg)) return fail(A8_ERR_USAGE, "a8_encode: schedule overflow");
    const int64_t grid = std::min<int64_t>((int64_t)di.sms * di.enc_occ, std::max<int64_t>(1, p.total));
    if (nseg <= kInlineSegs && (int)blks.size() <= kInlineBlks) {
        std::copy(d.begin(), d.end(), p.segs);
        std::copy(blks.begin(), blks.end(), p.blks);
        if (pre) premax_tables_kernel<<<nbig, kConsumers, 0, st>>>(p);
        if (amax_in)
            launch_premax(p, (unsigned)grid, pre, st);
        else
            encode_kernel<false><<<(unsigned)grid, kEncThreads, kEncDynSmem, st>>>(p);
    } else {
        // the plan goes through the workspace: upload + launch must not be
        // interleaved with another thread's upload to the same workspace
        std::lock_guard<std::mutex> lk(g_plan_mu);
        uint8_t* plan = ws + plan_off(cap);
        const size_t sb = sizeof(EncSegD) * nseg;
        cudaMemcpyAsync(plan, d.data(), sb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(plan + sb, blks.data(), sizeof(EncBlk) * blks.size(), cudaMemcpyHostToDevice, st);
        p.segs_dev = reinterpret_cast<const EncSegD*>(plan);
        p.blks_dev = reinterpret_cast<const EncBlk*>(plan + sb);
        if (pre) premax_tables_kernel<<<nbig, kConsumers, 0, st>>>(p);
        if (amax_in)
            launch_premax(p, (unsigned)grid, pre, st);
        else
            encode_kernel<false><<<(unsigned)grid, kEncThreads, kEncDynSmem, st>>>(p);
    }
    return cuda_check("a8_encode");
}

extern "C" int a8_encode(const a8_enc_seg_t* segs, int nseg, const void* book_dev, int norm,
                         const void* static_lut_dev, a8_layout_t layout, void* workspace,
                         size_t workspace_bytes, const uint32_t* status_in, uint32_t* status_out,
                         void* stream) {
    return encode_impl(segs, nseg, book_dev, norm, static_lut_dev, layout, workspace, workspace_bytes, status_in,
                       status_out, stream, nullptr);
}

extern "C" int a8_encode_premax(const a8_enc_seg_t* segs, int nseg, const void* book_dev, const uint32_t* amax_dev,
                                a8_layout_t layout, void* workspace, size_t workspace_bytes,
                                const uint32_t* status_in, uint32_t* status_out, void* stream) {
    if (!amax_dev) return fail(A8_ERR_USAGE, "a8_encode_premax: null amax_dev");
    return encode_impl(segs, nseg, book_dev, A8_NORM_ABSMAX, nullptr, layout, workspace, workspace_bytes, status_in,
                       status_out, stream, amax_dev);
}

static int decode_impl(const a8_dec_seg_t* segs, const float* const* locals, int local_rank, int nseg,
                       const void* book_dev, a8_layout_t layout, int nranks, int op, int status_idx,
                       int status_blocks, uint32_t* status_out, void* workspace, size_t workspace_bytes,
                       void* stream, const void* const* rank_bases = nullptr) {
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

    std::vector<DecSegD> d(std::max(nseg, 1));
    int64_t chunks = 0;
    for (int i = 0; i < nseg; ++i) {
        const a8_dec_seg_t& s = segs[i];
        if (s.n < 0 || (s.n > 0 && !s.out)) return fail(A8_ERR_USAGE, "a8_decode: bad segment");
        if (s.flat_off % 16 || s.flat_off < 0) return fail(A8_ERR_USAGE, "a8_decode: flat_off must be a multiple of 16");
        if (s.n > 0 && (s.flat_off / layout.block_len) != ((s.flat_off + s.n - 1) / layout.block_len))
            return fail(A8_ERR_USAGE, "a8_decode: a segment may not straddle blocks");
        d[i].out = s.out;
        d[i].n = s.n;
        d[i].flat_off = s.flat_off;
        d[i].scale_idx = s.scale_idx;
        d[i].local = locals ? locals[i] : nullptr;
        if (locals && s.n > 0 && !d[i].local) return fail(A8_ERR_USAGE, "a8_decode_local: null local input");
        d[i].aligned = (reinterpret_cast<uintptr_t>(s.out) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(d[i].local) % 16) == 0;
        d[i].cstart = chunks;
        chunks += (s.n + kDecChunkD - 1) / kDecChunkD;
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
    p.local_rank = locals ? local_rank : -1;
    for (int r = 0; r < nranks; ++r) {
        if (rank_bases) {
            if (!rank_bases[r] || reinterpret_cast<uintptr_t>(rank_bases[r]) % 16)
                return fail(A8_ERR_USAGE, "a8_decode_peers: rank bases must be non-null and 16-byte aligned");
            p.rank_off[r] = reinterpret_cast<const uint8_t*>(rank_bases[r]) - reinterpret_cast<const uint8_t*>(rank_bases[0]);
        } else {
            p.rank_off[r] = (int64_t)r * layout.rank_stride;
        }
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto launch = [&](unsigned grid, size_t smem) {
        if (locals)
            decode_kernel<true><<<grid, kDecThreads, smem, st>>>(p);
        else
            decode_kernel<false><<<grid, kDecThreads, smem, st>>>(p);
    };
    static const int dt_env = [] {
        const char* v = getenv("A8_DEC_TMA");
        return v ? atoi(v) : 1;
    }();
    bool tma = dt_env && !locals && nranks <= kDtMaxRanks && nseg <= kInlineSegs && chunks > 0;
    for (int i = 0; tma && i < nseg; ++i) tma = d[i].aligned;
    if (tma) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(decode_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dt_smem(kDtMaxRanks));
            attr = true;
        }
        std::copy(d.begin(), d.begin() + nseg, p.segs);
        static const int rp = [] {
            const char* v = getenv("A8_DEC_RPOL");
            return v ? atoi(v) : 0;
        }();
        static const int wp = [] {
            const char* v = getenv("A8_DEC_WPOL");
            return v ? atoi(v) : 0;
        }();
        p.rpol = rp;
        p.wpol = wp;
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)di.sms * kDtCtas, chunks));
        decode_tma_kernel<<<(unsigned)grid, kDtCons + 32, dt_smem(nranks), st>>>(p);
    } else if (nseg <= kInlineSegs) {
        std::copy(d.begin(), d.begin() + nseg, p.segs);
        const size_t smem = dec_smem(nranks);
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)di.sms * di.dec_occ, chunks));
        launch((unsigned)grid, smem);
    } else {
        const int cap = ws_capacity(workspace_bytes);
        if (cap < nseg) return fail(A8_ERR_USAGE, "a8_decode: workspace too small for the segment count");
        std::lock_guard<std::mutex> lk(g_plan_mu);  // upload + launch, not interleaved
        uint8_t* plan = static_cast<uint8_t*>(workspace) + plan_off(cap);
        cudaMemcpyAsync(plan, d.data(), sizeof(DecSegD) * nseg, cudaMemcpyHostToDevice, st);
        p.segs_dev = reinterpret_cast<const DecSegD*>(plan);
        const size_t smem = dec_smem(nranks);
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)di.sms * di.dec_occ, chunks));
        launch((unsigned)grid, smem);
    }
    return cuda_check("a8_decode");
}

extern "C" int a8_decode(const a8_dec_seg_t* segs, int nseg, const void* book_dev, a8_layout_t layout,
                         int nranks, int op, int status_idx, int status_blocks, uint32_t* status_out,
                         void* workspace, size_t workspace_bytes, void* stream) {
    return decode_impl(segs, nullptr, -1, nseg, book_dev, layout, nranks, op, status_idx, status_blocks,
                       status_out, workspace, workspace_bytes, stream);
}

extern "C" int a8_decode_peers(const a8_dec_seg_t* segs, int nseg, const void* book_dev, a8_layout_t layout,
                               const void* const* rank_bases, int nranks, int op, int status_idx, int status_blocks,
                               uint32_t* status_out, void* workspace, size_t workspace_bytes, void* stream) {
    if (!rank_bases) return fail(A8_ERR_USAGE, "a8_decode_peers: null rank bases");
    return decode_impl(segs, nullptr, -1, nseg, book_dev, layout, nranks, op, status_idx, status_blocks, status_out,
                       workspace, workspace_bytes, stream, rank_bases);
}

extern "C" int a8_decode_local(const a8_dec_seg_t* segs, const float* const* locals, int local_rank, int nseg,
                               const void* book_dev, a8_layout_t layout, int nranks, int op, int status_idx,
                               int status_blocks, uint32_t* status_out, void* workspace, size_t workspace_bytes,
                               void* stream) {
    if (nseg > 0 && !locals) return fail(A8_ERR_USAGE, "a8_decode_local: null locals");
    if (local_rank < 0 || local_rank >= nranks) return fail(A8_ERR_USAGE, "a8_decode_local: local_rank out of range");
    return decode_impl(segs, locals, local_rank, nseg, book_dev, layout, nranks, op, status_idx, status_blocks,
                       status_out, workspace, workspace_bytes, stream);
}

// ---------------------------------------------------------------------------
// float64 input: the reference decision restated directly (codecs.py:254-268)
//   y = fl64(|x| / s), s = float32(max|x|) (absmax) | float32(10^d) | 1
//   idx = clip(searchsorted_left(values, y), 1, D-1)
//   pick = fl64(y - v[idx-1]) <= fl64(v[idx] - y) ? idx-1 : idx
// Two launches for absmax (max over the 64-bit |x| patterns, then encode).

namespace a8 {

struct F64Seg {
    const double* x;
    int64_t n;
    int64_t flat_off;
    int32_t scale_idx;
    int32_t pad;
    int64_t cstart;
};

struct F64Params {
    a8_layout_t lay;
    const a8_book_t* book;
    WsHead* head;
    SegCtl* ctl;
    const unsigned int* status_in;
    unsigned int* status_out;
    float fixed_scale;
    int absmax;
    int nseg;
    int pad;
    int64_t total;
    F64Seg segs[kInlineSegs];
};

constexpr int kF64Chunk = 4096;

__device__ __forceinline__ int f64_seg_of(const F64Params& p, int64_t c) {
    int lo = 0, hi = p.nseg;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (p.segs[mid].cstart <= c)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) f64_absmax_kernel(const __grid_constant__ F64Params p) {
    __shared__ unsigned long long red[8];
    for (int64_t c = blockIdx.x; c < p.total; c += gridDim.x) {
        const int s = f64_seg_of(p, c);
        const F64Seg& sg = p.segs[s];
        const int64_t base = (c - sg.cstart) * kF64Chunk;
        const int64_t cnt = min((int64_t)kF64Chunk, sg.n - base);
        unsigned long long m = 0;
        const double* xs = sg.x + base;
        if (cnt == kF64Chunk && (reinterpret_cast<uintptr_t>(xs) & 15) == 0) {
            // 8 double2 loads per thread, all in flight before the max
            double2 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldcs(reinterpret_cast<const double2*>(xs) + q * 256 + threadIdx.x);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                m = max(m, (unsigned long long)__double_as_longlong(v[q].x) & 0x7fffffffffffffffull);
                m = max(m, (unsigned long long)__double_as_longlong(v[q].y) & 0x7fffffffffffffffull);
            }
        } else {
            for (int64_t i = threadIdx.x; i < cnt; i += 256)
                m = max(m, (unsigned long long)__double_as_longlong(xs[i]) & 0x7fffffffffffffffull);
        }
        for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long mm = 0;
            for (int w = 0; w < 8; ++w) mm = max(mm, red[w]);
            if (mm) atomicMax(reinterpret_cast<unsigned long long*>(&p.ctl[s].amax), mm);
        }
        __syncthreads();
    }
}

// The reference decision for float64 |x| (bits a) at scale s: picks the upper
// value of the pair (v_lo, v_hi) (codecs.py:260-265).
__device__ __forceinline__ bool picks_upper64(unsigned long long a, double s, double v_lo, double v_hi) {
    const double y = __ddiv_rn(__longlong_as_double((long long)a), s);
    return !(__dsub_rn(y, v_lo) <= __dsub_rn(v_hi, y));
}

// T64: the smallest float64 bit pattern (of |x|) whose decision resolves
// upward.  The decision is monotone in |x|, so the code of x is
// #{i : T64_i <= bits(|x|)}.  Walk from the rounded midpoint, then bisect.
__device__ unsigned long long threshold64(double s, double v_lo, double v_hi) {
    constexpr unsigned long long kInf64 = 0x7ff0000000000000ull;
    const double m = 0.5 * (v_lo + v_hi) * s;
    const unsigned long long g = (unsigned long long)__double_as_longlong(m);
    unsigned long long lo = 0ull, hi = kInf64;  // pred(lo) false (pred(0) is), pred(hi) true
    if (g > 0ull && g < kInf64) {
        if (picks_upper64(g, s, v_lo, v_hi)) {
            hi = g;
            for (int k = 0; k < 8 && hi > 0ull; ++k) {
                if (!picks_upper64(hi - 1ull, s, v_lo, v_hi)) return hi;
                --hi;
            }
        } else {
            lo = g;
            for (int k = 0; k < 8 && lo + 1ull < kInf64; ++k) {
                if (picks_upper64(lo + 1ull, s, v_lo, v_hi)) return lo + 1ull;
                ++lo;
            }
        }
    }
    while (hi - lo > 1ull) {
        const unsigned long long mid = lo + ((hi - lo) >> 1);
        if (picks_upper64(mid, s, v_lo, v_hi))
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

__global__ void __launch_bounds__(256) f64_encode_kernel(const __grid_constant__ F64Params p) {
    __shared__ double sV[128];
    __shared__ uint8_t sC[128];
    __shared__ unsigned long long sT64[128];  // thresholds of the current segment's scale
    __shared__ int sFinal;
    const int tid = threadIdx.x;
    const int D = p.book->ndistinct;
    if (tid < 128) {
        sV[tid] = tid < D ? p.book->values[tid] : __longlong_as_double(0x7ff0000000000000ll);  // +inf pad
        sC[tid] = p.book->codes[tid];
    }
    __syncthreads();
    unsigned int bad = 0;
    const int64_t L = p.lay.block_len;
    const int64_t gap = p.lay.block_stride - p.lay.block_len;
    int cur = -1;
    float sf = p.fixed_scale;
    for (int64_t c = blockIdx.x; c < p.total; c += gridDim.x) {
        const int s = f64_seg_of(p, c);
        const F64Seg& sg = p.segs[s];
        if (s != cur) {  // thresholds of this segment's scale, once per CTA and segment
            sf = p.fixed_scale;
            if (p.absmax) {
                const unsigned long long mb = __ldcg(reinterpret_cast<const unsigned long long*>(&p.ctl[s].amax));
                if (mb >= 0x7ff0000000000000ull) bad = 1;
                const double peak = __longlong_as_double((long long)mb);
                sf = peak > 0.0 ? __double2float_rn(peak) : 1.0f;  // codecs.py:234-241
            }
            __syncthreads();  // the previous segment's thresholds are no longer read
            if (tid < 128) {
                unsigned long long t = 0x7ff0000000000000ull;
                if (scale_ok(sf) && tid + 1 < D) t = threshold64((double)sf, sV[tid], sV[tid + 1]);
                sT64[tid] = t;
            }
            __syncthreads();
            cur = s;
        }
        const int64_t base = (c - sg.cstart) * kF64Chunk;
        const int64_t cnt = min((int64_t)kF64Chunk, sg.n - base);
        if (base == 0 && tid < p.lay.scale_reps) p.lay.scales[tid * p.lay.scale_block_stride + sg.scale_idx] = sf;
        auto code_of = [&](double xv) -> uint32_t {
            if (!isfinite(xv)) bad = 1;
            const unsigned long long a = (unsigned long long)__double_as_longlong(xv) & 0x7fffffffffffffffull;
            int pick = 0;  // #{i : T64_i <= |x|} = the reference's pick (codecs.py:262-266)
#pragma unroll
            for (int step = 64; step; step >>= 1)
                if (sT64[pick + step - 1] <= a) pick += step;
            uint32_t code = sC[pick];
            if (xv < 0.0 && pick != 0) code |= 0x80u;  // codecs.py:267-268
            return code;
        };
        const double* xs = sg.x + base;
        const int64_t f0 = sg.flat_off + base;
        if (cnt == kF64Chunk && (reinterpret_cast<uintptr_t>(xs) & 15) == 0) {
            // 8 consecutive elements per thread and group (4 double2 loads,
            // one 8-byte store of codes; a group never straddles a block)
#pragma unroll
            for (int grp = 0; grp < 2; ++grp) {
                const int e0 = grp * 2048 + tid * 8;
                double2 v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = __ldcs(reinterpret_cast<const double2*>(xs + e0) + q);
                unsigned long long w = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w |= ((unsigned long long)code_of(v[q].x) << (16 * q)) | ((unsigned long long)code_of(v[q].y) << (16 * q + 8));
                const int64_t f = f0 + e0;
                *reinterpret_cast<unsigned long long*>(p.lay.codes + f + (f / L) * gap) = w;
            }
        } else {
            for (int64_t i = tid; i < cnt; i += 256) {
                const int64_t f = f0 + i;
                p.lay.codes[f + (f / L) * gap] = (uint8_t)code_of(xs[i]);
            }
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&p.head->status, A8_STATUS_NONFINITE);
    if (tid == 0) {
        __threadfence();
        sFinal = atomicAdd(&p.head->ctas_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sFinal) {
        __threadfence();
        for (int i = tid; i < p.nseg; i += 256) *reinterpret_cast<unsigned long long*>(&p.ctl[i].amax) = 0ull;
        if (tid < p.lay.scale_reps) {
            const unsigned int stt = atomicAdd(&p.head->status, 0u) | (p.status_in ? *p.status_in : 0u);
            p.status_out[(int64_t)tid * p.lay.scale_block_stride] = stt;
        }
        __syncthreads();
        if (tid == 0) {
            p.head->ctas_done = 0u;
            p.head->status = 0u;
        }
        __threadfence();
    }
}

}  // namespace a8

extern "C" int a8_encode_f64(const a8_enc_seg64_t* segs, int nseg, const void* book_dev, int norm,
                             float fixed_scale, a8_layout_t layout, void* workspace, size_t workspace_bytes,
                             const uint32_t* status_in, uint32_t* status_out, void* stream) {
    if (nseg <= 0 || nseg > kInlineSegs) return fail(A8_ERR_USAGE, "a8_encode_f64: 1..32 segments per call");
    if (!segs || !book_dev || !workspace || !status_out) return fail(A8_ERR_USAGE, "a8_encode_f64: null argument");
    if (int rc = check_layout(layout)) return rc;
    if (layout.scale_reps < 1 || layout.scale_reps > 256) return fail(A8_ERR_USAGE, "a8_encode_f64: scale_reps out of range");
    if (ws_capacity(workspace_bytes) < nseg) return fail(A8_ERR_USAGE, "a8_encode_f64: workspace too small");
    int device = 0;
    cudaGetDevice(&device);
    DevInfo di;
    if (int rc = dev_info(device, &di)) return rc;
    F64Params p;
    memset(&p, 0, sizeof(p));
    p.lay = layout;
    p.book = static_cast<const a8_book_t*>(book_dev);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    p.head = reinterpret_cast<WsHead*>(ws);
    p.ctl = reinterpret_cast<SegCtl*>(ws + ctl_off());
    p.status_in = status_in;
    p.status_out = status_out;
    p.fixed_scale = fixed_scale;
    p.absmax = norm == A8_NORM_ABSMAX;
    p.nseg = nseg;
    int64_t ch = 0;
    for (int i = 0; i < nseg; ++i) {
        if (segs[i].n < 0 || (segs[i].n > 0 && !segs[i].x) || segs[i].flat_off % 16)
            return fail(A8_ERR_USAGE, "a8_encode_f64: bad segment");
        p.segs[i] = F64Seg{segs[i].x, segs[i].n, segs[i].flat_off, segs[i].scale_idx, 0, ch};
        ch += std::max<int64_t>(1, (segs[i].n + kF64Chunk - 1) / kF64Chunk);
    }
    p.total = ch;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)di.sms * 8, ch);
    if (p.absmax) {
        f64_absmax_kernel<<<grid, 256, 0, st>>>(p);
        if (int rc = cuda_check("a8_encode_f64(absmax)")) return rc;
    }
    f64_encode_kernel<<<grid, 256, 0, st>>>(p);
    return cuda_check("a8_encode_f64");
}
