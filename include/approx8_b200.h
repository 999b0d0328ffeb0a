/*
 * approx8_b200 -- C ABI of the B200-native 8-bit approximation codec.
 *
 * Drop-in boundary for the hot path of the reference package `approx8`
 * (/root/reference/pkg/src/approx8/codecs.py).  The reference is pure
 * Python/NumPy, so "the FFI a maintainer would bind" is a ctypes binding
 * from Python; every entry point below names the
 * reference function it replaces.
 *
 * Conventions
 *   - plain pointers and sizes only; device pointers are CUDA global memory,
 *     `stream` is a cudaStream_t passed as void*;
 *   - every call returns an int status (A8_OK or one of the A8_ERR_* codes,
 *     mirroring approx8/errors.py:16-33); a8_last_error() gives the message;
 *   - compute entry points are asynchronous on `stream`; the non-finite
 *     input condition (codecs.py:251-252, InputError) is reported through a
 *     device status word because detecting it needs the data.
 *
 * Flat index space and slab layout (shared by encode and decode)
 *   A call covers `nseg` segments (tensors).  Segment s occupies flat
 *   elements [flat_off_s, flat_off_s + n_s); flat_off_s is a multiple of 16.
 *   The codes for flat element e live at
 *       codes + (e / block_len) * block_stride + (e % block_len)
 *   and the float32 scale of segment s as seen from block j at
 *       scales + j * scale_block_stride + scale_idx_s           (floats)
 *   For decode, rank r's copy is offset by r * rank_stride bytes (codes and
 *   scales alike).  One block (block_len >= total) is the plain layout.
 */
#ifndef APPROX8_B200_H
#define APPROX8_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define A8_ABI_VERSION 1

/* status codes: approx8/errors.py:16-33 */
#define A8_OK 0
#define A8_ERR_INPUT 1  /* InputError  -- non-finite data (codecs.py:251-252) */
#define A8_ERR_CONFIG 2 /* ConfigError -- invalid spec (codecs.py:112-123)   */
#define A8_ERR_USAGE 3  /* UsageError  -- bad call (codecs.py:274-280)        */
#define A8_ERR_CUDA 4   /* CUDA launch / runtime failure                      */

/* codebook kinds: codecs.py:73-77 (DataTypeKind) */
#define A8_DYNAMIC_TREE 0
#define A8_STATIC_TREE 1
#define A8_LINEAR 2
#define A8_MANTISSA 3

/* normalisations: codecs.py:80-83 (NormKind) */
#define A8_NORM_NONE 0
#define A8_NORM_ABSMAX 1
#define A8_NORM_DECADE 2

/* device status bits (a8_encode) */
#define A8_STATUS_NONFINITE 1u
#define A8_STATUS_AMAX_MISMATCH 2u /* a8_encode_premax: a supplied max != max|x| */

#define A8_LUT_MAX 4096

/* Codebook of one kind: codecs.py:161-204 (Codebook / build_codebook). */
typedef struct a8_book {
    double values[128]; /* distinct non-negative values, ascending (codecs.py:194-199) */
    float table[256];   /* decode table, -0 folded to +0 (codecs.py:189-192)          */
    uint8_t codes[128]; /* lowest code byte per distinct value (codecs.py:195-200)    */
    int32_t ndistinct;  /* D: 128, or 114 for mantissa                                 */
    int32_t kind;
    int32_t pad[2];
} a8_book_t;

/* Per-scale decision table.  T[i] is the smallest float32 bit pattern whose
 * reference decision (codecs.py:260-265) picks a value above index i;
 * e[] buckets |x| by its top 15 bits (exponent + 7 mantissa bits) with at
 * most one distinct threshold per bucket.  valid == 0 means the bucket table
 * does not apply (e.g. subnormal scales) and T[] is searched instead. */
typedef struct a8_lut {
    uint32_t len;     /* used entries of e[]            */
    int32_t kbase;    /* key of e[0]                    */
    uint32_t valid;   /* 1: bucket table usable         */
    uint32_t nfinite; /* thresholds below 0x7f800000    */
    float scale;      /* the scale the table encodes    */
    uint32_t pad[3];
    uint32_t T[128];  /* thresholds, padded with 0x7f800000 */
    uint32_t e[A8_LUT_MAX]; /* t_low << 16 | code_hi << 8 | code_lo; an element of
                             * the bucket takes code_hi iff lo16(bits) >= t_low */
} a8_lut_t;

/* Encode segment: a float32 tensor (contiguous). */
typedef struct a8_enc_seg {
    const float* x;
    int64_t n;
    int64_t flat_off;  /* multiple of 16 */
    int32_t scale_idx; /* slot of this segment's scale in each block's scale array */
    int32_t pad;
} a8_enc_seg_t;

/* Encode segment with float64 input (a8_encode_f64). */
typedef struct a8_enc_seg64 {
    const double* x;
    int64_t n;
    int64_t flat_off;  /* multiple of 16 */
    int32_t scale_idx;
    int32_t pad;
} a8_enc_seg64_t;

/* Decode segment: a float32 output tensor (contiguous). */
typedef struct a8_dec_seg {
    float* out;
    int64_t n;
    int64_t flat_off;  /* multiple of 16; the piece lies inside one block */
    int32_t scale_idx;
    int32_t pad;
} a8_dec_seg_t;

typedef struct a8_layout {
    uint8_t* codes;
    float* scales;
    int64_t block_len;          /* elements per block, multiple of 16           */
    int64_t block_stride;       /* bytes between consecutive blocks of codes    */
    int64_t scale_block_stride; /* floats between consecutive blocks' scales    */
    int64_t rank_stride;        /* bytes between ranks' copies (decode only)    */
    int32_t scale_reps;         /* encode: write the scale into blocks [0, reps) */
    int32_t flags;              /* decode: A8_LAYOUT_* bits (0 = defaults)      */
} a8_layout_t;

/* a8_layout_t.flags (decode).  A8_LAYOUT_STATUS_COUNT: status_out counts
 * non-finite calls -- *status_out += (status != 0) -- instead of being
 * overwritten with the status bits, so a word shared by many launches (one
 * CUDA graph replayed many times) never loses a report between host reads. */
#define A8_LAYOUT_STATUS_COUNT 1

int a8_abi_version(void);
const char* a8_last_error(void);

/* build_codebook (codecs.py:186-204): fills `out` on the host. */
int a8_codebook(int kind, a8_book_t* out);

/* _scale_for (codecs.py:232-241) for the data-independent normalisations:
 * none -> 1, decade d -> float32(10^d).  absmax is data dependent (device). */
int a8_fixed_scale(int norm, int decades, float* scale_out);

/* Host construction of the decision table for a fixed scale (used for the
 * none/decade specs and by the CPU tests of the table logic). */
int a8_build_lut_host(const a8_book_t* book, float scale, a8_lut_t* out);

/* Device scratch needed by a8_encode / a8_decode for up to `nseg` segments.
 * Must be zero-filled once after allocation; the kernels leave it zeroed.
 * Calls pass the workspace's byte size: its layout is a function of that
 * capacity only, so calls with different segment counts can share it (in
 * stream order). */
size_t a8_workspace_bytes(int nseg);

/* encode_buffer (codecs.py:244-269) for nseg tensors in one launch.
 *   book_dev    device copy of a8_codebook(kind)
 *   norm        A8_NORM_ABSMAX: per-segment absmax scale computed on device;
 *               otherwise `static_lut_dev` (device copy of a8_build_lut_host
 *               for the fixed scale) is used for every segment.
 *   segs        host array of nseg descriptors (copied into the launch, or
 *               into `workspace` when nseg is large)
 *   status_in   optional device uint32 OR-ed into the result (chaining)
 *   status_out  device uint32, OVERWRITTEN with this call's A8_STATUS_* bits
 *               (| *status_in) once the kernel finishes; replicated to
 *               status_out[k * scale_block_stride] for k < scale_reps      */
int a8_encode(const a8_enc_seg_t* segs, int nseg, const void* book_dev, int norm,
              const void* static_lut_dev, a8_layout_t layout, void* workspace,
              size_t workspace_bytes, const uint32_t* status_in, uint32_t* status_out,
              void* stream);

/* a8_encode for an absmax spec whose per-segment maxima are already known --
 * computed by the kernel that produced the tensors (a8_produce_absmax, or
 * any producer that writes float32 bits of max|x|).  The segment's scale is
 * amax_dev[i] (codecs.py:237-241), so the encode is ONE pass over x (4 B read
 * + 1 B written per element) instead of max pass + encode pass.  The kernel
 * still computes max|x| of each segment as it encodes; if it differs from
 * amax_dev[i] the status gets A8_STATUS_AMAX_MISMATCH (the codes of that
 * call are then unspecified, but every access stays in bounds).  Two
 * non-finite maxima (Inf / any NaN) agree: that input is reported with
 * A8_STATUS_NONFINITE as by a8_encode.  Same
 * layout / workspace / status conventions as a8_encode.  Launches: one, or
 * for calls beyond the resident kernel a table prologue (one CTA per
 * multi-chunk segment) plus the encode as its programmatic dependent.
 * Replaces the max pass of codecs.py:237-241 when the producer supplies it
 * (the encode fused with its producer).                  */
int a8_encode_premax(const a8_enc_seg_t* segs, int nseg, const void* book_dev, const uint32_t* amax_dev,
                     a8_layout_t layout, void* workspace, size_t workspace_bytes, const uint32_t* status_in,
                     uint32_t* status_out, void* stream);

/* Producer pass with the absmax fused into it: for each segment,
 *   A8_PRODUCE_SCALE      y = fl(alpha * x)   (alpha == 1 and y == x: max only)
 *   A8_PRODUCE_RELU       y = x >= 0 || x is NaN ? x : 0      (mlp.py:205)
 *   A8_PRODUCE_RELU_MASK  y = fl(relu(x) * mask)               (mlp.py:205-207)
 * and amax_out[i] = bits(max|y|) (NaN bits when y holds a NaN), ready for
 * a8_encode_premax.  y may alias x.  1 launch (+ a 4 B/segment memset) per
 * 32 segments; the pass streams 8 B (12 B with a mask) per element.         */
#define A8_PRODUCE_SCALE 0
#define A8_PRODUCE_RELU 1
#define A8_PRODUCE_RELU_MASK 2
typedef struct a8_prod_seg {
    const float* x;
    float* y;
    const float* mask; /* A8_PRODUCE_RELU_MASK only */
    int64_t n;
} a8_prod_seg_t;
int a8_produce_absmax(const a8_prod_seg_t* segs, int nseg, int op, float alpha, uint32_t* amax_out, void* stream);

/* roundtrip (codecs.py:285-288) fused: decode(encode(x)) for nseg float32
 * tensors in one launch, written to outs[i] (same length as segs[i]); the
 * codes are never stored.  scales_out[scale_idx] receives each scale,
 * status_out (device uint32) the A8_STATUS_* bits.  Only for calls that fit
 * in the GPU's shared memory (<= 32 tensors, ~7.5M elements); otherwise it
 * returns A8_ERR_USAGE and the caller uses a8_encode + a8_decode.        */
int a8_roundtrip(const a8_enc_seg_t* segs, float* const* outs, int nseg, const void* book_dev, int norm,
                 const void* static_lut_dev, float* scales_out, uint32_t* status_out, void* workspace,
                 size_t workspace_bytes, void* stream);
/* encode_buffer for float64 input, bit-exact with the reference's float64
 * arithmetic (codecs.py:254-268): absmax over the float64 values rounded to
 * float32, y = |x|/s in float64, searchsorted + clip + tie rule per element.
 * 1..32 segments; `fixed_scale` is used for none/decade (see a8_fixed_scale).
 * Same layout / workspace / status conventions as a8_encode.               */
int a8_encode_f64(const a8_enc_seg64_t* segs, int nseg, const void* book_dev, int norm, float fixed_scale,
                  a8_layout_t layout, void* workspace, size_t workspace_bytes, const uint32_t* status_in,
                  uint32_t* status_out, void* stream);

/* decode_buffer (codecs.py:272-282) fused with the cross-rank reduction:
 *   out = sum_{r<nranks} table[c_r] * s_r, accumulated in rank order in
 *   float32 (round-to-nearest, no FMA contraction); op = 1 divides by
 *   float32(nranks) (the data-parallel average), op = 0 keeps the sum.
 *   nranks = 1 is exactly decode_buffer.
 *   status_idx >= 0: status_out = OR of the uint32 words at
 *   scales[r * rank_stride/4 + j * scale_block_stride + status_idx] for
 *   r < nranks, j < status_blocks (the encoders' replicated status words);
 *   with layout.flags & A8_LAYOUT_STATUS_COUNT it is incremented instead. */
int a8_decode(const a8_dec_seg_t* segs, int nseg, const void* book_dev, a8_layout_t layout,
              int nranks, int op, int status_idx, int status_blocks, uint32_t* status_out,
              void* workspace, size_t workspace_bytes, void* stream);

/* a8_decode over peers' slabs that are not one strided buffer: rank r's
 * codes and scales are at the layout's offsets from rank_bases[r] instead
 * of from layout.codes/scales + r * rank_stride (layout.codes/scales are
 * given for rank 0, i.e. relative to rank_bases[0]).  With NVLink peer
 * mappings (CUDA IPC / torch symmetric memory: buffer_ptrs) the decode-sum
 * reads the other GPUs' codes directly -- the all-gather and the decode in
 * one kernel, with no gathered copy in HBM.  rank_bases: host array of
 * nranks 16-byte aligned device pointers (UVA).                           */
int a8_decode_peers(const a8_dec_seg_t* segs, int nseg, const void* book_dev, a8_layout_t layout,
                    const void* const* rank_bases, int nranks, int op, int status_idx, int status_blocks,
                    uint32_t* status_out, void* workspace, size_t workspace_bytes, void* stream);

/* a8_decode with rank local_rank's term taken from its own float32 input:
 * out = sum_r t_r, t_r = locals[i][k] for r == local_rank, else
 * table[c_r] * s_r (same order, rounding and op as a8_decode).  The paper's
 * "8-bit for incoming GPUs, 32-bit for the local GPU" (PAPER.md:194,
 * SURVEY 8(e)); the reference has no multi-GPU path, so there is no
 * reference function it replaces.  locals[i] holds segs[i].n floats and may
 * be segs[i].out itself (in place).                                        */
int a8_decode_local(const a8_dec_seg_t* segs, const float* const* locals, int local_rank, int nseg,
                    const void* book_dev, a8_layout_t layout, int nranks, int op, int status_idx,
                    int status_blocks, uint32_t* status_out, void* workspace, size_t workspace_bytes,
                    void* stream);

/* 1-bit error-feedback quantizer: onebit_quantize (codecs.py:306-339).
 *   g          n gradients, float32 (g_is_f64 = 0) or float64 (1)
 *   residual   n float64, updated in place: corrected - reconstruction
 *   bits       ceil(n/8) bytes, np.packbits order (first element in the MSB)
 *   levels     device float[2] = {pos_level, neg_level}: float32 means of the
 *              corrected values on each side of 0 (0 for an empty side)
 *   status_out device uint32, overwritten (A8_STATUS_NONFINITE)
 *   workspace  a8_onebit_workspace_bytes() bytes of device scratch          */
size_t a8_onebit_workspace_bytes(void);
int a8_onebit_quantize(const void* g, int g_is_f64, double* residual, int64_t n, uint8_t* bits,
                       float* levels, uint32_t* status_out, void* workspace, size_t workspace_bytes,
                       void* stream);

/* a8_onebit_quantize for up to 32 tensors in two launches (stats, apply)
 * instead of two per tensor: the 1-bit exchange quantizes every gradient of
 * a step at once.  Each segment is computed exactly as a8_onebit_quantize
 * computes it alone (same partial layout and summation order), so the
 * results are bit-identical.  workspace: a8_onebit_multi_workspace_bytes(nseg)
 * bytes.                                                                    */
typedef struct a8_ob_q_seg {
    const void* g;
    double* residual;
    int64_t n;
    uint8_t* bits;
    float* levels;
    uint32_t* status;
} a8_ob_q_seg_t;
size_t a8_onebit_multi_workspace_bytes(int nseg);
int a8_onebit_quantize_multi(const a8_ob_q_seg_t* segs, int nseg, int g_is_f64, void* workspace,
                             size_t workspace_bytes, void* stream);

/* onebit_decode (codecs.py:342-348): out[i] = bit ? levels[0] : levels[1]. */
int a8_onebit_decode(const uint8_t* bits, int64_t n, const float* levels, float* out, void* stream);

/* 1-bit data-parallel exchange, decode side (the DP seam mlp.py:313-321
 * across N ranks; the reference has no multi-rank function).  Rank r's slab
 * starts at slabs + r * rank_stride and holds, for segment s, its packed
 * bits at segs[s].bit_off, its {pos, neg} levels (float32) at levels_off +
 * 8 s and its quantizer status word at status_off + 4 s.
 *   out_s[i] = sum_r (bit_r(i) ? pos_r : neg_r), rank order, float32
 *   (round-to-nearest); op = 1 then divides by float32(nranks).
 * status_out (optional, device uint32): OR of every rank's first nstatus
 * status words.  At most 32 segments per call; bit_off a multiple of 16.   */
typedef struct a8_ob_seg {
    float* out;
    int64_t n;
    int64_t bit_off; /* bytes from the slab start */
} a8_ob_seg_t;
int a8_onebit_reduce(const a8_ob_seg_t* segs, int nseg, const uint8_t* slabs, int64_t rank_stride,
                     int64_t levels_off, int64_t status_off, int nstatus, int nranks, int op, uint32_t* status_out,
                     void* stream);

/* Per-block max-abs codec (north star: "optional per-block max-abs"; not a
 * reference feature).  Block b = elements [b*block, (b+1)*block) is encoded
 * exactly as encode_buffer(x[block b]) with absmax normalisation
 * (codecs.py:232-269): scales[b] = float32(max |x| of the block), 0 -> 1.
 * block is 1024, 2048 or 4096; codes 4-byte aligned; scales holds
 * ceil(n/block) floats; status_out (device uint32) is overwritten with
 * A8_STATUS_* bits.  Single pass: 4 B read + 1 B written per element.     */
int a8_encode_blocked(const float* x, int64_t n, int64_t block, const void* book_dev, uint8_t* codes,
                      float* scales, uint32_t* status_out, void* stream);
/* decode of a8_encode_blocked: out[i] = table[codes[i]] * scales[i / block]
 * (one RN multiply, codecs.py:281).                                          */
int a8_decode_blocked(const uint8_t* codes, int64_t n, int64_t block, const float* scales, const void* book_dev,
                      float* out, void* stream);
/* Round-trip error aggregates: measure_error (errorbench.py:79-99) and the
 * hook statistics _HookStats.record (mlp.py:146-153).  Over n elements:
 *   d      = float32(table[codes[i]] * *scale_dev)  (codes != NULL, the
 *            decode of codecs.py:281), else after[i] (a decoded float32 tensor)
 *   out[0] = sum |x - d|, out[1] = sum over x != 0 of |x - d| / |x|,
 *   out[2] = #(x != 0), all float64 (x widened exactly from float32, or
 *            float64 when x_is_f64); accumulate = 1 adds to out[] instead.
 * Deterministic for a given device (fixed-order reduction).  workspace:
 * a8_error_workspace_bytes() bytes, zero-filled once (left zeroed).         */
size_t a8_error_workspace_bytes(void);
int a8_error_stats(const void* x, int x_is_f64, int64_t n, const uint8_t* codes, const float* scale_dev,
                   const void* book_dev, const float* after, double* out_dev, int accumulate, void* workspace,
                   size_t workspace_bytes, void* stream);
/* Diagnostics: globaltimer trace of the last ticket-kernel a8_encode on
 * `workspace` (synchronous device->host copy).  out[0..3] = kernel start
 * ns, end ns, total CTA time spent waiting for a segment's max to be final
 * (ns), number of such waits; out[4 + 4k .. 7 + 4k] are reserved (zero: the
 * per-segment tables are built by the CTAs that use them).  Needs
 * 4 + 4*nseg entries.                                                      */
int a8_encode_trace(const void* workspace, int nseg, uint64_t* out);

/* Number of SMs and the persistent grid sizes the kernels use on `device`. */
int a8_device_info(int device, int* num_sms, int* enc_ctas_per_sm, int* dec_ctas_per_sm);

#ifdef __cplusplus
}
#endif

#endif /* APPROX8_B200_H */
