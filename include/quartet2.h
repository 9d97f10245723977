/*
 * quartet2.h — C ABI of the B200-native Quartet II NVFP4 linear-layer kernels.
 *
 * The reference (nvfp4emu, /root/reference/pkg/src/nvfp4emu) has no FFI: its
 * boundary is a pure-Python function API.  Each entry point below replaces one
 * of those functions (cited per declaration); the Python package
 * paper_2601_22813_b200 binds them with ctypes and keeps the reference's names,
 * argument meanings and exceptions.  See INTEGRATION.md for the binding.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers; every call is stream-ordered on
 *    `stream` (a cudaStream_t passed as void*), asynchronous, and allocates
 *    nothing.  Callers own every buffer.
 *  - Return value: Q2_OK, Q2_EINVAL (bad shape / argument; nothing launched)
 *    or Q2_ECUDA (launch error).
 *  - Data-dependent failures that the reference raises as ValueError /
 *    OverflowError are OR-ed into the device word `err` (Q2_ERR_* bits); the
 *    host wrapper reads it and raises with the reference's message.
 *  - Reentrant: no global mutable state.  Concurrent calls are safe on
 *    distinct streams with distinct workspaces.
 *
 * NVFP4 tensor in HBM (q2_nvfp4): a logical [R, K] tensor quantized along K.
 *  codes   uint8 [R, K/2], row-major, two E2M1 codes per byte, low nibble =
 *          even k (the NV4T packing of quantizers.py:339).
 *  sf      UE4M3 group scales (one per 16 along K), unreplicated, in the tcgen05
 *          block-scale vector layout: one 1 KiB block per (256-row block,
 *          64-element K block), blocks K-fastest; rows padded to 256.  Block
 *          byte (L/8)*256 + h*128 + (L%8)*16 + c*4 + i holds scale i of row
 *          128*h + 32*c + L of the block (L = TMEM lane 0..31).  Each 512 B half
 *          h is the shared-memory source of one tcgen05.cp.32x128b.warpx4, which
 *          broadcasts it to the four TMEM subpartitions.  Byte of (r, j):
 *            ((r/256)*ceil(K/64) + j/4)*1024 + ((r%32)/8)*256 + ((r/128)%2)*128
 *              + (r%8)*16 + ((r%128)/32)*4 + j%4
 *          Size: q2_sf_bytes(R, K) = ceil(R/256)*ceil(K/64)*1024.
 *  scale32 float32 device scalar (the reference's np.float32 tensor scale).
 */
#ifndef QUARTET2_H_
#define QUARTET2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { Q2_OK = 0, Q2_EINVAL = 1, Q2_ECUDA = 2 };
enum { Q2_BF16 = 0, Q2_F32 = 1, Q2_F64 = 2 };   /* Q2_F64: q2_rht input only */

/* err-word bits (device uint32) */
enum {
  Q2_ERR_NONFINITE = 1u,  /* "input must be finite"              quantizers.py:118-119 */
  Q2_ERR_SCALE448  = 2u,  /* corrected scale exceeds 448         ms_eden.py:144-149, posthoc.py:115-122 */
  Q2_ERR_NAN_SCALE = 4u,  /* NaN reached encode_fp8_rtn          formats.py:167-168 */
  Q2_ERR_E8M3_OVF  = 8u,  /* round_e8m3_rtn overflow             formats.py:223-224 */
  Q2_ERR_SR_CLIP   = 16u  /* SR group quotient above 6 (AssertionError "encoder bug") quantizers.py:153-157 */
};

typedef struct {
  uint8_t* codes;
  uint8_t* sf;
  float*   scale32;
  int64_t  R, K;
} q2_nvfp4;

/* Bytes of the scale-factor buffer for a [R, K] tensor. */
size_t q2_sf_bytes(int64_t R, int64_t K);

/* Library build info (arch string); used by the loader's self-check. */
const char* q2_version(void);

/* Per-tensor |x| max as float bits (x is bf16/fp32, exact), OR-ing
 * Q2_ERR_NONFINITE into err.  amax must be zeroed by the caller (or use
 * q2_quant_fwd which does it).                                                  */
int q2_amax(const void* x, int dtype, int64_t R, int64_t K, int64_t ld,
            uint32_t* amax_bits, uint32_t* err, void* stream);

/* Forward quantizer family (one pass over x after the amax pass).
 *  quantize_rtn_46(x, caps, scale_cap)   quantizers.py:206-234
 *      ncaps = 2, caps = {c0, c1}, scale_div = c0*scale_cap (host float64)
 *  quantize_rtn(x, s)                    quantizers.py:164-181
 *      ncaps = 1, caps = {s}, scale_div = s*256
 *  scale32 = (float)(absmax / scale_div); per group s8 = E4M3_RTN(gmax /
 *  (scale32*c)); codes by ties-to-even RTN; with two caps the branch with the
 *  strictly lower sequential float64 squared error wins (ties keep caps[0]).
 *  ws: q2_quant_fwd_ws_bytes(R, K) bytes of device scratch (tensor absmax and
 *  the list of groups the certified fp32 fast path hands to the exact
 *  float64 fix-up kernel).                                                     */
size_t q2_quant_fwd_ws_bytes(int64_t R, int64_t K);
int q2_quant_fwd(const void* x, int dtype, int64_t R, int64_t K, int64_t ld,
                 int ncaps, double cap0, double cap1, double scale_div,
                 const q2_nvfp4* out, void* ws, uint32_t* err, void* stream);
/* q2_quant_fwd with the tensor absmax supplied by the producer of x (e.g. an
 * RMSNorm or activation epilogue that atomicMax-es the float bits of |x|):
 * the amax pass is skipped; `amax_bits` is device memory holding the float
 * bits of max|x|.                                           */
int q2_quant_fwd_amax(const void* x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps, double cap0,
                      double cap1, double scale_div, const uint32_t* amax_bits, const q2_nvfp4* out, void* ws,
                      uint32_t* err, void* stream);

/* MS-EDEN backward quantizer (randomized 128-Hadamard + clipping RTN cap 256 +
 * per-chunk EDEN factor + stochastic E4M3 scale rounding).
 *  ms_eden_quantize(x, seeds, s, tensor_id, rotation_id, pow2_scale)
 *      ms_eden.py:116-153     mode Q2_MSED_EXACT / Q2_MSED_POW2
 *  pass2(pass1(x, seed_rht, s, tensor_id, rotation_id), seed_sr, tensor_id)
 *      posthoc.py:74-125      mode Q2_MSED_POSTHOC (single read of x)
 * The quantized logical tensor is [R, K], grouped/rotated along K:
 *  Q2_SRC_ROWS     x is bf16/fp32 [R, K] with row stride ld (elements).
 *  Q2_SRC_COLS     x is bf16/fp32 [K, R] with row stride ld: quantizes x^T
 *                  (E^T for the wgrad GEMM) without materialising it.
 *  Q2_SRC_TAPE_COLS x is an NVFP4 tensor `tape` of logical shape [K, R]
 *                  (qW or qX saved by the forward); quantizes dequant(tape)^T
 *                  (W^T / X^T of linear_graph.py:293-294, 304, 322-323).
 * sign_mask: 128-bit sign vector (4 x u32, bit i = sign i negative) for the
 * rotation stream (rht.py:99-106); sr_stream = derive_stream(0x5343414C,
 * tensor_id) (ms_eden.py:150).  inv_sqrt_chunk is 128**-0.5 as the host
 * computes it.  ws: q2_msed_ws_bytes(R, K) bytes of device scratch.           */
enum { Q2_SRC_ROWS = 0, Q2_SRC_COLS = 1, Q2_SRC_TAPE_COLS = 2 };
enum { Q2_MSED_EXACT = 0, Q2_MSED_POW2 = 1, Q2_MSED_POSTHOC = 2 };
size_t q2_msed_ws_bytes(int64_t R, int64_t K);
int q2_msed_quant(const void* x, int dtype, const q2_nvfp4* tape, int src_kind,
                  int64_t R, int64_t K, int64_t ld, const uint32_t sign_mask[4],
                  double s, double inv_sqrt_chunk, uint64_t seed_sr, uint64_t sr_stream,
                  int mode, const q2_nvfp4* out, void* ws, uint32_t* err, void* stream);

/* Post-hoc pass 1 alone (posthoc.py:74-95): codes written to out->codes,
 * E8M3 pseudo-scales as bf16 [R, K/16], EDEN factors as float64 [R, K/128],
 * rotated absmax and pseudo-scale max as float bits in red[0], red[1].
 * pass 2 alone (posthoc.py:98-125) reads pseudo/corr/red and writes out->sf,
 * out->scale32.                                                              */
int q2_posthoc_pass1(const void* x, int dtype, const q2_nvfp4* tape, int src_kind,
                     int64_t R, int64_t K, int64_t ld, const uint32_t sign_mask[4],
                     double s, double inv_sqrt_chunk, uint8_t* codes,
                     uint16_t* pseudo_bf16, double* corr, uint32_t* red,
                     uint32_t* err, void* stream);
int q2_posthoc_pass2(const uint16_t* pseudo_bf16, const double* corr, const uint32_t* red,
                     int64_t R, int64_t K, uint64_t seed_sr, uint64_t sr_stream,
                     const q2_nvfp4* out, uint32_t* err, void* stream);

/* Both backward operands that read E, from ONE read of E (tensor-core kernel):
 *  out_rows = MS(E)    rows of E along N  (dgrad operand, pair_dx)   linear_graph.py:306
 *  out_cols = MS(E^T)  rows of E^T along T (wgrad operand, pair_dw)  linear_graph.py:325
 * with the ms_eden_quantize (ms_eden.py:116-153) semantics of `mode`
 * (Q2_MSED_EXACT / Q2_MSED_POW2) or pass2(pass1(.)) (posthoc.py:74-125,
 * Q2_MSED_POSTHOC).  E is bf16 [T, N] (row stride ld), T % 128 == N % 128 == 0.
 * Each 128x128 tile of E is read once; its row chunks and column chunks are
 * rotated by two tensor-core MMAs from the same shared-memory tile.
 * ws: q2_msed_dual_ws_bytes(T, N).
 * q2_msed_dual_posthoc: the same in post-hoc mode with the per-operand
 * workspaces of q2_msed_quant (q2_msed_ws_bytes(T, N) and (N, T)).            */
size_t q2_msed_dual_ws_bytes(int64_t T, int64_t N);
int q2_msed_dual(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t sign_rows[4],
                 const uint32_t sign_cols[4], double s, double inv_sqrt_chunk, uint64_t seed_sr,
                 uint64_t sr_stream_rows, uint64_t sr_stream_cols, int mode, const q2_nvfp4* out_rows,
                 const q2_nvfp4* out_cols, void* ws, uint32_t* err, void* stream);
int q2_msed_dual_posthoc(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t sign_rows[4],
                         const uint32_t sign_cols[4], double s, double inv_sqrt_chunk, uint64_t seed_sr,
                         uint64_t sr_stream_rows, uint64_t sr_stream_cols, const q2_nvfp4* out_rows,
                         const q2_nvfp4* out_cols, void* ws_rows, void* ws_cols, uint32_t* err, void* stream);
/* Engine selection for q2_msed_quant / q2_msed_dual (process-wide setting):
 * 0 auto (tensor-core kernel for the one-read dual E source; the literal
 * float64 kernels for single-operand sources, faster there today), 1 the
 * tensor-core kernel wherever eligible (bf16 or tape sources, dims multiples
 * of 128), 2 the literal float64 kernels everywhere.  Results are identical. */
int q2_set_msed_engine(int engine);
/* Counters of the tensor-core MS-EDEN path since load (host-synchronous):
 * out[0] = 128-chunks quantized, out[1] = chunks whose certification failed and
 * that were recomputed by the literal float64 path.  reset != 0 zeroes them.   */
int q2_msed_stats(unsigned long long out[2], int reset);
/* Kernel launches this library issued since load (host counter, incremented per
 * launch); reset != 0 zeroes it.  Used by bench.py for its gpu_launches figure.  */
unsigned long long q2_launch_count(int reset);

/* Stochastic-rounding baselines.
 *   q2_quant_sr: quantize_sr (quantizers.py:139-161; ncaps 1, cap0 6) and
 *   quantize_sr_46 (:237-262; ncaps 2, caps 6/4) on bf16/fp32 rows [R, K]
 *   (ld == K, 32-byte aligned):
 *     scale32 = (float)(absmax / scale_div)
 *     s8_b    = E4M3_RTN(gmax / ((scale32 * cap_b) * margin))   float64
 *     codes   = _nb_sr (_kernels.py:130-157) with
 *               u = prng_uniform(seed, stream_b, flat index)  (rht.py:89-96)
 *     46: per group the branch with strictly lower float64 error (ties: 0).
 *   The caller passes scale_div and margin evaluated in the reference's
 *   float64 order (6 * (16/17) * 448 for quantize_sr, 6 * (448 * 16/17) for
 *   quantize_sr_46; margin 16/17).  A group quotient above 6 (ncaps 1) sets
 *   Q2_ERR_SR_CLIP.  ws: q2_quant_sr_ws_bytes() bytes.
 *   q2_rht_sr_quant: the sr_rht operand quantizer (linear_graph.py:259-274):
 *   x_rot = rht_apply(x, sign_mask) along K (rht.py:144-155), then quantize_sr
 *   of x_rot with the same constants; sources as q2_msed_quant.  Two passes
 *   over x (absmax of x_rot, then quantize).  ws: q2_msed_ws_bytes(R, K).    */
/*   q2_sr_quant_src: the general SR operand quantizer of _sr_pair: rotate 0/1
 *   (sr / sr_46 vs sr_rht / sr_rht_46), ncaps 1 (quantize_sr) or 2
 *   (quantize_sr_46 with branch streams stream0, stream1), any source.       */
int q2_sr_quant_src(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R, int64_t K, int64_t ld,
                    int rotate, const uint32_t sign_mask[4], int ncaps, double cap0, double cap1, double margin,
                    double scale_div, double inv_sqrt_chunk, uint64_t seed, uint64_t stream0, uint64_t stream1,
                    const q2_nvfp4* out, void* ws, uint32_t* err, void* stream);
size_t q2_quant_sr_ws_bytes(void);
int q2_quant_sr(const void* x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps, double cap0, double cap1,
                double margin, double scale_div, uint64_t seed, uint64_t stream0, uint64_t stream1,
                const q2_nvfp4* out, void* ws, uint32_t* err, void* stream);
int q2_rht_sr_quant(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R, int64_t K,
                    int64_t ld, const uint32_t sign_mask[4], double cap, double margin, double scale_div,
                    double inv_sqrt_chunk, uint64_t seed, uint64_t stream, const q2_nvfp4* out, void* ws,
                    uint32_t* err, void* stream_);

/* 16x16 square-block quantizer (quantize_square_block, quantizers.py:265-312):
 * one E4M3 scale per 16x16 block, scale32 = (float)(absmax / (6 * 256)), codes
 * by the literal float64 quotient; use46 picks 6 or 4 per block on the float64
 * squared error summed in numpy's sum(axis=(1, 3)) order.  Writes the result
 * twice for the GEMM -- `out` [R, C] and `out_t` = its transpose [C, R], both
 * with the block scale expanded into the per-16 scale layout -- and the
 * compact block scales `scales8` uint8 [R/16, C/16].  x bf16/fp32 [R, C]
 * contiguous, 32-byte aligned.  ws: 16 bytes.                                 */
int q2_quant_square_block(const void* x, int dtype, int64_t R, int64_t C, int use46, const q2_nvfp4* out,
                          const q2_nvfp4* out_t, uint8_t* scales8, void* ws, uint32_t* err, void* stream);

/* NVFP4 "TN" GEMM on tcgen05 block-scaled MMAs (kind::mxf4nvf4, UE4M3 scales
 * per 16, FP32 accumulation in TMEM):  D[M, N] = alpha * A[M,K] . B[N,K]^T
 * with alpha = *a->scale32 * *b->scale32 (+ beta*D if accumulate).  CTA pairs
 * (cta_group::2) compute 256x256 tiles; M, N tails are masked by TMA.
 * Replaces gemm_emulated (linear_graph.py:190-205) for the fprop, dgrad and
 * wgrad GEMMs.  d_dtype Q2_BF16 or Q2_F32; d row stride ldd (elements).
 * K % 64 == 0; K/2 % 16 == 0.                                                */
int q2_gemm_tn(const q2_nvfp4* a, const q2_nvfp4* b, void* d, int d_dtype, int64_t ldd,
               int accumulate, void* stream);
/* accumulate (fp32 output only beyond Q2_ACC_STORE):
 *   Q2_ACC_STORE    D = A.B^T
 *   Q2_ACC_ADD      D += A.B^T (read-add-store; this launch is D's only writer)
 *   Q2_ACC_RED      D += A.B^T by red.global.add.v4.f32 (concurrent writers allowed)
 *   Q2_ACC_MULTIMEM d is an NVLS multicast address (cuMulticast / torch symmetric memory):
 *                   multimem.red.add.v4.f32 adds the tile into every member GPU's copy of D,
 *                   i.e. the data-parallel dW all-reduce fused into the wgrad epilogue
 *                   (replaces the dist.all_reduce after linear_graph.py:322-326).  The caller
 *                   zeroes D on every rank and barriers before, and barriers after, the launches.
 * Reductions flush fp32 subnormals (REDG .FTZ).                                              */
enum { Q2_ACC_STORE = 0, Q2_ACC_ADD = 1, Q2_ACC_RED = 2, Q2_ACC_MULTIMEM = 3 };

/* Helpers used by the host mirror: dequantize (quantizers.py:315-323) into
 * float64 [R, K]; unpack codes/scales into the reference's unpacked layout
 * (fp4 uint8 [R, K], scales8 uint8 [R, K/16]).                               */
int q2_dequant(const q2_nvfp4* t, double* out, void* stream);
int q2_unpack(const q2_nvfp4* t, uint8_t* fp4, uint8_t* scales8, void* stream);
int q2_pack(const uint8_t* fp4, const uint8_t* scales8, const q2_nvfp4* t, void* stream);

/* Chunked randomized Hadamard in literal float64: rht_apply (rht.py:144-155),
 * rht_inverse (:158-163) and hadamard_128 (:121-130).  x: n elements (BF16, F32
 * or F64), n % chunk == 0, chunk a power of two in [16, 2048].  Per chunk
 * out = FWHT(x * signs_pre) * scale * signs_post (either sign vector may be
 * NULL; chunk doubles of +-1), butterflies in the reference order
 * (_kernels.py:175-187), so out equals the reference bit for bit.  out: n f64.  */
int q2_rht(const void* x, int dtype, int64_t n, int chunk, const double* signs_pre, const double* signs_post,
           double scale, double* out, void* stream);

/* Element formats (formats.py:76-229) over n float64 inputs / uint8 codes:
 * op 0 encode_fp4_rtn, 1 encode_fp4_sr (u), 2 encode_fp8_rtn, 3 encode_fp8_sr (u),
 * 4 round_e8m3_rtn (vals_out; overflow sets Q2_ERR_E8M3_OVF in err),
 * 5 decode_fp4 (codes_in 0..15), 6 decode_fp8 (codes_in 0..255).
 * The caller has applied the reference's input checks (NaN, negative, grid max). */
int q2_formats(int op, const double* x, const double* u, const uint8_t* codes_in, int64_t n, uint8_t* codes_out,
               double* vals_out, uint32_t* err, void* stream);

/* EDEN correction factors (chunk_correction_factors, ms_eden.py:75-83): for each of
 * nchunks contiguous 128-element float64 chunks, S = sum(x_rot^2) / sum(x_rot*x_rtn)
 * in numpy's summation order, 1.0 when degenerate.  out: nchunks doubles.         */
int q2_eden_factors(const double* x_rot, const double* x_rtn, int64_t nchunks, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QUARTET2_H_ */
