// Baseline-recipe quantizers (sm_100a): stochastic rounding quantize_sr /
// quantize_sr_46 (quantizers.py:139-161, :237-262) on bf16/fp32 rows, and the
// 16x16 square-block quantizer (quantizers.py:265-312) that emits W and W^T.  The rotated variant
// (sr_rht, linear_graph.py:259-274) is msed64_kernel<..., M64_SR> in msed.cu.
//
//   scale32 = (float)(absmax / scale_div)
//   s8_b    = E4M3_RTN(gmax / ((scale32 * cap_b) * margin))        float64, literal
//   code    = sr_elem(v, E4M3[s8_b] * scale32, u)                  _nb_sr
//   u       = prng_uniform(seed, stream_b, flat element index)
//   46: keep branch 1 iff its sequential float64 error is strictly lower.
// One thread per 16-group; every division is the literal IEEE float64 one, so
// codes and scales equal the reference's by construction.
#include "common.cuh"

namespace q2 {

template <int DT>
__global__ void __launch_bounds__(256) sr_quant_kernel(const void* __restrict__ x, int64_t R, int64_t K, int ncaps,
                                                       double cap0, double cap1, double margin, double scale_div,
                                                       const uint32_t* __restrict__ amax_bits, uint64_t head0,
                                                       uint64_t head1, uint8_t* __restrict__ codes,
                                                       uint8_t* __restrict__ sf, float* __restrict__ scale32_out,
                                                       uint32_t* __restrict__ err) {
  const float amax = __uint_as_float(*amax_bits);
  const float scale32 = amax == 0.f ? 0.f : __double2float_rn(__ddiv_rn((double)amax, scale_div));
  const int64_t gpr = K / GROUP, total = R * gpr, kpr = sf_kblocks(K);
  if (blockIdx.x == 0 && threadIdx.x == 0) *scale32_out = scale32;
  const double s32 = (double)scale32;
  bool clip = false;
  for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total; gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = gid / gpr, j = gid - r * gpr;
    float v[16];
    if (DT == Q2_BF16) {
      const uint4* p = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + gid * GROUP);
      const uint4 a = __ldg(p), b = __ldg(p + 1);
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) { v[2 * i] = __uint_as_float(w[i] << 16); v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u); }
    } else {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + gid * GROUP);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t = __ldg(p + i);
        v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
      }
    }
    uint32_t lo = 0, hi = 0, s8 = 0;
    if (amax != 0.f) {
      float gm = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) gm = fmaxf(gm, fabsf(v[i]));
      const double gmax = (double)gm;
      double best = 0.0;
      for (int b = 0; b < ncaps; ++b) {
        const double xq = __ddiv_rn(gmax, __dmul_rn(__dmul_rn(s32, b ? cap1 : cap0), margin));
        const uint32_t sb = e4m3_rtn(xq);
        const double d = __dmul_rn(e4m3_val(sb), s32);
        // non-clipping construction check (quantize_sr only, quantizers.py:153-157)
        if (ncaps == 1 && d > 0.0 && __ddiv_rn(gmax, d) > 6.0 * (1.0 + 1e-9)) clip = true;
        const uint64_t head = b ? head1 : head0;
        uint32_t l = 0, h = 0;
        double e = 0.0;
        for (int i = 0; i < 16; ++i) {
          const uint64_t u53 = mix64(head ^ ((uint64_t)(gid * GROUP + i) + GOLDEN)) >> 11;
          double dq;
          const uint32_t c = sr_elem((double)v[i], d, u53, &dq);
          if (i < 8) l |= c << (4 * i); else h |= c << (4 * (i - 8));
          const double df = __dsub_rn(dq, (double)v[i]);
          e = __dadd_rn(e, __dmul_rn(df, df));
        }
        if (b == 0 || e < best) { best = e; lo = l; hi = h; s8 = sb; }
      }
    }
    *reinterpret_cast<uint2*>(codes + gid * 8) = make_uint2(lo, hi);
    sf_store(sf, r, j, kpr, (uint8_t)s8);
  }
  if (clip) atomic_or_err(err, Q2_ERR_SR_CLIP);
}

// Square blocks: a warp covers two 16x16 blocks of one block row (lanes 0-15
// and 16-31, one row of 16 elements per lane).  Literal float64 divisions and
// codes (rtn_code_literal); the 4/6 error is numpy's sum(axis=(1, 3)) order:
// each row by the 8-accumulator pairwise rule, then the 16 rows in order (one
// 256-element pairwise sum when the tensor has a single block column).
__device__ __forceinline__ double pw16(const double (&q)[16]) {
  return ((__dadd_rn(q[0], q[8]) + __dadd_rn(q[1], q[9])) + (__dadd_rn(q[2], q[10]) + __dadd_rn(q[3], q[11]))) +
         ((__dadd_rn(q[4], q[12]) + __dadd_rn(q[5], q[13])) + (__dadd_rn(q[6], q[14]) + __dadd_rn(q[7], q[15])));
}

template <int DT>
__global__ void __launch_bounds__(256) sq_quant_kernel(const void* __restrict__ x, int64_t R, int64_t C, int use46,
                                                       const uint32_t* __restrict__ amax_bits,
                                                       uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                       float* __restrict__ scale_out, uint8_t* __restrict__ codes_t,
                                                       uint8_t* __restrict__ sf_t, float* __restrict__ scale_t_out,
                                                       uint8_t* __restrict__ s8c) {
  const float amax = __uint_as_float(*amax_bits);
  const float scale32 = amax == 0.f ? 0.f : __double2float_rn(__ddiv_rn((double)amax, 6.0 * 256.0));
  if (blockIdx.x == 0 && threadIdx.x == 0) { *scale_out = scale32; *scale_t_out = scale32; }
  const double s32 = (double)scale32;
  const int lane = threadIdx.x & 31, half = lane >> 4, a = lane & 15;
  const int64_t CB = C / GROUP, RB = R / GROUP, pairs = (CB + 1) / 2, tasks = RB * pairs;
  const int64_t kb = sf_kblocks(C), kbt = sf_kblocks(R);
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t task = wid; task < tasks; task += nw) {
    const int64_t rb = task / pairs, cb = (task - rb * pairs) * 2 + half, r = rb * GROUP + a;
    const bool live = cb < CB;
    double v[16];
    float gm = 0.f;
    if (live) {
      if (DT == Q2_BF16) {
        const uint4* p = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + r * C + cb * GROUP);
        const uint4 u0 = __ldg(p), u1 = __ldg(p + 1);
        const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[2 * i] = (double)__uint_as_float(w[i] << 16);
          v[2 * i + 1] = (double)__uint_as_float(w[i] & 0xFFFF0000u);
        }
      } else {
        const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + r * C + cb * GROUP);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 t = __ldg(p + i);
          v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) gm = fmaxf(gm, fabsf((float)v[i]));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.0;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xFFFFFFFFu, gm, o));
    const double bmax = (double)gm;
    uint32_t lo = 0, hi = 0, s8 = 0;
    double best = 0.0;
    for (int b = 0; b < (use46 ? 2 : 1); ++b) {
      const uint32_t sb = amax == 0.f ? 0u : e4m3_rtn(__ddiv_rn(bmax, __dmul_rn(s32, b ? 4.0 : 6.0)));
      const double d = __dmul_rn(e4m3_val(sb), s32);
      uint32_t l = 0, h = 0;
      double sq[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t c = rtn_code_literal(v[i], d);
        if (i < 8) l |= c << (4 * i); else h |= c << (4 * (i - 8));
        // deq = copysign(r/2, q) * d (quantizers.py:296); q = v/d or +0
        const bool neg = d > 0.0 && signbit(v[i]);
        const double m = fp4_val(c & 7u);
        const double dq = d > 0.0 ? __dmul_rn(neg ? -m : m, d) : 0.0;
        const double df = __dsub_rn(dq, v[i]);
        sq[i] = __dmul_rn(df, df);
      }
      double e = 0.0;
      if (use46) {
        if (CB == 1) {                                        // one block column: flat pairwise 256
          double hs[2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            double acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0;
            for (int rr = 0; rr < 8; ++rr) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                acc[j] = __dadd_rn(acc[j], __shfl_sync(0xFFFFFFFFu, sq[j], 8 * hh + rr));
                acc[j] = __dadd_rn(acc[j], __shfl_sync(0xFFFFFFFFu, sq[j + 8], 8 * hh + rr));
              }
            }
            hs[hh] = (__dadd_rn(acc[0], acc[1]) + __dadd_rn(acc[2], acc[3])) +
                     (__dadd_rn(acc[4], acc[5]) + __dadd_rn(acc[6], acc[7]));
          }
          e = __dadd_rn(hs[0], hs[1]);
        } else {
          const double er = pw16(sq);
          for (int rr = 0; rr < 16; ++rr) e = __dadd_rn(e, __shfl_sync(0xFFFFFFFFu, er, 16 * half + rr));
        }
      }
      if (b == 0 || e < best) { best = e; lo = l; hi = h; s8 = sb; }
    }
    // transposed codes: W^T row cb*16 + i, element r; even rows pack the byte
    const uint32_t plo = __shfl_xor_sync(0xFFFFFFFFu, lo, 1), phi = __shfl_xor_sync(0xFFFFFFFFu, hi, 1);
    if (!live) continue;
    *reinterpret_cast<uint2*>(codes + r * (C / 2) + cb * 8) = make_uint2(lo, hi);
    sf_store(sf, r, cb, kb, (uint8_t)s8);
    sf_store(sf_t, cb * GROUP + a, rb, kbt, (uint8_t)s8);
    if (a == 0) s8c[rb * CB + cb] = (uint8_t)s8;
    if ((a & 1) == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t c0 = ((i < 8 ? lo : hi) >> (4 * (i & 7))) & 0xFu, c1 = ((i < 8 ? plo : phi) >> (4 * (i & 7))) & 0xFu;
        codes_t[(cb * GROUP + i) * (R / 2) + r / 2] = (uint8_t)(c0 | (c1 << 4));
      }
    }
  }
}

}  // namespace q2

using namespace q2;

extern "C" size_t q2_quant_sr_ws_bytes(void) { return 16; }

extern "C" int q2_quant_sr(const void* x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps, double cap0,
                           double cap1, double margin, double scale_div, uint64_t seed, uint64_t stream0,
                           uint64_t stream1, const q2_nvfp4* out, void* ws, uint32_t* err, void* stream) {
  if (!out || !ws || (ncaps != 1 && ncaps != 2) || out->R != R || out->K != K || R < 0 || K % 16 || ld != K)
    return Q2_EINVAL;
  if (dtype != Q2_BF16 && dtype != Q2_F32) return Q2_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (R == 0 || K == 0)                                   // empty tensor: the zero tensor (quantizers.py:147-149)
    return cudaMemsetAsync(out->scale32, 0, 4, s) == cudaSuccess ? Q2_OK : Q2_ECUDA;
  if (!x || (reinterpret_cast<uintptr_t>(x) & 31u)) return Q2_EINVAL;
  uint32_t* amax = static_cast<uint32_t*>(ws);
  if (cudaMemsetAsync(amax, 0, 4, s) != cudaSuccess) return Q2_ECUDA;
  int rc = q2_amax(x, dtype, R, K, ld, amax, err, stream);
  if (rc) return rc;
  const int64_t groups = R * (K / 16);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((groups + 255) / 256, 148 * 16));
  const uint64_t h0 = prng_head(seed, stream0), h1 = prng_head(seed, stream1);
  count_launch();
  if (dtype == Q2_BF16)
    sr_quant_kernel<Q2_BF16><<<blocks, 256, 0, s>>>(x, R, K, ncaps, cap0, cap1, margin, scale_div, amax, h0, h1,
                                                    out->codes, out->sf, out->scale32, err);
  else
    sr_quant_kernel<Q2_F32><<<blocks, 256, 0, s>>>(x, R, K, ncaps, cap0, cap1, margin, scale_div, amax, h0, h1,
                                                   out->codes, out->sf, out->scale32, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_quant_square_block(const void* x, int dtype, int64_t R, int64_t C, int use46, const q2_nvfp4* out,
                                     const q2_nvfp4* out_t, uint8_t* scales8, void* ws, uint32_t* err, void* stream) {
  if (!x || !out || !out_t || !scales8 || !ws || R % 16 || C % 16 || R < 0 || C < 0) return Q2_EINVAL;
  if (out->R != R || out->K != C || out_t->R != C || out_t->K != R) return Q2_EINVAL;
  if (dtype != Q2_BF16 && dtype != Q2_F32) return Q2_EINVAL;
  if (reinterpret_cast<uintptr_t>(x) & 31u) return Q2_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* amax = static_cast<uint32_t*>(ws);
  if (cudaMemsetAsync(amax, 0, 4, s) != cudaSuccess) return Q2_ECUDA;
  if (R == 0 || C == 0) {
    if (cudaMemsetAsync(out->scale32, 0, 4, s) != cudaSuccess || cudaMemsetAsync(out_t->scale32, 0, 4, s) != cudaSuccess)
      return Q2_ECUDA;
    return Q2_OK;
  }
  int rc = q2_amax(x, dtype, R, C, C, amax, err, stream);
  if (rc) return rc;
  const int64_t tasks = (R / 16) * ((C / 16 + 1) / 2);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tasks + 7) / 8, 148 * 16));
  count_launch();
  if (dtype == Q2_BF16)
    sq_quant_kernel<Q2_BF16><<<blocks, 256, 0, s>>>(x, R, C, use46, amax, out->codes, out->sf, out->scale32,
                                                    out_t->codes, out_t->sf, out_t->scale32, scales8);
  else
    sq_quant_kernel<Q2_F32><<<blocks, 256, 0, s>>>(x, R, C, use46, amax, out->codes, out->sf, out->scale32,
                                                   out_t->codes, out_t->sf, out_t->scale32, scales8);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}
