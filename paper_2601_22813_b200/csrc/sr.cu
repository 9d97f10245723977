// Stochastic-rounding NVFP4 baselines (sm_100a): quantize_sr / quantize_sr_46
// (quantizers.py:139-161, :237-262) on bf16/fp32 rows.  The rotated variant
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

}  // namespace q2

using namespace q2;

extern "C" size_t q2_quant_sr_ws_bytes(void) { return 16; }

extern "C" int q2_quant_sr(const void* x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps, double cap0,
                           double cap1, double margin, double scale_div, uint64_t seed, uint64_t stream0,
                           uint64_t stream1, const q2_nvfp4* out, void* ws, uint32_t* err, void* stream) {
  if (!x || !out || !ws || (ncaps != 1 && ncaps != 2) || out->R != R || out->K != K || R < 0 || K % 16 || ld != K)
    return Q2_EINVAL;
  if (dtype != Q2_BF16 && dtype != Q2_F32) return Q2_EINVAL;
  if (reinterpret_cast<uintptr_t>(x) & 31u) return Q2_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* amax = static_cast<uint32_t*>(ws);
  if (cudaMemsetAsync(amax, 0, 4, s) != cudaSuccess) return Q2_ECUDA;
  if (R == 0) return cudaMemsetAsync(out->scale32, 0, 4, s) == cudaSuccess ? Q2_OK : Q2_ECUDA;
  int rc = q2_amax(x, dtype, R, K, ld, amax, err, stream);
  if (rc) return rc;
  const int64_t groups = R * (K / 16);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((groups + 255) / 256, 148 * 16));
  const uint64_t h0 = prng_head(seed, stream0), h1 = prng_head(seed, stream1);
  if (dtype == Q2_BF16)
    sr_quant_kernel<Q2_BF16><<<blocks, 256, 0, s>>>(x, R, K, ncaps, cap0, cap1, margin, scale_div, amax, h0, h1,
                                                    out->codes, out->sf, out->scale32, err);
  else
    sr_quant_kernel<Q2_F32><<<blocks, 256, 0, s>>>(x, R, K, ncaps, cap0, cap1, margin, scale_div, amax, h0, h1,
                                                   out->codes, out->sf, out->scale32, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}
