// Forward NVFP4 quantizers: tensor absmax + Four-over-Six RTN (sm_100a).
//
// Restates quantize_rtn_46 / quantize_rtn (quantizers.py:164-234) with the
// same float64 decisions:
//   scale32 = (float)(absmax / scale_div)                       quantizers.py:221
//   s8_c    = E4M3_RTN(gmax / (scale32 * c))                    quantizers.py:227
//   codes   = ties-to-even RTN of v / (E4M3[s8_c] * scale32)    _kernels.py:101-127
//   keep c1 iff err(c1) < err(c0) (sequential float64 sums)     quantizers.py:184-203
// Codes are decided by exact threshold comparisons (the float64 quotient of a
// bf16/fp32 value decides exactly like the rational one), the 4/6 choice by
// the literal sequential float64 error sum.
#include "common.cuh"

namespace q2 {

struct Vec16 { float v[16]; };

__device__ __forceinline__ void load_vec8(const void* base, int dtype, int64_t off, float* out) {
  if (dtype == Q2_BF16) {
    uint4 raw = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + off));
    uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      out[2 * i] = bf16_to_f32(w[i] & 0xFFFFu);
      out[2 * i + 1] = bf16_to_f32(w[i] >> 16);
    }
  } else {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    float4 a = __ldg(p), b = __ldg(p + 1);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  }
}

__device__ __forceinline__ bool nonfinite(float f) {
  return (__float_as_uint(f) & 0x7F800000u) == 0x7F800000u;
}

// |x| max over a [R, K] view (K % 8 == 0), as float bits; flags non-finite.
__global__ void amax_kernel(const void* __restrict__ x, int dtype, int64_t R, int64_t K, int64_t ld,
                            uint32_t* __restrict__ amax_bits, uint32_t* __restrict__ err) {
  const int64_t per_row = K / 8, total = R * per_row;
  float m = 0.f;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / per_row, c = (i - r * per_row) * 8;
    float v[8];
    load_vec8(x, dtype, r * ld + c, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      bad |= nonfinite(v[k]);
      m = fmaxf(m, fabsf(v[k]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  bad = __any_sync(0xFFFFFFFFu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (m > 0.f) atomicMax(amax_bits, __float_as_uint(m));
    if (bad) atomic_or_err(err, Q2_ERR_NONFINITE);
  }
}

// One thread per 16-group.  ncaps in {1, 2}.
__global__ void __launch_bounds__(256) quant_fwd_kernel(
    const void* __restrict__ x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps,
    double cap0, double cap1, double scale_div, const uint32_t* __restrict__ amax_bits,
    uint8_t* __restrict__ codes, uint8_t* __restrict__ sf, float* __restrict__ scale32_out,
    uint32_t* __restrict__ err) {
  const int64_t gpr = K / GROUP, total = R * gpr, kb64 = kblocks64(K);
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const float amax = __uint_as_float(*amax_bits);
  const float scale32 = amax == 0.f ? 0.f : __double2float_rn(__ddiv_rn((double)amax, scale_div));
  if (gid == 0) *scale32_out = scale32;
  if (gid >= total) return;
  const int64_t r = gid / gpr, j = gid - r * gpr;
  uint8_t* cout = codes + r * (K / 2) + j * 8;
  uint8_t* sfout = sf + sf_offset(r, j, kb64);
  if (amax == 0.f) {                                          // quantizers.py:219-220
    *reinterpret_cast<uint2*>(cout) = make_uint2(0u, 0u);
    *sfout = 0;
    return;
  }
  float v[16];
  load_vec8(x, dtype, r * ld + j * GROUP, v);
  load_vec8(x, dtype, r * ld + j * GROUP + 8, v + 8);
  float gmax = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) gmax = fmaxf(gmax, fabsf(v[k]));

  const double s32 = (double)scale32;
  const double tq[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
  uint32_t best_s8 = 0, best_lo = 0, best_hi = 0;
  double best_err = 0.0;
  for (int b = 0; b < ncaps; ++b) {
    const double c = b == 0 ? cap0 : cap1;
    const double xq = __ddiv_rn((double)gmax, __dmul_rn(s32, c));
    if (isnan(xq)) atomic_or_err(err, Q2_ERR_NAN_SCALE);     // formats.py:167-168
    const uint32_t s8 = isnan(xq) ? 0u : e4m3_rtn(xq);
    const double d = __dmul_rn(e4m3_val(s8), s32);
    double T[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) T[t] = __dmul_rn(tq[t], d);
    uint32_t lo = 0, hi = 0;
    double e = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double a = fabs((double)v[k]);
      uint32_t mag = 0, neg = 0;
      if (d > 0.0) {
        mag = rtn_mag_thresholds(a, T);
        neg = signbit(v[k]) ? 1u : 0u;
      }
      const uint32_t code = mag | (neg << 3);
      if (k < 8) lo |= code << (4 * k); else hi |= code << (4 * (k - 8));
      if (ncaps > 1) {                                        // literal _nb_rtn error
        double dq = neg ? -fp4_val(mag) : fp4_val(mag);
        dq = d > 0.0 ? __dmul_rn(dq, d) : 0.0;
        const double diff = __dsub_rn(dq, (double)v[k]);
        e = __dadd_rn(e, __dmul_rn(diff, diff));
      }
    }
    if (b == 0 || e < best_err) {                             // ties keep caps[0]
      best_err = e; best_s8 = s8; best_lo = lo; best_hi = hi;
    }
  }
  *reinterpret_cast<uint2*>(cout) = make_uint2(best_lo, best_hi);
  *sfout = (uint8_t)best_s8;
}

}  // namespace q2

using namespace q2;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" size_t q2_sf_bytes(int64_t R, int64_t K) {
  return (size_t)((R + 127) / 128) * (size_t)kblocks64(K) * 512u;
}

extern "C" const char* q2_version(void) { return "quartet2-b200 sm_100a"; }

extern "C" int q2_amax(const void* x, int dtype, int64_t R, int64_t K, int64_t ld,
                       uint32_t* amax_bits, uint32_t* err, void* stream) {
  if (!x || R < 0 || K % 16 || ld < K || (dtype != Q2_BF16 && dtype != Q2_F32)) return Q2_EINVAL;
  const int esz = dtype == Q2_BF16 ? 2 : 4;
  if (!aligned16(x) || (ld * esz) % 16) return Q2_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t vecs = R * (K / 8);
  int blocks = (int)std::min<int64_t>((vecs + 255) / 256, 148 * 16);
  if (blocks < 1) blocks = 1;
  amax_kernel<<<blocks, 256, 0, s>>>(x, dtype, R, K, ld, amax_bits, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" size_t q2_quant_fwd_ws_bytes(void) { return 16; }

extern "C" int q2_quant_fwd(const void* x, int dtype, int64_t R, int64_t K, int64_t ld, int ncaps,
                            double cap0, double cap1, double scale_div, const q2_nvfp4* out,
                            void* ws, uint32_t* err, void* stream) {
  if (!out || !ws || (ncaps != 1 && ncaps != 2) || out->R != R || out->K != K) return Q2_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* amax = static_cast<uint32_t*>(ws);
  if (cudaMemsetAsync(amax, 0, 4, s) != cudaSuccess) return Q2_ECUDA;
  int rc = q2_amax(x, dtype, R, K, ld, amax, err, stream);
  if (rc) return rc;
  int64_t groups = R * (K / 16);
  int64_t blocks = (groups + 255) / 256;
  if (blocks < 1) blocks = 1;
  quant_fwd_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, dtype, R, K, ld, ncaps, cap0, cap1, scale_div,
                                                   amax, out->codes, out->sf, out->scale32, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}
