// Layout helpers for the host mirror: dequantize (quantizers.py:315-323) and
// conversion between the packed/swizzled HBM form and the reference's
// unpacked NVFP4Tensor arrays (quantizers.py:83-98).
#include "common.cuh"

namespace q2 {

// one thread per 16-group
__global__ void dequant_kernel(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ sf,
                               const float* __restrict__ scale32, int64_t R, int64_t K, double* __restrict__ out) {
  const int64_t gpr = K / GROUP, g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= R * gpr) return;
  const int64_t r = g / gpr, j = g - r * gpr;
  const double d = __dmul_rn(e4m3_val(sf[sf_offset(r, j, sf_kblocks(K))]), (double)*scale32);
  const uint2 c = *reinterpret_cast<const uint2*>(codes + r * (K / 2) + j * 8);
  double* o = out + r * K + j * GROUP;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    uint32_t code = ((k < 8 ? c.x : c.y) >> (4 * (k & 7))) & 0xF;
    o[k] = __dmul_rn(fp4_val(code), d);
  }
}

__global__ void unpack_kernel(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ sf, int64_t R, int64_t K,
                              uint8_t* __restrict__ fp4, uint8_t* __restrict__ s8) {
  const int64_t gpr = K / GROUP, g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= R * gpr) return;
  const int64_t r = g / gpr, j = g - r * gpr;
  s8[g] = sf[sf_offset(r, j, sf_kblocks(K))];
  const uint2 c = *reinterpret_cast<const uint2*>(codes + r * (K / 2) + j * 8);
#pragma unroll
  for (int k = 0; k < 16; ++k) fp4[r * K + j * GROUP + k] = ((k < 8 ? c.x : c.y) >> (4 * (k & 7))) & 0xF;
}

__global__ void pack_kernel(const uint8_t* __restrict__ fp4, const uint8_t* __restrict__ s8, int64_t R, int64_t K,
                            uint8_t* __restrict__ codes, uint8_t* __restrict__ sf) {
  const int64_t gpr = K / GROUP, g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= R * gpr) return;
  const int64_t r = g / gpr, j = g - r * gpr;
  sf_store(sf, r, j, sf_kblocks(K), s8[g]);
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    uint32_t v = fp4[r * K + j * GROUP + k] & 0xF;
    if (k < 8) lo |= v << (4 * k); else hi |= v << (4 * (k - 8));
  }
  *reinterpret_cast<uint2*>(codes + r * (K / 2) + j * 8) = make_uint2(lo, hi);
}

}  // namespace q2

using namespace q2;

static unsigned nblocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

extern "C" int q2_dequant(const q2_nvfp4* t, double* out, void* stream) {
  if (!t || !out || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  dequant_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(t->codes, t->sf, t->scale32, t->R, t->K, out);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_unpack(const q2_nvfp4* t, uint8_t* fp4, uint8_t* scales8, void* stream) {
  if (!t || !fp4 || !scales8 || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  unpack_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(t->codes, t->sf, t->R, t->K, fp4, scales8);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_pack(const uint8_t* fp4, const uint8_t* scales8, const q2_nvfp4* t, void* stream) {
  if (!t || !fp4 || !scales8 || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  pack_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(fp4, scales8, t->R, t->K, t->codes, t->sf);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}
