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

// Chunked randomized Hadamard in literal float64 (rht_apply / rht_inverse /
// hadamard_128, rht.py:121-163; butterflies _kernels.py:175-187): per chunk,
// out = FWHT(x * pre) * c * post, stages h = 1, 2, ..., chunk/2, every output one
// IEEE op (a + b or a - b) of two stage inputs, so the bits equal the reference's.
// A block transforms a tile of 2 * blockDim.x elements (whole chunks) in shared
// memory; each thread owns one butterfly pair per stage.
template <int DT>
__global__ void rht_kernel(const void* __restrict__ x, int64_t total, int chunk, const double* __restrict__ pre,
                           const double* __restrict__ post, double c, double* __restrict__ out) {
  extern __shared__ double tile_sh[];
  const int tile = 2 * blockDim.x;
  const int64_t base = (int64_t)blockIdx.x * tile;
  for (int i = threadIdx.x; i < tile; i += blockDim.x) {
    const int64_t g = base + i;
    double v = 0.0;
    if (g < total)
      v = DT == Q2_BF16 ? (double)bf16_to_f32(static_cast<const uint16_t*>(x)[g])
          : DT == Q2_F32 ? (double)static_cast<const float*>(x)[g]
                         : static_cast<const double*>(x)[g];
    if (pre) v = __dmul_rn(v, pre[i & (chunk - 1)]);
    tile_sh[i] = v;
  }
  __syncthreads();
  const int t = threadIdx.x;
  for (int h = 1; h < chunk; h <<= 1) {
    const int i = (t / h) * 2 * h + (t % h), j = i + h;
    const double a = tile_sh[i], b = tile_sh[j];
    tile_sh[i] = __dadd_rn(a, b);
    tile_sh[j] = __dsub_rn(a, b);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < tile; i += blockDim.x) {
    const int64_t g = base + i;
    if (g >= total) continue;
    double v = __dmul_rn(tile_sh[i], c);
    if (post) v = __dmul_rn(v, post[i & (chunk - 1)]);
    out[g] = v;
  }
}

// Element formats (formats.py:85-229) as one elementwise kernel over float64
// inputs; every op is the device helper the quantizers use (common.cuh), so the
// standalone encoders equal the fused ones.  Input checks the reference raises
// for (NaN, negative, above the grid) are done by the host wrapper before launch.
enum { FMT_FP4_RTN = 0, FMT_FP4_SR = 1, FMT_FP8_RTN = 2, FMT_FP8_SR = 3, FMT_E8M3 = 4, FMT_DEC_FP4 = 5,
       FMT_DEC_FP8 = 6 };

__device__ __forceinline__ uint32_t fp4_code_of_doubled(double r) {  // doubled grid 0,1,2,3,4,6,8,12 -> 0..7
  const uint32_t ri = (uint32_t)r;
  return ri <= 4u ? ri : (ri == 6u ? 5u : (ri == 8u ? 6u : 7u));
}

__global__ void formats_kernel(int op, const double* __restrict__ x, const double* __restrict__ u,
                               const uint8_t* __restrict__ cin, int64_t n, uint8_t* __restrict__ cout,
                               double* __restrict__ vout, uint32_t* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    switch (op) {
      case FMT_FP4_RTN:                                                   // formats.py:116-124
        cout[i] = (uint8_t)rtn_code_literal(x[i], 1.0);
        break;
      case FMT_FP4_SR: {                                                  // formats.py:127-157
        const double v = x[i], a2 = fmin(fabs(v) * 2.0, 12.0);
        const double lo = a2 < 4.0 ? floor(a2) : (a2 < 8.0 ? 2.0 * floor(a2 * 0.5) : 4.0 * floor(a2 * 0.25));
        const double step = lo < 4.0 ? 1.0 : (lo < 8.0 ? 2.0 : 4.0);
        const double p = __ddiv_rn(__dsub_rn(a2, lo), step);
        const double r = u[i] < p ? lo + step : lo;
        cout[i] = (uint8_t)(fp4_code_of_doubled(r) | (signbit(v) ? 8u : 0u));
        break;
      }
      case FMT_FP8_RTN:                                                   // formats.py:160-171
        cout[i] = (uint8_t)e4m3_rtn(x[i]);
        break;
      case FMT_FP8_SR:                                                    // formats.py:174-201
        cout[i] = (uint8_t)e4m3_sr(x[i], u[i]);
        break;
      case FMT_E8M3: {                                                    // formats.py:204-229
        bool ovf = false;
        vout[i] = e8m3_rtn(x[i], &ovf);
        if (ovf) atomic_or_err(err, Q2_ERR_E8M3_OVF);
        break;
      }
      case FMT_DEC_FP4:                                                   // formats.py:76-78
        vout[i] = fp4_val(cin[i]);
        break;
      default: {                                                          // FMT_DEC_FP8, formats.py:81-83
        const uint32_t c = cin[i];
        double v = (c & 0x7Fu) == 0x7Fu ? __longlong_as_double(0x7FF8000000000000ll) : e4m3_val(c & 0x7Fu);
        vout[i] = (c & 0x80u) ? -v : v;
      }
    }
  }
}

// EDEN correction factors per 128-chunk (chunk_correction_factors,
// ms_eden.py:75-83): num = sum(x_rot^2), den = sum(x_rot * x_rtn) with the
// products materialised and summed in numpy's order for a contiguous 128-row
// (8 strided accumulators, sequential; then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// SURVEY §8(c) E7); S = num/den unless num == 0 or |den| < 1e-30 num.  One thread
// per chunk (an API helper; the quantizers fuse this step).
__device__ __forceinline__ double np_sum128_products(const double* a, const double* b) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(a[j], b[j]);
  for (int k = 1; k < 16; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(a[8 * k + j], b[8 * k + j]));
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

__global__ void eden_factor_kernel(const double* __restrict__ xr, const double* __restrict__ xq, int64_t nchunks,
                                   double* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const double* a = xr + c * 128;
  const double num = np_sum128_products(a, a), den = np_sum128_products(a, xq + c * 128);
  const bool good = fabs(den) >= 1e-30 * num && num > 0.0;
  out[c] = good ? __ddiv_rn(num, den) : 1.0;
}

}  // namespace q2

using namespace q2;

extern "C" int q2_eden_factors(const double* x_rot, const double* x_rtn, int64_t nchunks, double* out, void* stream) {
  if (nchunks < 0) return Q2_EINVAL;
  if (nchunks == 0) return Q2_OK;
  if (!x_rot || !x_rtn || !out) return Q2_EINVAL;
  count_launch();
  eden_factor_kernel<<<(unsigned)((nchunks + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(x_rot, x_rtn,
                                                                                                      nchunks, out);
  return cudaGetLastError() == cudaSuccess ? Q2_OK : Q2_ECUDA;
}

extern "C" int q2_formats(int op, const double* x, const double* u, const uint8_t* codes_in, int64_t n,
                          uint8_t* codes_out, double* vals_out, uint32_t* err, void* stream) {
  if (op < FMT_FP4_RTN || op > FMT_DEC_FP8 || n < 0) return Q2_EINVAL;
  if (n == 0) return Q2_OK;
  const bool decode = op >= FMT_DEC_FP4, vals = decode || op == FMT_E8M3;
  if ((decode ? !codes_in : !x) || (vals ? !vals_out : !codes_out) || ((op == FMT_FP4_SR || op == FMT_FP8_SR) && !u) ||
      (op == FMT_E8M3 && !err))
    return Q2_EINVAL;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  count_launch();
  formats_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(op, x, u, codes_in, n, codes_out, vals_out,
                                                                        err);
  return cudaGetLastError() == cudaSuccess ? Q2_OK : Q2_ECUDA;
}

extern "C" int q2_rht(const void* x, int dtype, int64_t n, int chunk, const double* signs_pre,
                      const double* signs_post, double scale, double* out, void* stream) {
  if (chunk < 16 || (chunk & (chunk - 1)) || chunk > 2048 || n % chunk) return Q2_EINVAL;
  if (n == 0) return Q2_OK;
  if (!x || !out || (dtype != Q2_BF16 && dtype != Q2_F32 && dtype != Q2_F64)) return Q2_EINVAL;
  const int tile = std::max(chunk, 512), threads = tile / 2;
  const unsigned blocks = (unsigned)((n + tile - 1) / tile);
  const size_t smem = (size_t)tile * sizeof(double);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    count_launch();
    kern<<<blocks, threads, smem, s>>>(x, n, chunk, signs_pre, signs_post, scale, out);
  };
  if (dtype == Q2_BF16) launch(rht_kernel<Q2_BF16>);
  else if (dtype == Q2_F32) launch(rht_kernel<Q2_F32>);
  else launch(rht_kernel<Q2_F64>);
  return cudaGetLastError() == cudaSuccess ? Q2_OK : Q2_ECUDA;
}

static unsigned nblocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

extern "C" int q2_dequant(const q2_nvfp4* t, double* out, void* stream) {
  if (!t || !out || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  count_launch();
  dequant_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(t->codes, t->sf, t->scale32, t->R, t->K, out);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_unpack(const q2_nvfp4* t, uint8_t* fp4, uint8_t* scales8, void* stream) {
  if (!t || !fp4 || !scales8 || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  count_launch();
  unpack_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(t->codes, t->sf, t->R, t->K, fp4, scales8);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_pack(const uint8_t* fp4, const uint8_t* scales8, const q2_nvfp4* t, void* stream) {
  if (!t || !fp4 || !scales8 || t->K % 16) return Q2_EINVAL;
  int64_t n = t->R * (t->K / 16);
  if (n == 0) return Q2_OK;
  count_launch();
  pack_kernel<<<nblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(fp4, scales8, t->R, t->K, t->codes, t->sf);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

// Kernel launches issued by the library since load (or since the last reset).
extern "C" unsigned long long q2_launch_count(int reset) {
  const unsigned long long n = __atomic_load_n(&q2::launch_counter(), __ATOMIC_RELAXED);
  if (reset) __atomic_store_n(&q2::launch_counter(), 0ull, __ATOMIC_RELAXED);
  return n;
}
