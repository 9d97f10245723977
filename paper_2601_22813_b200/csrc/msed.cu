// MS-EDEN backward quantizer: randomized 128-Hadamard rotation fused with
// clipping RTN, the per-chunk EDEN correction factor and stochastic rounding
// of the E4M3 group scales (sm_100a).
//
// Restates ms_eden_quantize (ms_eden.py:116-153), its pow2 variant
// (ms_eden.py:86-113) and the post-hoc two-pass schedule pass1/pass2
// (posthoc.py:74-125).  One warp owns one (row, 128-chunk) unit; lane l holds
// elements 4l..4l+3.  A CTA stages a 64-row x 128-column tile of the logical
// tensor in shared memory, so row sources, transposed bf16 sources (E^T) and
// transposed NVFP4 tape sources (W^T, X^T) share the same compute path.
//
// The rotation is the literal float64 butterfly network of _nb_fwht
// (_kernels.py:175-187): every output of every stage is one IEEE add/sub of
// two stage inputs, so the result does not depend on which lane computes it.
#include <cuda_fp16.h>
#include "tc_common.cuh"

namespace q2 {

constexpr int TILE_ROWS = 64;
constexpr int TILE_LD = CHUNK + 4;   // floats per staged row
constexpr int MSED_THREADS = 256;

enum Pass { PASS_ABSMAX = 0, PASS_PMAX = 1, PASS_QUANT = 2, PASS_POSTHOC1 = 3 };

struct MsedArgs {
  const void* x; int dtype;
  const uint8_t* tape_codes; const uint8_t* tape_sf; const float* tape_scale32; int64_t tape_K;
  int64_t R, K, ld;
  uint32_t sign[4];
  double s, inv_sqrt;
  uint64_t sr_head;
  int pow2;                          // PASS_QUANT: scale32 from pmax (pow2) or absmax
  uint8_t* codes; uint8_t* sf; float* scale32;
  uint16_t* pseudo; double* corr;
  unsigned long long* red;           // [0] rotated absmax (f64 bits), [1] pseudo max (f64 bits)
  uint32_t* err;
};

// ------------------------------------------------------------ tile loads ----
template <int SRC>
__device__ __forceinline__ void load_tile(const MsedArgs& a, int64_t r0, int64_t c, float* tile,
                                          bool& bad) {
  const int t = threadIdx.x;
  if (SRC == Q2_SRC_ROWS) {
    // 64 rows x 16 vectors of 8 along K
    for (int v = t; v < TILE_ROWS * 16; v += MSED_THREADS) {
      int rr = v >> 4, kk = (v & 15) * 8;
      float vals[8];
      if (r0 + rr < a.R) {
        int64_t off = (r0 + rr) * a.ld + c * CHUNK + kk;
        if (a.dtype == Q2_BF16) {
          uint4 raw = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + off));
          uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) { vals[2 * i] = bf16_to_f32(w[i] & 0xFFFF); vals[2 * i + 1] = bf16_to_f32(w[i] >> 16); }
        } else {
          const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + off);
          float4 u = __ldg(p), w = __ldg(p + 1);
          vals[0] = u.x; vals[1] = u.y; vals[2] = u.z; vals[3] = u.w;
          vals[4] = w.x; vals[5] = w.y; vals[6] = w.z; vals[7] = w.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) vals[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bad |= (__float_as_uint(vals[i]) & 0x7F800000u) == 0x7F800000u;
        tile[rr * TILE_LD + kk + i] = vals[i];
      }
    }
  } else if (SRC == Q2_SRC_COLS) {
    // source [K, R] row-major: 128 source rows (k) x 64 source columns (rows of the tile)
    for (int v = t; v < CHUNK * 8; v += MSED_THREADS) {
      int kk = v >> 3, cc = (v & 7) * 8;
      float vals[8];
      if (r0 + cc < a.R) {
        int64_t off = (c * CHUNK + kk) * a.ld + r0 + cc;
        if (a.dtype == Q2_BF16) {
          uint4 raw = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + off));
          uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) { vals[2 * i] = bf16_to_f32(w[i] & 0xFFFF); vals[2 * i + 1] = bf16_to_f32(w[i] >> 16); }
        } else {
          const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + off);
          float4 u = __ldg(p), w = __ldg(p + 1);
          vals[0] = u.x; vals[1] = u.y; vals[2] = u.z; vals[3] = u.w;
          vals[4] = w.x; vals[5] = w.y; vals[6] = w.z; vals[7] = w.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) vals[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bad |= (__float_as_uint(vals[i]) & 0x7F800000u) == 0x7F800000u;
        tile[(cc + i) * TILE_LD + kk] = vals[i];
      }
    }
  } else {
    // NVFP4 tape of logical shape [K, R]: 128 tape rows x 64 tape columns
    // (32 code bytes + one 4-scale word per tape row).  Stores FP4*E4M3
    // (exact in fp32); the fp32 tensor scale is applied in float64 later.
    for (int v = t; v < CHUNK * 2; v += MSED_THREADS) {
      int kk = v >> 1, half = v & 1;
      int64_t trow = c * CHUNK + kk;
      int64_t tcol = r0 + half * 32;
      if (tcol >= a.R) {
        for (int i = 0; i < 32; ++i) tile[(half * 32 + i) * TILE_LD + kk] = 0.f;
        continue;
      }
      uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.tape_codes + trow * (a.R / 2) + tcol / 2));
      uint32_t sfw = __ldg(reinterpret_cast<const uint32_t*>(
          a.tape_sf + sf_offset(trow, r0 / 16, kpairs(a.R))));
      uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        uint32_t code = (w[i >> 3] >> (4 * (i & 7))) & 0xF;
        uint32_t s8 = (sfw >> (8 * (half * 2 + (i >> 4)))) & 0xFF;
        tile[(half * 32 + i) * TILE_LD + kk] = fp4_valf(code) * (float)e4m3_val(s8);
      }
    }
  }
}

// ------------------------------------------------------------ warp math -----
__device__ __forceinline__ void fwht_f64(double (&y)[4], int lane) {
  // h = 1, 2 inside the lane
  double a0 = __dadd_rn(y[0], y[1]), a1 = __dsub_rn(y[0], y[1]);
  double a2 = __dadd_rn(y[2], y[3]), a3 = __dsub_rn(y[2], y[3]);
  y[0] = __dadd_rn(a0, a2); y[2] = __dsub_rn(a0, a2);
  y[1] = __dadd_rn(a1, a3); y[3] = __dsub_rn(a1, a3);
  // h = 4 .. 64 across lanes (partner = lane ^ h/4)
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool top = (lane & m) == 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double o = __shfl_xor_sync(0xFFFFFFFFu, y[i], m);
      y[i] = top ? __dadd_rn(y[i], o) : __dsub_rn(o, y[i]);
    }
  }
}

__device__ __forceinline__ double group_max4(double v) {     // over lanes {4g..4g+3}
  v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, 1));
  return fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, 2));
}

// numpy's pairwise .sum over 128 contiguous float64 (8 strided accumulators,
// then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))) — ms_eden.py:79-80 on numpy 2.3.
// p: per-warp shared scratch holding the 128 products.
__device__ __forceinline__ double numpy_sum128(const double* p, int lane) {
  const int j = lane & 7;
  double acc = p[j];
#pragma unroll
  for (int k = 1; k < 16; ++k) acc = __dadd_rn(acc, p[8 * k + j]);
  double o = __shfl_xor_sync(0xFFFFFFFFu, acc, 1); acc = __dadd_rn(acc, o);
  o = __shfl_xor_sync(0xFFFFFFFFu, acc, 2); acc = __dadd_rn(acc, o);
  o = __shfl_xor_sync(0xFFFFFFFFu, acc, 4); acc = __dadd_rn(acc, o);
  return __shfl_sync(0xFFFFFFFFu, acc, 0);
}

__device__ __forceinline__ double ulong_as_double(unsigned long long b) { return __longlong_as_double((long long)b); }

// scale32 of the exact / pow2 single-pass constructions (quantizers.py:177, ms_eden.py:104-106)
__device__ __forceinline__ float msed_scale32(const MsedArgs& a) {
  double amax = ulong_as_double(a.red[0]);
  if (amax == 0.0) return 0.f;                                   // _zero_like
  if (a.pow2) {
    double pmax = ulong_as_double(a.red[1]);
    if (pmax <= 0.0) return 1.f;                                 // ms_eden.py:88-89: k = 0
    int e; double m = frexp(pmax / 256.0, &e);
    int k = (m == 0.5) ? e - 1 : e;
    return (float)ldexp(1.0, k);
  }
  return __double2float_rn(__ddiv_rn(amax, __dmul_rn(a.s, 256.0)));
}

template <int SRC, int PASS>
__global__ void __launch_bounds__(MSED_THREADS) msed_kernel(MsedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  double* scratch = reinterpret_cast<double*>(smem_raw + TILE_ROWS * TILE_LD * sizeof(float));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * TILE_ROWS, c = blockIdx.y;
  const int64_t gpr = a.K / GROUP, kpr = kpairs(a.K);

  bool bad = false;
  load_tile<SRC>(a, r0, c, tile, bad);
  if (PASS == PASS_ABSMAX || PASS == PASS_PMAX || PASS == PASS_POSTHOC1) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomic_or_err(a.err, Q2_ERR_NONFINITE);
  } else {
    __syncthreads();
  }
  const double tape_s = SRC == Q2_SRC_TAPE_COLS ? (double)*a.tape_scale32 : 1.0;
  const float scale32 = PASS == PASS_QUANT ? msed_scale32(a) : 0.f;
  if (PASS == PASS_QUANT && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.scale32 = scale32;

  double wmax = 0.0, pmx = 0.0;
  bool ovf = false;
  const bool zero = PASS == PASS_QUANT && ulong_as_double(a.red[0]) == 0.0;
  double* pn = scratch + warp * 256;
  double* pd = pn + 128;
  for (int u = 0; u < TILE_ROWS / 8; ++u) {
    const int rr = warp * (TILE_ROWS / 8) + u;
    const int64_t r = r0 + rr;
    if (r >= a.R) break;
    double y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double v = (double)tile[rr * TILE_LD + 4 * lane + i];
      if (SRC == Q2_SRC_TAPE_COLS) v = __dmul_rn(v, tape_s);   // fl64(FP4*E4M3*scale32), exact
      const int e = 4 * lane + i;
      y[i] = ((a.sign[e >> 5] >> (e & 31)) & 1u) ? -v : v;
    }
    fwht_f64(y, lane);
#pragma unroll
    for (int i = 0; i < 4; ++i) y[i] = __dmul_rn(y[i], a.inv_sqrt);   // rht.py:154

    double lmax = fmax(fmax(fabs(y[0]), fabs(y[1])), fmax(fabs(y[2]), fabs(y[3])));
    const double gmax = group_max4(lmax);
    const int64_t g = r * gpr + c * 8 + (lane >> 2);            // flat group index (ms_eden.py:150)
    if (PASS == PASS_ABSMAX) { wmax = fmax(wmax, lmax); continue; }
    if (PASS == PASS_PMAX) {
      wmax = fmax(wmax, lmax);
      pmx = fmax(pmx, e8m3_rtn(__ddiv_rn(gmax, a.s), &ovf));
      continue;
    }
    if (zero) {                                                  // quantizers.py:175-176
      *reinterpret_cast<uint16_t*>(a.codes + r * (a.K / 2) + c * 64 + 2 * lane) = 0;
      if ((lane & 3) == 0) sf_store(a.sf, r, c * 8 + (lane >> 2), kpr, 0);
      continue;
    }
    double d;
    uint32_t s8 = 0;
    if (PASS == PASS_QUANT) {
      double xq = __ddiv_rn(gmax, __dmul_rn((double)scale32, a.s));
      if (isnan(xq)) { atomic_or_err(a.err, Q2_ERR_NAN_SCALE); xq = 0.0; }
      s8 = e4m3_rtn(xq);
      d = __dmul_rn(e4m3_val(s8), (double)scale32);
    } else {                                                     // posthoc pass 1 (posthoc.py:83)
      d = e8m3_rtn(__ddiv_rn(gmax, a.s), &ovf);
      wmax = fmax(wmax, lmax);
      pmx = fmax(pmx, d);
    }
    uint32_t codes = 0;
    double dq[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t cd = rtn_code_literal(y[i], d);
      codes |= cd << (4 * i);
      dq[i] = __dmul_rn(fp4_val(cd), d);                         // dequant_elements
    }
    *reinterpret_cast<uint16_t*>(a.codes + r * (a.K / 2) + c * 64 + 2 * lane) = (uint16_t)codes;
    if (PASS == PASS_QUANT && scale32 == 0.f) {                  // ms_eden.py:139-140
      if ((lane & 3) == 0) sf_store(a.sf, r, c * 8 + (lane >> 2), kpr, (uint8_t)s8);
      continue;
    }
    // EDEN factor S = <x,x>/<x,q> in numpy pairwise order (ms_eden.py:75-83)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      pn[4 * lane + i] = __dmul_rn(y[i], y[i]);
      pd[4 * lane + i] = __dmul_rn(y[i], dq[i]);
    }
    __syncwarp();
    const double num = numpy_sum128(pn, lane);
    const double den = numpy_sum128(pd, lane);
    __syncwarp();
    const bool ok = (fabs(den) >= __dmul_rn(1e-30, num)) && (num > 0.0);
    const double S = ok ? __ddiv_rn(num, den) : 1.0;
    if (PASS == PASS_POSTHOC1) {
      if (lane == 0) a.corr[r * (a.K / CHUNK) + c] = S;
      if ((lane & 3) == 0) a.pseudo[g] = (uint16_t)(__float_as_uint((float)d) >> 16);
      continue;
    }
    if ((lane & 3) == 0) {
      const double corrected = __dmul_rn(S, e4m3_val(s8));       // ms_eden.py:142-143
      if (corrected > 448.0) atomic_or_err(a.err, Q2_ERR_SCALE448);
      const double uu = prng_uniform(a.sr_head, (uint64_t)g);
      sf_store(a.sf, r, c * 8 + (lane >> 2), kpr, (uint8_t)e4m3_sr(fmin(corrected, 448.0), uu));
    }
  }
  if (PASS != PASS_QUANT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xFFFFFFFFu, wmax, o));
    if (PASS == PASS_PMAX || PASS == PASS_POSTHOC1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pmx = fmax(pmx, __shfl_xor_sync(0xFFFFFFFFu, pmx, o));
    }
    if (lane == 0 && wmax > 0.0) atomicMax(&a.red[0], (unsigned long long)__double_as_longlong(wmax));
    if (lane == 0 && pmx > 0.0) atomicMax(&a.red[1], (unsigned long long)__double_as_longlong(pmx));
    if (ovf) atomic_or_err(a.err, Q2_ERR_E8M3_OVF);
  }
}

// --------------------------------------------------------- literal fix-ups --
// Warp-level gather of one (row, chunk) unit, signs applied: lane l holds
// elements 4l..4l+3 as float64 (tape: FP4*E4M3*scale32, exact).
template <int SRC>
__device__ __forceinline__ void load_chunk_lit(const MsedArgs& a, int64_t r, int64_t c, int lane, double (&y)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = 4 * lane + i;
    const int64_t k = c * CHUNK + e;
    double v;
    if (SRC == Q2_SRC_ROWS || SRC == Q2_SRC_COLS) {
      const int64_t off = SRC == Q2_SRC_ROWS ? r * a.ld + k : k * a.ld + r;
      v = a.dtype == Q2_BF16 ? (double)bf16_to_f32(static_cast<const uint16_t*>(a.x)[off])
                             : (double)static_cast<const float*>(a.x)[off];
    } else {
      const uint32_t byte = a.tape_codes[k * (a.R / 2) + r / 2];
      const uint32_t code = (r & 1) ? byte >> 4 : byte & 0xF;
      const uint32_t s8 = a.tape_sf[sf_offset(k, r / 16, kpairs(a.R))];
      v = __dmul_rn(__dmul_rn(fp4_val(code), e4m3_val(s8)), (double)*a.tape_scale32);
    }
    y[i] = ((a.sign[e >> 5] >> (e & 31)) & 1u) ? -v : v;
  }
}

// Literal posthoc pass 1 of one chunk (posthoc.py:74-95): returns S; writes
// codes and pseudo-scales when `write`; reduces the pseudo max into *pmx.
template <int SRC>
__device__ __forceinline__ double posthoc1_chunk_lit(const MsedArgs& a, int64_t r, int64_t c, int lane, double* pn,
                                                     double* pd, bool write, double* pmx, bool* ovf) {
  double y[4];
  load_chunk_lit<SRC>(a, r, c, lane, y);
  fwht_f64(y, lane);
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] = __dmul_rn(y[i], a.inv_sqrt);
  const double lmax = fmax(fmax(fabs(y[0]), fabs(y[1])), fmax(fabs(y[2]), fabs(y[3])));
  const double gmax = group_max4(lmax);
  const double d = e8m3_rtn(__ddiv_rn(gmax, a.s), ovf);
  *pmx = fmax(*pmx, d);
  uint32_t codes = 0;
  double dq[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t cd = rtn_code_literal(y[i], d);
    codes |= cd << (4 * i);
    dq[i] = __dmul_rn(fp4_val(cd), d);
  }
  if (write) {
    *reinterpret_cast<uint16_t*>(a.codes + r * (a.K / 2) + c * 64 + 2 * lane) = (uint16_t)codes;
    if ((lane & 3) == 0) a.pseudo[r * (a.K / GROUP) + c * 8 + (lane >> 2)] = (uint16_t)(__float_as_uint((float)d) >> 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    pn[4 * lane + i] = __dmul_rn(y[i], y[i]);
    pd[4 * lane + i] = __dmul_rn(y[i], dq[i]);
  }
  __syncwarp();
  const double num = numpy_sum128(pn, lane);
  const double den = numpy_sum128(pd, lane);
  __syncwarp();
  const bool ok = (fabs(den) >= __dmul_rn(1e-30, num)) && (num > 0.0);
  return ok ? __ddiv_rn(num, den) : 1.0;
}

// Fix-up of pass-1 chunks the fast path could not certify.
template <int SRC>
__global__ void __launch_bounds__(128) posthoc_fix1_kernel(MsedArgs a, float* dS, const uint32_t* listA_n,
                                                           const uint32_t* listA) {
  __shared__ double scratch[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n = *listA_n, cpr = (uint32_t)(a.K / CHUNK);
  double pmx = 0.0;
  bool ovf = false;
  for (uint32_t i = blockIdx.x * 4 + warp; i < n; i += gridDim.x * 4) {
    const uint32_t id = listA[i];
    const int64_t r = id / cpr, c = id % cpr;
    const double S = posthoc1_chunk_lit<SRC>(a, r, c, lane, scratch[warp], scratch[warp] + 128, true, &pmx, &ovf);
    if (lane == 0) { a.corr[id] = S; dS[id] = 0.f; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pmx = fmax(pmx, __shfl_xor_sync(0xFFFFFFFFu, pmx, o));
  if (lane == 0 && pmx > 0.0) atomicMax(&a.red[1], (unsigned long long)__double_as_longlong(pmx));
  if (ovf) atomic_or_err(a.err, Q2_ERR_E8M3_OVF);
}

__device__ __forceinline__ float posthoc_scale32(double pmax) {
  if (!(pmax > 0.0)) return 0.f;
  int e; const double m = frexp(pmax / 256.0, &e);
  return (float)ldexp(1.0, (m == 0.5) ? e - 1 : e);         // ms_eden.py:86-91
}

// Certified pass 2 (posthoc.py:98-125).  One thread per 4 consecutive groups
// of a row (one 32-bit store per scale replica).  shifted = pseudo / 2^k is an
// exact power-of-two multiply; the SR decision lo + (u < p) is taken when the
// bracket corr * (1 -+ dS) stays inside one E4M3 interval and u is outside the
// matching p bracket; otherwise the group goes to posthoc_fix2_kernel.
__device__ __forceinline__ uint32_t sr_certified(double c, double d, double u, bool& ok) {
  // E4M3 interval [a, b) of c (normal range; smaller values take the exact path)
  const double lo = c * (1.0 - d), hi = c * (1.0 + d);
  if (!(lo >= 0x1p-6) || !(hi <= 448.0)) { ok = false; return 0; }
  const int e = dexp(c);
  const double step = dpow2(e - 3);                               // b - a, a power of two
  const double fl = floor(__dmul_rn(c, dpow2(3 - e)));            // 8 + mantissa index
  const double a = __dmul_rn(fl, step);
  uint32_t code = ((uint32_t)(e + 7) << 3) + (uint32_t)fl - 8u;
  if (code > 125u) { ok = false; return 0; }
  if (!(lo >= a) || !(hi < a + step)) { ok = false; return 0; }  // bracket crosses a grid point
  const double rs = dpow2(3 - e);
  const double plo = (lo - a) * rs, phi = (hi - a) * rs;          // p range (monotone in c)
  if (u < plo) return code + 1;                                    // u < p for every c in the bracket
  if (u >= phi) return code;
  ok = false;
  return 0;
}

__global__ void __launch_bounds__(256) posthoc2_cert_kernel(
    const uint16_t* __restrict__ pseudo, const double* __restrict__ corr, const float* __restrict__ dS,
    const unsigned long long* __restrict__ red, int64_t R, int64_t K, FastDiv fq, uint64_t sr_head,
    uint8_t* __restrict__ sf, float* __restrict__ scale32_out, uint32_t* __restrict__ listB_n,
    uint32_t* __restrict__ listB, uint32_t* __restrict__ err) {
  const uint32_t qpr = (uint32_t)(K / 64), total = (uint32_t)(R * qpr);    // quads of groups per row
  const double pmax = ulong_as_double(red[1]);
  int k = 0;
  if (pmax > 0.0) {
    int e; const double m = frexp(pmax / 256.0, &e);
    k = (m == 0.5) ? e - 1 : e;                                             // ms_eden.py:86-91
  }
  const float scale32 = pmax > 0.0 ? (float)ldexp(1.0, k) : 0.f;
  const double inv_scale = pmax > 0.0 ? ldexp(1.0, -k) : 0.0;
  const uint32_t tq = blockIdx.x * blockDim.x + threadIdx.x;
  if (tq == 0) *scale32_out = scale32;
  if (tq >= total) return;
  const uint32_t r = fq.div(tq), jq = tq - r * qpr;                         // groups 4jq .. 4jq+3
  const int64_t kpr = kpairs(K);
  uint32_t* dst = reinterpret_cast<uint32_t*>(sf + sf_offset(r, 4 * jq, kpr));
  if (pmax == 0.0) { dst[0] = 0; dst[256] = 0; dst[512] = 0; dst[768] = 0; return; }
  const int64_t ch = (int64_t)r * (K / CHUNK) + (jq >> 1);
  const double S = corr[ch];
  const double d = (double)dS[ch] * 1.0001;
  const uint2 pw = *reinterpret_cast<const uint2*>(pseudo + (int64_t)r * (K / GROUP) + 4 * jq);
  const uint32_t pv[4] = {pw.x & 0xFFFF, pw.x >> 16, pw.y & 0xFFFF, pw.y >> 16};
  uint32_t word = 0;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t g = (uint64_t)r * (K / GROUP) + 4 * jq + i;
    const double ps = (double)__uint_as_float(pv[i] << 16);
    const double corrected = __dmul_rn(S, __dmul_rn(ps, inv_scale));
    const double u = prng_uniform(sr_head, g);
    bool ok = d > 0.0;
    uint32_t code = ok ? sr_certified(corrected, d, u, ok) : 0u;
    if (!ok) {
      if (d == 0.0) {                                                       // exact factor (fix-up 1)
        if (corrected > 448.0) bad = true;
        code = e4m3_sr(fmin(corrected, 448.0), u);
      } else {
        listB[atomicAdd(listB_n, 1u)] = (uint32_t)g;                        // exact re-do
        code = 0;
      }
    }
    word |= code << (8 * i);
  }
  if (bad) atomic_or_err(err, Q2_ERR_SCALE448);
  dst[0] = word; dst[256] = word; dst[512] = word; dst[768] = word;
}

// Exact re-do of pass-2 groups (exact float64 EDEN factor of their chunk).
template <int SRC>
__global__ void __launch_bounds__(128) posthoc_fix2_kernel(MsedArgs a, const uint32_t* listB_n, const uint32_t* listB,
                                                           uint64_t sr_head) {
  __shared__ double scratch[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n = *listB_n;
  const int64_t gpr = a.K / GROUP;
  const double pmax = ulong_as_double(a.red[1]);
  const float scale32 = posthoc_scale32(pmax);
  for (uint32_t i = blockIdx.x * 4 + warp; i < n; i += gridDim.x * 4) {
    const uint32_t g = listB[i];
    const int64_t r = g / gpr, j = g - r * gpr;
    double pm = 0.0;
    bool ovf = false;
    const double S = posthoc1_chunk_lit<SRC>(a, r, j / 8, lane, scratch[warp], scratch[warp] + 128, false, &pm, &ovf);
    if (lane == 0) {
      const double ps = (double)__uint_as_float((uint32_t)a.pseudo[g] << 16);
      const double corrected = __dmul_rn(S, __ddiv_rn(ps, (double)scale32));
      if (corrected > 448.0) atomic_or_err(a.err, Q2_ERR_SCALE448);
      sf_store(a.sf, r, j, kpairs(a.K), (uint8_t)e4m3_sr(fmin(corrected, 448.0), prng_uniform(sr_head, (uint64_t)g)));
    }
  }
}

// posthoc pass 2: scales only (posthoc.py:98-125).  One thread per group.
__global__ void posthoc2_kernel(const uint16_t* __restrict__ pseudo, const double* __restrict__ corr,
                                const unsigned long long* __restrict__ red, int64_t R, int64_t K,
                                uint64_t sr_head, uint8_t* __restrict__ sf, float* __restrict__ scale32_out,
                                uint32_t* __restrict__ err) {
  const int64_t gpr = K / GROUP, total = R * gpr;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double pmax = ulong_as_double(red[1]);
  float scale32 = 0.f;
  if (pmax > 0.0) {
    int e; double m = frexp(pmax / 256.0, &e);
    scale32 = (float)ldexp(1.0, (m == 0.5) ? e - 1 : e);
  }
  if (g == 0) *scale32_out = scale32;
  if (g >= total) return;
  const int64_t r = g / gpr, j = g - r * gpr;
  const int64_t kpr = kpairs(K);
  if (pmax == 0.0) { sf_store(sf, r, j, kpr, 0); return; }
  const double ps = (double)__uint_as_float((uint32_t)pseudo[g] << 16);
  const double shifted = __ddiv_rn(ps, (double)scale32);
  const double corrected = __dmul_rn(corr[r * (K / CHUNK) + j / 8], shifted);
  if (corrected > 448.0) atomic_or_err(err, Q2_ERR_SCALE448);
  sf_store(sf, r, j, kpr, (uint8_t)e4m3_sr(fmin(corrected, 448.0), prng_uniform(sr_head, (uint64_t)g)));
}

}  // namespace q2
#include "msed_fast.cuh"
#include "msed_tc.cuh"
namespace q2 {

constexpr size_t MSED_SMEM = TILE_ROWS * TILE_LD * sizeof(float) + 8 * 256 * sizeof(double);

template <int SRC, int PASS>
static int launch_msed(const MsedArgs& a, cudaStream_t s) {
  auto k = msed_kernel<SRC, PASS>;
  static bool attr_set = false;   // benign race: idempotent
  if (!attr_set) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MSED_SMEM) != cudaSuccess)
      return Q2_ECUDA;
    attr_set = true;
  }
  dim3 grid((unsigned)((a.R + TILE_ROWS - 1) / TILE_ROWS), (unsigned)(a.K / CHUNK));
  k<<<grid, MSED_THREADS, MSED_SMEM, s>>>(a);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

template <int PASS>
static int dispatch_src(int src, const MsedArgs& a, cudaStream_t s) {
  switch (src) {
    case Q2_SRC_ROWS: return launch_msed<Q2_SRC_ROWS, PASS>(a, s);
    case Q2_SRC_COLS: return launch_msed<Q2_SRC_COLS, PASS>(a, s);
    case Q2_SRC_TAPE_COLS: return launch_msed<Q2_SRC_TAPE_COLS, PASS>(a, s);
  }
  return Q2_EINVAL;
}

static int fill_args(MsedArgs& a, const void* x, int dtype, const q2_nvfp4* tape, int src, int64_t R,
                     int64_t K, int64_t ld, const uint32_t sign_mask[4], double s, double inv_sqrt) {
  if (R < 0 || K % CHUNK || !sign_mask) return Q2_EINVAL;
  a = MsedArgs{};
  a.x = x; a.dtype = dtype; a.R = R; a.K = K; a.ld = ld;
  for (int i = 0; i < 4; ++i) a.sign[i] = sign_mask[i];
  a.s = s; a.inv_sqrt = inv_sqrt;
  if (src == Q2_SRC_TAPE_COLS) {
    if (!tape || tape->R != K || tape->K != R || R % 64) return Q2_EINVAL;
    a.tape_codes = tape->codes; a.tape_sf = tape->sf; a.tape_scale32 = tape->scale32; a.tape_K = tape->K;
  } else {
    if (!x || (dtype != Q2_BF16 && dtype != Q2_F32)) return Q2_EINVAL;
    const int esz = dtype == Q2_BF16 ? 2 : 4;
    if ((reinterpret_cast<uintptr_t>(x) & 15u) || (ld * esz) % 16) return Q2_EINVAL;
    if (src == Q2_SRC_ROWS && ld < K) return Q2_EINVAL;
    if (src == Q2_SRC_COLS && (ld < R || R % 8)) return Q2_EINVAL;
    if (src != Q2_SRC_ROWS && src != Q2_SRC_COLS) return Q2_EINVAL;
  }
  return Q2_OK;
}

template <int SRC, int DT>
static int launch_fast1(const MsedArgs& a, const FastArgs& f, cudaStream_t st) {
  const int smem = F_ROWS * (DT == Q2_BF16 ? 256 : 512) + 256 + 64;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(msed_fast1_kernel<SRC, DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return Q2_ECUDA;
    attr = true;
  }
  dim3 grid((unsigned)((a.R + F_ROWS - 1) / F_ROWS), (unsigned)(a.K / CHUNK));
  msed_fast1_kernel<SRC, DT><<<grid, F_THREADS, smem, st>>>(a, f);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

static int num_sms() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

// Fix-ups and certified pass 2 after any pass-1 producer.
template <int SRC>
static int posthoc_tail(const MsedArgs& a, const FastArgs& f, uint32_t* listB_n, uint32_t* listB, uint64_t sr_head,
                        cudaStream_t st) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  posthoc_fix1_kernel<SRC><<<2 * nsm, 128, 0, st>>>(a, f.dS, f.listA_n, f.listA);
  Q2_CHECK_LAUNCH();
  const int64_t quads = a.R * (a.K / 64);
  posthoc2_cert_kernel<<<(unsigned)std::max<int64_t>(1, (quads + 255) / 256), 256, 0, st>>>(
      a.pseudo, a.corr, f.dS, a.red, a.R, a.K, FastDiv((uint32_t)(a.K / 64)), sr_head, a.sf, a.scale32, listB_n,
      listB, a.err);
  Q2_CHECK_LAUNCH();
  posthoc_fix2_kernel<SRC><<<2 * nsm, 128, 0, st>>>(a, listB_n, listB, sr_head);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

// Single-read post-hoc MS-EDEN with certified fast paths and exact fix-ups.
template <int SRC>
static int posthoc_fast(MsedArgs a, FastArgs f, uint32_t* listB_n, uint32_t* listB, uint64_t sr_head,
                        cudaStream_t st) {
  int rc = (SRC == Q2_SRC_TAPE_COLS || a.dtype == Q2_BF16) ? launch_fast1<SRC, Q2_BF16>(a, f, st)
                                                            : launch_fast1<SRC, Q2_F32>(a, f, st);
  if (rc) return rc;
  return posthoc_tail<SRC>(a, f, listB_n, listB, sr_head, st);
}

// Workspace carve-up shared by the post-hoc drivers.
struct PosthocWs {
  uint32_t* red; uint16_t* pseudo; double* corr; FastArgs f; uint32_t* listB; uint32_t* listB_n;
};
static size_t al256(size_t v) { return (v + 255) & ~size_t(255); }
static PosthocWs carve_ws(void* ws, int64_t R, int64_t K) {
  PosthocWs w;
  char* b = static_cast<char*>(ws);
  const size_t g = (size_t)R * (K / 16), ch = (size_t)R * (K / 128);
  w.red = reinterpret_cast<uint32_t*>(b);
  w.pseudo = reinterpret_cast<uint16_t*>(b + 256);
  w.corr = reinterpret_cast<double*>(b + 256 + al256(g * 2));
  char* p = b + 256 + al256(g * 2) + al256(ch * 8);
  w.f.dS = reinterpret_cast<float*>(p);
  p += al256(ch * 4);
  w.f.listA = reinterpret_cast<uint32_t*>(p);
  p += al256(ch * 4);
  w.listB = reinterpret_cast<uint32_t*>(p);
  w.f.listA_n = w.red + 4;
  w.listB_n = w.red + 5;
  return w;
}

// Tensor-core pass 1 for bf16 rows / E^T of the same tile; do_rows / do_cols select outputs.
static int tc_pass1(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t* sign_rows,
                    const uint32_t* sign_cols, double s, double inv_sqrt, const q2_nvfp4* out_rows,
                    const q2_nvfp4* out_cols, const PosthocWs* w_rows, const PosthocWs* w_cols, uint32_t* err,
                    cudaStream_t st) {
  TcArgs t{};
  t.do_rows = out_rows != nullptr;
  t.do_cols = out_cols != nullptr;
  t.tiles_r = (int)(T / 128);
  t.tiles_c = (int)(N / 128);
  t.c_eff = inv_sqrt;
  t.s = s;
  t.err = err;
  for (int j = 0; j < 2; ++j) {
    const q2_nvfp4* o = j ? out_cols : out_rows;
    const PosthocWs* w = j ? w_cols : w_rows;
    const uint32_t* sg = j ? sign_cols : sign_rows;
    if (!o) continue;
    t.out[j] = TcOut{o->codes, w->pseudo, w->corr, w->f.dS, reinterpret_cast<unsigned long long*>(w->red),
                     w->f.listA_n, w->f.listA, j ? N : T, j ? T : N, 0};
    for (int i = 0; i < 4; ++i) t.sign[j][i] = sg[i];
  }
  CUtensorMap mx;
  if (!make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, (uint64_t)N, (uint64_t)T, (uint64_t)ld * 2, 64, 128))
    return Q2_ECUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(msed_dual_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM) != cudaSuccess)
      return Q2_ECUDA;
    attr = true;
  }
  const int ntiles = t.tiles_r * t.tiles_c;
  msed_dual_tc_kernel<<<std::min(ntiles, num_sms()), TC_THREADS, TC_SMEM, st>>>(mx, t);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

static bool tc_ok(const void* x, int dtype, int64_t T, int64_t N, int64_t ld) {
  return dtype == Q2_BF16 && T % 128 == 0 && N % 128 == 0 && T > 0 && N > 0 && (ld * 2) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(x) & 15) == 0;
}

}  // namespace q2

using namespace q2;

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// ws: red | pseudo bf16 [R,K/16] | corr f64 [R,K/128] | dS f32 [R,K/128] | listA | listB
extern "C" size_t q2_msed_ws_bytes(int64_t R, int64_t K) {
  const size_t g = (size_t)R * (K / 16), ch = (size_t)R * (K / 128);
  return 256 + align256(g * 2) + align256(ch * 8) + align256(ch * 4) + align256(ch * 4) + align256(g * 4);
}

extern "C" int q2_posthoc_pass1(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R,
                                int64_t K, int64_t ld, const uint32_t sign_mask[4], double s,
                                double inv_sqrt_chunk, uint8_t* codes, uint16_t* pseudo_bf16, double* corr,
                                uint32_t* red, uint32_t* err, void* stream) {
  MsedArgs a;
  int rc = fill_args(a, x, dtype, tape, src_kind, R, K, ld, sign_mask, s, inv_sqrt_chunk);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  a.codes = codes; a.pseudo = pseudo_bf16; a.corr = corr;
  a.red = reinterpret_cast<unsigned long long*>(red); a.err = err;
  if (cudaMemsetAsync(red, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  if (R == 0) return Q2_OK;
  return dispatch_src<PASS_POSTHOC1>(src_kind, a, st);
}

extern "C" int q2_posthoc_pass2(const uint16_t* pseudo_bf16, const double* corr, const uint32_t* red,
                                int64_t R, int64_t K, uint64_t seed_sr, uint64_t sr_stream,
                                const q2_nvfp4* out, uint32_t* err, void* stream) {
  if (!out || out->R != R || out->K != K || K % CHUNK) return Q2_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t groups = R * (K / 16);
  unsigned blocks = (unsigned)std::max<int64_t>(1, (groups + 255) / 256);
  posthoc2_kernel<<<blocks, 256, 0, st>>>(pseudo_bf16, corr, reinterpret_cast<const unsigned long long*>(red),
                                          R, K, prng_head(seed_sr, sr_stream), out->sf, out->scale32, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

extern "C" int q2_msed_quant(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R,
                             int64_t K, int64_t ld, const uint32_t sign_mask[4], double s,
                             double inv_sqrt_chunk, uint64_t seed_sr, uint64_t sr_stream, int mode,
                             const q2_nvfp4* out, void* ws, uint32_t* err, void* stream) {
  if (!out || !ws || out->R != R || out->K != K) return Q2_EINVAL;
  MsedArgs a;
  int rc = fill_args(a, x, dtype, tape, src_kind, R, K, ld, sign_mask, s, inv_sqrt_chunk);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  uint32_t* red = reinterpret_cast<uint32_t*>(w);
  uint16_t* pseudo = reinterpret_cast<uint16_t*>(w + 256);
  double* corr = reinterpret_cast<double*>(w + 256 + align256((size_t)R * (K / 16) * 2));
  if (mode == Q2_MSED_POSTHOC) {
    const size_t g = (size_t)R * (K / 16), ch = (size_t)R * (K / 128);
    char* p = w + 256 + align256(g * 2) + align256(ch * 8);
    FastArgs f;
    f.dS = reinterpret_cast<float*>(p);
    p += align256(ch * 4);
    f.listA = reinterpret_cast<uint32_t*>(p);
    p += align256(ch * 4);
    uint32_t* listB = reinterpret_cast<uint32_t*>(p);
    uint32_t* cnt = red + 4;                 // red[0..3]: two f64 maxima; [4] listA_n, [5] listB_n
    f.listA_n = cnt;
    if (cudaMemsetAsync(red, 0, 32, st) != cudaSuccess) return Q2_ECUDA;
    if (R == 0) return Q2_OK;
    a.red = reinterpret_cast<unsigned long long*>(red); a.err = err;
    a.codes = out->codes; a.sf = out->sf; a.scale32 = out->scale32;
    a.pseudo = pseudo; a.corr = corr;
    const uint64_t head = prng_head(seed_sr, sr_stream);
    // Tensor-core rotations are opt-in (Q2_TC_MSED=1): their error bound assumes
    // fp32-accurate MMA accumulation (see msed_tc.cuh); the CUDA-core path's is proven.
    if (src_kind != Q2_SRC_TAPE_COLS && getenv("Q2_TC_MSED")) {
      const int64_t T = src_kind == Q2_SRC_ROWS ? R : K, N = src_kind == Q2_SRC_ROWS ? K : R;
      if (tc_ok(x, dtype, T, N, ld)) {
        const PosthocWs w = carve_ws(ws, R, K);
        rc = src_kind == Q2_SRC_ROWS
                 ? tc_pass1(x, T, N, ld, a.sign, a.sign, s, inv_sqrt_chunk, out, nullptr, &w, nullptr, err, st)
                 : tc_pass1(x, T, N, ld, a.sign, a.sign, s, inv_sqrt_chunk, nullptr, out, nullptr, &w, err, st);
        if (rc) return rc;
        return src_kind == Q2_SRC_ROWS ? posthoc_tail<Q2_SRC_ROWS>(a, f, cnt + 1, listB, head, st)
                                       : posthoc_tail<Q2_SRC_COLS>(a, f, cnt + 1, listB, head, st);
      }
    }
    switch (src_kind) {
      case Q2_SRC_ROWS: return posthoc_fast<Q2_SRC_ROWS>(a, f, cnt + 1, listB, head, st);
      case Q2_SRC_COLS: return posthoc_fast<Q2_SRC_COLS>(a, f, cnt + 1, listB, head, st);
      default: return posthoc_fast<Q2_SRC_TAPE_COLS>(a, f, cnt + 1, listB, head, st);
    }
  }
  if (mode != Q2_MSED_EXACT && mode != Q2_MSED_POW2) return Q2_EINVAL;
  a.red = reinterpret_cast<unsigned long long*>(red); a.err = err;
  a.codes = out->codes; a.sf = out->sf; a.scale32 = out->scale32;
  a.sr_head = prng_head(seed_sr, sr_stream);
  a.pow2 = mode == Q2_MSED_POW2;
  if (cudaMemsetAsync(red, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  if (R == 0) return Q2_OK;
  rc = a.pow2 ? dispatch_src<PASS_PMAX>(src_kind, a, st) : dispatch_src<PASS_ABSMAX>(src_kind, a, st);
  if (rc) return rc;
  return dispatch_src<PASS_QUANT>(src_kind, a, st);
}

// Both backward operands that read E in one pass: MS(E) along rows (dgrad, pair
// sign_rows / sr_stream_rows) and MS(E^T) (wgrad, pair sign_cols /
// sr_stream_cols), post-hoc schedule.  x is bf16 [T, N], T % 128 == N % 128 == 0.
extern "C" int q2_msed_dual_posthoc(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t sign_rows[4],
                                    const uint32_t sign_cols[4], double s, double inv_sqrt_chunk, uint64_t seed_sr,
                                    uint64_t sr_stream_rows, uint64_t sr_stream_cols, const q2_nvfp4* out_rows,
                                    const q2_nvfp4* out_cols, void* ws_rows, void* ws_cols, uint32_t* err,
                                    void* stream) {
  if (!x || !out_rows || !out_cols || !ws_rows || !ws_cols || out_rows->R != T || out_rows->K != N ||
      out_cols->R != N || out_cols->K != T || !tc_ok(x, Q2_BF16, T, N, ld))
    return Q2_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const PosthocWs wr = carve_ws(ws_rows, T, N), wc = carve_ws(ws_cols, N, T);
  if (cudaMemsetAsync(wr.red, 0, 32, st) != cudaSuccess || cudaMemsetAsync(wc.red, 0, 32, st) != cudaSuccess)
    return Q2_ECUDA;
  int rc = tc_pass1(x, T, N, ld, sign_rows, sign_cols, s, inv_sqrt_chunk, out_rows, out_cols, &wr, &wc, err, st);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j) {
    MsedArgs a;
    rc = fill_args(a, x, Q2_BF16, nullptr, j ? Q2_SRC_COLS : Q2_SRC_ROWS, j ? N : T, j ? T : N, ld,
                   j ? sign_cols : sign_rows, s, inv_sqrt_chunk);
    if (rc) return rc;
    const q2_nvfp4* o = j ? out_cols : out_rows;
    const PosthocWs& w = j ? wc : wr;
    a.red = reinterpret_cast<unsigned long long*>(w.red); a.err = err;
    a.codes = o->codes; a.sf = o->sf; a.scale32 = o->scale32;
    a.pseudo = w.pseudo; a.corr = w.corr;
    const uint64_t head = prng_head(seed_sr, j ? sr_stream_cols : sr_stream_rows);
    rc = j ? posthoc_tail<Q2_SRC_COLS>(a, w.f, w.listB_n, w.listB, head, st)
           : posthoc_tail<Q2_SRC_ROWS>(a, w.f, w.listB_n, w.listB, head, st);
    if (rc) return rc;
  }
  return Q2_OK;
}
