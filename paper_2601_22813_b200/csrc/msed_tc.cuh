// MS-EDEN post-hoc pass 1 on the tensor cores (included by msed.cu after
// msed_fast.cuh).
//
// The randomized 128-point Hadamard rotation of every chunk is a GEMM against
// the resident operand B = H . diag(signs) (bf16, +-1 entries, exact):
//   rows of x   : D1[r, i] = sum_k x[r, k]  B[i, k]   A = x tile, K-major
//   rows of x^T : D2[c, i] = sum_k x[k, c]  B'[i, k]  A = the SAME tile read
//                 MN-major, so E^T is quantized straight from E (no copy).
// One TMA-loaded 128x128 bf16 tile of E therefore feeds both backward GEMM
// operands (dgrad: rows of E with pair_dx; wgrad: rows of E^T with pair_dw):
// E is read once (3.125 B/elem).  tcgen05.mma kind::f16 accumulates in fp32
// TMEM (two 128x256 accumulator stages); four epilogue warps own one chunk per
// thread and apply the certified decisions of msed_fast.cuh.
//
// STATUS: opt-in (Q2_TC_MSED=1).  The bound used below, |y - y*| <= 2^-18
// ||y||_2, assumes each K=16 MMA adds at most 2^-21 of the L1 mass it sums;
// PTX only guarantees "at least single precision" accumulation, which allows
// up to ~2^-16.  Until a per-chunk exactness certificate (exponent span <= 9
// binades => every partial sum fits 24 bits => exact under any rounding) gates
// eps = 0, the proven CUDA-core path (msed_fast.cuh) is the default.  Measured
// on E 16384x11264: 5.3% of chunks / 1.5% of scale groups need the fix-ups.

namespace q2 {

constexpr int TC_STAGES = 3;
constexpr int TC_TILE_BYTES = 32768;   // [2 column halves][128 rows][128 B], 128B swizzle
constexpr int TC_B_BYTES = 32768;
constexpr int TC_OFF_B0 = TC_STAGES * TC_TILE_BYTES;
constexpr int TC_OFF_B1 = TC_OFF_B0 + TC_B_BYTES;
constexpr int TC_OFF_BAR = TC_OFF_B1 + TC_B_BYTES;
constexpr int TC_SMEM = TC_OFF_BAR + 256 + 1024;
constexpr int TC_THREADS = 256;
// kind::f16 instruction descriptor: fp32 D (bit 4), bf16 A/B ([7,10)=1, [10,13)=1),
// N = 128 (>>3 at 17), M = 128 (>>4 at 24); bit 15 = A MN-major.
constexpr uint32_t TC_IDESC_K = (1u << 4) | (1u << 7) | (1u << 10) | (16u << 17) | (8u << 24);
constexpr uint32_t TC_IDESC_MN = TC_IDESC_K | (1u << 15);

struct TcOut {
  uint8_t* codes; uint16_t* pseudo; double* corr; float* dS;
  unsigned long long* red; uint32_t* listA_n; uint32_t* listA;
  int64_t R, K;              // logical shape of this quantized output
  uint32_t err_dummy;
};

struct TcArgs {
  TcOut out[2];              // [0] rows (x), [1] rows of x^T
  uint32_t sign[2][4];
  int do_rows, do_cols;
  int tiles_r, tiles_c;      // tiles along rows (T/128) and columns (N/128) of x
  double c_eff, s;
  uint32_t* err;
};

// byte offset of element (row, col) of a 128x128 bf16 tile in the TMA 128B-swizzled layout
__device__ __forceinline__ uint32_t tc_tile_off(int row, int col) {
  const int half = col >> 6, byte = (col & 63) * 2;
  return (uint32_t)(half * 16384 + row * 128 + ((((byte >> 4) ^ (row & 7))) << 4) + (byte & 15));
}

// One chunk per thread: 128 rotated values from TMEM -> certified pass-1 products.
__device__ __forceinline__ void tc_chunk(uint32_t taddr, const TcOut& o, int64_t r, int64_t c, double c_eff, float cs,
                                         float cef, float& pmx_out, bool& ovf) {
  float y[128];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t v[32];
    Q2_LD32(v, taddr + 32 * q);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) y[32 * q + i] = __uint_as_float(v[i]);
  }
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const uint64_t p = f2pack(y[2 * i], y[2 * i + 1]);
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(p));
  }
  float n0, n1;
  f2unpack(acc, n0, n1);
  const float num = n0 + n1;
  const float eps = 0x1p-18f * 1.001f * sqrtf(num) + 0x1p-120f;
  bool unc = false;
  float den = 0.f, pmx = 0.f, psum = 0.f;
  uint32_t cw[16];
  uint32_t pb[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    float gm = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) gm = fmaxf(gm, fabsf(y[16 * g + i]));
    const float glo = fmaxf(gm - eps, 0.f) * cs * (1.f - 0x1p-21f), ghi = (gm + eps) * cs * (1.f + 0x1p-21f);
    const uint32_t plo = rne4(glo), phi = rne4(ghi);
    unc |= (plo != phi) | !(glo >= 0x1p-125f) | !(ghi < 0x1p126f);
    const float p = __uint_as_float(phi);
    pmx = fmaxf(pmx, p);
    psum += p;
    pb[g] = phi >> 16;
    float inv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(p));
    inv *= cef;
    const float il = inv * (1.f - 0x1p-19f), ih = inv * (1.f + 0x1p-19f);
    const uint64_t il2 = f2pack(il, il), ih2 = f2pack(ih, ih);
    float dsum0 = 0.f, dsum1 = 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint64_t lo[4], hi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = y[16 * g + 8 * half + 2 * i], b = y[16 * g + 8 * half + 2 * i + 1];
        const uint64_t v = f2pack(a, b);
        const uint64_t e2 = f2pack(__uint_as_float((__float_as_uint(a) & 0x80000000u) | __float_as_uint(eps)),
                                   __uint_as_float((__float_as_uint(b) & 0x80000000u) | __float_as_uint(eps)));
        const uint64_t ylo = sub2(v, e2), yhi = add2(v, e2);
        asm("mul.rz.f32x2 %0, %1, %2;" : "=l"(lo[i]) : "l"(ylo), "l"(il2));
        asm("mul.rz.f32x2 %0, %1, %2;" : "=l"(hi[i]) : "l"(yhi), "l"(ih2));
      }
      uint32_t wlo, whi;
      codes8(lo, hi, wlo, whi);
      unc |= wlo != whi;
      cw[2 * g + half] = wlo;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t h2;
        asm("{\n\t.reg .b8 t;\n\tcvt.u8.u32 t, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, t;\n\t}" : "=r"(h2) : "r"(wlo >> (8 * i)));
        float r0, r1;
        asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
            : "=f"(r0), "=f"(r1) : "r"(h2));
        dsum0 = fmaf(y[16 * g + 8 * half + 2 * i], r0, dsum0);
        dsum1 = fmaf(y[16 * g + 8 * half + 2 * i + 1], r1, dsum1);
      }
    }
    den = fmaf(p, dsum0 + dsum1, den);
  }
  // outputs (posthoc pass-1 products of this chunk)
  uint4* cp = reinterpret_cast<uint4*>(o.codes + r * (o.K / 2) + c * 64);
#pragma unroll
  for (int i = 0; i < 4; ++i) cp[i] = make_uint4(cw[4 * i], cw[4 * i + 1], cw[4 * i + 2], cw[4 * i + 3]);
  *reinterpret_cast<uint4*>(o.pseudo + r * (o.K / GROUP) + c * 8) =
      make_uint4(pb[0] | (pb[1] << 16), pb[2] | (pb[3] << 16), pb[4] | (pb[5] << 16), pb[6] | (pb[7] << 16));
  const int64_t ch = r * (o.K / CHUNK) + c;
  const bool good = !unc && num > 0.f && den != 0.f;
  // |dnum| <= 2 eps sqrt(128 num) + 128 eps^2 + accumulation; |dden| <= 6 eps sum_g 16 p_g + accumulation
  const float dn = (2.f * eps * sqrtf(128.f * num) + 128.f * eps * eps) / num + 0x1p-18f;
  const float dd = (eps * 96.f * psum) / fabsf(den) + 0x1p-18f;
  o.corr[ch] = c_eff * (double)num / (double)den;
  o.dS[ch] = good ? 1.001f * (dn + dd) + 0x1p-20f : 1e30f;
  if (!good) o.listA[atomicAdd(o.listA_n, 1u)] = (uint32_t)ch;
  pmx_out = good ? fmaxf(pmx_out, pmx) : pmx_out;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    msed_dual_tc_kernel(const __grid_constant__ CUtensorMap tmX, TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_r * a.tiles_c;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TC_OFF_BAR);
  const uint32_t bar_full = smem_u32(bars), bar_empty = smem_u32(bars + TC_STAGES);
  const uint32_t bar_accf = smem_u32(bars + 2 * TC_STAGES), bar_acce = smem_u32(bars + 2 * TC_STAGES + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TC_STAGES + 4);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) { mbar_init(bar_full + 8 * s, 1); mbar_init(bar_empty + 8 * s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(bar_accf + 8 * s, 1); mbar_init(bar_acce + 8 * s, 4); }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  // B_j[i][k] = H[i][k] * sign_j[k] (Sylvester order), K-major in the swizzled tile layout
  for (int idx = threadIdx.x; idx < 2 * 128 * 16; idx += TC_THREADS) {
    const int j = idx >> 11, i = (idx >> 4) & 127, kc = idx & 15;         // 8 k per 16-byte chunk
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t hw = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int k = kc * 8 + 2 * e + t;
        const bool neg = (__popc(i & k) & 1) ^ ((a.sign[j][k >> 5] >> (k & 31)) & 1);
        hw |= (neg ? 0xBF80u : 0x3F80u) << (16 * t);                         // bf16 -1 / +1
      }
      w[e] = hw;
    }
    *reinterpret_cast<uint4*>(smem + (j ? TC_OFF_B1 : TC_OFF_B0) + tc_tile_off(i, kc * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % TC_STAGES;
        if (it >= TC_STAGES) mbar_wait(bar_empty + 8 * s, ((it / TC_STAGES) - 1) & 1);
        const int tr = t / a.tiles_c, tc = t - tr * a.tiles_c;
        mbar_expect_tx(bar_full + 8 * s, TC_TILE_BYTES);
        tma_load_2d(smem_u32(smem + s * TC_TILE_BYTES), &tmX, tc * 128, tr * 128, bar_full + 8 * s);
        tma_load_2d(smem_u32(smem + s * TC_TILE_BYTES + 16384), &tmX, tc * 128 + 64, tr * 128, bar_full + 8 * s);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                   // MMA issuer
      const uint32_t b0 = smem_u32(smem + TC_OFF_B0), b1 = smem_u32(smem + TC_OFF_B1);
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % TC_STAGES, as = it & 1;
        if (it >= 2) mbar_wait(bar_acce + 8 * as, ((it >> 1) - 1) & 1);
        mbar_wait(bar_full + 8 * s, (it / TC_STAGES) & 1);
        tc_fence_after();
        const uint32_t tile = smem_u32(smem + s * TC_TILE_BYTES);
        const uint32_t d = tmem + as * 256;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {                // K = 16 per MMA
          const uint32_t koff = (ks >> 2) * 16384 + (ks & 3) * 32;
          if (a.do_rows)
            tc_mma_f16(d, desc_sw128(tile + koff), desc_sw128(b0 + koff), TC_IDESC_K, ks > 0);
          if (a.do_cols)
            tc_mma_f16(d + 128, desc_mn_sw128(tile + ks * 2048, 16384, 1024), desc_sw128(b1 + koff), TC_IDESC_MN, ks > 0);
        }
        tc_commit(bar_empty + 8 * s);
        tc_commit(bar_accf + 8 * as);
      }
    }
  } else if (warp >= 4) {                              // epilogue: one chunk per thread per output
    const int ew = warp - 4, row = ew * 32 + lane;
    const float cs = (float)(a.c_eff / a.s), cef = (float)a.c_eff;
    float pm0 = 0.f, pm1 = 0.f;
    bool ovf = false;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int as = it & 1;
      const int tr = t / a.tiles_c, tc = t - tr * a.tiles_c;
      mbar_wait(bar_accf + 8 * as, (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tl = tmem + ((uint32_t)(ew * 32) << 16) + as * 256;
      if (a.do_rows) tc_chunk(tl, a.out[0], (int64_t)tr * 128 + row, tc, a.c_eff, cs, cef, pm0, ovf);
      if (a.do_cols) tc_chunk(tl + 128, a.out[1], (int64_t)tc * 128 + row, tr, a.c_eff, cs, cef, pm1, ovf);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_acce + 8 * as);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pm0 = fmaxf(pm0, __shfl_xor_sync(0xFFFFFFFFu, pm0, o));
      pm1 = fmaxf(pm1, __shfl_xor_sync(0xFFFFFFFFu, pm1, o));
    }
    if (lane == 0 && pm0 > 0.f) atomicMax(&a.out[0].red[1], (unsigned long long)__double_as_longlong((double)pm0));
    if (lane == 0 && pm1 > 0.f) atomicMax(&a.out[1].red[1], (unsigned long long)__double_as_longlong((double)pm1));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

}  // namespace q2
