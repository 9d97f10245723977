// MS-EDEN post-hoc pass 1, certified fp32 fast path (included by msed.cu).
//
// Two threads own one (row, 128-chunk) unit, 64 elements each.  A CTA stages a
// 64-row x 128-column tile of the logical tensor in shared memory (rows, E^T
// columns or decoded NVFP4 tape columns, random signs already applied), then:
//   y      = H_128 (s . x) in fp32: six in-thread butterfly stages + one
//            partner exchange; |y - y*| <= eps = 7 * 2^-24 * ||x||_1
//            <= 7 * 2^-24 * ||y||_2 (disjoint-support argument + Cauchy-Schwarz).
//   pseudo = E8M3_RTN(gmax * c / s): both ends of the gmax +- eps bracket must
//            round to the same E8M3 value.
//   codes  = E2M1 RTN of y * c / pseudo: the codes of the lower and upper
//            magnitude brackets (y -+ eps, rz products with 1/pseudo * (1 -+ 2^-19))
//            must agree.
//   S      = c <y,y> / sum_g pseudo_g <y, rho>_g with a relative bound dS that
//            pass 2 uses to certify the stochastic scale rounding.
// Chunks that fail any certificate are appended to a list and recomputed by
// the literal float64 fix-up (msed.cu), so outputs equal the reference's.

namespace q2 {

constexpr int F_ROWS = 64, F_THREADS = 128;

struct FastArgs {
  float* dS;           // [R, K/128] relative bound of corr
  uint32_t* listA_n;   // uncertain chunks
  uint32_t* listA;
};

__device__ __forceinline__ int f_swz(int row) { return (row & 7) ^ ((row >> 3) & 7); }

// Stage the tile (signs applied) as bf16 (DT == Q2_BF16, tape) or fp32.
template <int SRC, int DT>
__device__ __forceinline__ void fast_load_tile(const MsedArgs& a, int64_t r0, int64_t c, unsigned char* tile,
                                               const uint32_t* sgnw, bool& bad, int* espan) {
  const int t = threadIdx.x;
  constexpr int ROWB = DT == Q2_BF16 ? 256 : 512;       // bytes per staged row
  if (SRC == Q2_SRC_ROWS) {
    constexpr int SEGS = ROWB / 16;
    constexpr int NV = F_ROWS * SEGS / F_THREADS;
    uint4 q[NV];
#pragma unroll
    for (int it = 0; it < NV; ++it) {                      // issue every load first
      const int v = t + it * F_THREADS, rr = v / SEGS, sg = v % SEGS;
      q[it] = make_uint4(0, 0, 0, 0);
      if (r0 + rr < a.R) {
        const char* src = static_cast<const char*>(a.x) + ((r0 + rr) * a.ld + c * CHUNK) * (DT == Q2_BF16 ? 2 : 4);
        q[it] = __ldg(reinterpret_cast<const uint4*>(src) + sg);
      }
    }
    uint32_t m16 = 0, m32 = 0;
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const int v = t + it * F_THREADS, rr = v / SEGS, sg = v % SEGS;
      uint4 w = q[it];
      if (DT == Q2_BF16) {                               // 8 elements: positions 8sg .. 8sg+7
        const uint4 m = *reinterpret_cast<const uint4*>(sgnw + 4 * sg);
        w.x ^= m.x; w.y ^= m.y; w.z ^= m.z; w.w ^= m.w;
        const uint32_t ww[4] = {w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu, w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu};
#pragma unroll
        for (int i = 0; i < 4; ++i) asm("max.u16x2 %0, %0, %1;" : "+r"(m16) : "r"(ww[i]));
      } else {                                           // 4 elements: positions 4sg .. 4sg+3
        const uint32_t bits = (a.sign[sg >> 3] >> ((4 * sg) & 31)) & 0xF;
        w.x ^= (bits & 1) << 31; w.y ^= ((bits >> 1) & 1) << 31;
        w.z ^= ((bits >> 2) & 1) << 31; w.w ^= ((bits >> 3) & 1) << 31;
        m32 = max(m32, max(max(w.x & 0x7FFFFFFFu, w.y & 0x7FFFFFFFu), max(w.z & 0x7FFFFFFFu, w.w & 0x7FFFFFFFu)));
      }
      *reinterpret_cast<uint4*>(tile + rr * ROWB + ((sg ^ f_swz(rr)) << 4)) = w;
    }
    bad |= (m16 & 0xFFFFu) >= 0x7F80u || (m16 >> 16) >= 0x7F80u || m32 >= 0x7F800000u;
  } else if (SRC == Q2_SRC_COLS) {
    // source [K, R]: a 16-byte source segment holds 8 (bf16) / 4 (fp32) tile rows at one k
    constexpr int EPS = DT == Q2_BF16 ? 8 : 4;
    constexpr int CSEG = F_ROWS / EPS;
    constexpr int NV = CHUNK * CSEG / F_THREADS;
    uint4 q[NV];
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const int v = t + it * F_THREADS, kk = v / CSEG, cs = v % CSEG;
      q[it] = make_uint4(0, 0, 0, 0);
      if (r0 + cs * EPS < a.R) {
        const char* src = static_cast<const char*>(a.x) + ((c * CHUNK + kk) * a.ld + r0 + cs * EPS) * (DT == Q2_BF16 ? 2 : 4);
        q[it] = __ldg(reinterpret_cast<const uint4*>(src));
      }
    }
    uint32_t m16 = 0, m32 = 0;
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const int v = t + it * F_THREADS, kk = v / CSEG, cs = v % CSEG;
      const bool neg = (a.sign[kk >> 5] >> (kk & 31)) & 1;
      const uint32_t ww[4] = {q[it].x, q[it].y, q[it].z, q[it].w};
      if (DT == Q2_BF16) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t w = ww[i] ^ (neg ? 0x80008000u : 0u);
          const uint32_t aw = w & 0x7FFF7FFFu;
          asm("max.u16x2 %0, %0, %1;" : "+r"(m16) : "r"(aw));
          const int ra = cs * 8 + 2 * i, rb = ra + 1;
          *reinterpret_cast<uint16_t*>(tile + ra * ROWB + (((kk >> 3) ^ f_swz(ra)) << 4) + (kk & 7) * 2) = (uint16_t)w;
          *reinterpret_cast<uint16_t*>(tile + rb * ROWB + (((kk >> 3) ^ f_swz(rb)) << 4) + (kk & 7) * 2) = (uint16_t)(w >> 16);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t w = ww[i] ^ (neg ? 0x80000000u : 0u);
          m32 = max(m32, w & 0x7FFFFFFFu);
          const int ra = cs * 4 + i;
          *reinterpret_cast<uint32_t*>(tile + ra * ROWB + (((kk >> 2) ^ f_swz(ra)) << 4) + (kk & 3) * 4) = w;
        }
      }
    }
    bad |= (m16 & 0xFFFFu) >= 0x7F80u || (m16 >> 16) >= 0x7F80u || m32 >= 0x7F800000u;
  } else {
    // NVFP4 tape [K, R]: thread t decodes tape row k = t (64 codes + 4 scales), stores FP4*E4M3 as bf16 (exact)
    const int kk = t;
    const int64_t trow = c * CHUNK + kk;
    const bool neg = (a.sign[kk >> 5] >> (kk & 31)) & 1;
    uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
    uint32_t sfw = 0;
    const bool live = r0 < a.R;
    if (live) {
      const uint4* src = reinterpret_cast<const uint4*>(a.tape_codes + trow * (a.R / 2) + r0 / 2);
      q0 = __ldg(src);
      q1 = __ldg(src + 1);
      sfw = __ldg(reinterpret_cast<const uint32_t*>(a.tape_sf + sf_offset(trow, r0 / 16, kpairs(a.R))));
    }
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    // exponent span of the nonzero group scales per column group: values are
    // multiples of 2^(E_min-11) below 2^(E_max-3), so the fp32 Hadamard of the
    // chunk is exact when E_max - E_min <= 9 (SURVEY E6 tape certificate).
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t s8 = (sfw >> (8 * q)) & 0xFF;
      const int e = max(1, (int)(s8 >> 3));
      int emin = s8 ? e : 64, emax = s8 ? e : -64;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
        emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
      }
      if ((t & 31) == 0) { atomicMin(&espan[2 * q], emin); atomicMax(&espan[2 * q + 1], emax); }
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const uint32_t code = (w[i >> 3] >> (4 * (i & 7))) & 0xF;
      const uint32_t s8 = (sfw >> (8 * (i >> 4))) & 0xFF;
      const float v = fp4_valf(code) * (float)e4m3_val(s8);
      const uint32_t bits = (__float_as_uint(v) >> 16) ^ (neg ? 0x8000u : 0u);
      *reinterpret_cast<uint16_t*>(tile + i * 256 + (((kk >> 3) ^ f_swz(i)) << 4) + (kk & 7) * 2) = (uint16_t)bits;
    }
  }
}

__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t p, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Round a positive normal float to 4 significant bits (E8M3 grid), ties to even.
__device__ __forceinline__ uint32_t rne4(float g) {
  const uint32_t b = __float_as_uint(g);
  return (b + 0x7FFFFu + ((b >> 20) & 1u)) & 0xFFF00000u;
}

// Codes of 8 elements (4 packed pairs) from the magnitude brackets; returns
// both code words; rho - q_lo residual is not needed here (den uses rho * y).
__device__ __forceinline__ void codes8(const uint64_t (&lo)[4], const uint64_t (&hi)[4], uint32_t& wlo, uint32_t& whi) {
  asm("{\n\t.reg .b8 a0, a1, a2, a3, b0, b1, b2, b3;\n\t.reg .f32 x<8>, z<8>;\n\t"
      "mov.b64 {x0, x1}, %2;\n\tmov.b64 {x2, x3}, %3;\n\tmov.b64 {x4, x5}, %4;\n\tmov.b64 {x6, x7}, %5;\n\t"
      "mov.b64 {z0, z1}, %6;\n\tmov.b64 {z2, z3}, %7;\n\tmov.b64 {z4, z5}, %8;\n\tmov.b64 {z6, z7}, %9;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 a0, x1, x0;\n\tcvt.rn.satfinite.e2m1x2.f32 a1, x3, x2;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 a2, x5, x4;\n\tcvt.rn.satfinite.e2m1x2.f32 a3, x7, x6;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, z1, z0;\n\tcvt.rn.satfinite.e2m1x2.f32 b1, z3, z2;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, z5, z4;\n\tcvt.rn.satfinite.e2m1x2.f32 b3, z7, z6;\n\t"
      "mov.b32 %0, {a0, a1, a2, a3};\n\tmov.b32 %1, {b0, b1, b2, b3};\n\t}"
      : "=r"(wlo), "=r"(whi)
      : "l"(lo[0]), "l"(lo[1]), "l"(lo[2]), "l"(lo[3]), "l"(hi[0]), "l"(hi[1]), "l"(hi[2]), "l"(hi[3]));
}
template <int SRC, int DT>
__global__ void __launch_bounds__(F_THREADS, 4) msed_fast1_kernel(MsedArgs a, FastArgs f) {
  extern __shared__ __align__(16) unsigned char fsm[];
  constexpr int ROWB = DT == Q2_BF16 ? 256 : 512;
  unsigned char* tile = fsm;
  uint32_t* sgnw = reinterpret_cast<uint32_t*>(fsm + F_ROWS * ROWB);   // 64 bf16-pair sign words
  const int64_t r0 = (int64_t)blockIdx.x * F_ROWS, c = blockIdx.y;
  int* espan = reinterpret_cast<int*>(fsm + F_ROWS * ROWB + 256);      // [4][min, max]
  if (threadIdx.x < 8) espan[threadIdx.x] = (threadIdx.x & 1) ? -64 : 64;
  if (threadIdx.x < 64) {
    const int e = 2 * threadIdx.x;
    sgnw[threadIdx.x] = (((a.sign[e >> 5] >> (e & 31)) & 1u) << 15) | (((a.sign[(e + 1) >> 5] >> ((e + 1) & 31)) & 1u) << 31);
  }
  __syncthreads();
  bool bad = false;
  fast_load_tile<SRC, DT>(a, r0, c, tile, sgnw, bad, espan);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomic_or_err(a.err, Q2_ERR_NONFINITE);

  const double c_eff = SRC == Q2_SRC_TAPE_COLS ? a.inv_sqrt * (double)*a.tape_scale32 : a.inv_sqrt;
  const float cs = (float)(c_eff / a.s), cef = (float)c_eff;
  const int rr = threadIdx.x >> 1, h = threadIdx.x & 1;
  const int64_t r = r0 + rr;
  const bool live = r < a.R;
  // ---- read the 64 values of this half into packed pairs
  uint64_t y[32];
  if (DT == Q2_BF16) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const uint4 q = *reinterpret_cast<const uint4*>(tile + rr * ROWB + (((8 * h + s) ^ f_swz(rr)) << 4));
      const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) y[4 * s + i] = f2pack(__uint_as_float(ww[i] << 16), __uint_as_float(ww[i] & 0xFFFF0000u));
    }
  } else {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const uint4 q = *reinterpret_cast<const uint4*>(tile + rr * ROWB + (((16 * h + s) ^ f_swz(rr)) << 4));
      y[2 * s] = f2pack(__uint_as_float(q.x), __uint_as_float(q.y));
      y[2 * s + 1] = f2pack(__uint_as_float(q.z), __uint_as_float(q.w));
    }
  }
  // ---- H_64 in-thread.  h = 1: inside each packed pair.
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float p0, p1;
    f2unpack(y[i], p0, p1);
    y[i] = f2pack(p0 + p1, p0 - p1);
  }
  // h = 2 .. 32: pairs of packed pairs (stride hp = h/2 in pair units)
#pragma unroll
  for (int hp = 1; hp < 32; hp <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & hp) continue;
      const uint64_t u = y[i], v = y[i + hp];
      y[i] = add2(u, v);
      y[i + hp] = sub2(u, v);
    }
  }
  // h = 64: partner exchange (thread h=0 holds positions [0,64), h=1 [64,128))
  {
    const float sg = h ? -1.f : 1.f;
    const uint64_t sg2 = f2pack(sg, sg);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, y[i], 1);
      asm("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(y[i]) : "l"(sg2), "l"(o));   // top: o + y, bottom: o - y
    }
  }
  // ---- ||y||^2 and the rotation error bound
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(y[i]));
  float n0, n1;
  f2unpack(acc, n0, n1);
  float num = n0 + n1;
  num += __shfl_xor_sync(0xFFFFFFFFu, num, 1);
  float eps = 7.0f * 0x1p-24f * 1.001f * sqrtf(num) + 0x1p-120f;   // sqrtf: <= 1 ulp
  if (SRC == Q2_SRC_TAPE_COLS && espan[2 * (rr >> 4) + 1] - espan[2 * (rr >> 4)] <= 9) eps = 0.f;
  // ---- per group: pseudo-scale, codes, <y, rho>
  bool unc = !live;
  float den = 0.f, pmx = 0.f;
  uint32_t cw[8];
  uint16_t pbits[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float gm = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float p0, p1;
      f2unpack(y[8 * g + i], p0, p1);
      gm = fmaxf(gm, fmaxf(fabsf(p0), fabsf(p1)));
    }
    const float glo = fmaxf(gm - eps, 0.f) * cs * (1.f - 0x1p-21f), ghi = (gm + eps) * cs * (1.f + 0x1p-21f);
    const uint32_t plo = rne4(glo), phi = rne4(ghi);
    unc |= (plo != phi) | !(glo >= 0x1p-125f) | !(ghi < 0x1p126f);
    const float p = __uint_as_float(phi);
    pmx = fmaxf(pmx, p);
    pbits[g] = (uint16_t)(phi >> 16);
    float inv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(p));
    inv *= cef;
    const float ilo = inv * (1.f - 0x1p-19f), ihi = inv * (1.f + 0x1p-19f);
    const uint64_t il2 = f2pack(ilo, ilo), ih2 = f2pack(ihi, ihi);
    uint64_t dacc = 0;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint64_t lo[4], hi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t v = y[8 * g + 4 * half + i];
        const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
        const uint32_t el = (vl & 0x80000000u) | __float_as_uint(eps), eh = (vh & 0x80000000u) | __float_as_uint(eps);
        const uint64_t e2 = ((uint64_t)eh << 32) | el;                         // copysign(eps, y)
        const uint64_t ylo = sub2(v, e2), yhi = add2(v, e2);
        asm("mul.rz.f32x2 %0, %1, %2;" : "=l"(lo[i]) : "l"(ylo), "l"(il2));
        asm("mul.rz.f32x2 %0, %1, %2;" : "=l"(hi[i]) : "l"(yhi), "l"(ih2));
      }
      uint32_t wlo, whi;
      codes8(lo, hi, wlo, whi);
      unc |= wlo != whi;
      cw[2 * g + half] = wlo;
uint32_t h4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm("{\n\t.reg .b8 t;\n\tcvt.u8.u32 t, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, t;\n\t}" : "=r"(h4[i]) : "r"(wlo >> (8 * i)));
      float dsum0 = 0.f, dsum1 = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float y0, y1, r0, r1;
        f2unpack(y[8 * g + 4 * half + i], y0, y1);
        asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
            : "=f"(r0), "=f"(r1) : "r"(h4[i]));
        dsum0 = fmaf(y0, r0, dsum0);
        dsum1 = fmaf(y1, r1, dsum1);
      }
      dacc = add2(dacc, f2pack(dsum0, dsum1));
    }
    float d0, d1;
    f2unpack(dacc, d0, d1);
    den = fmaf(p, d0 + d1, den);
  }
  den += __shfl_xor_sync(0xFFFFFFFFu, den, 1);
  unc |= __shfl_xor_sync(0xFFFFFFFFu, (int)unc, 1) != 0;
  const float pmx2 = fmaxf(pmx, __shfl_xor_sync(0xFFFFFFFFu, pmx, 1));
  // ---- outputs
  if (live) {
    uint4* cp = reinterpret_cast<uint4*>(a.codes + r * (a.K / 2) + c * 64 + 32 * h);
    cp[0] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
    cp[1] = make_uint4(cw[4], cw[5], cw[6], cw[7]);
    *reinterpret_cast<uint2*>(a.pseudo + r * (a.K / GROUP) + c * 8 + 4 * h) =
        make_uint2(pbits[0] | ((uint32_t)pbits[1] << 16), pbits[2] | ((uint32_t)pbits[3] << 16));
    if (h == 0) {
      // S = c <y,y> / sum_g p_g <y, rho>_g.  Relative bound: |dnum| <= 2 eps sqrt(128 num) + 128 eps^2
      // + 2^-21 num; |dden| <= eps * sum_g p_g * 96 + 2^-20 * |den|-ish accumulation.
      const double S = c_eff * (double)num / (double)den;
      const float pl1 = 8.f * pmx2;   // sum_g p_g over the chunk
      const float dn = (2.f * eps * sqrtf(128.f * num) + 128.f * eps * eps) / num + 0x1p-18f;
      const float dd = (eps * 96.f * pl1) / fabsf(den) + 0x1p-18f;
#ifdef Q2_DEBUG_S
      a.corr[r * (a.K / CHUNK) + c] = (double)den;
      f.dS[r * (a.K / CHUNK) + c] = num;
      return;
#endif
      a.corr[r * (a.K / CHUNK) + c] = S;
      f.dS[r * (a.K / CHUNK) + c] = (num > 0.f && den != 0.f) ? 1.001f * (dn + dd) + 0x1p-20f : 1e30f;
      if (unc || !(num > 0.f) || !(den != 0.f)) f.listA[atomicAdd(f.listA_n, 1u)] = (uint32_t)(r * (a.K / CHUNK) + c);
    }
  }
  // ---- pseudo-scale max (certified chunks only; the fix-up reduces its own exactly)
  float wm = (live && !unc) ? pmx : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xFFFFFFFFu, wm, o));
  if ((threadIdx.x & 31) == 0 && wm > 0.f)
    atomicMax(&a.red[1], (unsigned long long)__double_as_longlong((double)wm));
}

}  // namespace q2
