// MS-EDEN on the tensor cores: certified fp32 fast path, exact fallback
// (included by msed.cu after msed64.cuh, whose float64 helpers it reuses).
//
// Restates ms_eden_quantize (ms_eden.py:116-153, exact and pow2 scale32) and the
// post-hoc schedule pass2(pass1(.)) (posthoc.py:74-125) for bf16 sources E
// (rows: MS(E) along N; cols: MS(E^T) along T; dual: both from ONE read of E)
// and for the NVFP4 tape (MS(dequant(tape)^T): W^T / X^T of linear_graph.py:
// 293-294, 304, 322-323).  Codes and scales equal the reference's bit for bit.
//
// Rotation.  A 128x128 tile of E lands in shared memory by TMA.  The 128-point
// Hadamard of every row chunk and every column chunk is one tcgen05.mma
// kind::f16 each (bf16 operands, fp32 accumulation in TMEM): rows D = X.H,
// columns D = X^T.H (X^T as an MN-major operand of the same tile).  The signs
// of both rotations are folded into X (x' = x * s_col[n] * s_row[t]); a row
// result then carries the extra factor s_row[t] and a column result s_col[n],
// removed by flipping code sign bits.  H[k][j + 64] = H[k][j] * (-1)^[k >= 64],
// so one 64-column half of H serves both output halves (b_negate on K >= 64).
//
// Exactness of the rotation.  Tensor-core fp32 accumulation truncates
// (tools/tc_rot_probe.cu measured |err| up to 13 * 2^-24 * sum|x| on wide-range
// data), so X is split per tile: with E the tile's max binade, "main" values
// (|x| >= 2^(E-8), plus zeros) all lie on the 2^(E-15) grid and every partial
// sum of 128 of them fits 24 bits -> Y1 = H.main is EXACT (probe family
// grid15); "small" values (0 < |x| < 2^(E-8), ~1% of normal data) go to a
// second MMA Y2 = H.small whose error is bounded by 32 * 2^-24 * L1(small)
// (2.5x the worst measured ratio), and L1(small) <= ||H.small||_2 per chunk
// (Parseval), read off the Y2 accumulator.  Chunks without small values are
// exact.
//
// Certification.  Every decision of the reference is taken in fp32 against a
// rigorous margin: the E8M3 pseudo-scale / E4M3 group scale (brackets of gmax),
// the E2M1 codes (brackets of y/d through cvt.rn.satfinite.e2m1x2, the same
// ties-to-even rule), the EDEN factor S (fp32 sums with a running bound) and the
// SR decision u < p (interval of p against the 53-bit draw).  An undecided code
// of an exact chunk is settled in float64 on the spot (y64 = fl64(Y1 * c) is
// the reference's value); any other undecided chunk is deferred to a CTA-local
// list and recomputed at the end of the kernel by tc_literal_warp, a literal
// float64 restatement (FWHT in the reference's butterfly order, numpy's
// summation order, the reference's PRNG draw).  No global fix-up lists.
//
// CTA (one per SM, persistent, 448 threads):
//   warp 0      TMA producer (bf16 tiles) / bulk loads (tape codes + scales)
//   warp 1      TMEM owner; lane 0 issues the MMAs: per tile and orientation
//               two jobs (64-output halves), each Y1 + Y2 = 2 x 64 columns in
//               its own TMEM slot, so the next tile's half-0 MMAs overlap the
//               epilogue's half 1
//   warps 2-5   split warps: tile max, main/small split (tape: decode NVFP4
//               -> bf16 first)
//   warps 6-9   epilogue group 0, warps 10-13 epilogue group 1: one thread
//               per chunk (TMEM lane), half 0 then half 1.  Dual: group o =
//               orientation o.  Single orientation: groups alternate tiles.
namespace q2 {

enum { TC_ABSMAX = 0, TC_QUANT = 1, TC_POSTHOC = 2 };
enum { TC_ROWS = 1, TC_COLS = 2, TC_DUAL = 3, TC_TAPE = 6 };   // bit 0 rows, bit 1 cols, bit 2 tape

constexpr int TC_THREADS = 448;                  // 6 + 8 epilogue warps
constexpr int TC_TILE = 32768;                   // 128 x 128 bf16
constexpr int TC_RAW = 10240;                    // tape raw tile: codes 8 KB + scales 2 KB
constexpr int TC_NRAW = 3;
constexpr int TC_META = 4;                       // metadata ring (tile flags)
constexpr int TC_META_BYTES = 320;               // words: [0] flags, [1..4] rows z0 mask, [5..8] cols z0 mask, [9] tile max
                                                 // bits; bytes 64..191 small count per row chunk, 192..319 per column chunk
constexpr int TC_DEF_CAP = 4096;                 // deferred chunks per CTA before the epilogue must settle them inline
constexpr int TC_PF = 6;                         // tiles prefetched into L2 ahead of the TMA ring
// Shared memory: B operands diag(s) H per orientation (32 KB each) | NS stages of main + small (64 KB each) | tape raw ring |
// metadata ring | deferred list | misc | barriers.  bf16 sources: 3 stages
// (TMA writes the main buffer in place); tape: 2 stages + a 3-deep raw ring.
template <bool TAPE>
struct TcLayout {
  static constexpr int NS = 2;
  static constexpr int OFF_B = 0;                  // [orientation] 128 x 128 bf16, K-major, 128B swizzle
  static constexpr int OFF_ST = TAPE ? 32768 : 65536;
  static constexpr int OFF_RAW = OFF_ST + NS * 2 * TC_TILE;
  static constexpr int OFF_META = OFF_RAW + (TAPE ? TC_NRAW * TC_RAW : 0);
  static constexpr int OFF_DEF = OFF_META + TC_META * TC_META_BYTES;
  static constexpr int OFF_MISC = OFF_DEF + TC_DEF_CAP * 4;
  static constexpr int OFF_S4 = OFF_MISC + 256;    // epilogue group scales: float2 [4][256 threads]
  static constexpr int OFF_BAR = OFF_S4 + 8192;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
};
static_assert(TcLayout<false>::SMEM <= 232448 && TcLayout<true>::SMEM <= 232448, "shared memory budget");

struct TcOut {
  uint8_t* codes; uint8_t* sf; float* scale32;     // final tensor (QUANT) / codes (POSTHOC)
  uint16_t* aw;                                    // POSTHOC: aword per group [R, K/16]
  unsigned long long* red;                         // [0] |y| max f64 bits, [1] pseudo max f64 bits
  uint32_t sign[4];
  uint64_t sr_head;
  int64_t R, K;                                    // logical tensor
};

struct TcArgs {
  TcOut o[2];                                      // [0] rows orientation, [1] cols orientation
  const uint16_t* x; int64_t ld;                   // bf16 source [T, N] (ld elements)
  const uint8_t* tape_codes; const uint8_t* tape_sf; const float* tape_scale32;  // tape [T = Kt, N = Rt]
  int64_t T, N;
  int tiles_r, tiles_c;                            // T/128, N/128
  FastDiv fc;
  double s, inv_sqrt;
  uint32_t* err;
  int dbg;                                         // timing probes: 1 epilogue drains only, 2 + no split work
};
// chunks processed / deferred to the literal path since load (q2_msed_stats)
__device__ unsigned long long g_tc_stats[2];

__device__ __forceinline__ uint32_t tc_sw(int row, int piece) { return row * 128 + ((piece ^ (row & 7)) << 4); }

// E2M1 codes of 8 fp32 values (byte i = values 2i, 2i+1, low nibble = even)
__device__ __forceinline__ uint32_t e2m1x8(const float* v) {
  uint32_t w;
  asm("{\n\t.reg .b8 a0, a1, a2, a3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 a0, %2, %1;\n\tcvt.rn.satfinite.e2m1x2.f32 a1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 a2, %6, %5;\n\tcvt.rn.satfinite.e2m1x2.f32 a3, %8, %7;\n\t"
      "mov.b32 %0, {a0, a1, a2, a3};\n\t}"
      : "=r"(w) : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
  return w;
}
// signed E2M1 values of the 8 codes of a word as 4 packed f16x2 (value 2i in the low half)
__device__ __forceinline__ void e2m1x8_f16s(uint32_t w, uint32_t (&h)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{\n\t.reg .b8 t;\n\tcvt.u8.u32 t, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, t;\n\t}" : "=r"(h[i]) : "r"(w >> (8 * i)));
}
// |E2M1 value| of the 8 codes of a word as 4 packed f16x2 (value 2i in the low half)
__device__ __forceinline__ void e2m1x8_f16(uint32_t w, uint32_t (&h)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{\n\t.reg .b8 t;\n\tcvt.u8.u32 t, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, t;\n\t}" : "=r"(h[i]) : "r"((w >> (8 * i)) & 0x77u));
}
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t p, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(p)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float amax3(float a, float b, float c) {
  float r;
  asm("max.abs.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float amin3(float a, float b, float c) {
  float r;
  asm("min.abs.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void tmem_ld16(uint32_t* r, uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// ---------------------------------------------------------------------------
// Literal float64 restatement of one chunk by one warp (the deferred path).
// Lane l holds elements 4l..4l+3.  y = FWHT(x * signs) * c with every butterfly
// output one IEEE add/sub of the same two operands as the reference's loop
// (_kernels.py:175-187), then MODE's outputs exactly as the reference computes
// them: scales (posthoc.py:82-83 / quantizers.py:177-178), codes (_nb_rtn),
// the EDEN factor in numpy's 8-accumulator order (ms_eden.py:75-83), the
// reference's PRNG draw and SR (formats.py:174-201).  Returns (warp-uniform)
// max |y| bits (ABSMAX) or the pseudo-scale max bits (POSTHOC).
__device__ __noinline__ uint64_t tc_literal_warp(const TcArgs& a, int MODE, int o, int tile, int rt, double scale32,
                                                 bool* ovf, bool* nanscale) {
  const int lane = threadIdx.x & 31;
  const int tr = (int)a.fc.div((uint32_t)tile), tcl = tile - tr * a.tiles_c;
  const TcOut& out = a.o[o];
  const bool tape = a.tape_codes != nullptr;
  double y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = 4 * lane + i;
    const int64_t t = o == 0 ? (int64_t)tr * 128 + rt : (int64_t)tr * 128 + k;
    const int64_t n = o == 0 ? (int64_t)tcl * 128 + k : (int64_t)tcl * 128 + rt;
    double v;
    if (!tape) {
      v = (double)bf16_to_f32(a.x[t * a.ld + n]);
    } else {       // dequant(tape)[t][n] = FP4 * (E4M3 * scale32) (quantizers.py:315-323)
      const uint8_t cb = a.tape_codes[t * (a.N / 2) + (n >> 1)];
      const uint32_t code = (n & 1) ? (cb >> 4) : (cb & 15u);
      const uint8_t s8 = a.tape_sf[sf_offset(t, n >> 4, sf_kblocks(a.N))];
      v = __dmul_rn(fp4_val(code), __dmul_rn(e4m3_val(s8), (double)__ldg(a.tape_scale32)));
    }
    y[i] = ((out.sign[k >> 5] >> (k & 31)) & 1u) ? -v : v;
  }
  {
    double u;
    u = y[0]; y[0] = __dadd_rn(u, y[1]); y[1] = __dsub_rn(u, y[1]);     // h = 1
    u = y[2]; y[2] = __dadd_rn(u, y[3]); y[3] = __dsub_rn(u, y[3]);
    u = y[0]; y[0] = __dadd_rn(u, y[2]); y[2] = __dsub_rn(u, y[2]);     // h = 2
    u = y[1]; y[1] = __dadd_rn(u, y[3]); y[3] = __dsub_rn(u, y[3]);
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {                                     // h = 4m: partner lane ^ m
    const bool lower = (lane & m) == 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double p = __shfl_xor_sync(0xFFFFFFFFu, y[i], m);
      y[i] = lower ? __dadd_rn(y[i], p) : __dsub_rn(p, y[i]);           // (a + b, a - b), a the lower element
    }
  }
  uint64_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    y[i] = __dmul_rn(y[i], a.inv_sqrt);
    m = umax64(m, dbits(y[i]) & 0x7FFFFFFFFFFFFFFFull);
  }
  if (MODE == TC_ABSMAX) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = umax64(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
    return m;
  }
  // group g = lane / 4: exact group max from the abs bits
  m = umax64(m, __shfl_xor_sync(0xFFFFFFFFu, m, 1));
  m = umax64(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
  const double gmax = bitsd(m);
  double d, s4;
  if (MODE == TC_POSTHOC) {
    bool o2 = false;
    d = e8m3_rtn(__ddiv_rn(gmax, a.s), &o2);
    if (o2) *ovf = true;
    s4 = d;
  } else {
    double xq = scale32 == 0.0 ? 0.0 : __ddiv_rn(gmax, __dmul_rn(scale32, a.s));
    if (isnan(xq)) { *nanscale = true; xq = 0.0; }
    s4 = e4m3_val(e4m3_rtn(xq));
    d = __dmul_rn(s4, scale32);
  }
  uint32_t cw = 0;
  double pn[4], pd[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t c = d > 0.0 ? rtn_code_exact(y[i], d) : 0u;
    cw |= c << (4 * i);
    pn[i] = __dmul_rn(y[i], y[i]);
    pd[i] = __dmul_rn(y[i], __dmul_rn(fp4_val(c), d));
  }
  // numpy's sum of 128: r[j] = p[j] + p[8 + j] + ... in order, j = k % 8 lives in lanes
  // 2k' + (j >> 2), register j & 3; lane j < 8 accumulates r[j]
  double rn = 0.0, rd = 0.0;
#pragma unroll 1
  for (int kp = 0; kp < 16; ++kp) {
    double vn = 0.0, vd = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int src = 2 * kp + ((lane >> 2) & 1);
      const double a0 = __shfl_sync(0xFFFFFFFFu, pn[i], src), a1 = __shfl_sync(0xFFFFFFFFu, pd[i], src);
      if ((lane & 3) == i) { vn = a0; vd = a1; }
    }
    rn = kp == 0 ? vn : __dadd_rn(rn, vn);
    rd = kp == 0 ? vd : __dadd_rn(rd, vd);
  }
  // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
#pragma unroll
  for (int st = 1; st < 8; st <<= 1) {
    const double on = __shfl_down_sync(0xFFFFFFFFu, rn, st), od = __shfl_down_sync(0xFFFFFFFFu, rd, st);
    rn = __dadd_rn(rn, on);
    rd = __dadd_rn(rd, od);
  }
  const double num = __shfl_sync(0xFFFFFFFFu, rn, 0), den = __shfl_sync(0xFFFFFFFFu, rd, 0);
  const bool okS = (fabs(den) >= __dmul_rn(1e-30, num)) && (num > 0.0);
  const double S = okS ? __ddiv_rn(num, den) : 1.0;
  const int64_t r = o == 0 ? (int64_t)tr * 128 + rt : (int64_t)tcl * 128 + rt;
  const int ci = o == 0 ? tcl : tr;
  reinterpret_cast<uint16_t*>(out.codes + r * (out.K / 2) + (int64_t)ci * 64)[lane] = (uint16_t)cw;
  const int64_t g0 = r * (out.K / GROUP) + (int64_t)ci * 8;
  // group g's scales from lane 4g; lanes 0..7 round group `lane`
  const double dg = __shfl_sync(0xFFFFFFFFu, d, 4 * (lane & 7)), sg = __shfl_sync(0xFFFFFFFFu, s4, 4 * (lane & 7));
  uint64_t pm = dbits(dg);
  uint32_t code = 0;
  if (lane < 8) {
    const uint64_t u53 = mix64(out.sr_head ^ ((uint64_t)(g0 + lane) + GOLDEN)) >> 11;
    if (MODE == TC_POSTHOC) {
      out.aw[g0 + lane] = pack_aword(__dmul_rn(S, dg), u53);
    } else {
      bool o2 = false;
      code = scale32 == 0.0 ? 0u : sr_code_direct(__dmul_rn(S, sg), u53, &o2);
      if (o2) *ovf = true;
    }
  }
  if (MODE == TC_QUANT) {
    uint32_t w = code << (8 * (lane & 3));
    w |= __shfl_xor_sync(0xFFFFFFFFu, w, 1);
    w |= __shfl_xor_sync(0xFFFFFFFFu, w, 2);
    const int64_t kb = sf_kblocks(out.K);
    if (lane == 0 || lane == 4)
      *reinterpret_cast<uint32_t*>(out.sf + sf_offset(r, (int64_t)ci * 8 + lane, kb)) = w;
  }
#pragma unroll
  for (int off = 1; off < 8; off <<= 1) pm = umax64(pm, __shfl_xor_sync(0xFFFFFFFFu, pm, off));
  return pm;
}

// scale32 of the QUANT pass from the reductions of the first pass:
// exact   (float)(absmax / (s * 256))        quantizers.py:177
// pow2    2^k, k from E8M3(absmax / s)        ms_eden.py:86-113 (max of rounded = rounded max)
__device__ __forceinline__ double tc_scale32(const TcOut& o, double s, int pow2) {
  const double amax = bitsd(o.red[0]);
  if (!(amax > 0.0)) return 0.0;
  if (!pow2) return (double)__double2float_rn(__ddiv_rn(amax, __dmul_rn(s, 256.0)));
  bool ovf = false;
  const double pmax = e8m3_rtn(__ddiv_rn(amax, s), &ovf);
  int e;
  const double m = frexp(pmax / 256.0, &e);
  return ldexp(1.0, (m == 0.5) ? e - 1 : e);
}

// E4M3 code of an SR word: normal range by one shift-add of the word, aword_code otherwise
__device__ __forceinline__ uint32_t aword_code_fast(uint32_t w, int k, bool* ovf) {
  const int E = (int)(w >> 7) - 256 - k;
  if ((w >> 7) != 0u && E >= -6 && E < 8) return (w >> 4) + ((w >> 3) & 1u) - ((uint32_t)(249 + k) << 3);
  return aword_code(w, k, ovf);
}

template <int SRC, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1) msed_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ TcArgs a,
                                                                 int pow2) {
  constexpr bool DUAL = SRC == TC_DUAL, TAPE = SRC == TC_TAPE;
  constexpr int ONLY = SRC == TC_ROWS ? 0 : 1;                // orientation of single-orientation sources
  constexpr int NB = DUAL ? 2 : 1;                            // orientations (B operands, accumulators) per tile
  using LY = TcLayout<TAPE>;
  constexpr int NS = LY::NS;
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char* smem = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);   // stays a shared-space pointer (LDS/STS, not generic LD/ST)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LY::OFF_BAR);
  const uint32_t bar_full = smem_u32(bars);                   // [3] TMA landed (main stage / tape raw slot)
  const uint32_t bar_rawe = smem_u32(bars + 3);               // [3] tape raw slot decoded (4 warps)
  const uint32_t bar_split = smem_u32(bars + 6);              // [NS] split done (4 warps)
  const uint32_t bar_sempty = smem_u32(bars + 9);             // [NS] stage free (MMA commit)
  const uint32_t bar_tfull = smem_u32(bars + 12);             // [4] TMEM slot (buffer b, half h) = 2b + h ready
  const uint32_t bar_tempty = smem_u32(bars + 16);            // [4] TMEM slot drained (4 warps)
  const uint32_t bar_mfull = smem_u32(bars + 20);             // [4] tile metadata written (4 warps)
  const uint32_t bar_mempty = smem_u32(bars + 24);            // [4] tile metadata read (8 warps)
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + LY::OFF_MISC);
  // misc: [0] deferred count, [1] tmem base, [2..3] pmax (f32 bits, per orientation), [4..5] running L,
  //       [8..11] split-warp maxima (tape: scale ranges), [12] flags (bit0 nonfinite, bit1 ovf, bit2
  //       nanscale), [14..17] split-warp "any small" flags
  uint32_t* deflist = reinterpret_cast<uint32_t*>(smem + LY::OFF_DEF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_r * a.tiles_c;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_rawe + 8 * s, 4);
      mbar_init(bar_split + 8 * s, 4);
      mbar_init(bar_sempty + 8 * s, 1);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(bar_tfull + 8 * b, 1);
      mbar_init(bar_tempty + 8 * b, 4);
      mbar_init(bar_mfull + 8 * b, 4);
      mbar_init(bar_mempty + 8 * b, 8);
    }
    for (int i = 0; i < 24; ++i) misc[i] = 0;
    mbar_fence_init();
  }
  // B operands: B_o[j][k] = s_o[k] H[k][j] (the sign vector of orientation o folded into the
  // Hadamard matrix), bf16 +-1, K-major rows j, two 64-k slabs of 16 KB, 128B swizzle
  for (int i = threadIdx.x; i < NB * 128 * 16; i += TC_THREADS) {
    const int bi = i >> 11, j = (i >> 4) & 127, p = i & 15;
    const uint32_t* sg = a.o[DUAL ? bi : ONLY].sign;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k0 = p * 8 + 2 * e, k1 = k0 + 1;
      const uint32_t n0 = (__popc(k0 & j) + (sg[k0 >> 5] >> (k0 & 31))) & 1u;
      const uint32_t n1 = (__popc(k1 & j) + (sg[k1 >> 5] >> (k1 & 31))) & 1u;
      const uint32_t one = TAPE ? 0x3C00u : 0x3F80u, mone = TAPE ? 0xBC00u : 0xBF80u;   // +-1 in f16 / bf16
      w[e] = (n0 ? mone : one) | ((n1 ? mone : one) << 16);
    }
    *reinterpret_cast<uint4*>(smem + LY::OFF_B + bi * 32768 + (p >> 3) * 16384 + tc_sw(j, p & 7)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(misc + 1)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  pdl_trigger();
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[1];

  double qscale[2] = {0.0, 0.0};                              // QUANT: scale32 per orientation
  if (MODE == TC_QUANT) {
#pragma unroll
    for (int o = 0; o < 2; ++o)
      if ((SRC >> o) & 1) qscale[o] = tc_scale32(a.o[o], a.s, pow2);
  }
  bool ovf = false, nanscale = false;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
      int it = 0;
      // L2 prefetch runs TC_PF tiles ahead of the TMA ring: HBM needs ~25 MB in flight at
      // full bandwidth, more than 148 x NS shared-memory stages hold
      auto prefetch = [&](int tp) {
        if (tp >= ntiles) return;
        const int pr = (int)a.fc.div((uint32_t)tp), pc = tp - pr * a.tiles_c;
        if (!TAPE) {
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(&tm)),
                       "r"(pc * 128), "r"(pr * 128) : "memory");
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(&tm)),
                       "r"(pc * 128 + 64), "r"(pr * 128) : "memory");
        } else {
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(&tm)),
                       "r"(pc * 64), "r"(pr * 128) : "memory");
        }
      };
      for (int i = 0; i < TC_PF; ++i) prefetch(blockIdx.x + i * gridDim.x);
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int tr = (int)a.fc.div((uint32_t)t), tcl = t - tr * a.tiles_c;
        prefetch(t + TC_PF * gridDim.x);
        if (!TAPE) {
          const int s = it % NS;
          if (it >= NS) mbar_wait_sleep(bar_sempty + 8 * s, ((it / NS) - 1) & 1);
          const uint32_t fb = bar_full + 8 * s;
          const uint32_t dst = smem_u32(smem + LY::OFF_ST + s * 2 * TC_TILE);
          mbar_expect_tx(fb, TC_TILE);
          tma_load_2d(dst, &tm, tcl * 128, tr * 128, fb);
          tma_load_2d(dst + 16384, &tm, tcl * 128 + 64, tr * 128, fb);
        } else {
          const int s = it % TC_NRAW;
          if (it >= TC_NRAW) mbar_wait_sleep(bar_rawe + 8 * s, ((it / TC_NRAW) - 1) & 1);
          const uint32_t fb = bar_full + 8 * s;
          const uint32_t dst = smem_u32(smem + LY::OFF_RAW + s * TC_RAW);
          mbar_expect_tx(fb, 8192 + 2048);
          tma_load_2d(dst, &tm, tcl * 64, tr * 128, fb);                  // codes: 128 tape rows x 64 B
          const int64_t kb = sf_kblocks(a.N);
          bulk_load(dst + 8192, a.tape_sf + ((((int64_t)tr >> 1) * kb + 2 * tcl) << 10), 2048, fb);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------------- MMA
    // whole warp in the loop, one elected lane issues (warp-uniform descriptors stay in
    // uniform registers; a lone-lane loop paid an elect/R2UR sequence per MMA)
    {
      // M = 128 (chunks), N = 64 (one output half), bf16 x bf16 -> f32
      const uint32_t ab_fmt = TAPE ? 0u : 1u;                 // f16 (tape) / bf16 operands
      const uint32_t idk = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      int it = 0;
      uint32_t ubuf0 = 0, ubuf1 = 0;                         // uses of the two accumulator buffers
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % NS;
        mbar_wait_sleep(bar_split + 8 * s, (it / NS) & 1);
        tc_fence_after();
        const uint32_t flags = reinterpret_cast<const uint32_t*>(smem + LY::OFF_META + (it % TC_META) * TC_META_BYTES)[0];
        const bool has_small = flags & 1u;
        const uint32_t mainb = smem_u32(smem + LY::OFF_ST + s * 2 * TC_TILE), smallb = mainb + TC_TILE;
        // buffer b (dual: orientation; single orientation: tile parity) = 256 TMEM columns, two
        // slots 2b + h of 128 columns: Y1 = H.main (64) | Y2 = H.small (64) of output half h
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
#pragma unroll 1
          for (int jj = 0; jj < NB; ++jj) {
            const int o = DUAL ? jj : ONLY, buf = DUAL ? jj : (it & 1);
            const uint32_t ub = buf ? ubuf1 : ubuf0;
            if (ub > 0) mbar_wait_sleep(bar_tempty + 8 * (2 * buf + h), (ub - 1) & 1);
            if (h == 1) { if (buf) ++ubuf1; else ++ubuf0; }
            tc_fence_after();
            const uint32_t id = idk | (o ? (1u << 15) : 0u);
            const uint32_t bb = smem_u32(smem + LY::OFF_B + jj * 32768) + 8192 * h;   // B rows 64h..64h+63
            if (elect_one()) {
#pragma unroll
              for (int part = 0; part < 2; ++part) {
                if (part == 1 && (!has_small || a.dbg == 3)) break;
                if (a.dbg == 4) break;
                const uint32_t ab = part ? smallb : mainb;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                  const uint64_t ad = o == 0 ? desc_sw128(ab + (kk >> 2) * 16384 + (kk & 3) * 32)
                                             : desc_mn_sw128(ab + kk * 2048, 16384, 1024);
                  const uint64_t bd = desc_sw128(bb + (kk >> 2) * 16384 + (kk & 3) * 32);
                  tc_mma_f16(tmem + 256 * buf + 128 * h + 64 * part, ad, bd, id, kk > 0);
                }
              }
              tc_commit(bar_tfull + 8 * (2 * buf + h));
            }
            __syncwarp();
          }
        }
        if (elect_one()) tc_commit(bar_sempty + 8 * s);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------- split
    const int sw = warp - 2, st = threadIdx.x - 64;          // split thread 0..127
    const int piece = st & 7;                                 // fixed 16-B column piece
    // (the rotation signs live in the B operands: the split only separates main / small)
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % NS, m = it % TC_META;
      unsigned char* mainp = smem + LY::OFF_ST + s * 2 * TC_TILE;
      unsigned char* smallp = mainp + TC_TILE;
      uint32_t* metau = reinterpret_cast<uint32_t*>(smem + LY::OFF_META + m * TC_META_BYTES);
      if (!TAPE) mbar_wait_sleep(bar_full + 8 * s, (it / NS) & 1);
      if (it >= TC_META) mbar_wait_sleep(bar_mempty + 8 * m, ((it / TC_META) - 1) & 1);
      if (TAPE) {
        // decode the NVFP4 tape tile: tape row kr = st, 128 tape columns; FP4 * E4M3 has
        // <= 6 significant bits (exact in f16 and bf16); the row's rotation sign applied
        const int rs = it % TC_NRAW;
        mbar_wait_sleep(bar_full + 8 * rs, (it / TC_NRAW) & 1);
        if (it >= NS) mbar_wait_sleep(bar_sempty + 8 * s, ((it / NS) - 1) & 1);
        const int tr = (int)a.fc.div((uint32_t)t);
        const unsigned char* raw = smem + LY::OFF_RAW + rs * TC_RAW;
        const int kr = st, L = kr & 31;
        uint32_t scmax = 0u, scmin = 255u;                        // E4M3 scale codes of the row (min over nonzero)
#pragma unroll 1
        for (int qd = 0; qd < (a.dbg == 6 ? 0 : 4); ++qd) {                       // 32 tape columns per quarter
          const uint4 cw = *reinterpret_cast<const uint4*>(raw + kr * 64 + qd * 16);
          const uint32_t sfw = *reinterpret_cast<const uint32_t*>(raw + 8192 + (qd >> 1) * 1024 + ((L >> 3) << 8) +
                                                                  ((tr & 1) << 7) + ((L & 7) << 4) + ((kr >> 5) << 2));
          uint32_t sc[2];
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const uint32_t s8 = (sfw >> (8 * (2 * (qd & 1) + g))) & 0xFF;
            scmax = max(scmax, s8);
            scmin = min(scmin, s8 ? s8 : 255u);
            asm("{\n\t.reg .b16 t;\n\tmov.b16 t, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, t;\n\t}" : "=r"(sc[g])
                : "h"((unsigned short)(s8 | (s8 << 8))));
          }
          const uint32_t ww[4] = {cw.x, cw.y, cw.z, cw.w};
          // the tape operand is f16: FP4 x E4M3 (2^-10 .. 2688, <= 6 significant bits) is exact
          uint32_t ov[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            uint32_t hv;
            asm("{\n\t.reg .b8 t;\n\tcvt.u8.u32 t, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, t;\n\t}" : "=r"(hv) : "r"(ww[i >> 2] >> (8 * (i & 3))));
            // fma with +0 turns the -0 of code 8 into +0 (FP4_VALUES[8] = 0.0)
            asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(ov[i]) : "r"(hv), "r"(sc[i >> 3]), "r"(0u));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(mainp + (qd >> 1) * 16384 + tc_sw(kr, 4 * (qd & 1) + j)) =
                make_uint4(ov[4 * j], ov[4 * j + 1], ov[4 * j + 2], ov[4 * j + 3]);
          if (kr == 0) {            // z0 of the 32 chunks (tile columns) whose input 0 is in this quarter
            uint32_t zm = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              zm |= (((ov[i] & 0x7FFFu) == 0u ? 1u : 0u) | ((ov[i] & 0x7FFF0000u) == 0u ? 2u : 0u)) << (2 * i);
            metau[5 + qd] = (a.o[1].sign[0] & 1u) ? zm : 0u;   // tape zeros are +0: -0 iff s[0] < 0
          }
        }
        scmax = __reduce_max_sync(0xFFFFFFFFu, scmax);
        scmin = __reduce_min_sync(0xFFFFFFFFu, scmin);
        if (lane == 0) misc[8 + sw] = (scmax << 8) | scmin;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_rawe + 8 * rs);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // No small values are possible when the tile's nonzero scales span <= 5 binades: every
        // nonzero value is >= 0.5 E(min) while the split threshold is <= 6 E(max) / 2^10 (E(max) /
        // E(min) < 64 < 85).  Then the split passes are skipped: main = the decoded tile.
        uint32_t cmax = 0u, cmin = 255u;
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) { cmax = max(cmax, misc[8 + w4] >> 8); cmin = min(cmin, misc[8 + w4] & 255u); }
        const bool no_small = cmax == 0u || (cmin >= 8u && (cmax >> 3) - (cmin >> 3) <= 5u);
        asm volatile("bar.sync 1, 128;" ::: "memory");          // misc[8..11] is reused by pass 1
        if (no_small && a.dbg < 2) {
          if (st == 0) { metau[0] = 0u; metau[9] = 0u; }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (lane == 0) { mbar_arrive(bar_split + 8 * s); mbar_arrive(bar_mfull + 8 * m); }
          continue;
        }
      }
      if (a.dbg >= 2) {
        if (st == 0) metau[0] = 1u;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (lane == 0) { mbar_arrive(bar_split + 8 * s); mbar_arrive(bar_mfull + 8 * m); }
        continue;
      }
      // pass 1: tile max of |x| (bf16 bits), and the z0 masks: chunk input 0 (rows: column 0,
      // cols: row 0 of the tile) is -0 after the orientation's sign s[0] (see the epilogue)
      uint32_t mx = 0, zrow = 0, zcol = 0;
      // x * s[0] == -0 iff x == (s[0] < 0 ? +0 : -0)
      const uint32_t sneg0 = (a.o[0].sign[0] & 1u) ? 0u : 0x8000u, sneg1 = (a.o[1].sign[0] & 1u) ? 0u : 0x8000u;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int p = st + 128 * i, sl = p >> 10, row = (p & 1023) >> 3;
        const uint4 v = *reinterpret_cast<const uint4*>(mainp + sl * 16384 + tc_sw(row, piece));
        if (!TAPE && sl == 0 && piece == 0 && (v.x & 0xFFFFu) == sneg0) zrow |= 1u << (i & 31);
        if (!TAPE && row == 0) {
          const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (((vv[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) == sneg1) zcol |= 1u << (8 * (i >> 3) + e);
        }
        uint32_t m2;
        asm("max.u16x2 %0, %1, %2;" : "=r"(m2) : "r"(v.x & 0x7FFF7FFFu), "r"(v.y & 0x7FFF7FFFu));
        asm("max.u16x2 %0, %0, %1;" : "+r"(m2) : "r"(v.z & 0x7FFF7FFFu));
        asm("max.u16x2 %0, %0, %1;" : "+r"(m2) : "r"(v.w & 0x7FFF7FFFu));
        asm("max.u16x2 %0, %0, %1;" : "+r"(mx) : "r"(m2));
      }
      mx = max(mx & 0xFFFFu, mx >> 16);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
      if (lane == 0) misc[8 + sw] = mx;
      if (!TAPE && st < 8) metau[1 + st] = 0u;
      if (st < 32) metau[48 + st] = 0u;                          // column small counts (atomic byte sums)
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (!TAPE) {
        // rows: thread st (piece 0) saw rows st/8 + 16 i at bit i; cols: thread st < 8 saw columns
        // 64 (i/8) + 8 st + e at bit 8 (i/8) + e
        if (zrow)
          for (int i = 0; i < 8; ++i)
            if ((zrow >> i) & 1u) { const int r = st / 8 + 16 * i; atomicOr(&metau[1 + (r >> 5)], 1u << (r & 31)); }
        if (zcol)
          for (int b = 0; b < 16; ++b)
            if ((zcol >> b) & 1u) { const int c = 64 * (b >> 3) + 8 * st + (b & 7); atomicOr(&metau[5 + (c >> 5)], 1u << (c & 31)); }
      }
      const uint32_t M = max(max(misc[8], misc[9]), max(misc[10], misc[11]));
      // biased binade of the tile max (bf16: 8-bit exponent at bit 7; the tape's f16: 5 bits at 10).
      // Tape values are finite and >= 2^-10 (never tiny).
      const int Ef = TAPE ? (int)(M >> 10) : (int)(M >> 7);
      const bool nonfin = !TAPE && M >= 0x7F80u;
      const bool tiny = !TAPE && M != 0u && Ef < 80;             // tile below 2^-47: literal path for all chunks
      // main values lie on the 2^(E-15) grid: bf16 (8 significant bits) from 2^(E-8), the decoded
      // tape (FP4 x E4M3: <= 6 significant bits) from 2^(E-10)
      constexpr int SPLIT = TAPE ? 10 : 8;
      const uint32_t thr = Ef >= SPLIT + 1 ? (uint32_t)(Ef - SPLIT) << (TAPE ? 10 : 7) : 0u;
      const uint32_t thr2 = thr | (thr << 16);
      // pass 2: main/small split (the absmax pass rotates the raw tile: no split), and the
      // number of nonzero small values of every row and column chunk (byte counters: the
      // flag bytes of four elements at a time)
      uint32_t anys = 0, rc[8], cc[2][2] = {{0u, 0u}, {0u, 0u}};
#pragma unroll
      for (int j = 0; j < 8; ++j) rc[j] = 0u;
#pragma unroll
      for (int i = 0; i < (MODE == TC_ABSMAX ? 0 : 16); ++i) {
        const int p = st + 128 * i, sl = p >> 10, row = (p & 1023) >> 3;
        const uint32_t off = sl * 16384 + tc_sw(row, piece);
        const uint4 v = *reinterpret_cast<const uint4*>(mainp + off);
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
        uint32_t mo[4], so[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t w = vv[e];
          // big: |x| >= 2^(E-8) per half (bit 15 / 31 of (|x| | 0x8000) - thr)
          // bit 15 / 31 of (|x| | 0x8000) - thr: 1 = big; PRMT replicates each half's sign byte
          const uint32_t tb = (w | 0x80008000u) - thr2;
          uint32_t mask;
          asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(mask) : "r"(tb));
          mo[e] = w & mask;
          so[e] = w & ~mask;
          anys |= so[e];
        }
        *reinterpret_cast<uint4*>(mainp + off) = make_uint4(mo[0], mo[1], mo[2], mo[3]);
        *reinterpret_cast<uint4*>(smallp + off) = make_uint4(so[0], so[1], so[2], so[3]);
        uint32_t t4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t4[e] = ((so[e] & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x80008000u;   // nonzero small
        uint32_t fa, fb;                                         // flag bytes of elements 0-3 / 4-7
        asm("prmt.b32 %0, %1, %2, 0x7531;" : "=r"(fa) : "r"(t4[0]), "r"(t4[1]));
        asm("prmt.b32 %0, %1, %2, 0x7531;" : "=r"(fb) : "r"(t4[2]), "r"(t4[3]));
        fa = (fa >> 7) & 0x01010101u;
        fb = (fb >> 7) & 0x01010101u;
        rc[i & 7] += __popc(fa | (fb << 1));
        cc[i >> 3][0] += fa;
        cc[i >> 3][1] += fb;
      }
      if (MODE != TC_ABSMAX) {
        // rows st/8 + 16 j: the eight lanes 8k..8k+7 hold their pieces
        uint8_t* const rcnt = reinterpret_cast<uint8_t*>(metau + 16);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t v = rc[j];
          v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
          v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
          v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
          if (piece == 0) rcnt[st / 8 + 16 * j] = (uint8_t)v;
        }
        // columns 64 sl + 8 piece + e: lanes piece + 8 m of the four warps (byte sums <= 128)
#pragma unroll
        for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 2; ++b2) {
            uint32_t v = cc[a2][b2];
            v += __shfl_xor_sync(0xFFFFFFFFu, v, 8);
            v += __shfl_xor_sync(0xFFFFFFFFu, v, 16);
            if (lane < 8 && v) atomicAdd(&metau[48 + (a2 * 8 + piece) * 2 + b2], v);
          }
      }
      const bool anyw = __any_sync(0xFFFFFFFFu, (anys & 0x7FFF7FFFu) != 0u);
      // separate slots from the maxima in misc[8..11]: a warp past pass 2 must not overwrite a
      // maximum another split warp has not read yet (the absmax pass has no pass 2 in between)
      if (lane == 0) misc[14 + sw] = anyw ? 1u : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (st == 0) {
        const bool hs = (misc[14] | misc[15] | misc[16] | misc[17]) != 0u;
        metau[0] = (hs ? 1u : 0u) | (nonfin ? 2u : 0u) | (tiny ? 4u : 0u);
        metau[9] = M;                                            // tile max |x| bits (bf16 / the tape's f16)
        if (nonfin) misc[12] |= 1u;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane == 0) {
        mbar_arrive(bar_split + 8 * s);
        mbar_arrive(bar_mfull + 8 * m);
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // 8 warps.  Warp e = warp - 6 reads TMEM lanes 32q..32q+31 (q = warp & 3; one lane = one
    // chunk rt) of buffer grp = e >> 2: half 0 (groups 0-3) from slot 2 grp, then half 1
    // (groups 4-7) from slot 2 grp + 1; each slot is released as soon as it is read, so the
    // MMAs of the next tile overlap the rest of this one.  Dual: grp = orientation.  Single
    // orientation: grp = tile parity.
    const int e = warp - 6, q = warp & 3, grp = e >> 2;
    const int rt = 32 * q + lane;
    const int o = DUAL ? grp : ONLY;
    // per-thread constants of this thread's orientation (no dynamic indexing of the params)
    uint8_t* const ocodes = o ? a.o[1].codes : a.o[0].codes;
    uint8_t* const osf = o ? a.o[1].sf : a.o[0].sf;
    uint16_t* const oaw = o ? a.o[1].aw : a.o[0].aw;
    const uint64_t ohead = o ? a.o[1].sr_head : a.o[0].sr_head;
    const uint32_t oK = (uint32_t)(o ? a.o[1].K : a.o[0].K);
    const uint32_t okb = (oK + 63) / 64;
    const int b = grp;                                        // TMEM buffer: slots 2b (half 0), 2b + 1 (half 1)
    float2* const s4s = reinterpret_cast<float2*>(smem + LY::OFF_S4) + (threadIdx.x - 192) * 4;   // [4] this thread
    uint32_t use = 0;
    const double C64 = TAPE ? __dmul_rn((double)__ldg(a.tape_scale32), a.inv_sqrt) : a.inv_sqrt;
    const float C = (float)C64;
    const float invC = __frcp_ru(C) * 1.0001f;                          // upper bound of 1/C
    const float is_lo = __frcp_rd((float)a.s), is_hi = __frcp_ru((float)a.s); // brackets of 1/s
    const double qs = MODE == TC_QUANT ? qscale[o] : 0.0;
    const float qsf = (float)qs;                              // scale32 is a float value: exact
    const float isd_lo = qs > 0.0 ? __double2float_rd(__drcp_rd(__dmul_rn(qs, a.s))) : 0.f;
    const float isd_hi = qs > 0.0 ? __double2float_ru(__drcp_ru(__dmul_rn(qs, a.s))) : 0.f;
    auto push_deferred = [&](bool want, int t) {            // warp-collective
      uint32_t need = __ballot_sync(0xFFFFFFFFu, want);
      if (!need) return;
      bool inl = false;
      if (want) {
        const uint32_t sl = atomicAdd(misc, 1u);
        if (sl < TC_DEF_CAP) deflist[sl] = ((uint32_t)t << 8) | ((uint32_t)o << 7) | (uint32_t)rt;
        else inl = true;
      }
      uint32_t todo = __ballot_sync(0xFFFFFFFFu, inl);
      while (todo) {
        const int l = __ffs(todo) - 1;
        todo &= todo - 1;
        bool o2 = false, ns = false;
        const uint64_t pm = tc_literal_warp(a, MODE, o, t, 32 * q + l, qs, &o2, &ns);
        if (lane == 0) {
          if (MODE == TC_POSTHOC && pm) atomicMax(misc + 2 + o, __float_as_uint((float)bitsd(pm)));
          if (MODE == TC_ABSMAX && pm) atomicMax(a.o[o].red, (unsigned long long)pm);
        }
        ovf |= o2; nanscale |= ns;
      }
    };
    auto release = [&](int h) {                               // slot 2b + h fully read
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_tempty + 8 * (2 * b + h));
    };
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int m = it % TC_META;
      const bool mine = DUAL || ((it & 1) == grp);
      mbar_wait_sleep(bar_mfull + 8 * m, (it / TC_META) & 1);
      const uint32_t* meta = reinterpret_cast<const uint32_t*>(smem + LY::OFF_META + m * TC_META_BYTES);
      const uint32_t flags = meta[0], tmaxb = meta[9];
      const uint32_t nsmall = reinterpret_cast<const uint8_t*>(meta + 16)[(o ? 128 : 0) + rt];   // small values in the chunk
      // z0: input 0 of this chunk is -0 after the rotation sign.  Only then can an exactly
      // zero output of the reference's butterflies be -0 (every output's left operand chain
      // ends at input 0; a zero from cancellation is +0), i.e. carry code sign 1.
      const bool z0 = (meta[(o ? 5 : 1) + (rt >> 5)] >> (rt & 31)) & 1u;
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_mempty + 8 * m);
      if (!mine) continue;
      const uint32_t tr = a.fc.div((uint32_t)t), tcl = (uint32_t)t - tr * (uint32_t)a.tiles_c;
      const uint32_t r = o == 0 ? tr * 128 + rt : tcl * 128 + rt;        // logical row
      const uint32_t ci = o == 0 ? tcl : tr;                             // chunk along K
      const bool tiny = (flags & 4u) != 0, has_small = (flags & 1u) != 0;
      const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + 256 * b;  // slot 2b + h at + 128 h: Y1 | Y2 (+64)
      if (a.dbg) {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait_sleep(bar_tfull + 8 * (2 * b + h), use & 1);
          tc_fence_after();
          release(h);
        }
        ++use;
        continue;
      }
      if (MODE == TC_ABSMAX) {
        // Absmax pass: the raw tile was rotated in one chain, so |Y^ - Y| <= 32 2^-24 L1(x)
        // <= 2^-19 ||Y||_2 (Parseval, ||Y||_2 = sqrt(128) ||x||_2 >= L1(x)); a chunk whose upper
        // bound reaches the CTA's running lower bound of the maximum is recomputed exactly
        // by the literal warp, so the tensor's exact max |y| is among those (quantizers.py:177).
        float ym = 0.f, sa = 0.f, sb = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait_sleep(bar_tfull + 8 * (2 * b + h), use & 1);
          tc_fence_after();
          uint32_t v1[64];
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_ld16(v1 + 16 * c, tb + 128 * h + 16 * c);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          release(h);
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            ym = amax3(ym, __uint_as_float(v1[i]), __uint_as_float(v1[i + 1]));
            sa = fmaf(__uint_as_float(v1[i]), __uint_as_float(v1[i]), sa);
            sb = fmaf(__uint_as_float(v1[i + 1]), __uint_as_float(v1[i + 1]), sb);
          }
        }
        ++use;
        const float ss = (sa + sb) * 1.0001f;
        const float bt = __fmul_ru(__fadd_ru(__fmul_ru(__fsqrt_ru(ss), 0x1p-19f * 1.001f), 0x1p-118f), C * 1.0001f);
        const float yv = ym * C, ee = __fmaf_ru(yv, 0x1p-21f, bt);
        const float yu = __fadd_ru(yv, ee), yl = fmaxf(__fsub_rd(yv, ee), 0.f);
        atomicMax(misc + 4 + o, __float_as_uint(yl));
        // no barrier: Lrun may miss this tile's lower bounds (any value <= the true max is a valid
        // threshold; a stale one only sends a few more chunks to the literal path)
        const float Lrun = __uint_as_float(misc[4 + o]);
        push_deferred(tiny || yu >= Lrun, t);
        continue;
      }
      // beta: bound (y units) of |Y2 - H.small| over the chunk: 32 * 2^-24 * L1(small),
      // L1(small) <= ||H.small||_2 (Parseval; both halves of Y2), plus flush-to-zero slack
      // beta: bound (y units) of |Y2 - H.small| over the chunk: 32 * 2^-24 * L1(small), with
      // L1(small) <= n * thr (the split warps counted the chunk's n small values, each below
      // the split threshold thr), plus flush-to-zero slack.  A chunk without small values is
      // exact.
      float beta = 0.f;
      // A chunk with at most one small value has an exact Y2 (one nonzero product per output):
      // beta = 0, although Y = fl32(Y1 + Y2) still rounds (inside the 2^-21 margins), so only
      // chunks without small values are exact.
      if (has_small && nsmall > 1u) {
        const int Eb = TAPE ? (int)(tmaxb >> 10) - 15 - 10 : (int)(tmaxb >> 7) - 127 - 8;   // log2 thr
        const float thr = __uint_as_float((uint32_t)max(Eb + 127, 1) << 23);
        beta = __fmul_ru(__fadd_ru(__fmul_ru(thr * (float)nsmall, 0x1p-19f * 1.0001f), 0x1p-118f), C * 1.0001f);
      }
      const bool exact_chunk = (!has_small || nsmall == 0u) && !tiny;   // y64 = fl64(fl64(Y * scale) * c) exactly
      // the sign of a zero / tiny value needs |Y| > betaY -- except an exact zero of an exact
      // chunk without z0, which is +0 in the reference (the fma below makes it +0 here as well)
      const bool sign_chk = !exact_chunk || z0;
      const float betaY = beta * invC;
      bool defer = tiny;
      float nh = 0.f, dh = 0.f;
      uint32_t pmaxb = 0;
      // group pairs gp = 0..3 (half h = gp / 2); one loop body keeps the kernel's code small
#pragma unroll 1
      for (int gp = 0; gp < 4; ++gp) {
        const int h = gp >> 1;
        if ((gp & 1) == 0) {
          mbar_wait_sleep(bar_tfull + 8 * (2 * b + h), use & 1);
          tc_fence_after();
        }
        {
          float Yp[32];
          {
            uint32_t v1[32], v2[32];
            const uint32_t ta = tb + 128 * h + 32 * (gp & 1);
            tmem_ld16(v1, ta);
            tmem_ld16(v1 + 16, ta + 16);
            if (has_small) {
              tmem_ld16(v2, ta + 64);
              tmem_ld16(v2 + 16, ta + 80);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (gp & 1) release(h);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              if (has_small) {
                uint64_t s2;
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s2) : "l"(pk2(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1]))),
                    "l"(pk2(__uint_as_float(v2[i]), __uint_as_float(v2[i + 1]))));
                upk2(s2, Yp[i], Yp[i + 1]);
              } else {
                Yp[i] = __uint_as_float(v1[i]);
                Yp[i + 1] = __uint_as_float(v1[i + 1]);
              }
            }
          }
          // two groups side by side, branch-free (independent chains the scheduler can
          // interleave); the rare exact-chunk code fix runs after both
          float gmv[2], mnv[2], s4v[2], dv[2], numv[2], denv[2];
          bool uncv[2], dokv[2];
          uint32_t c0v[2], c1v[2], mm0[2], mm1[2];
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            const float* Y = Yp + 16 * gq;
            float gm = amax3(Y[0], Y[1], Y[2]), gm2 = amax3(Y[3], Y[4], Y[5]);
            float mn = amin3(Y[0], Y[1], Y[2]), mn2 = amin3(Y[3], Y[4], Y[5]);
            gm = amax3(gm, Y[6], Y[7]);
            mn = amin3(mn, Y[6], Y[7]);
            gm2 = amax3(gm2, Y[8], Y[9]);
            mn2 = amin3(mn2, Y[8], Y[9]);
            gm = amax3(gm, Y[10], Y[11]);
            mn = amin3(mn, Y[10], Y[11]);
            gm2 = amax3(gm2, Y[12], Y[13]);
            mn2 = amin3(mn2, Y[12], Y[13]);
            gm = amax3(gm, Y[14], Y[15]);
            mn = amin3(mn, Y[14], Y[15]);
            gmv[gq] = fmaxf(gm, gm2);
            mnv[gq] = fminf(mn, mn2);
          }
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            const float gm = gmv[gq];
            const float gy = gm * C;                            // ~ gmax
            const float eg = __fmaf_ru(gy, 0x1p-21f, beta);     // |gy - gmax| bound
            float d = 0.f, s4 = 0.f;
            bool unc = !(gy < 0x1p120f) || (gm == 0.f && beta > 0.f);
            if (MODE == TC_POSTHOC) {
              // pseudo = E8M3_RTN(fl64(gmax / s))  (posthoc.py:82-83)
              const float lo = __fmul_rd(__fsub_rd(gy, eg), is_lo), hi = __fmul_ru(__fadd_ru(gy, eg), is_hi);
              const uint32_t pl = rne4(fmaxf(lo, 0.f)), ph = rne4(hi);
              unc |= gm != 0.f && (pl != ph || !(lo >= 0x1p-125f));
              d = __uint_as_float(pl);
              s4 = d;
              pmaxb = max(pmaxb, pl);
            } else {
              // s8 = E4M3_RTN(fl64(gmax / (scale32 * s)))  (quantizers.py:177-178)
              const float lo = __fmul_rd(__fsub_rd(gy, eg), isd_lo), hi = __fmul_ru(__fadd_ru(gy, eg), isd_hi);
              uint32_t cl, ch;
              asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %3;\n\tcvt.u32.u16 %0, t;\n\t}\n\t"
                  "{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %4;\n\tcvt.u32.u16 %1, t;\n\t}"
                  : "=r"(cl), "=r"(ch) : "f"(0.f), "f"(fmaxf(lo, 0.f)), "f"(hi));
              const bool live = qsf != 0.f && gm != 0.f;          // float test: a double one ran per group on the FP64 pipe
              unc |= live && (cl != ch || !(isd_hi < 0x1p120f));
              s4 = live ? e4m3_valf(cl) : 0.f;
              // E4M3 (4 significant bits) x scale32 (a float) is exact in double, so its float
              // rounding is one fp32 product; the double value is only needed by the fix path
              d = __fmul_rn(s4, qsf);                           // rounded: inside the code margin
            }
            // the sign of a zero / tiny value: |Y| > betaY (see sign_chk)
            unc |= sign_chk && !(mnv[gq] > betaY);
            s4v[gq] = s4;
            dv[gq] = d;
            uncv[gq] = unc;
            dokv[gq] = d > 0.f && !unc;
          }
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            const float* Y = Yp + 16 * gq;
            // codes: q = y / d through cvt (ties-to-even) on the brackets q (1 -+ eps); eps covers
            // the fp32 roundings (2^-21 |q|) and the small-part bound for |q| >= 1/8; below 1/8
            // the magnitude code is 0 on both sides and only the sign needs |y| > beta.  The
            // fma with +0 turns an exact -0 into +0.
            float rd;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rd) : "f"(dokv[gq] ? dv[gq] : 1.f));
            const float invc = C * rd;                          // rcp: <= 1 ulp; inside the 2^-21 budget
            const float eps = __fmaf_ru(8.02f * beta, rd, 0x1p-21f);
            const float il = invc * (1.f - eps), ih = invc * (1.f + eps);
            const uint64_t il2 = pk2(il, il), ih2 = pk2(ih, ih);
            uint32_t ca[2], cb[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              float qa[8], qb[8];
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                const uint64_t y2 = pk2(Y[8 * hf + i], Y[8 * hf + i + 1]);
                uint64_t ra, rb;
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(ra) : "l"(y2), "l"(il2), "l"(0ull));
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rb) : "l"(y2), "l"(ih2), "l"(0ull));
                upk2(ra, qa[i], qa[i + 1]);
                upk2(rb, qb[i], qb[i + 1]);
              }
              ca[hf] = e2m1x8(qa);
              cb[hf] = e2m1x8(qb);
            }
            const bool ok = dokv[gq];
            c0v[gq] = ok ? ca[0] : 0u;
            c1v[gq] = ok ? ca[1] : 0u;
            mm0[gq] = ok ? ca[0] ^ cb[0] : 0u;
            mm1[gq] = ok ? ca[1] ^ cb[1] : 0u;
          }
          if ((mm0[0] | mm1[0] | mm0[1] | mm1[1]) != 0u) {      // rare: codes on a threshold
#pragma unroll
            for (int gq = 0; gq < 2; ++gq) {
              if (!(mm0[gq] | mm1[gq])) continue;
              if (!exact_chunk) { uncv[gq] = true; continue; }
              // y64 = fl64(Y * c) (tape: fl64(fl64(Y * scale32) * c)) is the reference's value
              const float* Y = Yp + 16 * gq;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const uint32_t sh = 4 * (i & 7);
                if (!(((i < 8 ? mm0[gq] : mm1[gq]) >> sh) & 15u)) continue;
                const double y64 = TAPE ? __dmul_rn(__dmul_rn((double)Y[i], (double)__ldg(a.tape_scale32)), a.inv_sqrt)
                                        : __dmul_rn((double)Y[i], C64);
                const double d64 = MODE == TC_POSTHOC ? (double)dv[gq] : (double)s4v[gq] * (double)qsf;   // exact
                const uint32_t nc = rtn_code_exact(y64, d64);
                if (i < 8) c0v[gq] = (c0v[gq] & ~(15u << sh)) | (nc << sh);
                else c1v[gq] = (c1v[gq] & ~(15u << sh)) | (nc << sh);
              }
            }
          }
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            const float* Y = Yp + 16 * gq;
            // EDEN partial sums: num += Y^2, den += |Y| |q| (times d per group), 4-long fp32 chains
            uint64_t na2 = 0, nb2 = 0, qa2 = 0, qb2 = 0;
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              uint32_t hv[4];
              e2m1x8_f16s(w ? c1v[gq] : c0v[gq], hv);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int k = 8 * w + 2 * i;
                float f0, f1;
                asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
                    : "=f"(f0), "=f"(f1) : "r"(hv[i]));
                const uint64_t y2 = pk2(Y[k], Y[k + 1]);        // Y and its code share the sign
                if (w) { nb2 = ffma2(y2, y2, nb2); qb2 = ffma2(y2, pk2(f0, f1), qb2); }
                else { na2 = ffma2(y2, y2, na2); qa2 = ffma2(y2, pk2(f0, f1), qa2); }
              }
            }
            uint64_t n2, q2;
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(n2) : "l"(na2), "l"(nb2));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(q2) : "l"(qa2), "l"(qb2));
            float n0, n1, d0, d1;
            upk2(n2, n0, n1);
            upk2(q2, d0, d1);
            numv[gq] = n0 + n1;
            denv[gq] = d0 + d1;
          }
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            if (uncv[gq]) defer = true;
            nh += numv[gq];
            const float s4 = s4v[gq];
            dh = fmaf(denv[gq], MODE == TC_POSTHOC ? s4 : dv[gq], dh);   // s4 = 0 gives d = 0
          }
          s4s[gp] = make_float2(s4v[0], s4v[1]);
          // codes of the two groups: 16 bytes
          *reinterpret_cast<uint4*>(ocodes + (size_t)r * (oK / 2) + ci * 64 + 16 * gp) =
              make_uint4(c0v[0], c1v[0], c0v[1], c1v[1]);
        }
      }
      ++use;
      // S = num64 / den64 = C * num / den (num = sum Y^2, den = sum d_g sum |Y| |q|).  Relative
      // bounds: fp32 group sums of positive terms (<= 6 roundings) and the cross-group sums
      // (<= 7), the rounding of Y (2^-24 |Y|) and the small part (|dY| <= betaY, sum |Y| <=
      // sqrt(128 num)); then S, v in fp32 (rcp <= 2 ulp, products 1 ulp each)
      uint32_t srdef = 0u;
      if (!defer) {
        const float nf = nh, df = dh;
        bool ok = nf > 0x1p-100f && df > 0x1p-100f && nf < 0x1p100f && df < 0x1p100f;
        const bool sure_deg = nf == 0.f && betaY == 0.f;
        float S = 1.f, es = 0.f;
        if (ok) {
          float rn_, rdn;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rn_) : "f"(nf));
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rdn) : "f"(df));
          const float sq = sqrtf(128.f * nf) * 1.001f;
          const float en = 16.f * 0x1p-24f + (2.f * betaY * sq + 128.f * betaY * betaY) * rn_ * 1.01f;
          // |d den| <= betaY sum_g d_g sum |sval| <= betaY 2 C sum |Y| <= 2 beta sq (|sval| <= 2 |q|,
          // q = C Y / d_g, beta = C betaY)
          const float ed = 20.f * 0x1p-24f + 2.f * beta * sq * rdn * 1.01f;
          // the reference's degenerate test |den| >= 1e-30 num, decided with margin
          ok = df * (1.f - ed) >= 1.001e-30f * (C * nf) * (1.f + en);
          S = C * nf * rdn;
          es = en + ed + 6.f * 0x1p-24f;
        }
        if (!ok && !sure_deg) srdef = 1u;
        if (!ok) { S = 1.f; es = 0.f; }
        if (!srdef) {
          // SR of v = S * scale value: E4M3-style truncation a, p = (v - a) / ulp and u < p
          // (pack_aword) certified on [v (1 - es), v (1 + es)] against the draw's top 20 bits
          const uint32_t g0 = r * (oK / GROUP) + ci * 8;
          uint32_t aws[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            // branch-free over the eight groups (a zero scale gives word 0)
            const float sv = g & 1 ? s4s[g >> 1].y : s4s[g >> 1].x;
            const bool live = sv > 0.f;
            const float v = S * sv;
            const uint32_t bl = __float_as_uint(__fmul_rd(v, 1.f - es)), bh = __float_as_uint(__fmul_ru(v, 1.f + es));
            const uint32_t u20 = mix64_top20(ohead ^ ((uint64_t)(g0 + g) + GOLDEN)), lo20 = bl & 0xFFFFFu,
                           hi20 = bh & 0xFFFFFu;
            const bool same = (bl >> 20) == (bh >> 20) && lo20 > 0u && bl >= 0x02000000u && bh < 0x7E000000u;
            if (live && (!same || (u20 >= lo20 && u20 <= hi20))) srdef = 1u;
            const uint32_t up = u20 < lo20 ? 1u : 0u;
            aws[g] = live ? ((bl >> 23) + 129u) << 7 | (((bl >> 20) & 7u) << 4) | (up << 3) : 0u;   // E + 256 = (bl >> 23) + 129
          }
          if (!srdef) {
            if (MODE == TC_POSTHOC) {
              *reinterpret_cast<uint4*>(oaw + g0) = make_uint4(aws[0] | (aws[1] << 16), aws[2] | (aws[3] << 16),
                                                               aws[4] | (aws[5] << 16), aws[6] | (aws[7] << 16));
            } else {
              // E4M3 codes: the normal range (E in [-6, 8): eb in [250, 264)) by one shift-add of
              // each word, branch-free; a chunk with any other live word redoes all eight through
              // aword_code (subnormal RTN, overflow)
              uint32_t w0 = 0, w1 = 0;
              bool slow = false;
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const uint32_t w = aws[g], eb = w >> 7;
                slow |= w != 0u && (eb < 250u || eb >= 264u);
                const uint32_t c = w == 0u ? 0u : (w >> 4) + ((w >> 3) & 1u) - (249u << 3);
                if (g < 4) w0 |= (c & 0xFFu) << (8 * g);
                else w1 |= (c & 0xFFu) << (8 * (g - 4));
              }
              if (slow) {
                w0 = 0u; w1 = 0u;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                  bool o2 = false, o3 = false;
                  w0 |= aword_code_fast(aws[g], 0, &o2) << (8 * g);
                  w1 |= aword_code_fast(aws[g + 4], 0, &o3) << (8 * g);
                  if (o2 || o3) ovf = true;
                }
              }
              *reinterpret_cast<uint32_t*>(osf + sf_offset(r, ci * 8, okb)) = w0;
              *reinterpret_cast<uint32_t*>(osf + sf_offset(r, ci * 8 + 4, okb)) = w1;
            }
          }
        }
      }
      defer = defer || srdef != 0u;
      if (MODE == TC_POSTHOC && !defer && pmaxb) atomicMax(misc + 2 + o, pmaxb);
      push_deferred(defer, t);
    }
  }

  // ----------------------------------------------------- deferred chunks
  tc_fence_before();
  __syncthreads();
  const uint32_t ndef = min(misc[0], (uint32_t)TC_DEF_CAP);
  if (threadIdx.x == 0) {
    const int mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    atomicAdd(&g_tc_stats[0], (unsigned long long)mine * 128ull * (DUAL ? 2ull : 1ull));
    atomicAdd(&g_tc_stats[1], (unsigned long long)misc[0]);
  }
  for (uint32_t i = warp; i < ndef; i += TC_THREADS / 32) {
    const uint32_t ent = deflist[i];
    const int t = (int)(ent >> 8), o = (ent >> 7) & 1, rt = ent & 127;
    bool o2 = false, ns = false;
    const uint64_t pm = tc_literal_warp(a, MODE, o, t, rt, qscale[o], &o2, &ns);
    if (lane == 0) {
      if (MODE == TC_POSTHOC && pm) atomicMax(misc + 2 + o, __float_as_uint((float)bitsd(pm)));
      if (MODE == TC_ABSMAX && pm) atomicMax(a.o[o].red, (unsigned long long)pm);
    }
    ovf |= o2; nanscale |= ns;
  }
  __syncthreads();
  if (threadIdx.x < 2 && MODE == TC_POSTHOC) {
    const uint32_t pb = misc[2 + threadIdx.x];
    if (pb && ((SRC >> threadIdx.x) & 1)) atomicMax(&a.o[threadIdx.x].red[1], (unsigned long long)dbits((double)__uint_as_float(pb)));
  }
  if (threadIdx.x == 0) {
    if (misc[12] & 1u) atomic_or_err(a.err, Q2_ERR_NONFINITE);
    if (MODE == TC_QUANT && blockIdx.x == 0) {
#pragma unroll
      for (int o = 0; o < 2; ++o)
        if ((SRC >> o) & 1) *a.o[o].scale32 = (float)qscale[o];
    }
  }
  if (ovf) atomic_or_err(a.err, MODE == TC_QUANT ? Q2_ERR_SCALE448 : Q2_ERR_E8M3_OVF);
  if (nanscale) atomic_or_err(a.err, Q2_ERR_NAN_SCALE);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// Post-hoc pass 2 for the tensor-core pass 1: k from the pseudo-scale max,
// each group's SR word re-biased to the E4M3 code of x = v 2^-k (aword_code).
__global__ void __launch_bounds__(256) tc_pass2_kernel(const uint16_t* __restrict__ aw,
                                                       const unsigned long long* __restrict__ red, uint32_t R,
                                                       uint32_t K, FastDiv fq, uint8_t* __restrict__ sf,
                                                       float* __restrict__ scale32_out, uint32_t* __restrict__ err) {
  pdl_trigger();
  pdl_wait();
  const uint32_t qpr = K / 64, total = R * qpr;
  const uint64_t pb = red[1];
  const double pmax = __longlong_as_double((long long)pb);
  const int E = (int)(pb >> 52) - 1023;
  const int k = (pb & ((1ull << 52) - 1)) == 0 ? E - 8 : E - 7;
  const uint32_t tq = blockIdx.x * blockDim.x + threadIdx.x;
  if (tq == 0) *scale32_out = pmax > 0.0 ? (float)ldexp(1.0, k) : 0.f;
  if (tq >= total) return;
  const uint32_t r = fq.div(tq), jq = tq - r * qpr;
  uint32_t word = 0;
  bool ovf = false;
  if (pmax > 0.0) {
    const uint2 w2 = *reinterpret_cast<const uint2*>(aw + (uint64_t)r * (K / GROUP) + 4 * jq);
    const uint32_t ws[4] = {w2.x & 0xFFFFu, w2.x >> 16, w2.y & 0xFFFFu, w2.y >> 16};
#pragma unroll
    for (int i = 0; i < 4; ++i) word |= aword_code(ws[i], k, &ovf) << (8 * i);
  }
  if (ovf) atomic_or_err(err, Q2_ERR_SCALE448);
  *reinterpret_cast<uint32_t*>(sf + sf_offset(r, 4 * jq, sf_kblocks(K))) = word;
}


// Post-hoc pass 2, tiled: one block per (256-row block, 4 K64 blocks).  Thread t reads
// the 16 SR words of row 256 rb + t (32 contiguous bytes), turns them into E4M3 codes
// (normal range: one shift-add of the word, aword_code otherwise), places them at their
// position in the scale layout in shared memory, and the block writes its 4 KiB of
// scales contiguously (rows past R get scale 0: deterministic padding).
struct Pass2Op {
  const uint16_t* aw; const unsigned long long* red; uint32_t R, K; uint8_t* sf; float* scale32_out;
};

// Post-hoc pass 2 of one operand: block (bx, by) covers rows 256 by .. and scale blocks 4 bx ..
__device__ __forceinline__ void pass2t_body(const uint16_t* __restrict__ aw, const unsigned long long* __restrict__ red,
                                            uint32_t R, uint32_t K, uint8_t* __restrict__ sf,
                                            float* __restrict__ scale32_out, uint32_t* __restrict__ err,
                                            uint32_t bx, uint32_t by, uint32_t (&tile)[4 * 256]) {
  const uint64_t pb = red[1];
  const double pmax = __longlong_as_double((long long)pb);
  const int E = (int)(pb >> 52) - 1023;
  const int k = (pb & ((1ull << 52) - 1)) == 0 ? E - 8 : E - 7;
  if (bx == 0 && by == 0 && threadIdx.x == 0) *scale32_out = pmax > 0.0 ? (float)ldexp(1.0, k) : 0.f;
  const uint32_t kb = (K + 63) / 64, jb0 = 4 * bx, nj = min(4u, kb - jb0);
  const uint32_t t = threadIdx.x, r = 256 * by + t;
  // word of row t within a 1 KiB block: byte (L/8)*256 + h*128 + (L%8)*16 + c*4, row = 128h + 32c + L
  const uint32_t L = t & 31, c = (t >> 5) & 3, h = t >> 7;
  const uint32_t widx = (L >> 3) * 64 + h * 32 + (L & 7) * 4 + c;
  bool ovf = false;
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q) {
    if (q >= nj) break;
    uint32_t word = 0;
    if (r < R && pmax > 0.0) {
      const uint2 w2 = *reinterpret_cast<const uint2*>(aw + (uint64_t)r * (K / GROUP) + 4 * (jb0 + q));
      word = aword_code_fast(w2.x & 0xFFFFu, k, &ovf) | (aword_code_fast(w2.x >> 16, k, &ovf) << 8) |
             (aword_code_fast(w2.y & 0xFFFFu, k, &ovf) << 16) | (aword_code_fast(w2.y >> 16, k, &ovf) << 24);
    }
    tile[256 * q + widx] = word;
  }
  if (ovf) atomic_or_err(err, Q2_ERR_SCALE448);
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(sf + (((uint64_t)by * kb + jb0) << 10));
  const uint4* src = reinterpret_cast<const uint4*>(tile);
  for (uint32_t i = t; i < nj * 64; i += 256) dst[i] = src[i];
}

__global__ void __launch_bounds__(256) tc_pass2t_kernel(const uint16_t* __restrict__ aw,
                                                        const unsigned long long* __restrict__ red, uint32_t R,
                                                        uint32_t K, uint8_t* __restrict__ sf,
                                                        float* __restrict__ scale32_out, uint32_t* __restrict__ err) {
  __shared__ __align__(16) uint32_t tile[4 * 256];
  pdl_trigger();
  pdl_wait();
  pass2t_body(aw, red, R, K, sf, scale32_out, err, blockIdx.x, blockIdx.y, tile);
}

// Both orientations of a dual post-hoc call in one launch (one launch and one tail instead
// of two): a 1-D grid, the first gx0 * gy0 blocks cover operand 0's (scale blocks / 4) x
// (rows / 256) grid, the rest operand 1's (the two grids are transposes of each other, so a
// 2-D grid of their maxima would be mostly empty blocks for skinny shapes).
__global__ void __launch_bounds__(256) tc_pass2t_dual_kernel(Pass2Op o0, Pass2Op o1, uint32_t* __restrict__ err) {
  __shared__ __align__(16) uint32_t tile[4 * 256];
  pdl_trigger();
  pdl_wait();
  const uint32_t gx0 = ((o0.K + 63) / 64 + 3) / 4, n0 = gx0 * ((o0.R + 255) / 256);
  const bool second = blockIdx.x >= n0;
  const Pass2Op& o = second ? o1 : o0;
  const uint32_t gx = second ? ((o1.K + 63) / 64 + 3) / 4 : gx0;
  const uint32_t b = second ? blockIdx.x - n0 : blockIdx.x;
  pass2t_body(o.aw, o.red, o.R, o.K, o.sf, o.scale32_out, err, b % gx, b / gx, tile);
}

}  // namespace q2
