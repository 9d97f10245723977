// MS-EDEN backward quantizer: randomized 128-Hadamard rotation fused with
// clipping RTN, the per-chunk EDEN correction factor and stochastic rounding
// of the E4M3 group scales (sm_100a).
//
// Restates ms_eden_quantize (ms_eden.py:116-153), its pow2 variant
// (ms_eden.py:86-113) and the post-hoc two-pass schedule pass1/pass2
// (posthoc.py:74-125).  The compute kernel is msed64_kernel (msed64.cuh): a
// persistent, TMA-fed, literal-float64 restatement whose outputs equal the
// reference's by construction.  Row sources, transposed bf16/fp32 sources (E^T)
// and transposed NVFP4 tape sources (W^T, X^T) share one kernel template.
//
// Schedules
//   posthoc  msed64<POSTHOC> (codes + per-group SR words + pseudo max), then
//            msed64_pass2_kernel (exponent re-bias to scale32 = 2^k).  One read.
//   exact    msed64<ABSMAX> (rotated absmax), msed64<QUANT>.  Two reads, as the
//            reference's non-pow2 scale32 needs the absmax before any code.
//   pow2     msed64<PMAX> (pseudo max), msed64<QUANT, pow2>.
#include <cuda_fp16.h>
#include <cstdio>
#include "tc_common.cuh"
#include "msed64.cuh"
#include "msed_tc.cuh"

namespace q2 {

// posthoc pass 2 from the pass-1 API outputs (pseudo-scales + EDEN factors):
// literal float64 restatement of posthoc.py:98-125, one thread per group.
__global__ void posthoc2_kernel(const uint16_t* __restrict__ pseudo, const double* __restrict__ corr,
                                const unsigned long long* __restrict__ red, int64_t R, int64_t K,
                                uint64_t sr_head, uint8_t* __restrict__ sf, float* __restrict__ scale32_out,
                                uint32_t* __restrict__ err) {
  const int64_t gpr = K / GROUP, total = R * gpr;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double pmax = __longlong_as_double((long long)red[1]);
  float scale32 = 0.f;
  if (pmax > 0.0) {
    int e; double m = frexp(pmax / 256.0, &e);
    scale32 = (float)ldexp(1.0, (m == 0.5) ? e - 1 : e);
  }
  if (g == 0) *scale32_out = scale32;
  if (g >= total) return;
  const int64_t r = g / gpr, j = g - r * gpr;
  const int64_t kpr = sf_kblocks(K);
  if (pmax == 0.0) { sf_store(sf, r, j, kpr, 0); return; }
  const double ps = (double)__uint_as_float((uint32_t)pseudo[g] << 16);
  const double shifted = __ddiv_rn(ps, (double)scale32);
  const double corrected = __dmul_rn(corr[r * (K / CHUNK) + j / 8], shifted);
  if (corrected > 448.0) atomic_or_err(err, Q2_ERR_SCALE448);
  sf_store(sf, r, j, kpr, (uint8_t)e4m3_sr(fmin(corrected, 448.0), prng_uniform(sr_head, (uint64_t)g)));
}

static int num_sms() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

struct M64Src {
  const void* x; int dtype; int64_t ld;             // bf16/fp32 sources
  const q2_nvfp4* tape;                             // NVFP4 tape source
  int kind;
};

static int check_src(const M64Src& s, int64_t R, int64_t K) {
  if (R < 0 || K < 0 || K % CHUNK) return Q2_EINVAL;
  if (s.kind == Q2_SRC_TAPE_COLS) {
    if (!s.tape || s.tape->R != K || s.tape->K != R || R % 64) return Q2_EINVAL;
    if (reinterpret_cast<uintptr_t>(s.tape->codes) & 15) return Q2_EINVAL;
    return Q2_OK;
  }
  if (s.dtype != Q2_BF16 && s.dtype != Q2_F32) return Q2_EINVAL;
  if (R == 0 || K == 0) return Q2_OK;                   // empty: nothing is read
  if (!s.x) return Q2_EINVAL;
  const int esz = s.dtype == Q2_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(s.x) & 15u) || (s.ld * esz) % 16) return Q2_EINVAL;
  if (s.kind == Q2_SRC_ROWS && s.ld < K) return Q2_EINVAL;
  if (s.kind == Q2_SRC_COLS && (s.ld < R || R % 8)) return Q2_EINVAL;
  if (s.kind != Q2_SRC_ROWS && s.kind != Q2_SRC_COLS) return Q2_EINVAL;
  return Q2_OK;
}

template <int SRC, int DT, int MODE>
static int launch_m64(const M64Src& s, const M64Args& a, cudaStream_t st) {
  using TL = M64Tile<SRC, DT>;
  auto k = msed64_kernel<SRC, DT, MODE>;
  static unsigned attr = 0;                     // per-device opt-in
  if (!smem_opt_in(k, TL::SMEM, attr)) return Q2_ECUDA;
  CUtensorMap tm;
  bool ok;
  if (SRC == Q2_SRC_TAPE_COLS) {
    ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, s.tape->codes, (uint64_t)(a.R / 2), (uint64_t)a.K,
                  (uint64_t)(a.R / 2), 64, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    const CUtensorMapDataType dt = DT == Q2_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const int esz = DT == Q2_BF16 ? 2 : 4, bi = DT == Q2_BF16 ? 64 : 32;
    if (SRC == Q2_SRC_ROWS)
      ok = make_map(&tm, dt, s.x, (uint64_t)a.K, (uint64_t)a.R, (uint64_t)s.ld * esz, bi, M64_ROWS);
    else
      ok = make_map(&tm, dt, s.x, (uint64_t)a.R, (uint64_t)a.K, (uint64_t)s.ld * esz, bi, CHUNK);
  }
  if (!ok) return Q2_ECUDA;
  const int ntiles = a.tiles_r * a.tiles_c;
  if (launch_pdl(k, dim3(std::min(ntiles, num_sms())), dim3(M64_THREADS), TL::SMEM, st, tm, a) != cudaSuccess)
    return Q2_ECUDA;
  return Q2_OK;
}

template <int MODE>
static int dispatch_m64(const M64Src& s, const M64Args& a, cudaStream_t st) {
  if (a.R == 0 || a.K == 0) return Q2_OK;
  switch (s.kind) {
    case Q2_SRC_ROWS:
      return s.dtype == Q2_BF16 ? launch_m64<Q2_SRC_ROWS, Q2_BF16, MODE>(s, a, st)
                                : launch_m64<Q2_SRC_ROWS, Q2_F32, MODE>(s, a, st);
    case Q2_SRC_COLS:
      return s.dtype == Q2_BF16 ? launch_m64<Q2_SRC_COLS, Q2_BF16, MODE>(s, a, st)
                                : launch_m64<Q2_SRC_COLS, Q2_F32, MODE>(s, a, st);
    case Q2_SRC_TAPE_COLS: return launch_m64<Q2_SRC_TAPE_COLS, Q2_BF16, MODE>(s, a, st);
  }
  return Q2_EINVAL;
}

static M64Args base_args(const M64Src& s, int64_t R, int64_t K, const uint32_t sign_mask[4], double sgrid,
                         double inv_sqrt) {
  M64Args a{};
  a.R = R; a.K = K;
  for (int i = 0; i < 4; ++i) a.sign[i] = sign_mask[i];
  a.s = sgrid; a.inv_sqrt = inv_sqrt;
  if (s.kind == Q2_SRC_TAPE_COLS) { a.tape_sf = s.tape->sf; a.tape_scale32 = s.tape->scale32; }
  a.tiles_r = (int)((R + M64_ROWS - 1) / M64_ROWS);
  a.tiles_c = (int)(K / CHUNK);
  a.fc = FastDiv((uint32_t)a.tiles_c);
  a.rotate = 1;
  a.sr_ncaps = 1;
  return a;
}


// ------------------------------------------------ tensor-core MS-EDEN launches
// Engine of q2_msed_quant for single-operand sources: 0 auto (tensor-core kernel for the
// dual E source and the NVFP4 tape, where it is fastest; literal float64 kernels for the
// single-orientation bf16 sources), 1 tensor-core kernel wherever eligible, 2 literal
// float64 kernels everywhere.
static int g_msed_engine = -1;
static int msed_engine() {
  if (g_msed_engine < 0) g_msed_engine = getenv("Q2_MSED_LITERAL") ? 2 : 0;
  return g_msed_engine;
}
static bool tc_disabled() { return msed_engine() == 2; }

template <int SRC, int MODE>
static int launch_tc(const TcArgs& a, int pow2, cudaStream_t st) {
  using LY = TcLayout<SRC == TC_TAPE>;
  auto k = msed_tc_kernel<SRC, MODE>;
  static unsigned attr = 0;                     // per-device opt-in
  if (!smem_opt_in(k, LY::SMEM, attr)) return Q2_ECUDA;
  CUtensorMap tm;
  bool ok;
  if (SRC == TC_TAPE)
    ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.tape_codes, (uint64_t)(a.N / 2), (uint64_t)a.T,
                  (uint64_t)(a.N / 2), 64, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  else
    ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.x, (uint64_t)a.N, (uint64_t)a.T, (uint64_t)a.ld * 2, 64, 128);
  if (!ok) return Q2_ECUDA;
  const int ntiles = a.tiles_r * a.tiles_c;
  if (launch_pdl(k, dim3(std::min(ntiles, num_sms())), dim3(TC_THREADS), LY::SMEM, st, tm, a, pow2) != cudaSuccess)
    return Q2_ECUDA;
  return Q2_OK;
}

template <int MODE>
static int dispatch_tc(int src, const TcArgs& a, int pow2, cudaStream_t st) {
  switch (src) {
    case TC_ROWS: return launch_tc<TC_ROWS, MODE>(a, pow2, st);
    case TC_COLS: return launch_tc<TC_COLS, MODE>(a, pow2, st);
    case TC_DUAL: return launch_tc<TC_DUAL, MODE>(a, pow2, st);
    case TC_TAPE: return launch_tc<TC_TAPE, MODE>(a, pow2, st);
  }
  return Q2_EINVAL;
}

static int tc_pass2(const TcOut& o, uint32_t* err, cudaStream_t st) {
  const int64_t quads = o.R * (o.K / 64);
  if (quads >= (1ll << 31)) return Q2_EINVAL;
  static const bool old = getenv("Q2_PASS2_OLD") != nullptr;   // A/B timing of the per-quad kernel
  if (!old && (o.R + 255) / 256 < 65535) {
    const int64_t kb = (o.K + 63) / 64;
    return launch_pdl(tc_pass2t_kernel, dim3((unsigned)((kb + 3) / 4), (unsigned)((o.R + 255) / 256)), dim3(256), 0, st,
                      (const uint16_t*)o.aw, (const unsigned long long*)o.red, (uint32_t)o.R, (uint32_t)o.K, o.sf,
                      o.scale32, err) == cudaSuccess ? Q2_OK : Q2_ECUDA;
  }
  if (launch_pdl(tc_pass2_kernel, dim3((unsigned)std::max<int64_t>(1, (quads + 255) / 256)), dim3(256), 0, st,
                 (const uint16_t*)o.aw, (const unsigned long long*)o.red, (uint32_t)o.R, (uint32_t)o.K,
                 FastDiv((uint32_t)(o.K / 64)), o.sf, o.scale32, err) != cudaSuccess)
    return Q2_ECUDA;
  return Q2_OK;
}

// Run the tensor-core MS-EDEN for source kind src (TC_ROWS / TC_COLS / TC_DUAL / TC_TAPE) over
// E [T, N] (or the tape [T, N]); outputs a.o[0] (rows) / a.o[1] (cols) already filled in.
static int tc_run(int src, TcArgs& a, int mode, cudaStream_t st) {
  static const int dbg = getenv("Q2_TC_DBG") ? atoi(getenv("Q2_TC_DBG")) : 0;
  a.dbg = dbg;
  a.tiles_r = (int)(a.T / 128);
  a.tiles_c = (int)(a.N / 128);
  a.fc = FastDiv((uint32_t)a.tiles_c);
  for (int o = 0; o < 2; ++o)
    if ((src >> o) & 1)
      if (cudaMemsetAsync(a.o[o].red, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  int rc;
  if (mode == Q2_MSED_POSTHOC) {
    if ((rc = dispatch_tc<TC_POSTHOC>(src, a, 0, st))) return rc;
    static const bool split2 = getenv("Q2_PASS2_SPLIT") != nullptr;   // A/B: one pass-2 launch per orientation
    if (src == TC_DUAL && !split2 && (a.o[0].R + 255) / 256 < 65535 && (a.o[1].R + 255) / 256 < 65535) {
      Pass2Op p[2];
      for (int o = 0; o < 2; ++o)
        p[o] = Pass2Op{(const uint16_t*)a.o[o].aw, (const unsigned long long*)a.o[o].red, (uint32_t)a.o[o].R,
                       (uint32_t)a.o[o].K, a.o[o].sf, a.o[o].scale32};
      int64_t nb = 0;
      for (int o = 0; o < 2; ++o) nb += ((((a.o[o].K + 63) / 64) + 3) / 4) * ((a.o[o].R + 255) / 256);
      if (nb < (1ll << 31))
        return launch_pdl(tc_pass2t_dual_kernel, dim3((unsigned)nb), dim3(256), 0, st, p[0], p[1],
                          a.err) == cudaSuccess ? Q2_OK : Q2_ECUDA;
    }
    for (int o = 0; o < 2; ++o)
      if ((src >> o) & 1)
        if ((rc = tc_pass2(a.o[o], a.err, st))) return rc;
    return Q2_OK;
  }
  if ((rc = dispatch_tc<TC_ABSMAX>(src, a, 0, st))) return rc;
  return dispatch_tc<TC_QUANT>(src, a, mode == Q2_MSED_POW2 ? 1 : 0, st);
}

static void tc_fill_out(TcOut& o, const q2_nvfp4* out, const uint32_t sign[4], uint64_t seed_sr, uint64_t stream,
                        void* red, void* aw) {
  o.codes = out->codes; o.sf = out->sf; o.scale32 = out->scale32;
  o.R = out->R; o.K = out->K;
  for (int i = 0; i < 4; ++i) o.sign[i] = sign[i];
  o.sr_head = prng_head(seed_sr, stream);
  o.red = static_cast<unsigned long long*>(red);
  o.aw = static_cast<uint16_t*>(aw);
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace q2

using namespace q2;

// ws: red (256 B) | pseudo-scales bf16 [R, K/16] | EDEN factors f64 [R, K/128]
extern "C" size_t q2_msed_ws_bytes(int64_t R, int64_t K) {
  return 256 + align256((size_t)R * (K / 16) * 2) + align256((size_t)R * (K / 128) * 8);
}

extern "C" int q2_msed_quant(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R,
                             int64_t K, int64_t ld, const uint32_t sign_mask[4], double s,
                             double inv_sqrt_chunk, uint64_t seed_sr, uint64_t sr_stream, int mode,
                             const q2_nvfp4* out, void* ws, uint32_t* err, void* stream) {
  if (!out || !ws || !sign_mask || out->R != R || out->K != K) return Q2_EINVAL;
  if (mode != Q2_MSED_EXACT && mode != Q2_MSED_POW2 && mode != Q2_MSED_POSTHOC) return Q2_EINVAL;
  const M64Src src{x, dtype, ld, tape, src_kind};
  int rc = check_src(src, R, K);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  // tensor-core path: bf16 or tape sources with 128-multiple dims
  const bool tc_ok = (msed_engine() == 1 || (msed_engine() == 0 && src_kind == Q2_SRC_TAPE_COLS)) && R > 0 && K > 0 && R % 128 == 0 && K % 128 == 0 &&
                     (src_kind == Q2_SRC_TAPE_COLS || dtype == Q2_BF16) && R / 128 < (1 << 16) && K / 128 < (1 << 16);
  if (tc_ok) {
    TcArgs ta{};
    const int osel = src_kind == Q2_SRC_ROWS ? 0 : 1;
    tc_fill_out(ta.o[osel], out, sign_mask, seed_sr, sr_stream, w, w + 256);
    ta.s = s; ta.inv_sqrt = inv_sqrt_chunk; ta.err = err;
    int kind;
    if (src_kind == Q2_SRC_ROWS) { ta.x = static_cast<const uint16_t*>(x); ta.ld = ld; ta.T = R; ta.N = K; kind = TC_ROWS; }
    else if (src_kind == Q2_SRC_COLS) { ta.x = static_cast<const uint16_t*>(x); ta.ld = ld; ta.T = K; ta.N = R; kind = TC_COLS; }
    else {
      ta.tape_codes = tape->codes; ta.tape_sf = tape->sf; ta.tape_scale32 = tape->scale32;
      ta.T = K; ta.N = R; kind = TC_TAPE;
    }
    if ((int64_t)(ta.T / 128) * (ta.N / 128) < (1ll << 24)) return tc_run(kind, ta, mode, st);
  }
  M64Args a = base_args(src, R, K, sign_mask, s, inv_sqrt_chunk);
  a.red = reinterpret_cast<unsigned long long*>(w);
  a.err = err;
  a.codes = out->codes; a.sf = out->sf; a.scale32 = out->scale32;
  a.sr_head = prng_head(seed_sr, sr_stream);
  if (cudaMemsetAsync(w, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  if (mode == Q2_MSED_POSTHOC) {
    a.pseudo = reinterpret_cast<uint16_t*>(w + 256);
    a.corr = reinterpret_cast<double*>(w + 256 + align256((size_t)R * (K / 16) * 2));
    if ((rc = dispatch_m64<M64_POSTHOC>(src, a, st))) return rc;
    const int64_t quads = R * (K / 64);
    if (quads >= (1ll << 31)) return Q2_EINVAL;
    if (launch_pdl(msed64_pass2_kernel, dim3((unsigned)std::max<int64_t>(1, (quads + 255) / 256)), dim3(256), 0, st,
                   (const uint16_t*)a.pseudo, (const double*)a.corr, (const unsigned long long*)a.red, (uint32_t)R,
                   (uint32_t)K, FastDiv((uint32_t)(K / 64)), a.sr_head, out->sf, out->scale32, err) != cudaSuccess)
      return Q2_ECUDA;
    return Q2_OK;
  }
  a.pow2 = mode == Q2_MSED_POW2;
  if (R == 0 || K == 0) {                               // empty tensor: scale32 of a zero tensor
    if (cudaMemsetAsync(out->scale32, 0, 4, st) != cudaSuccess) return Q2_ECUDA;
    return Q2_OK;
  }
  rc = a.pow2 ? dispatch_m64<M64_PMAX>(src, a, st) : dispatch_m64<M64_ABSMAX>(src, a, st);
  if (rc) return rc;
  return dispatch_m64<M64_QUANT>(src, a, st);
}

extern "C" int q2_sr_quant_src(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R, int64_t K,
                               int64_t ld, int rotate, const uint32_t sign_mask[4], int ncaps, double cap0,
                               double cap1, double margin, double scale_div, double inv_sqrt_chunk, uint64_t seed,
                               uint64_t stream0, uint64_t stream1, const q2_nvfp4* out, void* ws, uint32_t* err,
                               void* stream) {
  if (!out || !ws || !sign_mask || out->R != R || out->K != K || (ncaps != 1 && ncaps != 2)) return Q2_EINVAL;
  const M64Src src{x, dtype, ld, tape, src_kind};
  int rc = check_src(src, R, K);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  const uint32_t none[4] = {0u, 0u, 0u, 0u};
  M64Args a = base_args(src, R, K, rotate ? sign_mask : none, cap0, inv_sqrt_chunk);
  a.rotate = rotate ? 1 : 0;
  a.red = reinterpret_cast<unsigned long long*>(w);
  a.err = err;
  a.codes = out->codes; a.sf = out->sf; a.scale32 = out->scale32;
  a.sr_head = prng_head(seed, stream0);
  a.sr_head1 = prng_head(seed, stream1);
  a.sr_ncaps = ncaps; a.sr_cap1 = cap1;
  a.sr_div = scale_div; a.sr_margin = margin;
  if (cudaMemsetAsync(w, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  if (R == 0 || K == 0) return cudaMemsetAsync(out->scale32, 0, 4, st) == cudaSuccess ? Q2_OK : Q2_ECUDA;
  if ((rc = dispatch_m64<M64_ABSMAX>(src, a, st))) return rc;
  return dispatch_m64<M64_SR>(src, a, st);
}

extern "C" int q2_rht_sr_quant(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R, int64_t K,
                               int64_t ld, const uint32_t sign_mask[4], double cap, double margin, double scale_div,
                               double inv_sqrt_chunk, uint64_t seed, uint64_t sr_stream, const q2_nvfp4* out,
                               void* ws, uint32_t* err, void* stream) {
  return q2_sr_quant_src(x, dtype, tape, src_kind, R, K, ld, 1, sign_mask, 1, cap, 0.0, margin, scale_div,
                         inv_sqrt_chunk, seed, sr_stream, 0, out, ws, err, stream);
}

extern "C" int q2_posthoc_pass1(const void* x, int dtype, const q2_nvfp4* tape, int src_kind, int64_t R,
                                int64_t K, int64_t ld, const uint32_t sign_mask[4], double s,
                                double inv_sqrt_chunk, uint8_t* codes, uint16_t* pseudo_bf16, double* corr,
                                uint32_t* red, uint32_t* err, void* stream) {
  if (!codes || !pseudo_bf16 || !corr || !red || !sign_mask) return Q2_EINVAL;
  const M64Src src{x, dtype, ld, tape, src_kind};
  int rc = check_src(src, R, K);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  M64Args a = base_args(src, R, K, sign_mask, s, inv_sqrt_chunk);
  a.codes = codes; a.pseudo = pseudo_bf16; a.corr = corr; a.want_absmax = 1;
  a.red = reinterpret_cast<unsigned long long*>(red); a.err = err;
  if (cudaMemsetAsync(red, 0, 16, st) != cudaSuccess) return Q2_ECUDA;
  return dispatch_m64<M64_POSTHOC>(src, a, st);
}

extern "C" int q2_posthoc_pass2(const uint16_t* pseudo_bf16, const double* corr, const uint32_t* red,
                                int64_t R, int64_t K, uint64_t seed_sr, uint64_t sr_stream,
                                const q2_nvfp4* out, uint32_t* err, void* stream) {
  if (!out || out->R != R || out->K != K || K % CHUNK) return Q2_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t groups = R * (K / 16);
  unsigned blocks = (unsigned)std::max<int64_t>(1, (groups + 255) / 256);
  count_launch();
  posthoc2_kernel<<<blocks, 256, 0, st>>>(pseudo_bf16, corr, reinterpret_cast<const unsigned long long*>(red),
                                          R, K, prng_head(seed_sr, sr_stream), out->sf, out->scale32, err);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

// Both backward operands that read E, from ONE read of E (tensor-core kernel,
// TC_DUAL): MS(E) along rows (dgrad operand, pair sign_rows / sr_stream_rows)
// and MS(E^T) (wgrad operand, pair sign_cols / sr_stream_cols), in any mode.
// x is bf16 [T, N], T % 128 == N % 128 == 0.  ws: q2_msed_dual_ws_bytes(T, N).
extern "C" int q2_set_msed_engine(int engine) {
  if (engine < 0 || engine > 2) return Q2_EINVAL;
  g_msed_engine = engine;
  return Q2_OK;
}

// Chunk counters of the tensor-core MS-EDEN since load: out[0] chunks quantized,
// out[1] chunks deferred to the literal float64 path.  reset != 0 zeroes them.
extern "C" int q2_msed_stats(unsigned long long* out, int reset) {
  unsigned long long h[2] = {0ull, 0ull};
  if (cudaMemcpyFromSymbol(h, g_tc_stats, sizeof(h)) != cudaSuccess) return Q2_ECUDA;
  if (out) { out[0] = h[0]; out[1] = h[1]; }
  if (reset) {
    const unsigned long long z[2] = {0ull, 0ull};
    if (cudaMemcpyToSymbol(g_tc_stats, z, sizeof(z)) != cudaSuccess) return Q2_ECUDA;
  }
  return Q2_OK;
}

extern "C" size_t q2_msed_dual_ws_bytes(int64_t T, int64_t N) {
  return 256 + 2 * align256((size_t)T * (N / 16) * 2);
}

extern "C" int q2_msed_dual(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t sign_rows[4],
                            const uint32_t sign_cols[4], double s, double inv_sqrt_chunk, uint64_t seed_sr,
                            uint64_t sr_stream_rows, uint64_t sr_stream_cols, int mode, const q2_nvfp4* out_rows,
                            const q2_nvfp4* out_cols, void* ws, uint32_t* err, void* stream) {
  if (!x || !ws || !out_rows || !out_cols || !sign_rows || !sign_cols || T <= 0 || N <= 0 || T % CHUNK || N % CHUNK)
    return Q2_EINVAL;
  if (mode != Q2_MSED_EXACT && mode != Q2_MSED_POW2 && mode != Q2_MSED_POSTHOC) return Q2_EINVAL;
  if (out_rows->R != T || out_rows->K != N || out_cols->R != N || out_cols->K != T) return Q2_EINVAL;
  if (ld < N || (reinterpret_cast<uintptr_t>(x) & 15u) || (ld * 2) % 16) return Q2_EINVAL;
  if ((T / 128) * (N / 128) >= (1ll << 24)) return Q2_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  if (tc_disabled()) {
    // the literal kernels run the two operands one after the other on the same workspace
    int rc = q2_msed_quant(x, Q2_BF16, nullptr, Q2_SRC_ROWS, T, N, ld, sign_rows, s, inv_sqrt_chunk, seed_sr,
                           sr_stream_rows, mode, out_rows, w, err, stream);
    if (rc) return rc;
    return q2_msed_quant(x, Q2_BF16, nullptr, Q2_SRC_COLS, N, T, ld, sign_cols, s, inv_sqrt_chunk, seed_sr,
                         sr_stream_cols, mode, out_cols, w, err, stream);
  }
  TcArgs ta{};
  const size_t awb = align256((size_t)T * (N / 16) * 2);
  tc_fill_out(ta.o[0], out_rows, sign_rows, seed_sr, sr_stream_rows, w, w + 256);
  tc_fill_out(ta.o[1], out_cols, sign_cols, seed_sr, sr_stream_cols, w + 64, w + 256 + awb);
  ta.x = static_cast<const uint16_t*>(x); ta.ld = ld; ta.T = T; ta.N = N;
  ta.s = s; ta.inv_sqrt = inv_sqrt_chunk; ta.err = err;
  return tc_run(TC_DUAL, ta, mode, st);
}

extern "C" int q2_msed_dual_posthoc(const void* x, int64_t T, int64_t N, int64_t ld, const uint32_t sign_rows[4],
                                    const uint32_t sign_cols[4], double s, double inv_sqrt_chunk, uint64_t seed_sr,
                                    uint64_t sr_stream_rows, uint64_t sr_stream_cols, const q2_nvfp4* out_rows,
                                    const q2_nvfp4* out_cols, void* ws_rows, void* ws_cols, uint32_t* err,
                                    void* stream) {
  // workspaces sized q2_msed_ws_bytes(T, N) / (N, T): red + words of each operand
  if (!x || !ws_rows || !ws_cols || !out_rows || !out_cols || T <= 0 || N <= 0 || T % CHUNK || N % CHUNK)
    return Q2_EINVAL;
  if (out_rows->R != T || out_rows->K != N || out_cols->R != N || out_cols->K != T) return Q2_EINVAL;
  if (ld < N || (reinterpret_cast<uintptr_t>(x) & 15u) || (ld * 2) % 16) return Q2_EINVAL;
  if (tc_disabled() || (T / 128) * (N / 128) >= (1ll << 24)) {
    int rc = q2_msed_quant(x, Q2_BF16, nullptr, Q2_SRC_ROWS, T, N, ld, sign_rows, s, inv_sqrt_chunk, seed_sr,
                           sr_stream_rows, Q2_MSED_POSTHOC, out_rows, ws_rows, err, stream);
    if (rc) return rc;
    return q2_msed_quant(x, Q2_BF16, nullptr, Q2_SRC_COLS, N, T, ld, sign_cols, s, inv_sqrt_chunk, seed_sr,
                         sr_stream_cols, Q2_MSED_POSTHOC, out_cols, ws_cols, err, stream);
  }
  TcArgs ta{};
  char* wr = static_cast<char*>(ws_rows);
  char* wc = static_cast<char*>(ws_cols);
  tc_fill_out(ta.o[0], out_rows, sign_rows, seed_sr, sr_stream_rows, wr, wr + 256);
  tc_fill_out(ta.o[1], out_cols, sign_cols, seed_sr, sr_stream_cols, wc, wc + 256);
  ta.x = static_cast<const uint16_t*>(x); ta.ld = ld; ta.T = T; ta.N = N;
  ta.s = s; ta.inv_sqrt = inv_sqrt_chunk; ta.err = err;
  return tc_run(TC_DUAL, ta, Q2_MSED_POSTHOC, static_cast<cudaStream_t>(stream));
}
