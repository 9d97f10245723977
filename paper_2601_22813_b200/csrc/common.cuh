// Shared device helpers for the Quartet II kernels (sm_100a).
//
// Everything here reproduces a float64 decision of the reference emulator
// bit-for-bit; the reference line each helper restates is cited.  Literal
// float64 arithmetic uses __d*_rn intrinsics so nvcc never contracts it into
// an FMA (the reference is numpy/numba without fastmath).
#pragma once
#include <utility>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/quartet2.h"

namespace q2 {

constexpr int GROUP = 16;
constexpr int CHUNK = 128;

// ---------------------------------------------------------------- layout ----
// Group scales (UE4M3, one per 16 along K) are stored unreplicated in the
// tcgen05 block-scale vector layout: one 1 KiB block per (256-row block,
// 64-element K block), blocks K-fastest.  Block byte
//   (L/8)*256 + half*128 + (L%8)*16 + c*4 + i      (L = TMEM lane 0..31)
// holds scale i (= j%4) of row 128*half + 32*c + L.  Each half is the smem
// source of one tcgen05.cp.32x128b.warpx4 (core matrices of 8 lanes x 16 B,
// SBO 256 B), which broadcasts it to the four TMEM subpartitions.
__host__ __device__ __forceinline__ int64_t sf_kblocks(int64_t K) { return (K + 63) / 64; }
__host__ __device__ __forceinline__ int64_t sf_offset(int64_t r, int64_t j, int64_t kb) {
  const int64_t L = r & 31;
  return (((r >> 8) * kb + (j >> 2)) << 10) + ((L >> 3) << 8) + (((r >> 7) & 1) << 7) + ((L & 7) << 4) +
         (((r >> 5) & 3) << 2) + (j & 3);
}
__device__ __forceinline__ void sf_store(uint8_t* sf, int64_t r, int64_t j, int64_t kb, uint8_t v) {
  sf[sf_offset(r, j, kb)] = v;
}

// ------------------------------------------------------------------ E2M1 ----
// code -> value (formats.py:43-46) by bit construction (no local-memory table):
// |value| = 2^((m>>1)-1) * (1 or 1.5); code 8 decodes to +0.
__device__ __forceinline__ double fp4_val(uint32_t code) {
  const uint32_t m = code & 7u;
  uint32_t hi = m <= 1u ? (m ? 0x3FE00000u : 0u) : (((0x3FEu + (m >> 1)) << 20) | ((m & 1u) << 19));
  hi |= m ? (code & 8u) << 28 : 0u;
  return __longlong_as_double((long long)((uint64_t)hi << 32));
}

// ------------------------------------------------------------------ E4M3 ----
// Decode a non-negative E4M3 code (0..126) (formats.py:53-66).
__host__ __device__ __forceinline__ double e4m3_val(uint32_t code) {
  const uint32_t e = (code >> 3) & 0xF, m = code & 7;
  if (e == 0) return (double)m * 0x1p-9;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)((((uint64_t)(e + 1016)) << 52) | ((uint64_t)m << 49)));
#else
  return (double)(8 + m) * ldexp(1.0, (int)e - 10);
#endif
}
// The same value as a float (exact): code < 8 is k * 2^-9, else (8 + m) 2^(e-10).
__host__ __device__ __forceinline__ float e4m3_valf(uint32_t k) {
#ifdef __CUDA_ARCH__
  // k * 2^-9 as one exact FMA on (2^23 + k) (no int->float conversion on the XU pipe)
  return k < 8 ? __fmaf_rn(__uint_as_float(0x4B000000u | k), 0x1p-9f, -0x1p14f)
               : __uint_as_float((((k >> 3) + 120u) << 23) | ((k & 7u) << 20));
#else
  return (float)e4m3_val(k);
#endif
}
// Bit-level helpers for positive normal doubles (no libm calls on the hot path).
__device__ __forceinline__ int dexp(double x) { return (int)((__double_as_longlong(x) >> 52) & 0x7FF) - 1023; }
__device__ __forceinline__ double dpow2(int e) { return __longlong_as_double((long long)((uint64_t)(e + 1023) << 52)); }

// Nearest E4M3 code, ties to the even code, saturating at 448 (code 126).
// Restates formats._nearest_even_index over the 126 exact midpoints
// (formats.py:85-94, 160-171).  x >= 0, not NaN.
__device__ __forceinline__ uint32_t e4m3_rtn(double x) {
  if (!(x < 432.0)) return 126u;                       // 432 is the top midpoint (tie -> 126, even)
  if (x < 0x1p-6) return (uint32_t)rint(x * 512.0);    // subnormal spacing 2^-9, rint = RNE
  const int e = dexp(x);                               // x in [2^e, 2^(e+1)), e in [-6, 8]
  const double f = __dsub_rn(__dmul_rn(x, dpow2(-e)), 1.0);   // exact
  uint32_t q = (uint32_t)rint(f * 8.0);                // RNE on the mantissa; q == 8 carries
  uint32_t code = ((uint32_t)(e + 7) << 3) + q;
  return code > 126u ? 126u : code;
}

// Stochastic E4M3 rounding; RTN below 2^-6 (formats.py:174-201).  x <= 448(1+1e-9).
__device__ __forceinline__ uint32_t e4m3_sr(double x, double u) {
  if (x < 0x1p-6) return e4m3_rtn(x);
  x = fmin(x, 448.0);
  const int e = dexp(x);
  const double f = __dsub_rn(__dmul_rn(x, dpow2(-e)), 1.0);
  uint32_t lo = ((uint32_t)(e + 7) << 3) + (uint32_t)floor(f * 8.0);
  if (lo > 125u) lo = 125u;
  double a = e4m3_val(lo), b = e4m3_val(lo + 1);
  double p = __ddiv_rn(__dsub_rn(x, a), __dsub_rn(b, a));
  return lo + (u < p ? 1u : 0u);
}

// Round to the E8M3 grid (4 significant bits, bf16 exponent range)
// (formats.py:204-229).  Sets *ovf on overflow.
__device__ __forceinline__ double e8m3_rtn(double x, bool* ovf) {
  if (x < 0x1p-126) return (x <= 0x1p-127) ? 0.0 : 0x1p-126;
  int e = dexp(x) + 1;                    // frexp: x = m 2^e, m in [0.5, 1)
  const double m = __dmul_rn(x, dpow2(-e));
  double q = rint(16.0 * m);
  if (q >= 16.0) { q = 8.0; e += 1; }
  if (e - 1 > 127) { *ovf = true; return x; }
  return __dmul_rn(q * 0.0625, dpow2(e));
}

// ------------------------------------------------------------ element RTN ---
// Literal _nb_rtn (_kernels.py:101-127) for a float64 value: q = v/d (d<=0 ->
// q = +0), a2 = min(2|q|, 12), banker's rounding on the doubled grid.
__device__ __forceinline__ uint32_t rtn_code_literal(double v, double d) {
  double q = d > 0.0 ? __ddiv_rn(v, d) : 0.0;
  double a2 = fmin(fabs(q) * 2.0, 12.0);
  double r = a2 <= 4.0 ? rint(a2) : (a2 <= 8.0 ? 2.0 * rint(a2 * 0.5) : 4.0 * rint(a2 * 0.25));
  uint32_t ri = (uint32_t)r;               // 0,1,2,3,4,6,8,12
  uint32_t mag = ri <= 4 ? ri : (ri == 6 ? 5u : (ri == 8 ? 6u : 7u));
  return mag | (signbit(q) ? 8u : 0u);
}

// Exact-threshold RTN for a value whose float64 quotient v/d decides exactly
// like the rational (v an fp32/bf16, d = E4M3 * fp32): count the ties-to-even
// thresholds t*d with t in {.25 .75 1.25 1.75 2.5 3.5 5} (down, up, down, ...)
// crossed by |v|.  T[] holds t*d (exact in float64).
__device__ __forceinline__ uint32_t rtn_mag_thresholds(double a, const double* T) {
  uint32_t c = 0;
  c += a > T[0]; c += a >= T[1]; c += a > T[2]; c += a >= T[3];
  c += a > T[4]; c += a >= T[5]; c += a > T[6];
  return c;
}

// Stochastic E2M1 code of v/d with draw u = u53 * 2^-53 (_nb_sr, _kernels.py:130-157):
// q = fl64(v/d) (q = +0 when d <= 0), a2 = min(2|q|, 12), lo the doubled-grid
// point at or below a2, step 1/2/4; up iff u < (a2 - lo)/step (exact: a2 - lo is
// exact by Sterbenz and step a power of two).  *deq = the dequantized value.
__device__ __forceinline__ uint32_t sr_elem(double v, double d, uint64_t u53, double* deq) {
  const double q = d > 0.0 ? __ddiv_rn(v, d) : 0.0;
  const double a2 = fmin(fabs(q) * 2.0, 12.0);
  const double lo = a2 < 4.0 ? floor(a2) : (a2 < 8.0 ? 2.0 * floor(a2 * 0.5) : 4.0 * floor(a2 * 0.25));
  const double step = lo < 4.0 ? 1.0 : (lo < 8.0 ? 2.0 : 4.0);
  const double r = (double)u53 < ((a2 - lo) / step) * 0x1p53 ? lo + step : lo;
  const uint32_t ri = (uint32_t)r;
  const uint32_t mag = ri <= 4u ? ri : (ri == 6u ? 5u : (ri == 8u ? 6u : 7u));
  const bool neg = signbit(q);
  const double dq = neg ? -r * 0.5 : r * 0.5;
  *deq = d > 0.0 ? __dmul_rn(dq, d) : 0.0;
  return mag | (neg ? 8u : 0u);
}

// ------------------------------------------------------------------- PRNG ---
// splitmix64 finalizer chain (rht.py:36-39, 57-68, 89-96).
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// Top 20 bits of mix64(z) (= the top 20 bits of the 53-bit uniform draw): the second
// product only needs its high word, and the final z ^ (z >> 31) leaves bits >= 33 alone.
__device__ __forceinline__ uint32_t mix64_top20(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  const uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
  return (__umulhi(zl, 0x133111EBu) + zl * 0x94D049BBu + zh * 0x133111EBu) >> 12;
}
// The (seed, stream) prefix of _bits, shared by every index of one stream.
__host__ __device__ __forceinline__ uint64_t prng_head(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed + GOLDEN) ^ (stream + GOLDEN));
}
__device__ __forceinline__ double prng_uniform(uint64_t head, uint64_t index) {
  uint64_t z = mix64(head ^ (index + GOLDEN));
  return (double)(z >> 11) * 0x1p-53;
}

// ------------------------------------------------------ fast 32-bit divmod ---
// n / d for n, d < 2^31 via a 32x32->64 multiply-high (Granlund-Montgomery).
struct FastDiv {
  uint32_t d, m, s;
  FastDiv() = default;
  __host__ FastDiv(uint32_t div) : d(div) {
    s = 0;
    while ((1ull << s) < div) ++s;
    m = (uint32_t)(((1ull << 32) * ((1ull << s) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// ------------------------------------------------------- mbarrier / bulk ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// Non-blocking probe of a phase.
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  return done != 0;
}
// Blocking wait: the thread suspends in try_wait (time hint 1 ms) instead of spinning.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// ------------------------------------------------------------------ loads ---
__device__ __forceinline__ float bf16_to_f32(uint32_t bits16) { return __uint_as_float(bits16 << 16); }

__device__ __forceinline__ void atomic_or_err(uint32_t* err, uint32_t bits) {
  if (err) atomicOr(err, bits);
}

// ------------------------------------------------- programmatic launches ---
// Hot-path kernels are launched with programmatic stream serialization: each
// signals its dependents as soon as it starts and waits for its predecessor
// (griddepcontrol.wait) before touching global memory, so a kernel's launch
// and prologue (barrier init, TMEM allocation, tensor-map prefetch) overlap the
// previous kernel's tail.  Q2_NO_PDL=1 launches them plainly.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {}   // dependents launch as CTAs exit (an early trigger measured slower)

inline bool pdl_enabled() {
  static const int on = getenv("Q2_NO_PDL") ? 0 : 1;
  return on != 0;
}

// cudaFuncSetAttribute applies to the current device only: opt a kernel into its dynamic
// shared memory once per device (bit d of done_mask), so a process driving several GPUs
// launches correctly on each.
template <class F>
inline bool smem_opt_in(F* fn, int bytes, unsigned& done_mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32) return false;
  if (__atomic_load_n(&done_mask, __ATOMIC_ACQUIRE) & (1u << dev)) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  __atomic_fetch_or(&done_mask, 1u << dev, __ATOMIC_RELEASE);
  return true;
}

// Kernel launches issued by this library since load (q2_launch_count): the bench's
// gpu_launches figure.  One counter per process (inline function, single instance).
inline unsigned long long& launch_counter() {
  static unsigned long long n = 0;
  return n;
}
inline void count_launch() { __atomic_fetch_add(&launch_counter(), 1ull, __ATOMIC_RELAXED); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace q2

#define Q2_CHECK_LAUNCH()                                 \
  do {                                                    \
    if (cudaGetLastError() != cudaSuccess) return Q2_ECUDA; \
  } while (0)
