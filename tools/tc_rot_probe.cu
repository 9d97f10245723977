// Probe: numerics and operand layouts of the tensor-core 128-point rotation
// (tcgen05.mma kind::f16, bf16 operands, fp32 accumulation in TMEM).
//
// One CTA loads a 128x128 bf16 tile X into shared memory (128B swizzle, two
// 64-column slabs, the layout TMA writes), builds B = diag(s) H_128 as bf16
// +-1, and runs two M=128 N=128 K=128 MMAs:
//   rows: D_r[t][j] = sum_k X[t][k] s_k H[k][j]      (A = X, K-major)
//   cols: D_c[n][j] = sum_t X[t][n] s_t H[t][j]      (A = X^T, MN-major)
// The host compares with the exact sums (float64; bf16 inputs with a span of
// < 45 binades sum exactly) and reports the error in units of 2^-24 * sum|x|
// and of ulp(result), per data family, to calibrate the certification bound
// of the tensor-core MS-EDEN kernel.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>
#include "../paper_2601_22813_b200/csrc/tc_common.cuh"
using namespace q2;

__device__ __forceinline__ uint32_t sw128(int row, int col16) {   // byte of 16-B piece col16 of row in a slab
  return row * 128 + ((col16 ^ (row & 7)) << 4);
}

__global__ void probe(const uint16_t* X, const uint32_t* sign, float* out_r, float* out_c, int lbo_mode) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned char* A = sm;                 // 2 slabs x 16 KB: X[t][k], k in [64j, 64j+64)
  unsigned char* B = sm + 32768;         // 2 slabs x 16 KB: Bm[j][k] = s_k H[k][j]
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 16; i += blockDim.x) {     // 16 pieces of 8 bf16 per row
    const int r = i >> 4, p = i & 15, slab = p >> 3;
    uint4 v = *reinterpret_cast<const uint4*>(X + r * 128 + p * 8);
    *reinterpret_cast<uint4*>(A + slab * 16384 + sw128(r, p & 7)) = v;
    uint16_t h[8];
    for (int e = 0; e < 8; ++e) {
      const int k = p * 8 + e, j = r;
      int neg = (__popc(k & j) & 1) ^ ((sign[k >> 5] >> (k & 31)) & 1);
      h[e] = neg ? 0xBF80 : 0x3F80;
    }
    *reinterpret_cast<uint4*>(B + slab * 16384 + sw128(r, p & 7)) = *reinterpret_cast<uint4*>(h);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); mbar_fence_init(); }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  // kind::f16: D f32 (bit 4), A/B bf16 (bits 7, 10), N>>3 at 17, M>>4 at 24; bit 15 = A MN-major
  const uint32_t id_k = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t id_mn = id_k | (1u << 15);
  if (tid == 0) {
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    for (int kk = 0; kk < 8; ++kk) {       // K = 16 per MMA: 32 B within a slab
      const uint64_t ad = desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32);
      const uint64_t bd = desc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32);
      tc_mma_f16(tmem, ad, bd, id_k, kk > 0);
    }
    for (int kk = 0; kk < 8; ++kk) {       // A = X^T: MN-major; K step of 16 t-rows = 2 x 1024 B
      const uint32_t lbo = lbo_mode == 0 ? 16384 : 1024, sbo = lbo_mode == 0 ? 1024 : 16384;
      const uint64_t ad = desc_mn_sw128(a + kk * 2048, lbo, sbo);
      const uint64_t bd = desc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32);
      tc_mma_f16(tmem + 128, ad, bd, id_mn, kk > 0);
    }
    tc_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int w = tid >> 5, lane = tid & 31, row = 32 * w + lane;
  for (int half = 0; half < 2; ++half)
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      Q2_LD32(r, tmem + ((uint32_t)(32 * w) << 16) + half * 128 + c * 32);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float* o = half ? out_c : out_r;
      for (int i = 0; i < 32; ++i) o[row * 128 + c * 32 + i] = __uint_as_float(r[i]);
    }
  tc_fence_before(); __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

static uint16_t to_bf16(float f) {   // round to nearest even
  uint32_t u; memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static double from_bf16(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  std::mt19937_64 g(1234);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud;
  const char* fams[] = {"normal", "lognorm3", "t2", "span30", "outlier", "rowscale", "coarse", "grid15", "small8", "smallsp"};
  uint16_t *dX; uint32_t* dS; float *dR, *dC;
  cudaMalloc(&dX, 128 * 128 * 2); cudaMalloc(&dS, 16); cudaMalloc(&dR, 128 * 128 * 4); cudaMalloc(&dC, 128 * 128 * 4);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int lbo_mode = 0; lbo_mode < 1; ++lbo_mode) {
    printf("== MN-major descriptor mode %d (LBO %s)\n", lbo_mode, lbo_mode == 0 ? "16384, SBO 1024" : "1024, SBO 16384");
    for (int f = 0; f < 10; ++f) {
      double worst_model[2] = {0, 0}, worst_l1[2] = {0, 0}, worst_ulp[2] = {0, 0}, bias[2] = {0, 0}, worst_l2[2] = {0, 0};
      long nbad[2] = {0, 0};
      for (int trial = 0; trial < 40; ++trial) {
        std::vector<uint16_t> X(128 * 128);
        std::vector<double> xd(128 * 128);
        for (int t = 0; t < 128; ++t) {
          const double rs = f == 5 ? std::exp(3.0 * nd(g)) : 1.0;
          for (int k = 0; k < 128; ++k) {
            double v = nd(g);
            if (f == 1) v *= std::exp(3.0 * nd(g));
            if (f == 2) v = nd(g) / std::sqrt(0.5 * (std::pow(nd(g), 2) + std::pow(nd(g), 2)));
            if (f == 3) v *= std::ldexp(1.0, -(int)(ud(g) * 30));
            if (f == 4 && (k % 37) == 0) v *= 1e3;
            if (f == 6) v = std::round(v * 4) / 4;
            if (f == 7) { v = std::fabs(v) > 3.9 ? 0.0 : v; if (std::fabs(v) < 4.0 / 256) v = 0.0; }
            if (f == 8) v = v * std::ldexp(1.0, -10) * std::exp(2.0 * nd(g));
            if (f == 9) v = (ud(g) < 0.03) ? v * std::ldexp(1.0, -9) : 0.0;
            v *= rs;
            X[t * 128 + k] = to_bf16((float)v);
            xd[t * 128 + k] = from_bf16(X[t * 128 + k]);
          }
        }
        uint32_t sign[4];
        for (int i = 0; i < 4; ++i) sign[i] = (uint32_t)g();
        cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dS, sign, 16, cudaMemcpyHostToDevice);
        probe<<<1, 128, smem>>>(dX, dS, dR, dC, lbo_mode);
        std::vector<float> R(128 * 128), C(128 * 128);
        cudaMemcpy(R.data(), dR, R.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        auto sgn = [&](int k) { return ((sign[k >> 5] >> (k & 31)) & 1) ? -1.0 : 1.0; };
        for (int mode = 0; mode < 2; ++mode) {
          for (int a = 0; a < 128; ++a) {
            double l1 = 0, l2 = 0;
            for (int k = 0; k < 128; ++k) {
              const double v = mode == 0 ? xd[a * 128 + k] : xd[k * 128 + a];
              l1 += std::fabs(v); l2 += v * v;
            }
            l2 = std::sqrt(l2);
            for (int j = 0; j < 128; ++j) {
              double ex = 0, ulps = 0;
              for (int k = 0; k < 128; ++k) {
                const double v = mode == 0 ? xd[a * 128 + k] : xd[k * 128 + a];
                ex += v * sgn(k) * ((__builtin_popcount(k & j) & 1) ? -1.0 : 1.0);
                if ((k & 15) == 15 && ex != 0) { int e; std::frexp(ex, &e); ulps += std::ldexp(1.0, e - 24); }
              }
              const double got = mode == 0 ? R[a * 128 + j] : C[a * 128 + j];
              const double err = got - ex;
              if (l1 > 0) {
                worst_l1[mode] = std::max(worst_l1[mode], std::fabs(err) / (std::ldexp(1.0, -24) * l1));
                worst_l2[mode] = std::max(worst_l2[mode], std::fabs(err) / (std::ldexp(1.0, -24) * l2));
                bias[mode] += (ex >= 0 ? err : -err) / (std::ldexp(1.0, -24) * l1);
              }
              if (ex != 0) {
                int e; std::frexp(ex, &e);
                worst_ulp[mode] = std::max(worst_ulp[mode], std::fabs(err) / std::ldexp(1.0, e - 24));
              }
              if (std::fabs(err) > 1e-3 * (l1 + 1e-30)) nbad[mode]++;
              if (std::fabs(err) > 0) worst_model[mode] = std::max(worst_model[mode], ulps > 0 ? std::fabs(err) / ulps : 1e30);
            }
          }
        }
      }
      for (int mode = 0; mode < 2; ++mode)
        printf("%-9s %s: err/sum_s ulp(P_s) %.3f  max|err|/(2^-24 L1) %.3f  /(2^-24 L2) %.3f  max ulps %.2f  mean signed (toward 0 < 0) %.4f  gross %ld\n",
               fams[f], mode ? "cols" : "rows", worst_model[mode], worst_l1[mode], worst_l2[mode], worst_ulp[mode],
               bias[mode] / (40.0 * 128 * 128), nbad[mode]);
    }
  }
  printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
