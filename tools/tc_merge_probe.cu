// Probe: error of the MERGED tensor-core rotation used by the v2 MS-EDEN kernel.
// Per 128x128 bf16 tile with max binade E, "main" = |x| >= 2^(E-THR) (plus zeros),
// "small" = the rest.  One accumulator per orientation: 8 K-steps of main, then 8
// K-steps of small (accumulate), N = 128 (full H with the sign vector folded into B).
// Reports, per family and orientation:
//   exact: max |err| over chunks without small values (must be 0)
//   model: max |err| / (2^-20 |Y| + 2^-18 L1(small))  (must stay well below 1)
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstring>
#include <vector>
#include <random>
#include <algorithm>
#include "../paper_2601_22813_b200/csrc/tc_common.cuh"
using namespace q2;

__device__ __forceinline__ uint32_t sw128(int row, int col16) { return row * 128 + ((col16 ^ (row & 7)) << 4); }

// A: main (2 slabs) | small (2 slabs), B: rows-H (2 slabs), cols-H (2 slabs)
__global__ void probe(const uint16_t* M, const uint16_t* S, const uint32_t* sign, float* out_r, float* out_c) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned char* Am = sm;
  unsigned char* As = sm + 32768;
  unsigned char* Br = sm + 65536;
  unsigned char* Bc = sm + 98304;
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int r = i >> 4, p = i & 15, slab = p >> 3;
    *reinterpret_cast<uint4*>(Am + slab * 16384 + sw128(r, p & 7)) = *reinterpret_cast<const uint4*>(M + r * 128 + p * 8);
    *reinterpret_cast<uint4*>(As + slab * 16384 + sw128(r, p & 7)) = *reinterpret_cast<const uint4*>(S + r * 128 + p * 8);
    uint16_t hr[8], hc[8];
    for (int e = 0; e < 8; ++e) {
      const int k = p * 8 + e, j = r;
      const int hb = __popc(k & j) & 1;
      hr[e] = (hb ^ ((sign[k >> 5] >> (k & 31)) & 1)) ? 0xBF80 : 0x3F80;
      hc[e] = (hb ^ ((sign[4 + (k >> 5)] >> (k & 31)) & 1)) ? 0xBF80 : 0x3F80;
    }
    *reinterpret_cast<uint4*>(Br + slab * 16384 + sw128(r, p & 7)) = *reinterpret_cast<uint4*>(hr);
    *reinterpret_cast<uint4*>(Bc + slab * 16384 + sw128(r, p & 7)) = *reinterpret_cast<uint4*>(hc);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); mbar_fence_init(); }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t id_k = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t id_mn = id_k | (1u << 15);
  if (tid == 0) {
    for (int part = 0; part < 2; ++part) {
      const uint32_t a = smem_u32(part ? As : Am);
      for (int kk = 0; kk < 8; ++kk)
        tc_mma_f16(tmem, desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32),
                   desc_sw128(smem_u32(Br) + (kk >> 2) * 16384 + (kk & 3) * 32), id_k, part > 0 || kk > 0);
      for (int kk = 0; kk < 8; ++kk)
        tc_mma_f16(tmem + 128, desc_mn_sw128(a + kk * 2048, 16384, 1024),
                   desc_sw128(smem_u32(Bc) + (kk >> 2) * 16384 + (kk & 3) * 32), id_mn, part > 0 || kk > 0);
    }
    tc_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int w = tid >> 5, row = 32 * w + (tid & 31);
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

static uint16_t to_bf16(double d) {
  float f = (float)d; uint32_t u; memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static double from_bf16(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
  const int THR = argc > 1 ? atoi(argv[1]) : 9;
  std::mt19937_64 g(99);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud;
  const char* fams[] = {"normal", "lognorm3", "t2", "span30", "rowscale", "small8", "smallsp", "wide40", "nearbin"};
  const int NF = 9;
  uint16_t *dM, *dS; uint32_t* dSg; float *dR, *dC;
  cudaMalloc(&dM, 32768); cudaMalloc(&dS, 32768); cudaMalloc(&dSg, 32); cudaMalloc(&dR, 65536); cudaMalloc(&dC, 65536);
  const int smem = 131072 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("threshold 2^(E-%d)\n", THR);
  for (int f = 0; f < NF; ++f) {
    double worst_exact[2] = {0, 0}, worst_model[2] = {0, 0}, worst_rel[2] = {0, 0}, worst_l1[2] = {0, 0};
    long nsmall_chunks[2] = {0, 0}, nchunks[2] = {0, 0};
    for (int trial = 0; trial < 60; ++trial) {
      std::vector<double> xd(16384);
      for (int t = 0; t < 128; ++t) {
        const double rs = f == 4 ? std::exp(3.0 * nd(g)) : 1.0;
        for (int k = 0; k < 128; ++k) {
          double v = nd(g);
          if (f == 1) v *= std::exp(3.0 * nd(g));
          if (f == 2) v = nd(g) / std::sqrt(0.5 * (std::pow(nd(g), 2) + std::pow(nd(g), 2)));
          if (f == 3) v *= std::ldexp(1.0, -(int)(ud(g) * 30));
          if (f == 5) v = (ud(g) < 0.5) ? v * std::ldexp(1.0, -(int)(ud(g) * 12)) : v;
          if (f == 6) v = (ud(g) < 0.03) ? v * std::ldexp(1.0, -9 - (int)(ud(g) * 20)) : v;
          if (f == 7) v *= std::ldexp(1.0, -(int)(ud(g) * 40));
          if (f == 8) v = std::ldexp(1.0 - std::ldexp(ud(g), -7), (int)(ud(g) * 3)) * (ud(g) < 0.5 ? -1 : 1) *
                          (ud(g) < 0.1 ? std::ldexp(1.0, -9 - (int)(ud(g) * 8)) : 1.0);
          v *= rs;
          xd[t * 128 + k] = from_bf16(to_bf16(v));
        }
      }
      double mx = 0;
      for (double v : xd) mx = std::max(mx, std::fabs(v));
      int E; std::frexp(mx, &E); E -= 1;                    // mx in [2^E, 2^(E+1))
      const double thr = std::ldexp(1.0, E - THR);
      std::vector<uint16_t> M(16384), S(16384);
      std::vector<double> sd(16384);
      for (int i = 0; i < 16384; ++i) {
        const bool small = xd[i] != 0 && std::fabs(xd[i]) < thr;
        M[i] = small ? 0 : to_bf16(xd[i]);
        S[i] = small ? to_bf16(xd[i]) : 0;
        sd[i] = small ? xd[i] : 0;
      }
      uint32_t sign[8];
      for (int i = 0; i < 8; ++i) sign[i] = (uint32_t)g();
      cudaMemcpy(dM, M.data(), 32768, cudaMemcpyHostToDevice);
      cudaMemcpy(dS, S.data(), 32768, cudaMemcpyHostToDevice);
      cudaMemcpy(dSg, sign, 32, cudaMemcpyHostToDevice);
      probe<<<1, 128, smem>>>(dM, dS, dSg, dR, dC);
      std::vector<float> R(16384), C(16384);
      cudaMemcpy(R.data(), dR, 65536, cudaMemcpyDeviceToHost);
      cudaMemcpy(C.data(), dC, 65536, cudaMemcpyDeviceToHost);
      for (int mode = 0; mode < 2; ++mode) {
        for (int a = 0; a < 128; ++a) {
          double l1s = 0;
          for (int k = 0; k < 128; ++k) l1s += std::fabs(mode == 0 ? sd[a * 128 + k] : sd[k * 128 + a]);
          nchunks[mode]++;
          if (l1s > 0) nsmall_chunks[mode]++;
          for (int j = 0; j < 128; ++j) {
            double ex = 0;
            for (int k = 0; k < 128; ++k) {
              const double v = mode == 0 ? xd[a * 128 + k] : xd[k * 128 + a];
              const int sb = (sign[4 * mode + (k >> 5)] >> (k & 31)) & 1;
              ex += ((__builtin_popcount(k & j) + sb) & 1) ? -v : v;
            }
            const double got = mode == 0 ? R[a * 128 + j] : C[a * 128 + j];
            const double err = std::fabs(got - ex);
            if (l1s == 0) { worst_exact[mode] = std::max(worst_exact[mode], err); continue; }
            worst_model[mode] = std::max(worst_model[mode], err / (std::ldexp(std::fabs(got), -20) + std::ldexp(l1s, -18)));
            if (got != 0) worst_rel[mode] = std::max(worst_rel[mode], err / std::ldexp(std::fabs(got), -24));
            worst_l1[mode] = std::max(worst_l1[mode], err / std::ldexp(l1s, -24));
          }
        }
      }
    }
    for (int mode = 0; mode < 2; ++mode)
      printf("%-9s %s: chunks with small %5.1f%%  exact-chunk max|err| %g  model ratio %.4f  max err/(2^-24|Y|) %.2f  max err/(2^-24 L1s) %.2f\n",
             fams[f], mode ? "cols" : "rows", 100.0 * nsmall_chunks[mode] / nchunks[mode], worst_exact[mode],
             worst_model[mode], worst_rel[mode], worst_l1[mode]);
  }
  printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
