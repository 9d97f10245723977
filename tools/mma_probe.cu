// Calibrates tcgen05.mma kind::mxf4nvf4 throughput on resident smem (no TMA).
#include <cstdio>
#include <cstdint>
#include "../paper_2601_22813_b200/csrc/common.cuh"
using namespace q2;
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_sf(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint64_t desc_sf2(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
template <int N, bool CP>
__global__ void probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < (128 + N) * 128 + 16384; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); mbar_fence_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const uint32_t a = smem_u32(sm), b = a + 128 * 128, sfs = b + N * 128;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t ad = desc_sw128(a), bd = desc_sw128(b);
    for (int kk = 0; kk < 4; ++kk) {
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tmem + 256 + 4 * kk), "l"(desc_sf(sfs + kk * 512)));
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tmem + 272 + 4 * kk), "l"(desc_sf(sfs + 2048 + kk * 512)));
    }
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
      if (CP) {
        for (int p = 0; p < 2; ++p) {
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + 8 * p), "l"(desc_sf2(sfs + p * 4096)));
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 272 + 8 * p), "l"(desc_sf2(sfs + 8192 + p * 4096)));
        }
      }
      for (int kk = 0; kk < 4; ++kk)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                     ::"r"(tmem), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1), "r"(tmem + 256 + 4 * kk), "r"(tmem + 272 + 4 * kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    mbar_wait(smem_u32(&bar), 0);
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
template <int N, bool CP> void run(int blocks) {
  unsigned long long* d; cudaMalloc(&d, 8 * blocks);
  int smem = (128 + N) * 128 + 16384 + 1024;
  cudaFuncSetAttribute(probe<N, CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  probe<N, CP><<<blocks, 128, smem>>>(iters, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); probe<N, CP><<<blocks, 128, smem>>>(iters, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 256 * (double)iters * blocks;
  printf("N=%d cp=%d blocks=%d: %.1f cycles/MMA(K64)  %.0f TFLOP/s  err=%s\n", N, CP, blocks, (double)h[0] / (iters * 4),
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<128, false>(148); run<128, true>(148); run<256, false>(148); run<256, true>(148); run<64, false>(148);
  return 0;
}
