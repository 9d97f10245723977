#include <cstdio>
#include <cstdint>
#include "../paper_2601_22813_b200/csrc/common.cuh"
using namespace q2;
__device__ __forceinline__ uint64_t desc_sf(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
template <int SHAPE>
__global__ void probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (unsigned char)i;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); mbar_fence_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot, s0 = smem_u32(sm);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
      const uint32_t col = 256 + 8 * (i & 7);
      if (SHAPE == 0) asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tmem + col), "l"(desc_sf(s0, 128)));
      if (SHAPE == 1) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + col), "l"(desc_sf(s0, 256)));
      if (SHAPE == 2) asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + col), "l"(desc_sf(s0, 128)));
      if (SHAPE == 3) asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(tmem + col), "l"(desc_sf(s0, 128)));
      if (SHAPE == 4) asm volatile("tcgen05.cp.cta_group::1.4x256b [%0], %1;" ::"r"(tmem + col), "l"(desc_sf(s0, 128)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    mbar_wait(smem_u32(&bar), 0);
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
template <int S> void run(const char* name, int dst_bytes) {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17408);
  probe<S><<<148, 128, 17408>>>(4000, d);
  probe<S><<<148, 128, 17408>>>(4000, d);
  unsigned long long h; cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles/cp  (%d TMEM bytes)  %s\n", name, (double)h / 4000, dst_bytes, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("32x128b.warpx4", 2048); run<1>("128x256b", 4096); run<2>("128x128b", 2048);
  run<3>("64x128b.warpx2::02_13", 2048); run<4>("4x256b", 128);
  return 0;
}
