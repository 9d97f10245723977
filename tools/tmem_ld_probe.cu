// Probe: tcgen05.ld throughput per SM vs warps and shape (32x32b.xN), clock64-timed.
#include <cstdio>
#include <cstdint>
#include "../paper_2601_22813_b200/csrc/tc_common.cuh"
using namespace q2;

template <int N>
__device__ __forceinline__ void ldx(uint32_t taddr, uint32_t& acc) {
  uint32_t r[32];
  if (N == 16) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) acc += r[i];
  } else {
    Q2_LD32(r, taddr);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) acc += r[i];
  }
}

template <int N>
__global__ void probe(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) ldx<N>(tmem + ((i * N + (warp >> 2) * 64) & 511 & ~(N - 1)), acc);
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}

int main() {
  unsigned long long* dc; uint32_t* ds;
  cudaMalloc(&dc, 8 * 148); cudaMalloc(&ds, 4 * 148 * 1024);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int n : {16, 32}) {
      if (n == 16) probe<16><<<148, warps * 32>>>(iters, dc, ds); else probe<32><<<148, warps * 32>>>(iters, dc, ds);
      unsigned long long c;
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)iters * warps * 32 * n * 4;
      printf("warps %2d x%d: %.1f B/clk per SM (%llu cyc)\n", warps, n, bytes / c, c);
    }
  }
  printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
