// Throughput probe: f64 add/fma vs f32x2 on this B200 (148 SMs, 1 CTA of 1024 threads per SM x 2).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a0) {
  double x[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { x[i] = a0 + threadIdx.x + i; f[i] = (float)x[i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], 1.0000001);
      if (OP == 1) x[i] = __fma_rn(x[i], 0.9999999, 1e-7);
      if (OP == 2) f[i] = __fadd_rn(f[i], 1.0000001f);
      if (OP == 3) x[i] = (double)__float_as_uint(__uint_as_float((unsigned)x[i] ^ it));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i] + f[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"DADD", "DFMA", "FADD", "cvt"};
  for (int op = 0; op < 3; ++op) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<nsm * 2, 1024>>>(o, iters, 1.0);
      if (op == 1) k<1><<<nsm * 2, 1024>>>(o, iters, 1.0);
      if (op == 2) k<2><<<nsm * 2, 1024>>>(o, iters, 1.0);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)nsm * 2 * 1024 * iters * 8;
    printf("%s: %.1f Gop/s  (%.1f lane-ops/clk/SM at 1.965 GHz)\n", names[op], ops / ms / 1e6, ops / (ms * 1e-3) / nsm / 1.965e9);
  }
  return 0;
}
