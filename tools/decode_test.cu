#include <cstdio>
#include <cuda_fp16.h>
#include <cstdint>
__global__ void k(float* out) {
  uint32_t b = threadIdx.x;   // byte value 0..255
  uint32_t h;
  asm("{\n\t.reg .b8 a0;\n\tcvt.u8.u32 a0, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, a0;\n\t}" : "=r"(h) : "r"(b));
  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h));
  uint32_t h2;
  asm("{\n\t.reg .b8 a0, a1, a2, a3;\n\tmov.b32 {a0, a1, a2, a3}, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, a0;\n\t}" : "=r"(h2) : "r"(b | 0xAB00u));
  const float2 g = __half22float2(*reinterpret_cast<const __half2*>(&h2));
  out[4 * b] = f.x; out[4 * b + 1] = f.y; out[4 * b + 2] = g.x; out[4 * b + 3] = g.y;
}
int main() {
  float* d; cudaMalloc(&d, 4096); k<<<1, 256>>>(d); float hbuf[1024]; cudaMemcpy(hbuf, d, 4096, cudaMemcpyDeviceToHost);
  for (int b : {0x00, 0x01, 0x10, 0x21, 0x7F, 0x9A, 0xF7}) printf("byte %02x -> (%g, %g) via mov.b32: (%g, %g)\n", b, hbuf[4*b], hbuf[4*b+1], hbuf[4*b+2], hbuf[4*b+3]);
  return 0;
}
