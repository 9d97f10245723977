// Debug harness: the forward quantizer's fast-path decision for one 16-group
// (tools only; prints both branches' certified quantities).
#include "../paper_2601_22813_b200/csrc/quant_fwd.cu"
#include <cstdio>
__global__ void k(const float* g, float scale32, double cap0, double cap1, float* out, uint32_t* codes) {
  __shared__ float mids[128];
  for (int i = threadIdx.x; i < 127; i += blockDim.x)
    mids[i] = i < 126 ? 0.5f * (e4m3_valf(i) + e4m3_valf(i + 1)) : __int_as_float(0x7f800000);
  __syncthreads();
  if (threadIdx.x) return;
  uint64_t vv[8], vacc = 0;
  float gmax = 0.f;
  for (int i = 0; i < 8; ++i) { vv[i] = pack2(g[2 * i], g[2 * i + 1]); gmax = fmaxf(gmax, fmaxf(fabsf(g[2*i]), fabsf(g[2*i+1]))); }
  const double s32 = scale32, D0 = s32 * cap0, D1 = s32 * cap1;
  const float invD0 = (float)(1.0 / D0), invD1 = (float)(1.0 / D1), s32f = scale32;
  for (int k = 0; k < 8; ++k) asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(vacc) : "l"(vv[k]));
  const float V = hsum2(vacc);
  const BranchConst c0 = branch_const(gmax, invD0, (float)cap0, s32f, mids);
  bool unc0 = c0.bad, unc1 = false;
  float S0, S1; uint32_t lo0, hi0, lo1, hi1;
  run_branch(vv, c0, s32f, lo0, hi0, unc0, S0);
  const BranchConst c1 = branch_const(gmax, invD1, (float)cap1, s32f, mids);
  unc1 = c1.bad;
  run_branch(vv, c1, s32f, lo1, hi1, unc1, S1);
  const float Q0 = V * c0.inv * c0.inv * 1.001f, Q1 = V * c1.inv * c1.inv * 1.001f;
  const float E0 = c0.E * c0.E, E1 = c1.E * c1.E;
  const float A0 = E0 * S0, A1 = E1 * S1;
  const float M = E0 * s_bound(S0, Q0) + E1 * s_bound(S1, Q1) + 0x1p-22f * (A0 + A1);
  out[0] = S0; out[1] = S1; out[2] = A0; out[3] = A1; out[4] = M; out[5] = Q0; out[6] = Q1;
  codes[0] = lo0; codes[1] = hi0; codes[2] = lo1; codes[3] = hi1; codes[4] = c0.s8; codes[5] = c1.s8;
  codes[6] = unc0; codes[7] = unc1;
}
int main(int argc, char** argv) {
  float h[16]; float s32f = atof(argv[1]);
  for (int i = 0; i < 16; ++i) h[i] = atof(argv[2 + i]);
  float *g, *o; uint32_t* c;
  cudaMalloc(&g, 64); cudaMalloc(&o, 64); cudaMalloc(&c, 32);
  cudaMemcpy(g, h, 64, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(g, s32f, 6.0, 4.0, o, c);
  float ho[16]; uint32_t hc[8];
  cudaMemcpy(ho, o, 64, cudaMemcpyDeviceToHost); cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
  printf("S0=%.7g S1=%.7g A0=%.7g A1=%.7g M=%.7g Q0=%.5g Q1=%.5g | codes6 %08x %08x codes4 %08x %08x s8 %u %u unc %u %u\n",
         ho[0], ho[1], ho[2], ho[3], ho[4], ho[5], ho[6], hc[0], hc[1], hc[2], hc[3], hc[4], hc[5], hc[6], hc[7]);
}
