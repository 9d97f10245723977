// NVFP4 x NVFP4 "TN" GEMM on 5th-gen tensor cores (tcgen05, sm_100a).
//
//   D[M, N] = (scale32_a * scale32_b) * sum_k A[m, k] * B[n, k]   (+ D if accumulate)
//
// Replaces gemm_emulated (linear_graph.py:190-205), which dequantizes both
// operands to float32 and runs an sgemm, for the three Quartet II GEMMs:
// fprop Q(X).Q(W)^T, dgrad Q(E).Q(W^T)^T, wgrad Q(E^T).Q(X^T)^T.  Both operands
// are E2M1 codes packed two per byte along K with one UE4M3 scale per 16,
// which is exactly the operand format of tcgen05.mma kind::mxf4nvf4 with
// block16 scaling.
//
// Persistent, warp-specialized (256 threads, one CTA per SM):
//   warp 0  TMA producer: 128x256-fp4 slices of A and B (cp.async.bulk.tensor,
//           128B swizzle) + their scale-factor atoms (cp.async.bulk) into a
//           STAGES-deep ring guarded by full/empty mbarriers.
//   warp 1  MMA issuer (one thread): tcgen05.cp scale atoms smem->TMEM, four
//           tcgen05.mma (K = 64) per stage into one of two 128x128 fp32 TMEM
//           accumulators; tcgen05.commit releases smem stages and signals the
//           epilogue.
//   warp 2  owns the TMEM allocation.
//   warps 4-7  epilogue: tcgen05.ld the accumulator, scale, convert, write a
//           128B-swizzled smem tile, TMA-store it (TMA reduce-add when
//           accumulating).  The second accumulator lets the MMAs of the next
//           tile run under this epilogue.
// Tiles are visited in M-groups of 8 so concurrently running CTAs share B and A
// tiles in L2.
#include <cuda.h>
#include <cuda_bf16.h>
#include "tc_common.cuh"

namespace q2 {

constexpr int BM = 128, BN = 128, BKB = 128;             // BK = 256 fp4 = 128 bytes
constexpr int A_STAGE = BM * BKB;                         // 16 KB
constexpr int B_STAGE = BN * BKB;                         // 16 KB
constexpr int SF_STAGE = 2 * 4096;                        // two 128x256b TMEM-image blocks (K pairs)
constexpr int STAGE_BYTES = A_STAGE + B_STAGE + 2 * SF_STAGE;
constexpr int TMEM_COLS = 512;
constexpr int SFA_COL = 256, SFB_COL = 272;               // after two 128-column accumulators
constexpr int GEMM_THREADS = 256;
constexpr int GROUP_M = 8;

template <bool F32>
struct GemmCfg {
  static constexpr int STAGES = F32 ? 3 : 4;
  static constexpr int OUT_BYTES = BM * BN * (F32 ? 4 : 2);          // staging for the TMA store
  static constexpr int OFF_OUT = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_OUT + OUT_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int BOX_COLS = F32 ? 32 : 64;                     // 128-byte store boxes
};

// instruction descriptor, kind::mxf4nvf4 (cute InstrDescriptorBlockScaled):
// a/b format E2M1 (=1) at [7,10)/[10,13), K-major, N>>3 at [17,23),
// scale format UE4M3 (=0) at [23], M>>4 at [24,29).
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct GemmArgs {
  const uint8_t* sfa; const uint8_t* sfb;
  const float* sa; const float* sb;
  int M, N, K;
  int tiles_m, tiles_n;
  int accumulate;
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = GROUP_M * tiles_n;
  const int grp = t / per_group, first_m = grp * GROUP_M;
  const int gm = min(GROUP_M, tiles_m - first_m);
  const int r = t - grp * per_group;
  tm = first_m + r % gm;
  tn = r / gm;
}

template <bool F32>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    nvfp4_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmD, GemmArgs g) {
  using C = GemmCfg<F32>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsub_total = g.K / 64;                   // K = 64 MMAs
  const int nk = (nsub_total + 3) / 4;
  const int64_t kpr = (g.K + 127) / 128;             // scale image blocks per 128-row block
  const int ntiles = g.tiles_m * g.tiles_n;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  const uint32_t bar_full = smem_u32(bars), bar_empty = smem_u32(bars + C::STAGES);
  const uint32_t bar_accf = smem_u32(bars + 2 * C::STAGES), bar_acce = smem_u32(bars + 2 * C::STAGES + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(bar_full + 8 * s, 1); mbar_init(bar_empty + 8 * s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(bar_accf + 8 * s, 1); mbar_init(bar_acce + 8 * s, 4); }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmD)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int tm, tn;
        tile_coords(t, g.tiles_m, g.tiles_n, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % C::STAGES;
          if (it >= C::STAGES) mbar_wait(bar_empty + 8 * s, ((it / C::STAGES) - 1) & 1);
          const int nkp = (int)(kpr - 2 * kt < 2 ? kpr - 2 * kt : 2);
          unsigned char* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(bar_full + 8 * s, A_STAGE + B_STAGE + 2 * nkp * 4096);
          tma_load_2d(smem_u32(st), &tmA, kt * BKB, m0, bar_full + 8 * s);
          tma_load_2d(smem_u32(st + A_STAGE), &tmB, kt * BKB, n0, bar_full + 8 * s);
          bulk_load(smem_u32(st + A_STAGE + B_STAGE), g.sfa + (((int64_t)tm * kpr + 2 * kt) << 12), nkp * 4096,
                    bar_full + 8 * s);
          bulk_load(smem_u32(st + A_STAGE + B_STAGE + SF_STAGE), g.sfb + (((int64_t)tn * kpr + 2 * kt) << 12),
                    nkp * 4096, bar_full + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc) {
        const int as = tc & 1;
        if (tc >= 2) mbar_wait(bar_acce + 8 * as, ((tc >> 1) - 1) & 1);   // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t dacc = tmem + as * BN;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(bar_full + 8 * s, (it / C::STAGES) & 1);
          tc_fence_after();
          const int nsub = min(4, nsub_total - kt * 4);
          const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
          for (int p = 0; p < (nsub + 1) / 2; ++p) {
            tc_cp_sf(tmem + SFA_COL + 8 * p, desc_sf(st + A_STAGE + B_STAGE + p * 4096));
            tc_cp_sf(tmem + SFB_COL + 8 * p, desc_sf(st + A_STAGE + B_STAGE + SF_STAGE + p * 4096));
          }
          const uint64_t adesc = desc_sw128(st), bdesc = desc_sw128(st + A_STAGE);
          for (int kk = 0; kk < nsub; ++kk)
            tc_mma(dacc, adesc + 2 * kk, bdesc + 2 * kk, IDESC, tmem + SFA_COL + 4 * kk, tmem + SFB_COL + 4 * kk,
                   (kt | kk) != 0);
          tc_commit(bar_empty + 8 * s);
        }
        tc_commit(bar_accf + 8 * as);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;                       // TMEM lanes 32*ew .. 32*ew+31
    const int row = ew * 32 + lane;                // row within the tile
    const float alpha = __ldg(g.sa) * __ldg(g.sb);
    unsigned char* out = smem + C::OFF_OUT;
    constexpr int NBOX = BN / C::BOX_COLS;
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc) {
      int tm, tn;
      tile_coords(t, g.tiles_m, g.tiles_n, tm, tn);
      const int as = tc & 1;
      mbar_wait(bar_accf + 8 * as, (tc >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 128 && tc > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      named_bar(1, 128);                            // staging buffer free again
#pragma unroll
      for (int q = 0; q < BN / 32; ++q) {
        uint32_t r[32];
        Q2_LD32(r, tmem + ((uint32_t)(ew * 32) << 16) + as * BN + q * 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (F32) {
          // 32 fp32 = 128 B = one full swizzled row of box q
          unsigned char* base = out + q * (BM * 128) + row * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const float4 v = make_float4(alpha * __uint_as_float(r[4 * ch]), alpha * __uint_as_float(r[4 * ch + 1]),
                                         alpha * __uint_as_float(r[4 * ch + 2]), alpha * __uint_as_float(r[4 * ch + 3]));
            *reinterpret_cast<float4*>(base + ((ch ^ (row & 7)) << 4)) = v;
          }
        } else {
          // 32 bf16 = 64 B = half a swizzled row of box q/2
          unsigned char* base = out + (q >> 1) * (BM * 128) + row * 128;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(r[8 * ch + 2 * e]),
                                                       alpha * __uint_as_float(r[8 * ch + 2 * e + 1]));
              p[e] = *reinterpret_cast<uint32_t*>(&h);
            }
            const int chunk = (q & 1) * 4 + ch;
            *reinterpret_cast<uint4*>(base + ((chunk ^ (row & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_acce + 8 * as);   // MMA warp may reuse this accumulator
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(1, 128);
      if (threadIdx.x == 128) {
#pragma unroll
        for (int b = 0; b < NBOX; ++b)
          tma_store_2d(&tmD, smem_u32(out + b * (BM * 128)), tn * BN + b * C::BOX_COLS, tm * BM, g.accumulate != 0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

template <bool F32>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md, const GemmArgs& g,
                       cudaStream_t st) {
  using C = GemmCfg<F32>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(nvfp4_gemm_kernel<F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return Q2_ECUDA;
    attr = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int ntiles = g.tiles_m * g.tiles_n;
  nvfp4_gemm_kernel<F32><<<std::min(ntiles, nsm), GEMM_THREADS, C::SMEM, st>>>(ma, mb, md, g);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}

}  // namespace q2

using namespace q2;

extern "C" int q2_gemm_tn(const q2_nvfp4* a, const q2_nvfp4* b, void* d, int d_dtype, int64_t ldd, int accumulate,
                          void* stream) {
  if (!a || !b || !d || a->K != b->K || a->K % 64 || (a->K / 2) % 16 || a->R <= 0 || b->R <= 0) return Q2_EINVAL;
  if (d_dtype != Q2_BF16 && d_dtype != Q2_F32) return Q2_EINVAL;
  if (accumulate && d_dtype != Q2_F32) return Q2_EINVAL;
  const int esz = d_dtype == Q2_F32 ? 4 : 2;
  if (ldd < b->R || (ldd * esz) % 16 || (reinterpret_cast<uintptr_t>(d) & 15)) return Q2_EINVAL;
  if (a->R > INT32_MAX || b->R > INT32_MAX || a->K > INT32_MAX) return Q2_EINVAL;
  CUtensorMap ma, mb, md;
  if (!make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, a->codes, a->K / 2, a->R, a->K / 2, BKB, BM) ||
      !make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, b->codes, b->K / 2, b->R, b->K / 2, BKB, BN) ||
      !make_map(&md, d_dtype == Q2_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, d,
                b->R, a->R, ldd * esz, d_dtype == Q2_F32 ? 32 : 64, BM))
    return Q2_ECUDA;
  GemmArgs g{a->sf, b->sf, a->scale32, b->scale32, (int)a->R, (int)b->R, (int)a->K,
             (int)((a->R + BM - 1) / BM), (int)((b->R + BN - 1) / BN), accumulate};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d_dtype == Q2_F32 ? launch_gemm<true>(ma, mb, md, g, st) : launch_gemm<false>(ma, mb, md, g, st);
}
