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
// Structure (one 128x256 output tile per CTA, 128 threads):
//   warp 0 / lane 0  TMA producer: 128-byte (256 fp4) K slices of A and B via
//                    cp.async.bulk.tensor (128B swizzle) + the matching
//                    scale-factor atoms via cp.async.bulk, into a 4-stage ring
//                    guarded by full/empty mbarriers.
//   warp 1 / lane 0  MMA issuer: tcgen05.cp scale atoms smem->TMEM, then four
//                    tcgen05.mma (K = 64 each) per stage into a 128x256 fp32
//                    accumulator in TMEM; tcgen05.commit frees the stage.
//   warps 0..3       epilogue: tcgen05.ld accumulator rows, multiply by the
//                    two tensor scales, convert, store.
#include <cuda.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace q2 {

constexpr int BM = 128, BN = 256, BKB = 128;            // BK = 256 fp4 = 128 bytes
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BKB;                         // 16 KB
constexpr int B_STAGE = BN * BKB;                         // 32 KB
constexpr int SFA_STAGE = 4 * 512;                        // 4 atoms (128 rows x 16 scales)
constexpr int SFB_STAGE = 8 * 512;                        // 2 row blocks x 4 atoms
constexpr int OFF_A = 0;
constexpr int OFF_B = OFF_A + STAGES * A_STAGE;
constexpr int OFF_SFA = OFF_B + STAGES * B_STAGE;
constexpr int OFF_SFB = OFF_SFA + STAGES * SFA_STAGE;
constexpr int OFF_BAR = OFF_SFB + STAGES * SFB_STAGE;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;          // + alignment slack
constexpr int TMEM_COLS = 512;
constexpr int SFA_COL = 256, SFB_COL = 272;               // after the 256 accumulator columns

// instruction descriptor, kind::mxf4nvf4 (cute InstrDescriptorBlockScaled):
// a/b format E2M1 (=1) at [7,10)/[10,13), K-major, N>>3 at [17,23),
// scale format UE4M3 (=0) at [23], M>>4 at [24,29).
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// tcgen05.cp source descriptor: 32 rows x 16 B, no swizzle, 8-row groups 128 B apart.
__device__ __forceinline__ uint64_t desc_sf(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_cp_sf(uint32_t tmem, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tmem), "l"(desc) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t tsfa, uint32_t tsfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(tsfa), "r"(tsfb)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define Q2_LD32(r, taddr)                                                                                       \
  asm volatile(                                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                            \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
      : "r"(taddr))

struct GemmArgs {
  const uint8_t* sfa; const uint8_t* sfb;
  const float* sa; const float* sb;
  void* d; int64_t ldd;
  int M, N, K;
  int d_f32, accumulate;
};

__global__ void __launch_bounds__(128, 1)
    nvfp4_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int nsub_total = g.K / 64;                   // K = 64 MMAs
  const int nk = (nsub_total + 3) / 4;
  const int64_t kb64 = nsub_total;                   // scale atoms per 128-row block
  const int nrb_b = min(2, (g.N + 127) / 128 - n0 / 128);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  const uint32_t bar_full = smem_u32(bars), bar_empty = smem_u32(bars + STAGES), bar_acc = smem_u32(bars + 2 * STAGES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(bar_full + 8 * s, 1); mbar_init(bar_empty + 8 * s, 1); }
    mbar_init(bar_acc, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(bar_empty + 8 * s, ((kt / STAGES) - 1) & 1);
      const int nsub = min(4, nsub_total - kt * 4);
      const uint32_t bytes = A_STAGE + B_STAGE + nsub * 512 * (1 + nrb_b);
      mbar_expect_tx(bar_full + 8 * s, bytes);
      tma_load_2d(smem_u32(smem + OFF_A + s * A_STAGE), &tmA, kt * BKB, m0, bar_full + 8 * s);
      tma_load_2d(smem_u32(smem + OFF_B + s * B_STAGE), &tmB, kt * BKB, n0, bar_full + 8 * s);
      bulk_load(smem_u32(smem + OFF_SFA + s * SFA_STAGE), g.sfa + (((int64_t)(m0 / 128) * kb64 + kt * 4) << 9),
                nsub * 512, bar_full + 8 * s);
      for (int rb = 0; rb < nrb_b; ++rb)
        bulk_load(smem_u32(smem + OFF_SFB + s * SFB_STAGE + rb * 2048),
                  g.sfb + (((int64_t)(n0 / 128 + rb) * kb64 + kt * 4) << 9), nsub * 512, bar_full + 8 * s);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(bar_full + 8 * s, (kt / STAGES) & 1);
      tc_fence_after();
      const int nsub = min(4, nsub_total - kt * 4);
      const uint32_t sfa_s = smem_u32(smem + OFF_SFA + s * SFA_STAGE);
      const uint32_t sfb_s = smem_u32(smem + OFF_SFB + s * SFB_STAGE);
      for (int kk = 0; kk < nsub; ++kk) {
        tc_cp_sf(tmem + SFA_COL + 4 * kk, desc_sf(sfa_s + kk * 512));
        for (int rb = 0; rb < nrb_b; ++rb) tc_cp_sf(tmem + SFB_COL + 8 * kk + 4 * rb, desc_sf(sfb_s + rb * 2048 + kk * 512));
      }
      const uint64_t adesc = desc_sw128(smem_u32(smem + OFF_A + s * A_STAGE));
      const uint64_t bdesc = desc_sw128(smem_u32(smem + OFF_B + s * B_STAGE));
      for (int kk = 0; kk < nsub; ++kk)
        tc_mma(tmem, adesc + 2 * kk, bdesc + 2 * kk, IDESC, tmem + SFA_COL + 4 * kk, tmem + SFB_COL + 8 * kk,
               (kt | kk) != 0);
      tc_commit(bar_empty + 8 * s);
    }
    tc_commit(bar_acc);
  }
  __syncwarp();

  // ---------------- epilogue: all four warps ----------------
  mbar_wait(bar_acc, 0);
  tc_fence_after();
  const float alpha = __ldg(g.sa) * __ldg(g.sb);
  const int row = m0 + warp * 32 + lane;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    Q2_LD32(r, tmem + ((uint32_t)(warp * 32) << 16) + c0);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int n = n0 + c0;
    if (row >= g.M || n >= g.N) continue;
    const bool full = n + 32 <= g.N;
    if (g.d_f32) {
      float* out = static_cast<float*>(g.d) + (int64_t)row * g.ldd + n;
      if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          float4 v = make_float4(alpha * __uint_as_float(r[i]), alpha * __uint_as_float(r[i + 1]),
                                 alpha * __uint_as_float(r[i + 2]), alpha * __uint_as_float(r[i + 3]));
          if (g.accumulate) {
            float4 o = *reinterpret_cast<float4*>(out + i);
            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
          }
          *reinterpret_cast<float4*>(out + i) = v;
        }
      } else {
        for (int i = 0; i < 32 && n + i < g.N; ++i) {
          float v = alpha * __uint_as_float(r[i]);
          out[i] = g.accumulate ? out[i] + v : v;
        }
      }
    } else {
      uint16_t* out = static_cast<uint16_t*>(g.d) + (int64_t)row * g.ldd + n;
      if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t p[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(r[i + 2 * q]),
                                                     alpha * __uint_as_float(r[i + 2 * q + 1]));
            p[q] = *reinterpret_cast<uint32_t*>(&h);
          }
          *reinterpret_cast<uint4*>(out + i) = make_uint4(p[0], p[1], p[2], p[3]);
        }
      } else {
        for (int i = 0; i < 32 && n + i < g.N; ++i) {
          __nv_bfloat16 h = __float2bfloat16_rn(alpha * __uint_as_float(r[i]));
          out[i] = *reinterpret_cast<uint16_t*>(&h);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// ------------------------------------------------------------ host side -----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static bool make_codes_map(CUtensorMap* map, const uint8_t* codes, int64_t rows, int64_t K, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)(K / 2), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(K / 2)};
  cuuint32_t box[2] = {(cuuint32_t)BKB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(codes), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace q2

using namespace q2;

extern "C" int q2_gemm_tn(const q2_nvfp4* a, const q2_nvfp4* b, void* d, int d_dtype, int64_t ldd, int accumulate,
                          void* stream) {
  if (!a || !b || !d || a->K != b->K || a->K % 64 || (a->K / 2) % 16 || a->R <= 0 || b->R <= 0) return Q2_EINVAL;
  if (d_dtype != Q2_BF16 && d_dtype != Q2_F32) return Q2_EINVAL;
  if (accumulate && d_dtype != Q2_F32) return Q2_EINVAL;
  if (ldd < b->R || a->R > INT32_MAX || b->R > INT32_MAX || a->K > INT32_MAX) return Q2_EINVAL;
  CUtensorMap ma, mb;
  if (!make_codes_map(&ma, a->codes, a->R, a->K, BM) || !make_codes_map(&mb, b->codes, b->R, b->K, BN))
    return Q2_ECUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(nvfp4_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) !=
        cudaSuccess)
      return Q2_ECUDA;
    attr = true;
  }
  GemmArgs g{a->sf, b->sf, a->scale32, b->scale32, d, ldd, (int)a->R, (int)b->R, (int)a->K, d_dtype == Q2_F32,
             accumulate};
  dim3 grid((unsigned)((b->R + BN - 1) / BN), (unsigned)((a->R + BM - 1) / BM));
  nvfp4_gemm_kernel<<<grid, 128, SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(ma, mb, g);
  Q2_CHECK_LAUNCH();
  return Q2_OK;
}
