// NVFP4 x NVFP4 "TN" GEMM on 5th-gen tensor cores, CTA pairs (tcgen05
// cta_group::2, sm_100a).
//
//   D[M, N] = (scale32_a * scale32_b) * sum_k A[m, k] * B[n, k]   (+ D if accumulate)
//
// Replaces gemm_emulated (linear_graph.py:190-205), which dequantizes both
// operands to float32 and runs an sgemm, for the three Quartet II GEMMs:
// fprop Q(X).Q(W)^T, dgrad Q(E).Q(W^T)^T, wgrad Q(E^T).Q(X^T)^T.  Both operands
// are E2M1 codes packed two per byte along K with one UE4M3 scale per 16 --
// the operand format of tcgen05.mma kind::mxf4nvf4 with block16 scaling.
//
// Why CTA pairs: at 128x128 tiles the kernel streamed ~6300 B/clk out of L2
// (the chip's LTS limit, B300_MICROARCH.md) for 2.2 PFLOP/s.  A pair computes a
// 256x256 tile with one M=256, N=256 MMA per K=64 step: each CTA stages half of
// A and half of B (its 128 rows of each) and the tensor cores read both CTAs'
// shared memory, so operand bytes per FLOP halve.  Scale factors are fetched
// unreplicated; instead of tcgen05.cp (three copies per MMA measured at ~45% of
// the MMA time) four "scale warps" write them into TMEM with tcgen05.st, each
// warp filling its own 32-lane subpartition (the replication the block-scaled
// MMA needs comes for free), so the MMA thread issues only MMAs.
//
// Per CTA (512 threads, one CTA per SM, clusters of 2):
// Warps 0, 1 and 3 run their loops as whole warps and elect one lane to issue (TMA, MMA,
// tcgen05.cp): warp-uniform values then live in uniform registers.  A lone-lane issuer
// wrapped each MMA in an elect/R2UR sequence; with it the tensor pipe was idle ~45% of an
// MMA-only probe (Q2_GEMM_DBG=4: 4.8 -> 6.4 PFLOP/s once fixed).
//
//   warp 0   TMA producer: A/B slices (128 B of K x 128 rows, 128B swizzle)
//            complete on the LEADER's full barrier (cta_group::2 TMA); the raw
//            scale halves complete on this CTA's scale barrier.
//   warp 1   (leader only) MMA issuer: 4 tcgen05.mma per stage; commits
//            release both CTAs' stages and signal both epilogues.
//   warp 2   owns the TMEM allocation (cta_group::2, 512 columns: 256-column
//            accumulator + one 48-column scale slot per stage).
//   warps 4-7 scale warps (see above); arrive on the leader's scale-ready barrier.
//   warps 8-15 epilogue: warp 8+e drains TMEM lanes 32*(e%4).. of columns
//            128*(e/4)..+127 (two 64-column passes), releases the accumulator
//            (leader's barrier, 16 arrivals), scales, converts and stores
//            16-byte vectors straight to global (read-add-write when accumulating).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include "tc_common.cuh"

namespace q2 {

constexpr int PT = 256;                                   // pair tile (M and N)
constexpr int BKB = 128;                                  // K bytes per stage (256 fp4)
constexpr int A_ST = 128 * BKB, B_ST = 128 * BKB;         // 16 KB each
constexpr int SFA_ST = 2048;                              // 4 K64 blocks x the CTA's 512 B half
constexpr int SFB_ST = 4096;                              // 4 K64 blocks x both halves
constexpr int STAGE = A_ST + B_ST + SFA_ST + SFB_ST;      // 38 KB
constexpr int STAGES = 5;
constexpr int OFF_EPI = STAGES * STAGE;                   // bf16 epilogue staging: 4 KB per epilogue warp
constexpr int OFF_BAR = OFF_EPI + 8 * 4096;
constexpr int GEMM_SMEM = OFF_BAR + 256 + 1024;
constexpr int GEMM_THREADS = 512;
constexpr int TMEM_COLS = 512;
constexpr int SF_COL = 256, SF_SLOT = 48;                 // per stage: 4 x (SFA 4 + SFB 8) columns
#ifndef Q2_GROUP_M
#define Q2_GROUP_M 8
#endif
constexpr int GROUP_M = Q2_GROUP_M;
#ifndef Q2_GEMM_STAGE_EPI
#define Q2_GEMM_STAGE_EPI 1
#endif
#ifndef Q2_SF_BATCH
#define Q2_SF_BATCH 2
#endif
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;               // shared::cluster address of the leader's copy

// instruction descriptor, kind::mxf4nvf4 (cute InstrDescriptorBlockScaled): a/b E2M1 (=1)
// at [7,10)/[10,13), K-major, N>>3 at [17,23), scale UE4M3 (=0), M>>4 at [24,29).
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)(PT >> 3) << 17) | ((uint32_t)(PT >> 4) << 24);

struct GemmArgs {
  const float* sa; const float* sb;
  void* d; int64_t ldd;
  int M, N, K, kb;                                        // kb = ceil(K/64) scale blocks per row block
  int tiles_m, tiles_n, nk;
  int accumulate;
  int dbg;                                                // timing probes (wrong results): 1 = scale warps skip their
                                                          // TMEM writes, 4 = MMAs re-read the first stages (no feed)
  int sfcp;                                               // 1: the MMA thread copies all scales (tcgen05.cp), no scale warps
  int cpmask;                                             // sfcp == 0: bit s = stage s's scales by the copier thread
  unsigned long long* trace;                              // optional timeline probe (pair 0), else nullptr
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// fp32 epilogue writes by accumulate mode: 0 store, 1 read-add-store (one writer per element),
// Q2_ACC_RED: red.global.add (any number of concurrent writers, e.g. split work on this GPU),
// Q2_ACC_MULTIMEM: d is an NVLS multicast address; the switch adds the tile into every member
// GPU's replica (the fused wgrad all-reduce).  The reductions flush subnormals.
__device__ __forceinline__ void out_f32x4(float* dp, float4 o, int mode) {
  if (mode == 3) {
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(dp), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w) : "memory");
  } else if (mode == 2) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(dp), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w) : "memory");
  } else {
    if (mode == 1) { const float4 p = *reinterpret_cast<const float4*>(dp); o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w; }
    *reinterpret_cast<float4*>(dp) = o;
  }
}
__device__ __forceinline__ void out_f32(float* dp, float o, int mode) {
  if (mode == 3) asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" :: "l"(dp), "f"(o) : "memory");
  else if (mode == 2) asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" :: "l"(dp), "f"(o) : "memory");
  else *dp = mode == 1 ? *dp + o : o;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma2_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & PEER_MASK) : "memory");
}
// pair-mode load multicast to the CTAs in `mask` (same shared offset in each); the bytes complete
// on the barrier at `bar`'s offset in each destination's pair leader
__device__ __forceinline__ void tma2_load_2d_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                                uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.cta_group::2 [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & PEER_MASK), "h"(mask) : "memory");
}
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar & PEER_MASK) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc2_cp_sf(uint32_t tmem, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(tmem), "l"(desc) : "memory");
}
__device__ __forceinline__ void tc2_cp_sf256(uint32_t tmem, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tmem), "l"(desc) : "memory");
}
__device__ __forceinline__ void tc2_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tsfa,
                                        uint32_t tsfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %6, [%4], [%5], p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(accum), "r"(tsfa), "r"(tsfb), "r"(IDESC)
      : "memory");
}
__device__ __forceinline__ void tc2_commit(uint32_t bar, uint16_t mask) {   // arrive on `bar` in the CTAs of `mask`
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"(mask) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar & PEER_MASK) : "memory");
}
// scale-factor source descriptor: core matrices of 8 lanes x 16 B, `sbo` bytes apart
__device__ __forceinline__ uint64_t desc_sf32(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ void tmem_ld64(uint32_t* r, uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,"
      "%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = GROUP_M * tiles_n;
  const int grp = t / per_group, first_m = grp * GROUP_M;
  const int gm = min(GROUP_M, tiles_m - first_m);
  const int r = t - grp * per_group;
  tm = first_m + r % gm;
  tn = r / gm;
}
// Clusters of CL pairs share one operand: pair p of the cluster takes tile (tm, CL*j + p)
// (SHARE_A: the A rows are common) or (CL*i + p, tn) (B common).  A cluster walks "super
// tiles"; a pair whose tile falls past the matrix edge still loads and multiplies (zeros)
// because the others need its slice of the shared operand, and stores nothing.
template <int CL, bool SHARE_A>
__device__ __forceinline__ int super_count(const GemmArgs& g) {
  return SHARE_A ? g.tiles_m * ((g.tiles_n + CL - 1) / CL) : ((g.tiles_m + CL - 1) / CL) * g.tiles_n;
}
template <int CL, bool SHARE_A>
__device__ __forceinline__ void super_coords(int u, const GemmArgs& g, int p, int& tm, int& tn) {
  if (SHARE_A) {
    tile_coords(u, g.tiles_m, (g.tiles_n + CL - 1) / CL, tm, tn);
    tn = tn * CL + p;
  } else {
    tile_coords(u, (g.tiles_m + CL - 1) / CL, g.tiles_n, tm, tn);
    tm = tm * CL + p;
  }
}

template <bool F32, int CL, bool SHARE_A>
__global__ void __cluster_dims__(2 * CL, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    nvfp4_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                      GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays a shared-space pointer (LDS/STS, not generic LD/ST)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1, pp = crank >> 1;           // CTA within the pair, pair within the cluster
  const int clid = blockIdx.x / (2 * CL), ncl = gridDim.x / (2 * CL);
  const int nsuper = super_count<CL, SHARE_A>(g);
  const bool tr0 = clid == 0 && pp == 0;                      // the traced pair
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pp));
  const uint16_t all_mask = (uint16_t)((1u << (2 * CL)) - 1);
  constexpr uint32_t SL = 128 / CL;                           // rows of the shared operand each pair loads
  constexpr uint16_t MC = CL == 4 ? 0x55 : (CL == 2 ? 0x5 : 0x1);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  const uint32_t bar_full = smem_u32(bars);                   // A/B of both CTAs (leader's copy used)
  const uint32_t bar_sff = smem_u32(bars + STAGES);           // this CTA's raw scales landed
  const uint32_t bar_sfr = smem_u32(bars + 2 * STAGES);       // scales in TMEM, both CTAs (leader's copy)
  const uint32_t bar_empty = smem_u32(bars + 3 * STAGES);     // stage (and its TMEM scale slot) free
  const uint32_t bar_accf = smem_u32(bars + 4 * STAGES), bar_acce = smem_u32(bars + 4 * STAGES + 1);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * STAGES + 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_sff + 8 * s, 1);
      mbar_init(bar_sfr + 8 * s, (g.cpmask >> s) & 1 ? 1 : 8);  // copier commit / 4 scale warps x 2 CTAs
      mbar_init(bar_empty + 8 * s, CL);                        // one MMA commit per pair of the cluster
    }
    mbar_init(bar_accf, 1);
    mbar_init(bar_acce, 16);                                  // 8 epilogue warps x 2 CTAs
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmSFA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmSFB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  pdl_trigger();
  pdl_wait();                                                 // operands written by the previous kernels
  tc_fence_before();
  cluster_sync();                                             // barriers and TMEM of both CTAs ready
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {
      // ---------------- TMA producer (both CTAs) ----------------
      // whole warp in the loop, one elected lane issues (as the MMA issuer)
      int it = 0;
      const uint16_t mc = (uint16_t)(MC << rank);             // this CTA's counterparts in every pair
      for (int u = clid; u < nsuper; u += ncl) {
        int tm, tn;
        super_coords<CL, SHARE_A>(u, g, (int)pp, tm, tn);
        const int m0 = tm * PT + (int)rank * 128, n0 = tn * PT + (int)rank * 128;
        for (int kt = 0; kt < g.nk; ++kt, ++it) {
          const int s = it % STAGES;
          if (g.dbg >= 4 && it >= STAGES) break;              // probe: MMAs re-read the first stages
          // the stage is free in every CTA this one writes: each pair's MMA commit arrives here
          if (it >= STAGES) mbar_wait_sleep(bar_empty + 8 * s, ((it / STAGES) - 1) & 1);
          if (!elect_one()) { __syncwarp(); continue; }
          const uint32_t st = smem_u32(smem + s * STAGE), fb = bar_full + 8 * s, sb = bar_sff + 8 * s;
          const bool cps = g.sfcp || ((g.cpmask >> s) & 1);
          // scales of copier stages complete on the leader's full barrier with the operands
          if (rank == 0) mbar_expect_tx(fb, 2 * (A_ST + B_ST + (cps ? SFA_ST + SFB_ST : 0)));
          if (CL == 1) {
            tma2_load_2d(st, &tmA, kt * BKB, m0, fb);
            tma2_load_2d(st + A_ST, &tmB, kt * BKB, n0, fb);
          } else if (SHARE_A) {                                 // slice pp of the common A rows, to all pairs
            tma2_load_2d_mc(st + pp * SL * BKB, &tmA, kt * BKB, m0 + (int)(pp * SL), fb, mc);
            tma2_load_2d(st + A_ST, &tmB, kt * BKB, n0, fb);
          } else {
            tma2_load_2d(st, &tmA, kt * BKB, m0, fb);
            tma2_load_2d_mc(st + A_ST + pp * SL * BKB, &tmB, kt * BKB, n0 + (int)(pp * SL), fb, mc);
          }
          if (cps) {
            tma2_load_3d(st + A_ST + B_ST, &tmSFA, 0, (int)rank, (tm * g.kb + 4 * kt) * 4, fb);
            tma2_load_3d(st + A_ST + B_ST + SFA_ST, &tmSFB, 0, 0, (tn * g.kb + 4 * kt) * 4, fb);
          } else {
            mbar_expect_tx(sb, SFA_ST + SFB_ST);
            tma_load_3d(st + A_ST + B_ST, &tmSFA, 0, (int)rank, (tm * g.kb + 4 * kt) * 4, sb);
            tma_load_3d(st + A_ST + B_ST + SFA_ST, &tmSFB, 0, 0, (tn * g.kb + 4 * kt) * 4, sb);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader) ----------------
      // The whole warp runs the loop (warp-uniform values stay in uniform registers) and one
      // elected lane issues each stage's MMAs: a lone-lane loop wrapped every MMA in an
      // elect/R2UR sequence and left the tensor pipe idle ~45% of the time (ncu, MMA-only probe).
      int it = 0, tc = 0;
      for (int u = clid; u < nsuper; u += ncl, ++tc) {
        if (tc >= 1) mbar_wait(bar_acce, (tc - 1) & 1);       // both epilogues drained the accumulator
        tc_fence_after();
        if (g.trace && tr0 && tc < 64 && lane == 0) g.trace[4 * tc] = gtime();
        unsigned long long wf = 0, ws = 0;
        for (int kt = 0; kt < g.nk; ++kt, ++it) {
          const int s = it % STAGES;
          const unsigned long long t0 = g.trace ? gtime() : 0;
          if (g.dbg < 4 || it < STAGES) mbar_wait(bar_full + 8 * s, (it / STAGES) & 1);
          const unsigned long long t1 = g.trace ? gtime() : 0;
          if (!g.sfcp && (g.dbg < 4 || it < STAGES)) mbar_wait(bar_sfr + 8 * s, (it / STAGES) & 1);
          if (g.trace) { wf += t1 - t0; ws += gtime() - t1; }
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * STAGE);
          const uint64_t adesc = desc_sw128(st), bdesc = desc_sw128(st + A_ST);
          const uint32_t tsf = tmem + SF_COL + SF_SLOT * s;
          const int nsub = min(4, g.K / 64 - 4 * kt);          // K tail: no MMA past K
          const bool leader = elect_one();
          if (g.sfcp && leader) {
            // scales of this stage into its own TMEM slot (distinct per stage and K64 block, so
            // the copies never wait on an MMA still reading the previous contents); the tensor
            // pipe runs them in issue order ahead of the MMAs that read them.  32x128b.warpx4
            // replicates each 512 B half to the four subpartitions.
            const uint32_t sfa = st + A_ST + B_ST, sfb = sfa + SFA_ST;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nsub) break;
              tc2_cp_sf(tsf + 12 * kk, desc_sf32(sfa + 512 * kk, 128));
              tc2_cp_sf(tsf + 12 * kk + 4, desc_sf32(sfb + 1024 * kk, 256));
              tc2_cp_sf(tsf + 12 * kk + 8, desc_sf32(sfb + 1024 * kk + 128, 256));
            }
          }
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nsub) break;
              tc2_mma(tmem, adesc + 2 * kk, bdesc + 2 * kk, tsf + 12 * kk, tsf + 12 * kk + 4, (kt | kk) != 0);
            }
            tc2_commit(bar_empty + 8 * s, all_mask);
          }
          __syncwarp();
        }
        if (elect_one()) tc2_commit(bar_accf, pair_mask);
        __syncwarp();
        if (g.trace && tr0 && tc < 64 && lane == 0) { g.trace[4 * tc + 1] = gtime(); g.trace[256 + 2 * tc] = wf; g.trace[257 + 2 * tc] = ws; }
      }
    }
  } else if (warp == 3 && g.cpmask) {
    // ---------------- scale copier (leader, one thread): tcgen05.cp of the masked stages'
    // scales into their TMEM slots, off the MMA thread; a commit signals the MMA thread.
    // The copies cost tensor-pipe time (~60 cycles per 512 B) but no shared-memory reads
    // beyond the 6 KB of the stage, so splitting stages between this thread and the scale
    // warps balances the pipe against shared-memory bandwidth; with few K stages per tile
    // the copier runs ahead while the MMA waits for the accumulator drain.
    if (rank == 0) {
      const int my_tiles = clid < nsuper ? (nsuper - 1 - clid) / ncl + 1 : 0;
      const int total = my_tiles * g.nk;
      for (int it = 0; it < total; ++it) {
        const int s = it % STAGES, kt = it % g.nk;
        if (!((g.cpmask >> s) & 1)) continue;
        mbar_wait(bar_full + 8 * s, (it / STAGES) & 1);
        tc_fence_after();
        if (!elect_one()) { __syncwarp(); continue; }
        const uint32_t st = smem_u32(smem + s * STAGE), sfa = st + A_ST + B_ST, sfb = sfa + SFA_ST;
        const uint32_t tsf = tmem + SF_COL + SF_SLOT * s;
        const int nsub = min(4, g.K / 64 - 4 * kt);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kk >= nsub) break;
          tc2_cp_sf(tsf + 12 * kk, desc_sf32(sfa + 512 * kk, 128));
          tc2_cp_sf(tsf + 12 * kk + 4, desc_sf32(sfb + 1024 * kk, 256));
          tc2_cp_sf(tsf + 12 * kk + 8, desc_sf32(sfb + 1024 * kk + 128, 256));
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(bar_sfr + 8 * s), "h"((unsigned short)(1u << (2 * pp))) : "memory");
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 8 && !g.sfcp && g.cpmask != (1 << STAGES) - 1) {
    // ---------------- scale warps: raw scales -> TMEM (both CTAs) ----------------
    // Warp 4+sp writes TMEM lanes 32sp..32sp+31, i.e. one replica of every
    // scale vector; lane L holds rows 32c + L (c = column within a 4-group).
    const int sp = warp - 4;
    const uint32_t trow = (uint32_t)(sp * 32) << 16;
    // Stages are written two at a time with one tcgen05.wait::st: the per-stage chain
    // (LDS -> STTM -> wait -> fence -> remote arrive) is longer than a stage's MMAs, so
    // one stage per round left the MMA waiting on scales.
    const int my_tiles = clid < nsuper ? (nsuper - 1 - clid) / ncl + 1 : 0;
    const int total = my_tiles * g.nk;
    for (int it = 0; it < (g.dbg >= 4 ? min(total, STAGES) : total); it += Q2_SF_BATCH) {
      const int nb = min(Q2_SF_BATCH, (g.dbg >= 4 ? min(total, STAGES) : total) - it);
#pragma unroll
      for (int u = 0; u < Q2_SF_BATCH; ++u) {
        if (u >= nb) break;
        const int s = (it + u) % STAGES;
        if ((g.cpmask >> s) & 1) continue;                    // the copier's stage
        mbar_wait_sleep(bar_sff + 8 * s, ((it + u) / STAGES) & 1);
        const unsigned char* sfa = smem + s * STAGE + A_ST + B_ST;
        const unsigned char* sfb = sfa + SFA_ST;
        const uint32_t tsf = tmem + trow + SF_COL + SF_SLOT * s;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (g.dbg == 1 || (g.dbg == 2 && sp != 0) || (g.dbg == 3 && sp != (int)(rank * 0) + 0 && sp != 1)) break;
          const uint4 a4 = *reinterpret_cast<const uint4*>(sfa + 512 * kk + (lane >> 3) * 128 + (lane & 7) * 16);
          const uint4 b0 = *reinterpret_cast<const uint4*>(sfb + 1024 * kk + (lane >> 3) * 256 + (lane & 7) * 16);
          const uint4 b1 = *reinterpret_cast<const uint4*>(sfb + 1024 * kk + (lane >> 3) * 256 + 128 + (lane & 7) * 16);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                       ::"r"(tsf + 12 * kk), "r"(a4.x), "r"(a4.y), "r"(a4.z), "r"(a4.w) : "memory");
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                       ::"r"(tsf + 12 * kk + 4), "r"(b0.x), "r"(b0.y), "r"(b0.z), "r"(b0.w), "r"(b1.x), "r"(b1.y),
                       "r"(b1.z), "r"(b1.w) : "memory");
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        for (int u = 0; u < nb; ++u)
          if (!((g.cpmask >> ((it + u) % STAGES)) & 1)) mbar_arrive_leader(bar_sfr + 8 * ((it + u) % STAGES));
    }
  } else if (warp >= 8) {
    // ---------------- epilogue ----------------
    const int e = warp - 8, sp = e & 3, grp = e >> 2;
    const int row = sp * 32 + lane;                           // row within the CTA's 128
    const float alpha = __ldg(g.sa) * __ldg(g.sb);
    const uint32_t tbase = tmem + ((uint32_t)(sp * 32) << 16) + grp * 128;
    int tc = 0;
    for (int u = clid; u < nsuper; u += ncl, ++tc) {
      int tm, tn;
      super_coords<CL, SHARE_A>(u, g, (int)pp, tm, tn);
      mbar_wait_sleep(bar_accf, tc & 1);
      tc_fence_after();
      if (g.trace && tr0 && rank == 0 && warp == 8 && lane == 0 && tc < 64) g.trace[4 * tc + 2] = gtime();
      const int gm = tm * PT + (int)rank * 128 + row, gn0 = tn * PT + grp * 128;
      unsigned char* drow = static_cast<unsigned char*>(g.d) + (int64_t)gm * g.ldd * (F32 ? 4 : 2);
      if (!F32) {
        // bf16: pack the first 64 columns while the second 64 are loaded, release
        // the accumulator after the last TMEM read, then store (TMEM reads run at
        // ~64 B/clk, so no store sits between them)
        uint32_t pk[32], v[64];
        tmem_ld64(v, tbase);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(v[2 * i]), alpha * __uint_as_float(v[2 * i + 1]));
          pk[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        tmem_ld64(v, tbase + 64);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(bar_acce);          // MMA may overwrite the accumulator
        if (g.trace && tr0 && rank == 0 && warp == 8 && lane == 0 && tc < 64) g.trace[4 * tc + 3] = gtime();
        __nv_bfloat16* dr = reinterpret_cast<__nv_bfloat16*>(drow);
        if (Q2_GEMM_STAGE_EPI && tm * PT + (int)rank * 128 + 128 <= g.M && gn0 + 128 <= g.N) {
          // coalesced stores: the warp's 32 rows x 64 columns go through 4 KB of shared memory
          // (16-byte chunks swizzled by row) and leave as 4 full 128-byte row segments per
          // store instruction instead of 32 partial ones
          unsigned char* stg = smem + OFF_EPI + 4096 * e;
          const int lr = lane >> 3, lc = lane & 7;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              uint32_t p[4];
              if (hh == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) p[i] = pk[4 * c + i];
              } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int j = 8 * c + 2 * i;
                  __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(v[j]), alpha * __uint_as_float(v[j + 1]));
                  p[i] = *reinterpret_cast<uint32_t*>(&h);
                }
              }
              *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
            }
            __syncwarp();
            const int64_t row0 = (int64_t)(tm * PT + (int)rank * 128 + sp * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 4 * i + lr;
              const uint4 q = *reinterpret_cast<const uint4*>(stg + r * 128 + ((lc ^ (r & 7)) << 4));
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(g.d) + (row0 + r) * g.ldd + gn0 + 64 * hh + 8 * lc) = q;
            }
            __syncwarp();
          }
          continue;
        }
        if (gm >= g.M) continue;
#pragma unroll
        for (int c = 0; c < 16; ++c) {                        // 8 columns per 16-byte store
          uint32_t p[4];
          if (c < 8) {
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = pk[4 * c + i];
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = 8 * (c - 8) + 2 * i;
              __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(v[j]), alpha * __uint_as_float(v[j + 1]));
              p[i] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          const int n = gn0 + 8 * c;
          if (n + 8 <= g.N) {
            *reinterpret_cast<uint4*>(dr + n) = make_uint4(p[0], p[1], p[2], p[3]);
          } else {
            for (int i = 0; i < 8 && n + i < g.N; ++i) dr[n + i] = reinterpret_cast<const __nv_bfloat16*>(p)[i];
          }
        }
        continue;
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {                  // 64 columns per pass
        uint32_t v[2][32];
        tmem_ld64(&v[0][0], tbase + half * 64);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (half == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(bar_acce);        // MMA may overwrite the accumulator
          if (g.trace && tr0 && rank == 0 && warp == 8 && lane == 0 && tc < 64) g.trace[4 * tc + 3] = gtime();
        }
        if (F32 && Q2_GEMM_STAGE_EPI && tm * PT + (int)rank * 128 + 128 <= g.M && gn0 + 128 <= g.N) {
          // coalesced fp32 stores (and accumulate reads) through the warp's 4 KB of shared memory
          unsigned char* stg = smem + OFF_EPI + 4096 * e;
          const int lr = lane >> 3, lc = lane & 7;
          const int64_t row0 = (int64_t)(tm * PT + (int)rank * 128 + sp * 32);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_float4(alpha * __uint_as_float(v[q][4 * c]), alpha * __uint_as_float(v[q][4 * c + 1]),
                              alpha * __uint_as_float(v[q][4 * c + 2]), alpha * __uint_as_float(v[q][4 * c + 3]));
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 4 * i + lr;
              float4 o = *reinterpret_cast<const float4*>(stg + r * 128 + ((lc ^ (r & 7)) << 4));
              float* dp = static_cast<float*>(g.d) + (row0 + r) * g.ldd + gn0 + 64 * half + 32 * q + 4 * lc;
              out_f32x4(dp, o, g.accumulate);
            }
            __syncwarp();
          }
          continue;
        }
        if (gm >= g.M) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#pragma unroll
          for (int c8 = 0; c8 < 32; c8 += F32 ? 4 : 8) {
            const int n = gn0 + 64 * half + 32 * q + c8;
            if (F32) {
              float4 o = make_float4(alpha * __uint_as_float(v[q][c8]), alpha * __uint_as_float(v[q][c8 + 1]),
                                     alpha * __uint_as_float(v[q][c8 + 2]), alpha * __uint_as_float(v[q][c8 + 3]));
              float* dp = reinterpret_cast<float*>(drow) + n;
              if (n + 4 <= g.N) {
                out_f32x4(dp, o, g.accumulate);
              } else {
                const float oo[4] = {o.x, o.y, o.z, o.w};
                for (int i = 0; i < 4 && n + i < g.N; ++i) out_f32(dp + i, oo[i], g.accumulate);
              }
            } else {
              uint32_t p[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                __nv_bfloat162 h = __floats2bfloat162_rn(alpha * __uint_as_float(v[q][c8 + 2 * i]),
                                                         alpha * __uint_as_float(v[q][c8 + 2 * i + 1]));
                p[i] = *reinterpret_cast<uint32_t*>(&h);
              }
              __nv_bfloat16* dp = reinterpret_cast<__nv_bfloat16*>(drow) + n;
              if (n + 8 <= g.N) {
                *reinterpret_cast<uint4*>(dp) = make_uint4(p[0], p[1], p[2], p[3]);
              } else {
                for (int i = 0; i < 8 && n + i < g.N; ++i) dp[i] = reinterpret_cast<const __nv_bfloat16*>(p)[i];
              }
            }
          }
        }
      }
    }
  }
  // multicast reductions performed system-wide before the kernel retires, so the caller's
  // cross-GPU barrier after this launch orders them (release side of that barrier)
  if (F32 && g.accumulate == 3) asm volatile("fence.acq_rel.sys;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();                                             // peer's MMAs/arrivals done before teardown
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

static bool make_sf_map(CUtensorMap* map, const void* sf, int64_t R, int64_t K, uint32_t halves, uint32_t groups_box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  const uint64_t groups = (uint64_t)((R + 255) / 256) * (uint64_t)sf_kblocks(K) * 4;
  cuuint64_t dims[3] = {128, 2, (cuuint64_t)groups};
  cuuint64_t strides[2] = {128, 256};
  cuuint32_t box[3] = {128, halves, groups_box};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(sf), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Persistent grid: as many clusters as fit at once (clusters of 8 CTAs may not tile every
// GPC, so the count comes from the occupancy query, once per device).
template <bool F32, int CL, bool SHARE_A>
static int launch_gemm(const CUtensorMap* maps, const GemmArgs& g, cudaStream_t st) {
  auto kern = nvfp4_gemm_kernel<F32, CL, SHARE_A>;
  static unsigned attr = 0;                     // per-device opt-in
  static int max_cl[64] = {0};
  if (!smem_opt_in(kern, GEMM_SMEM, attr)) return Q2_ECUDA;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int& mc = max_cl[dev & 63];
  if (mc == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm / (2 * CL) * 2 * CL);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM_SMEM;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = nsm / (2 * CL);
    }
    mc = n;
    if (getenv("Q2_GEMM_VERBOSE")) fprintf(stderr, "gemm: clusters of %d pairs, %d resident\n", CL, n);
  }
  const int nsuper = SHARE_A ? g.tiles_m * ((g.tiles_n + CL - 1) / CL) : ((g.tiles_m + CL - 1) / CL) * g.tiles_n;
  const int ncl = std::max(1, std::min(nsuper, mc));
  if (launch_pdl(kern, dim3(2 * CL * ncl), dim3(GEMM_THREADS), GEMM_SMEM, st, maps[0], maps[1],
                 maps[2], maps[3], g) != cudaSuccess)
    return Q2_ECUDA;
  return Q2_OK;
}

// Pairs per cluster and the shared operand: clusters of CL pairs read the common operand
// from L2 once (TMA multicast) -- the kernel is L2-throughput bound otherwise (ncu: LTS at
// ~52% of its nominal peak = the chip's practical cap).  Prefer the side that divides evenly.
template <bool F32>
static int dispatch_gemm(const q2_nvfp4* a, const q2_nvfp4* b, const CUtensorMap* maps, GemmArgs& g,
                         cudaStream_t st, int cl) {
  const bool share_a = g.tiles_n % cl == 0 || g.tiles_m % cl != 0;
  if (cl > 1) {
    // the shared operand's map loads 128/cl-row slices
    const int sl = 128 / cl;
    CUtensorMap* m = const_cast<CUtensorMap*>(maps);
    const bool ok = share_a ? make_map(&m[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, a->codes, a->K / 2, a->R, a->K / 2, BKB, sl)
                            : make_map(&m[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, b->codes, b->K / 2, b->R, b->K / 2, BKB, sl);
    if (!ok) return Q2_ECUDA;
  }
  if (cl == 4) return share_a ? launch_gemm<F32, 4, true>(maps, g, st) : launch_gemm<F32, 4, false>(maps, g, st);
  if (cl == 2) return share_a ? launch_gemm<F32, 2, true>(maps, g, st) : launch_gemm<F32, 2, false>(maps, g, st);
  return launch_gemm<F32, 1, true>(maps, g, st);
}

}  // namespace q2

using namespace q2;

extern "C" int q2_gemm_tn(const q2_nvfp4* a, const q2_nvfp4* b, void* d, int d_dtype, int64_t ldd, int accumulate,
                          void* stream) {
  if (!a || !b || !d || a->K != b->K || a->K % 64 || (a->K / 2) % 16 || a->R <= 0 || b->R <= 0) return Q2_EINVAL;
  if (d_dtype != Q2_BF16 && d_dtype != Q2_F32) return Q2_EINVAL;
  if (accumulate < Q2_ACC_STORE || accumulate > Q2_ACC_MULTIMEM || (accumulate && d_dtype != Q2_F32)) return Q2_EINVAL;
  const int esz = d_dtype == Q2_F32 ? 4 : 2;
  if (ldd < b->R || (ldd * esz) % 16 || (reinterpret_cast<uintptr_t>(d) & 15)) return Q2_EINVAL;
  if (a->R > INT32_MAX || b->R > INT32_MAX || a->K > INT32_MAX) return Q2_EINVAL;
  CUtensorMap maps[4];
  if (!make_map(&maps[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, a->codes, a->K / 2, a->R, a->K / 2, BKB, 128) ||
      !make_map(&maps[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, b->codes, b->K / 2, b->R, b->K / 2, BKB, 128) ||
      !make_sf_map(&maps[2], a->sf, a->R, a->K, 1, 16) || !make_sf_map(&maps[3], b->sf, b->R, b->K, 2, 16))
    return Q2_ECUDA;
  static unsigned long long* trace = nullptr;
  if (getenv("Q2_GEMM_TRACE") && !trace) cudaMalloc(&trace, 64 * 8 * 8);
  // A/B option: scales copied by the MMA thread with tcgen05.cp (measured 1.3-1.7x slower: each
  // 512-byte 32x128b.warpx4 copy holds the tensor pipe ~60 cycles, 12 per stage > the stage's MMAs)
  static const int g_gemm_cp = getenv("Q2_GEMM_CP") ? atoi(getenv("Q2_GEMM_CP")) : 0;
  // stages whose scales the copier thread moves (the rest by the scale warps): three of five
  // measured best for short (<= 12 stages of 256 per tile) and long K alike once the epilogue
  // stores were staged (sweeps of 0x0A..0x1F, tools/gemm_c3.py); kept as two knobs
  static const int g_mask_long = getenv("Q2_GEMM_CPMASK_LONG") ? (int)strtol(getenv("Q2_GEMM_CPMASK_LONG"), nullptr, 0) : 0x15;
  static const int g_mask_short = getenv("Q2_GEMM_CPMASK_SHORT") ? (int)strtol(getenv("Q2_GEMM_CPMASK_SHORT"), nullptr, 0) : 0x15;
  const int nk_tiles = (int)((a->K / 2 + BKB - 1) / BKB);
  const int cpmask = g_gemm_cp ? 0 : (nk_tiles <= 12 ? g_mask_short : g_mask_long);
  GemmArgs g{a->scale32, b->scale32, d, ldd, (int)a->R, (int)b->R, (int)a->K, (int)sf_kblocks(a->K),
             (int)((a->R + PT - 1) / PT), (int)((b->R + PT - 1) / PT), (int)((a->K / 2 + BKB - 1) / BKB), accumulate, getenv("Q2_GEMM_DBG") ? atoi(getenv("Q2_GEMM_DBG")) : 0, g_gemm_cp, cpmask,
             getenv("Q2_GEMM_TRACE") ? trace : nullptr};
  if (g.trace) cudaMemsetAsync(trace, 0, 64 * 8 * 8, static_cast<cudaStream_t>(stream));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // clusters of 2 or 4 pairs multicasting the shared operand: measured slower (the occupancy
  // query gives 33 / 15 resident clusters = 132 / 120 SMs, and the per-SM rate does not rise:
  // multicast to <= 4 CTAs costs L2 like unicast), kept as an A/B option
  static const int g_cl = getenv("Q2_GEMM_CL") ? atoi(getenv("Q2_GEMM_CL")) : 1;
  const int cl = g_cl == 4 ? 4 : (g_cl == 2 ? 2 : 1);
  const int rc = d_dtype == Q2_F32 ? dispatch_gemm<true>(a, b, maps, g, st, cl) : dispatch_gemm<false>(a, b, maps, g, st, cl);
  if (g.trace) {
    unsigned long long h[512];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 12; ++i)
      fprintf(stderr, "tile %d: mma %.2f us (waits: operands %.2f, scales %.2f; scale warp: lds+st %.2f, wait::st+arrive %.2f), "
              "accf->wake %.2f, wake->release %.2f, release->next start %.2f\n", i, (h[4 * i + 1] - h[4 * i]) / 1e3,
              h[256 + 2 * i] / 1e3, h[257 + 2 * i] / 1e3, h[384 + 2 * i] / 1e3, h[385 + 2 * i] / 1e3, (h[4 * i + 2] - h[4 * i + 1]) / 1e3, (h[4 * i + 3] - h[4 * i + 2]) / 1e3,
              (h[4 * i + 4] - h[4 * i + 3]) / 1e3);
  }
  return rc;
}
