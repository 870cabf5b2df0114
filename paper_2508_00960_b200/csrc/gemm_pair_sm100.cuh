// 2-SM (cta_group::2) variant of the grouped GEMM for the bf16 tier.
//
// A CTA pair (cluster of 2) owns a 256 x BN output tile: each CTA stages 128 rows of A and BN/2
// rows of B; the leader issues M=256 tcgen05.mma into both CTAs' TMEM.  A stage carries
// K = PBK (default 128: two 64-wide SWIZZLE_128B atoms, 3 stages), so one stage is 8 MMAs = 1024
// tensor cycles per SM between barrier round trips (the 1-SM kernel's 4 MMAs / 512 cycles leaves the tensor pipe
// ~25% idle on barrier/issue latency).  Double-buffered TMEM accumulators (2 x 256 columns) keep
// the epilogue of tile i under the MMAs of tile i+1.  Problems, segments, slot-blocked K / N
// coordinates and the epilogue are shared with gemm_sm100.cuh (same GemmParams).
#pragma once
#include "gemm_sm100.cuh"

namespace ppx {

#ifndef PPX_PBK
#define PPX_PBK 128
#endif
constexpr int PBK = PPX_PBK;                     // K elements per stage (PKA 64-wide atoms)
constexpr int PKA = PBK / 64;
static_assert(PBK % 64 == 0 && PKA >= 1 && PKA <= 4, "stage K must be 1..4 whole atoms");
constexpr int PA_STAGE = BM * PKA * ROW_BYTES;   // [PKA K-atoms][128 rows][128 B] (32 KB at K 128)
constexpr int PB_STAGE = 128 * PKA * ROW_BYTES;  // [PKA K-atoms][<=128 rows][128 B]
constexpr int PSTAGES = (192 * 1024) / (PA_STAGE + PB_STAGE);   // 192 KB of operand ring
constexpr int PSMEM_BYTES = PSTAGES * (PA_STAGE + PB_STAGE) + 1024 + 256 + EPI_STAGE_BYTES;

__device__ __forceinline__ void tma4_pair(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma5_pair(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %3, "
      "%4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

// Operand maps for this kernel (host side, ppx.cu):
//   K-major:          4D {64, rows, K/64 atoms, slots}  box {64, rows_per_cta, PKA, 1}  -> [katom][rows][128B]
//   MN-major (mode1): 4D {64, K rows, MN atoms, slots}  box {64, PBK, natoms, 1}       -> [atom][PBK K rows][128B]
//   MN-major (mode2): 5D {64, 8, MN atoms, K/8, slots}  box {64, 8, natoms, PBK/8, 1}  -> [kgroup][atom][8][128B]
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_pair_kernel(const __grid_constant__ GemmParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base_u32;
  const uint32_t sB = sA + PSTAGES * PA_STAGE;
  const uint32_t sBar = sB + PSTAGES * PB_STAGE;
  auto full_bar = [&](int s) { return sBar + 8u * s; };
  auto empty_bar = [&](int s) { return sBar + 8u * (PSTAGES + s); };
  auto tfull_bar = [&](int s) { return sBar + 8u * (2 * PSTAGES + s); };
  auto tempty_bar = [&](int s) { return sBar + 8u * (2 * PSTAGES + 2 + s); };
  const uint32_t tmem_slot = sBar + 8u * (2 * PSTAGES + 4);
  uint8_t* smem_gen = smem_raw + (base_u32 - smem_u32(smem_raw));
  volatile uint32_t* tmem_slot_ptr = reinterpret_cast<volatile uint32_t*>(smem_gen + (tmem_slot - base_u32));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t* epi_stage = reinterpret_cast<uint32_t*>(smem_gen + (sBar + 256 - base_u32));
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  constexpr int CHA = 64;       // bf16 elements per 128-byte atom
  constexpr int KMMA = 16;      // K per tcgen05.mma (bf16)

  if (warp == W_TMA && lane == 0) {
    for (int i = 0; i < P.nmaps; ++i) prefetch_map(&P.maps[i]);
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull_bar(s), 1);
      mbar_init(tempty_bar(s), 2 * NUM_EPI_WARPS);   // the epilogue warps of both CTAs of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_ALLOC) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  // programmatic dependent launch: the prologue above (barrier init, TMEM alloc, tensor-map
  // prefetch) overlapped the previous kernel's tail; global memory is touched only once that
  // kernel has completed.  Our own dependents may start their prologue from here on.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int t0 = (int)(blockIdx.x >> 1);
  const int tstep = (int)(gridDim.x >> 1);

  if (is_epi_warp(warp)) {
    reg_alloc_epilogue();
    epilogue_loop<2 * BM, true>(P, tmem_base, tfull_bar(0), tempty_bar(0), t0, tstep, crank, warp, lane, epi_stage);
  } else {
  reg_dealloc_mainloop();
  if (warp >= W_PUB0) {
    publisher_loop<2 * BM>(P, t0, tstep, crank, warp, lane);
  } else if (warp == W_TMA) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long st_empty = 0;
      const int epoch = P.epoch ? *(volatile int*)P.epoch : 0;
      for (int i = 0, t; (t = tile_of(P, t0, tstep, i)) >= 0; ++i) {
        TileCoord tc = tile_coord<2 * BM>(P, t);
        const Problem& pr = P.probs[tc.prob];
        const int bnc = pr.BN / 2;
        const uint32_t bytes = (uint32_t)(BM + bnc) * (uint32_t)PKA * ROW_BYTES * 2u;   // both CTAs, PKA K-atoms each
        const int am0 = tc.m0 + (int)crank * BM;
        // a spanning tile gives each CTA of the pair one whole N block; otherwise the two CTAs
        // split one block's BN columns
        const bool span = pr.nspan > 1;
        const int bn0 = span ? tc.nin : tc.nin + (int)crank * bnc;
        const int qb = span ? tc.qn + (int)crank : tc.qn;
        for (int sg = 0; sg < pr.nsegs; ++sg) {
          const Segment& seg = pr.segs[sg];
          const CUtensorMap* ma = &P.maps[seg.a.map];
          const CUtensorMap* mb = &P.maps[seg.b.map];
          if (sg == pr.wait_seg && pr.wait_ctr) wait_dependency(P, pr, epoch);
          for (int kt = 0; kt < seg.k_tiles; ++kt) {
            const int kblk = kt / seg.kpb;
            const int kin = (kt - kblk * seg.kpb) * PBK;
            mbar_wait_t(empty_bar(stage), phase ^ 1u, kStats && P.stats != nullptr, st_empty);
            if (leader) mbar_expect_tx(full_bar(stage), bytes);
            const uint32_t fb = mapa_shared(full_bar(stage), 0);
            const uint32_t da = sA + stage * PA_STAGE;
            const uint32_t db = sB + stage * PB_STAGE;
            const int slot_a = op_slot(seg.a, kblk, tc.qn);
            const int slot_b = op_slot(seg.b, kblk, qb);
            if (!seg.a.mn) tma4_pair(ma, fb, da, 0, am0, kin / CHA, slot_a);
            else if (seg.a.atoms4d == 2) tma5_pair(ma, fb, da, am0 / CHA, kin / 8, slot_a);
            else tma4_pair(ma, fb, da, 0, kin, am0 / CHA, slot_a);
            if (!seg.b.mn) tma4_pair(mb, fb, db, 0, bn0, kin / CHA, slot_b);
            else if (seg.b.atoms4d == 2) tma5_pair(mb, fb, db, bn0 / CHA, kin / 8, slot_b);
            else tma4_pair(mb, fb, db, 0, kin, bn0 / CHA, slot_b);
            if (++stage == PSTAGES) { stage = 0; phase ^= 1u; }
          }
        }
      }
      if (kStats && P.stats) atomicAdd(P.stats + 2, st_empty);
    }
    __syncwarp();
  } else if (warp == W_MMA) {
    // ===================== MMA issuer (leader CTA, one lane) =====================
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      unsigned long long st_tempty = 0, st_full = 0;
      const unsigned long long c_start = kStats && P.stats ? clock64() : 0ull;
      for (int t; (t = tile_of(P, t0, tstep, iter)) >= 0; ++iter) {
        TileCoord tc = tile_coord<2 * BM>(P, t);
        const Problem& pr = P.probs[tc.prob];
        const int as = iter & 1;
        const uint32_t aphase = (iter >> 1) & 1;
        mbar_wait_t(tempty_bar(as), aphase ^ 1u, kStats && P.stats != nullptr, st_tempty);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + as * BN_MAX;
        const int bnc = pr.BN / 2;
        uint32_t accum = 0;
        for (int sg = 0; sg < pr.nsegs; ++sg) {
          const Segment& seg = pr.segs[sg];
          const uint32_t idesc = seg.idesc;
          // per-operand descriptor geometry (bytes): LBO, SBO, advance per MMA, advance per K atom
          uint32_t a_lbo, a_sbo, a_step, a_katom, b_lbo, b_sbo, b_step, b_katom;
          if (!seg.a.mn) { a_lbo = 16; a_sbo = 1024; a_step = 32; a_katom = BM * ROW_BYTES; }
          else if (seg.a.atoms4d == 2) {
            a_lbo = 1024; a_sbo = (BM / CHA) * 1024; a_step = 2 * a_sbo; a_katom = 4 * a_step;
          } else { a_lbo = PBK * ROW_BYTES; a_sbo = 1024; a_step = KMMA * ROW_BYTES; a_katom = 4 * a_step; }
          if (!seg.b.mn) { b_lbo = 16; b_sbo = 1024; b_step = 32; b_katom = bnc * ROW_BYTES; }
          else if (seg.b.atoms4d == 2) {
            b_lbo = 1024; b_sbo = (bnc / CHA) * 1024; b_step = 2 * b_sbo; b_katom = 4 * b_step;
          } else { b_lbo = PBK * ROW_BYTES; b_sbo = 1024; b_step = KMMA * ROW_BYTES; b_katom = 4 * b_step; }
          for (int kt = 0; kt < seg.k_tiles; ++kt) {
            mbar_wait_t(full_bar(stage), phase, kStats && P.stats != nullptr, st_full);
            tc_fence_after();
            const uint32_t da = sA + stage * PA_STAGE;
            const uint32_t db = sB + stage * PB_STAGE;
#pragma unroll
            for (int ka = 0; ka < PKA; ++ka) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = sdesc(da + ka * a_katom + kk * a_step, a_lbo, a_sbo);
                const uint64_t bd = sdesc(db + ka * b_katom + kk * b_step, b_lbo, b_sbo);
                mma_pair(tmem_d, ad, bd, idesc, accum);
                accum = 1;
              }
            }
            commit_pair(empty_bar(stage));
            if (++stage == PSTAGES) { stage = 0; phase ^= 1u; }
          }
        }
        commit_pair(tfull_bar(as));
      }
      if (kStats && P.stats) {
        atomicAdd(P.stats + 3, st_tempty);
        atomicAdd(P.stats + 4, st_full);
        atomicAdd(P.stats + 5, clock64() - c_start);
        atomicAdd(P.stats + 6, 1ull);
      }
    }
    __syncwarp();
  }
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == W_ALLOC) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
  end_epoch(P);
}

}  // namespace ppx
