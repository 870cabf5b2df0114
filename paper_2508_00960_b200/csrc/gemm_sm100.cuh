// Grouped, K-segmented tcgen05 GEMM for sm_100a with fused phantom-layer epilogues.
//
// One persistent kernel serves every dense contraction on the phantom-parallel hot path
// (reference call sites phantom.py:152-264, tensor_parallel.py:115-145):
//
//   D[m, n] = sum_seg  A_seg[m, :] . B_seg[n, :]        (fp32 accumulation in TMEM)
//
// * Operands are staged by TMA (cp.async.bulk.tensor.3d, SWIZZLE_128B) into a 4-stage smem
//   ring and consumed by tcgen05.mma issued from one thread; accumulators live in TMEM
//   (2 x 256 columns, double buffered so the epilogue of tile i overlaps the MMAs of i+1).
// * Each operand is either K-major or MN-major (the transposed-operand GEMMs of the backward
//   pass read activations [batch, features] as MN-major tiles, no transpose kernels).
// * A "problem" is one output matrix (or a stack of same-shaped blocks: the per-peer
//   decompressor blocks); up to MAX_PROBS problems share one launch (grouped GEMM).
// * A problem sums up to MAX_SEGS K-segments, each with its own tensor maps: this is how the
//   local block and the (p-1) incoming phantom blocks become ONE K-concatenated contraction
//   (phantom.py:152+156-157), how [delta | r] . [L ; C] is formed (phantom.py:228-229), and how
//   the fp32 tier runs 3xTF32 (hi*hi + hi*lo + lo*hi) on the same machinery.
// * Blocked coordinates: a segment's K range, or a problem's N range, can walk over "slots"
//   (the third tensor-map dimension) skipping the caller's own rank, which reads the
//   all-gathered phantom buffer [p, batch, k] directly (phantom.py:155-157, 202-205, 259-264).
// * The epilogue fuses bias, ReLU, pre-activation store, the ReLU'-mask of the error
//   recurrence, the output delta + half-squared loss, bias-gradient column sums, accumulate
//   into an existing output, and in-place SGD / Adam on fp32 master weights.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <type_traits>

namespace ppx {

constexpr int BM = 128;           // tcgen05 M (cta_group::1)
constexpr int BN_MAX = 256;       // max tcgen05 N per tile
constexpr int STAGES = 4;         // smem ring depth
constexpr int ROW_BYTES = 128;    // one SWIZZLE_128B row = one BK slice of K
constexpr int A_STAGE_BYTES = BM * ROW_BYTES;          // 16 KB
constexpr int B_STAGE_BYTES = BN_MAX * ROW_BYTES;      // 32 KB
// Warp roles: w0-7 epilogue (TMEM lane quadrant = warp % 4; warps 0-3 drain the even 32-column
// chunks of a tile, warps 4-7 the odd ones, so each SM sub-partition runs two independent
// epilogue instruction streams), w8 TMA producer + TMEM allocator, w9 MMA issuer. The SM's warp
// schedulers favour the higher warp id among eligible warps, so the producer and the MMA issuer
// never wait behind an epilogue warp for an issue slot.
// Warpgroups 0-1 (the epilogue) raise their register budget to 232 and warpgroup 2 (producer,
// MMA, two idle warps) drops to 40 (setmaxnreg), so the 32-wide epilogue math never spills.
constexpr int NUM_EPI_WARPS = 8;
constexpr int NUM_THREADS = 384;
constexpr int W_TMA = 8, W_MMA = 9, W_ALLOC = 8;
__device__ __forceinline__ bool is_epi_warp(int w) { return w < NUM_EPI_WARPS; }
__device__ __forceinline__ void reg_alloc_epilogue() { asm volatile("setmaxnreg.inc.sync.aligned.u32 232;"); }
__device__ __forceinline__ void reg_dealloc_mainloop() { asm volatile("setmaxnreg.dec.sync.aligned.u32 40;"); }
constexpr int TMEM_COLS = 512;    // 2 accumulator stages x 256 fp32 columns
constexpr int MAX_MAPS = 40;
constexpr int MAX_PROBS = 16;
constexpr int MAX_SEGS = 12;   // 4 contributing ranks x 3 TF32 passes (FP32-tier error slots)
constexpr int MAX_REP = 7;
constexpr int MAX_SCHED = 4096;    // tiles of one LPT-scheduled launch         // peer replicas of an epilogue output (world <= 8)
// per-epilogue-warp staging of one 32 x 32 bf16 output chunk (80-byte rows: 64 B data + 16 B pad),
// so the warp's stores leave as full 64-byte row segments instead of 32 half-filled sectors
constexpr int EPI_STAGE_ROW_WORDS = 20;
constexpr int EPI_STAGE_BYTES = NUM_EPI_WARPS * 32 * EPI_STAGE_ROW_WORDS * 4;
constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE_BYTES;

// epilogue flags
enum : uint32_t {
  EP_BIAS = 1u << 0,      // v += bias[col]
  EP_RELU = 1u << 1,      // y = max(v, 0)
  EP_PREACT = 1u << 2,    // store pre-activation (after bias) to `preact`
  EP_MASK = 1u << 3,      // v *= (mask[row, col] > 0)   (ReLU'(preact) from the layer output)
  EP_LOSS = 1u << 4,      // output layer: diff = y - target; aux = diff * act'(pre) * scale; loss += diff^2
  EP_COLSUM = 1u << 5,    // colsum[col] += delta value (bias gradient, phantom.py:253)
  EP_ACCUM = 1u << 6,     // out = out + v
  EP_SGD = 1u << 7,       // master -= lr * v ; out = cast(master)
  EP_ADAM = 1u << 8,      // Adam on master with m, v moments ; out = cast(master)
  EP_GRAD = 1u << 9,      // also store the raw gradient to `aux` (fp32)
  EP_FINITE = 1u << 10,   // flag non-finite accumulator values
  EP_BITS = 1u << 11,     // also store the ReLU'(pre) bit mask, bit i of word (row, col/32) = v > 0, to
                          // `preact` as uint32 words (ld in words; forward layers feeding a recurrence)
  EP_MASKBITS = 1u << 12, // EP_MASK from such a bit mask in `mask` instead of the bf16 layer output
};

struct Operand {
  int8_t map;        // tensor-map index
  int8_t mn;         // 0 = K-major, 1 = MN-major
  int8_t slot_src;   // 0 = const, 1 = K-block index, 2 = N-block index
  int8_t atoms4d;    // MN-major only: 1 = 4D map {atom, K, atoms, slots} (atom-major smem tile);
                     // 2 = 5D map {atom, 8 rows, atoms, K groups, slots}: canonical interleaved tile
  int slot_base;
  int slot_skip;     // raw slot index >= skip is shifted by one (own rank excluded); INT_MAX = none
                     // < 0: decompressor-stack mode of rank -skip-1 (see op_slot)
};

struct Segment {
  Operand a, b;
  int k_tiles;       // number of BK slices
  int kpb;           // BK slices per K block (K-blocked segments walk slots); == k_tiles otherwise
  uint32_t idesc;    // tcgen05 instruction descriptor (majors, N, M)
};

struct Tensor2 {     // epilogue side tensor: row-major with leading dim, optional slot stride
  void* ptr;
  long long ld;
  long long slot_stride;
  int f32;           // 0 = bf16, 1 = fp32
  int pad_;
};

struct Epilogue {
  uint32_t flags;
  int out_skip;      // N-block -> output slot skip (own rank)
  Tensor2 out, aux, preact, mask, target, master, adam_m, adam_v;
  const float* bias;
  float* colsum;
  float* loss;       // += sum diff^2 * loss_scale
  int* bad;          // non-finite flag
  const float* hyper;   // device scalars: [lr, beta1, beta2, eps, bias_corr1, bias_corr2]
  float scale;       // delta scale (1 or 1/B)
  float loss_scale;  // 0.5 or 0.5/B
  int nrep;          // plain stores only: also write every output element at out + rep_off[r] bytes
  int narrive;       // after each CTA's part of a tile is stored (incl. replicas): fence (system
                     // scope) and add to each arrive[i] (this GPU's and the peers' counters):
  int arrive_units;  //   0: 1 per CTA-tile; 1: rows * cols / 8 of the CTA's part (tiling-independent)
  int rep_per_half;  // spanning tiles whose two N blocks have different destinations: half h goes to
                     // out + rep_off[h] (0 = not sent) and counts on arrive[h] (null = none)
  int* arrive[MAX_REP + 1];
  long long rep_off[MAX_REP];   // (peer copies of the output buffer mapped over NVLink: the phantom
                                // all-gather fused into the compression GEMM's epilogue)
};

struct Problem {
  int M;             // rows of D
  int nb_extent;     // columns per N block
  int nblk;          // number of N blocks
  int BN;            // tile N (multiple of 16, <= 256)
  int m_tiles, npb;  // tiles along M, tiles per N block
  int m_base;        // first row covered by this problem's tiles (a split-off tail of a problem)
  int nspan;         // 2-SM kernel: N blocks per tile (2 = each CTA of the pair owns one whole N block)
  int tile_begin;    // prefix over problems
  // in-kernel dependency (fused compress + all-gather + forward): before loading segment
  // `wait_seg` the producers spin until *wait_ctr >= (*P.epoch + 1) * wait_per_epoch
  const int* wait_ctr;
  int wait_seg;
  int wait_per_epoch;
  int nsegs;
  Segment segs[MAX_SEGS];
  Epilogue epi;
};

struct alignas(64) GemmParams {
  CUtensorMap maps[MAX_MAPS];
  Problem probs[MAX_PROBS];
  int nmaps;
  int nprobs;
  int total_tiles;
  int dbg;             // debug: bit0 = skip the epilogue body (TMEM drain only by arrival)
  unsigned long long* stats;   // debug (PPX_DEBUG_STATS): per-role wait / busy clock sums, else null
  int nsched;          // > 0: static LPT schedule — cluster c runs tiles sched[sched_off[c] .. sched_off[c+1])
  uint16_t sched_off[76];
  uint16_t sched[MAX_SCHED];
  int* epoch;          // launches with waiting problems: *epoch += 1 by the last CTA to exit
  unsigned int* done;  //   (CTA exit counter, self-resetting)
  int* bad;            //   |= 2 when a wait timed out
};
static_assert(sizeof(GemmParams) <= 32764, "kernel parameter space");

// ------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Blocking wait with a watchdog: a pipeline bug traps after ~20 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity);
// per-role clock statistics (wait / busy cycles, PPX_DEBUG_STATS at run time) exist only in a
// build with -DPPX_STATS=1: the counters cost registers the 40-register mainloop warps lack
#ifndef PPX_STATS
#define PPX_STATS 0
#endif
constexpr bool kStats = PPX_STATS != 0;
// mbar_wait that adds the cycles spent to *acc when profiling statistics are on
__device__ __forceinline__ void mbar_wait_t(uint32_t bar, uint32_t parity, bool on, unsigned long long& acc) {
  if (!on) { mbar_wait(bar, parity); return; }
  const unsigned long long c0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - c0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++n & 0x3FFu) == 0 && global_ns() - t0 > 20000000000ull) asm volatile("trap;");
  }
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c2, int c3,
                                            int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor (version 1 for sm_100): layout 2 = SWIZZLE_128B (16-byte atoms),
// 1 = SWIZZLE_128B_BASE32B (32-byte atoms, 4-row pattern: the MN-major TF32 operand layout)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// accumulator-drained signals: only the (already waited) TMEM loads must precede them, not the
// epilogue's global stores, so the arrive is relaxed and never waits for stores to drain
__device__ __forceinline__ void mbar_arrive_relaxed(uint32_t bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <bool kTF32>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------------------------------
// epilogue element I/O (32 contiguous values of one row)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void load32(const Tensor2& t, long long off, int nvalid, float* v) {
  if (t.f32) {
    const float* p = reinterpret_cast<const float*>(t.ptr) + off;
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 q = reinterpret_cast<const float4*>(p)[i];
        v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = i < nvalid ? p[i] : 0.f;
    }
  } else {
    const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(t.ptr) + off;
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q = reinterpret_cast<const uint4*>(p)[i];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = __bfloat1622float2(h[j]);
          v[8 * i + 2 * j] = f.x; v[8 * i + 2 * j + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = i < nvalid ? __bfloat162float(p[i]) : 0.f;
    }
  }
}

// one warp's full 32 x 32 bf16 chunk (rows row0 .. row0+31 of lanes 0..31, columns col .. col+31)
// through the warp's smem staging: each global store instruction then writes 8 whole 64-byte row
// segments.  Needs every row and column of the chunk valid and a 16-byte aligned destination.
__device__ __forceinline__ void store32_bf16_coalesced(uint32_t* stage, const Tensor2& t, long long off_row0, int lane,
                                                       const float* v) {
  uint32_t* my = stage + lane * EPI_STAGE_ROW_WORDS;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
    *reinterpret_cast<uint4*>(my + 4 * i) = q;
  }
  __syncwarp();
  const int r = lane >> 2, seg = lane & 3;
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(t.ptr) + off_row0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = r + 8 * i;
    const uint4 q = *reinterpret_cast<const uint4*>(stage + rr * EPI_STAGE_ROW_WORDS + 4 * seg);
    *reinterpret_cast<uint4*>(base + (long long)rr * t.ld + 8 * seg) = q;
  }
  __syncwarp();
}

__device__ __forceinline__ void store32(const Tensor2& t, long long off, int nvalid, const float* v) {
  if (t.f32) {
    float* p = reinterpret_cast<float*>(t.ptr) + off;
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) p[i] = v[i];
    }
  } else {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(t.ptr) + off;
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
        reinterpret_cast<uint4*>(p)[i] = q;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) p[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

// one row's 32-value input chunk, loaded ahead of use: the 16-byte vector loads are issued one
// chunk early so their latency hides behind the TMEM drain of the chunk before
struct Pre32 {
  uint4 q[8];
  bool vec;
};

__device__ __forceinline__ void pre_issue(const Tensor2& t, long long off, int nvalid, bool active, Pre32& r) {
  r.vec = false;
  if (!active || nvalid != 32) return;
  const char* p = reinterpret_cast<const char*>(t.ptr) + off * (t.f32 ? 4 : 2);
  if (reinterpret_cast<uintptr_t>(p) & 15) return;
  const uint4* q = reinterpret_cast<const uint4*>(p);
  if (t.f32) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r.q[i] = q[i];
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) r.q[i] = q[i];
  }
  r.vec = true;
}

// values of a chunk issued by pre_issue (ragged / unaligned chunks load here, element-wise)
__device__ __forceinline__ void pre_finish(const Tensor2& t, long long off, int nvalid, bool active, const Pre32& r,
                                           float* v) {
  if (!active) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    return;
  }
  if (!r.vec) { load32(t, off, nvalid, v); return; }
  if (t.f32) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[4 * i] = __uint_as_float(r.q[i].x); v[4 * i + 1] = __uint_as_float(r.q[i].y);
      v[4 * i + 2] = __uint_as_float(r.q[i].z); v[4 * i + 3] = __uint_as_float(r.q[i].w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.q[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[8 * i + 2 * j] = f.x; v[8 * i + 2 * j + 1] = f.y;
      }
    }
  }
}

// Adam on 32 fp32 master values of one row (moments updated in place, 4 at a time to keep the
// epilogue's register footprint small); training.py:92-105
__device__ __forceinline__ void adam32(const Epilogue& E, long long moff, int nvalid, float lr, const float* g,
                                       float* w) {
  float* pm = reinterpret_cast<float*>(E.adam_m.ptr) + moff;
  float* pv = reinterpret_cast<float*>(E.adam_v.ptr) + moff;
  const float b1 = E.hyper[1], b2 = E.hyper[2], eps = E.hyper[3], bc1 = E.hyper[4], bc2 = E.hyper[5];
  const bool vec = nvalid == 32 && ((reinterpret_cast<uintptr_t>(pm) | reinterpret_cast<uintptr_t>(pv)) & 15) == 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float m4[4], v4[4];
    if (vec) {
      const float4 a = reinterpret_cast<const float4*>(pm)[q], b = reinterpret_cast<const float4*>(pv)[q];
      m4[0] = a.x; m4[1] = a.y; m4[2] = a.z; m4[3] = a.w;
      v4[0] = b.x; v4[1] = b.y; v4[2] = b.z; v4[3] = b.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        m4[e] = 4 * q + e < nvalid ? pm[4 * q + e] : 0.f;
        v4[e] = 4 * q + e < nvalid ? pv[4 * q + e] : 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * q + e;
      m4[e] = b1 * m4[e] + (1.f - b1) * g[i];
      v4[e] = b2 * v4[e] + (1.f - b2) * g[i] * g[i];
      w[i] -= lr * (m4[e] / bc1) / (sqrtf(v4[e] / bc2) + eps);
    }
    if (vec) {
      reinterpret_cast<float4*>(pm)[q] = make_float4(m4[0], m4[1], m4[2], m4[3]);
      reinterpret_cast<float4*>(pv)[q] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < nvalid) { pm[4 * q + e] = m4[e]; pv[4 * q + e] = v4[e]; }
    }
  }
}

// warm L2 with `ncols` values of one row starting at `off` (issued while the tile's MMAs run)
__device__ __forceinline__ void prefetch_row(const Tensor2& t, long long off, int ncols) {
  const char* p = reinterpret_cast<const char*>(t.ptr) + off * (t.f32 ? 4 : 2);
  const int bytes = ncols * (t.f32 ? 4 : 2);
  for (int b = 0; b < bytes; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + b));
}

// sum of v[i] over the 32 lanes of a warp; lane L returns the total for column L
__device__ __forceinline__ float warp_transpose_sum(float* v, int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      float send = up ? v[i] : v[i + off];
      float keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------
struct TileCoord {
  int prob, m0, qn, nin;
};

template <int MT>
__device__ __forceinline__ TileCoord tile_coord(const GemmParams& P, int t) {
  int pi = 0;
#pragma unroll 1
  while (pi + 1 < P.nprobs && t >= P.probs[pi + 1].tile_begin) ++pi;
  const Problem& pr = P.probs[pi];
  int local = t - pr.tile_begin;
  const int span = pr.nspan > 1 ? pr.nspan : 1;
  int ntn = (pr.nblk + span - 1) / span * pr.npb;
  int mt = local / ntn;
  int nt = local - mt * ntn;
  TileCoord c;
  c.prob = pi;
  c.m0 = pr.m_base + mt * MT;
  const int qt = nt / pr.npb;     // tile column over the N blocks (a spanning tile covers `span`)
  c.qn = qt * span;
  c.nin = (nt - qt * pr.npb) * pr.BN;
  return c;
}

// i-th tile of cluster (or CTA) c: the static LPT schedule when present, else round robin
__device__ __forceinline__ int tile_of(const GemmParams& P, int c, int step, int i) {
  if (P.nsched) {
    const int b = P.sched_off[c] + i;
    return b < P.sched_off[c + 1] ? (int)P.sched[b] : -1;
  }
  const int t = c + i * step;
  return t < P.total_tiles ? t : -1;
}

// producer-side wait of a fused launch (see Problem::wait_ctr); TMA reads what the generic proxy
// (local or NVLink stores) wrote, hence the proxy fence after the acquire
// (bounded: after ~20 s it flags bit 1 of *P.bad and proceeds — a lost peer never hangs the GPU)
__device__ __forceinline__ void wait_dependency(const GemmParams& P, const Problem& pr, int epoch) {
  const int target = (int)((unsigned)(epoch + 1) * (unsigned)pr.wait_per_epoch);
  int x;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(x) : "l"(pr.wait_ctr) : "memory");
    if ((int)((unsigned)x - (unsigned)target) >= 0) break;   // wrap-safe
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      if (P.bad) atomicOr(P.bad, 2);
      break;
    }
    __nanosleep(32);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void end_epoch(const GemmParams& P) {
  if (!P.epoch || threadIdx.x != 0) return;
  __threadfence();
  const unsigned int prev = atomicAdd(P.done, 1u);
  if (prev == gridDim.x - 1) {
    *P.done = 0u;
    atomicAdd(P.epoch, 1);
  }
}

__device__ __forceinline__ int op_slot(const Operand& o, int kblk, int qn) {
  int raw = o.slot_src == 1 ? kblk : (o.slot_src == 2 ? qn : 0);
  if (o.slot_skip < 0) {
    // decompressor stack of rank j = -slot_skip - 1 (sources ascending, j itself absent): the
    // absolute source slot maps to its stack index, and j's own slot to an index past the end,
    // which TMA fills with zeros (a slot-pair tile whose one half has no contribution from j)
    const int src = o.slot_base + raw, j = -o.slot_skip - 1;
    return src < j ? src : (src == j ? 0x7fff : src - 1);
  }
  return o.slot_base + raw + (raw >= o.slot_skip ? 1 : 0);
}

// ------------------------------------------------------------------------------------------
// epilogue warps (4 warps = the 4 TMEM lane quadrants): drain one accumulator stage per tile
// ------------------------------------------------------------------------------------------
// NVLink exchange tiles (compression / error compression with peer replicas or arrival counters)
// are published by the two otherwise idle warps (10, 11) while the epilogue warps move on: after
// storing such a tile the epilogue warps meet them at a named barrier; the publisher warps re-read the stored
// rows (L2-hot) and write them to every replica as consecutive 16-byte vectors (coalesced NVLink
// writes), then fence at system scope and bump the arrival counters.
constexpr int W_PUB0 = 10;
__device__ __forceinline__ bool publishes(const Epilogue& E) { return E.nrep || E.narrive; }

template <int MT>
__device__ __forceinline__ void publisher_loop(const GemmParams& P, int t0, int tstep, uint32_t crank, int warp,
                                               int lane) {
  const int tid = (warp - W_PUB0) * 32 + lane;
  for (int i = 0, t; (t = tile_of(P, t0, tstep, i)) >= 0; ++i) {
    TileCoord tc = tile_coord<MT>(P, t);
    const Problem& pr = P.probs[tc.prob];
    const Epilogue& E = pr.epi;
    if (!publishes(E)) continue;
    asm volatile("bar.sync 4, %0;" ::"n"(NUM_EPI_WARPS * 32 + 64) : "memory");
    const int rbase = tc.m0 + (int)crank * BM;
    int nrows = pr.M - rbase;
    nrows = nrows < 0 ? 0 : (nrows > BM ? BM : nrows);
    // a spanning tile holds two consecutive N blocks (slots); every block it covers is published
    const int nhalf = pr.nspan > 1 ? 2 : 1;
    const int ncols = pr.nspan > 1 ? pr.nb_extent
                                   : (pr.nb_extent - tc.nin < pr.BN ? pr.nb_extent - tc.nin : pr.BN);
    int cells = 0, cells_h[2] = {0, 0};
    for (int h = 0; h < nhalf; ++h) {
      const int q = tc.qn + h;
      if (q >= pr.nblk) break;
      cells += nrows * ncols;
      cells_h[h] = nrows * ncols;
      if (!E.nrep || (E.rep_per_half && !E.rep_off[h])) continue;
      const int es = E.out.f32 ? 4 : 2;
      const int upr = ncols * es / 16;
      const long long ldb = E.out.ld * es;
      const char* src = reinterpret_cast<const char*>(E.out.ptr) + (long long)q * E.out.slot_stride * es +
                        (long long)rbase * ldb + (long long)tc.nin * es;
      for (int u = tid; u < nrows * upr; u += 64) {
        const int r = u / upr;
        const long long off = r * ldb + (long long)(u - r * upr) * 16;
        const uint4 v = *reinterpret_cast<const uint4*>(src + off);
        if (E.rep_per_half) *reinterpret_cast<uint4*>(const_cast<char*>(src) + E.rep_off[h] + off) = v;
        else
          for (int i = 0; i < E.nrep; ++i) *reinterpret_cast<uint4*>(const_cast<char*>(src) + E.rep_off[i] + off) = v;
      }
    }
    asm volatile("bar.sync 5, 64;" ::: "memory");
    if (E.narrive && tid == 0) {
      __threadfence_system();
      if (E.rep_per_half) {
        for (int h = 0; h < 2; ++h)
          if (E.arrive[h] && cells_h[h])
            asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(E.arrive[h]), "r"(cells_h[h] / 8) : "memory");
      } else {
        const int amount = E.arrive_units ? cells / 8 : 1;
        for (int i = 0; i < E.narrive; ++i)
          asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(E.arrive[i]), "r"(amount) : "memory");
      }
    }
  }
}

template <int MT, bool kPair>
__device__ __forceinline__ void epilogue_loop(const GemmParams& P, uint32_t tmem_base, uint32_t tfull0,
                                              uint32_t tempty0, int t0, int tstep, uint32_t crank, int warp,
                                              int lane, uint32_t* epi_stage) {
  auto tfull_bar = [&](int s) { return tfull0 + 8u * s; };
  auto tempty_bar = [&](int s) { return tempty0 + 8u * s; };
  const int wq = warp & 3;    // TMEM lane quadrant
  const int grp = warp >> 2;  // chunk parity drained by this warp
  uint32_t* wstage = epi_stage + warp * 32 * EPI_STAGE_ROW_WORDS;
  const bool coalesce = !(P.dbg & 16);   // A/B (PPX_DEBUG_EPI=scatter): the per-lane row stores
  unsigned long long st_wait = 0, st_busy = 0, st_tmem = 0, st_body = 0;
  int iter = 0;
  for (int t; (t = tile_of(P, t0, tstep, iter)) >= 0; ++iter) {
    TileCoord tc = tile_coord<MT>(P, t);
    const Problem& pr = P.probs[tc.prob];
    const Epilogue& E = pr.epi;
    const int as = iter & 1;
    const uint32_t aphase = (iter >> 1) & 1;
    const int row0 = tc.m0 + (int)crank * BM + wq * 32;
    int rows_valid = pr.M - row0;
    rows_valid = rows_valid < 0 ? 0 : (rows_valid > 32 ? 32 : rows_valid);
    const int row = row0 + lane;
    const bool row_ok = lane < rows_valid;
    // debug A/B only (PPX_DEBUG_EPI, wrong results): bit 2 drops the ReLU'-mask read, bit 3 the
    // column sums
    const uint32_t flags = E.flags & ~((P.dbg & 4) ? EP_MASK : 0u) & ~((P.dbg & 8) ? EP_COLSUM : 0u);
    const bool upd = (flags & (EP_SGD | EP_ADAM)) != 0;
    // per-row input streamed one chunk ahead: target | fp32 master | ReLU mask | accumulated output
    const Tensor2* sa = (flags & EP_LOSS) ? &E.target
                        : upd            ? &E.master
                        : ((flags & EP_MASK) && !(flags & EP_MASKBITS)) ? &E.mask
                        : (flags & EP_ACCUM) ? &E.out : nullptr;
    const long long a_ss = sa && (upd || sa == &E.out) ? sa->slot_stride : 0;
    const long long a_rb = sa ? (long long)row * sa->ld : 0;
    const long long o_rb = (long long)row * E.out.ld, m_rb = (long long)row * E.master.ld;
    // chunk c -> (N block, column inside it): a spanning tile's two halves are consecutive N blocks
    const int half = pr.nspan > 1 ? pr.BN / 2 : (1 << 30);
    auto geom = [&](int c, int& col0, int& nvalid, int& oslot) {
      const int h = (c * 32) / half;
      const int q = tc.qn + h;
      col0 = tc.nin + c * 32 - h * half;
      nvalid = q < pr.nblk ? pr.nb_extent - col0 : 0;
      nvalid = nvalid > 32 ? 32 : nvalid;
      oslot = q + (q >= E.out_skip ? 1 : 0);
    };
    const int nchunks = (P.dbg & 1) ? 0 : (pr.BN + 31) / 32;
    const int ncols = pr.nb_extent - tc.nin < pr.BN ? pr.nb_extent - tc.nin : pr.BN;   // non-spanning tiles
    if (row_ok && nchunks && grp == 0) {    // warm L2 with this row's inputs while the MMAs run
      for (int h = 0; h * half < pr.BN; ++h) {
        int col0, nv, os;
        geom(h * half / 32, col0, nv, os);
        const int n = pr.nspan > 1 ? (nv > 0 ? pr.nb_extent - col0 : 0) : ncols;
        if (n <= 0) continue;
        if (sa) prefetch_row(*sa, os * a_ss + a_rb + col0, n);
        if (flags & EP_ADAM) {
          const long long mo = (long long)os * E.master.slot_stride + m_rb + col0;
          prefetch_row(E.adam_m, mo, n);
          prefetch_row(E.adam_v, mo, n);
        }
      }
    }
    // bit-mask words of this warp's chunks (c = grp, grp + 2, ...), loaded before the wait
    uint32_t mbits[BN_MAX / 64];
    if (flags & EP_MASKBITS) {
#pragma unroll
      for (int u = 0; u < BN_MAX / 64; ++u) {
        const int c = grp + 2 * u;
        mbits[u] = 0u;
        if (c < nchunks && row_ok) {
          int col0, nv, os;
          geom(c, col0, nv, os);
          if (nv > 0) mbits[u] = __ldg(reinterpret_cast<const uint32_t*>(E.mask.ptr) + row * E.mask.ld + (col0 >> 5));
        }
      }
    }
    mbar_wait_t(tfull_bar(as), aphase, kStats && P.stats != nullptr, st_wait);
    const unsigned long long c_busy = kStats && P.stats ? clock64() : 0ull;
    tc_fence_after();
    float loss_acc = 0.f;
    bool bad = false;
    Pre32 pa;
    if (grp < nchunks) {
      int col0, nv0, os;
      geom(grp, col0, nv0, os);
      pre_issue(sa ? *sa : E.out, os * a_ss + a_rb + col0, nv0, sa && row_ok && nv0 > 0, pa);
    }
    for (int c = grp; c < nchunks; c += 2) {
      int col0, nvalid, oslot;
      geom(c, col0, nvalid, oslot);
      const long long a_row = (long long)oslot * a_ss + a_rb;
      const long long o_row = (long long)oslot * E.out.slot_stride + o_rb;
      const long long m_row = (long long)oslot * E.master.slot_stride + m_rb;
      const bool live = row_ok && nvalid > 0;
      const float bl = ((flags & EP_BIAS) && lane < nvalid) ? E.bias[col0 + lane] : 0.f;
      Pre32 na;
      if (c + 2 < nchunks) {
        int col1, nv1, os1;
        geom(c + 2, col1, nv1, os1);
        pre_issue(sa ? *sa : E.out, os1 * a_ss + a_rb + col1, nv1, sa && row_ok && nv1 > 0, na);
      } else {
        na.vec = false;
      }
      float v[32];
      const unsigned long long c_t0 = kStats && P.stats ? clock64() : 0ull;
      tmem_ld32(tmem_base + as * BN_MAX + c * 32 + ((uint32_t)(wq * 32) << 16), v);
      if (kStats && P.stats) st_tmem += clock64() - c_t0;
      // full chunks (every row and column valid, the common case) compile without per-element masks
      auto body = [&](auto full_c) {
        constexpr bool F = decltype(full_c)::value;
        auto ok = [&](int i) { return F ? true : (row_ok && i < nvalid); };
        if (flags & EP_FINITE) {
#pragma unroll
          for (int i = 0; i < 32; ++i) bad |= ok(i) && !isfinite(v[i]);
        }
        if (flags & EP_BIAS) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bl, i);
        }
        const long long ooff = o_row + col0;
        if ((flags & EP_PREACT) && live)
          store32(E.preact, (long long)oslot * E.preact.slot_stride + (long long)row * E.preact.ld + col0, nvalid, v);
        if (upd) {
          if (live) {
            if (flags & EP_GRAD)
              store32(E.aux, (long long)oslot * E.aux.slot_stride + (long long)row * E.aux.ld + col0, nvalid, v);
            const long long moff = m_row + col0;
            float w[32];
            pre_finish(E.master, moff, nvalid, true, pa, w);
            const float lr = E.hyper[0];
            if (flags & EP_ADAM) {
              adam32(E, moff, nvalid, lr, v, w);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) w[i] -= lr * v[i];
            }
            store32(E.master, moff, nvalid, w);
            if (E.out.ptr) store32(E.out, ooff, nvalid, w);
          }
        } else if (flags & EP_LOSS) {
          float tg[32];   // target, then the output delta in place
          pre_finish(E.target, a_row + col0, nvalid, live, pa, tg);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float y = (flags & EP_RELU) ? fmaxf(v[i], 0.f) : v[i];
            const float diff = ok(i) ? (y - tg[i]) : 0.f;
            loss_acc += diff * diff;
            tg[i] = ((flags & EP_RELU) && !(v[i] > 0.f)) ? 0.f : diff * E.scale;
            v[i] = y;
          }
          if (live && E.out.ptr) store32(E.out, ooff, nvalid, v);
          const long long aoff = (long long)row * E.aux.ld + col0;
          if (F && coalesce && !E.aux.f32 && ((reinterpret_cast<uintptr_t>(E.aux.ptr) | (E.aux.ld * 2) |
                                                ((aoff - lane * E.aux.ld) * 2)) & 15) == 0)
            store32_bf16_coalesced(wstage, E.aux, aoff - (long long)lane * E.aux.ld, lane, tg);
          else if (live) store32(E.aux, aoff, nvalid, tg);
          if (flags & EP_COLSUM) {   // bias gradient: one global reduction per column and warp
            const float cs = warp_transpose_sum(tg, lane);
            if (lane < nvalid) atomicAdd(E.colsum + col0 + lane, cs);
          }
        } else {
          if (flags & EP_RELU) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
          }
          if (flags & EP_MASKBITS) {
            const uint32_t mw = mbits[(c - grp) >> 1];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (ok(i) && ((mw >> i) & 1u)) ? v[i] : 0.f;
          } else if (flags & EP_MASK) {
            float mk[32];
            pre_finish(E.mask, a_row + col0, nvalid, live, pa, mk);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (ok(i) && mk[i] > 0.f) ? v[i] : 0.f;
          }
          if (flags & EP_ACCUM) {
            float o[32];
            if (sa == &E.out) pre_finish(E.out, ooff, nvalid, live, pa, o);
            else if (live) load32(E.out, ooff, nvalid, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += (ok(i) && live) ? o[i] : 0.f;
          }
          if (F && coalesce && !E.out.f32 && ((reinterpret_cast<uintptr_t>(E.out.ptr) | (E.out.ld * 2) |
                                                  ((ooff - lane * E.out.ld) * 2)) & 15) == 0)
            store32_bf16_coalesced(wstage, E.out, ooff - (long long)lane * E.out.ld, lane, v);
          else if (live) store32(E.out, ooff, nvalid, v);
          if ((flags & EP_BITS) && live) {   // ReLU'(pre) = (y > 0) for the recurrence, 1 bit each
            uint32_t w = 0u;
#pragma unroll
            for (int i = 0; i < 32; ++i) w |= (ok(i) && v[i] > 0.f) ? (1u << i) : 0u;
            reinterpret_cast<uint32_t*>(E.preact.ptr)[row * E.preact.ld + (col0 >> 5)] = w;
          }
          if (flags & EP_COLSUM) {
            if (!F) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = ok(i) ? v[i] : 0.f;
            }
            const float cs = warp_transpose_sum(v, lane);
            if (lane < nvalid) atomicAdd(E.colsum + col0 + lane, cs);
          }
        }
      };
      const unsigned long long c_b0 = kStats && P.stats ? clock64() : 0ull;
      if (nvalid == 32 && rows_valid == 32) body(std::true_type{});
      else body(std::false_type{});
      if (kStats && P.stats) st_body += clock64() - c_b0;
      pa = na;
    }
    if (flags & EP_LOSS) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, off);
      if (lane == 0) atomicAdd(E.loss, loss_acc * E.loss_scale);
    }
    if ((flags & EP_FINITE) && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(E.bad, 1);
    // hand the stored tile to the publisher warps (a full barrier: it also waits until they took
    // the previous published tile, so barrier generations never mix)
    if (publishes(E)) asm volatile("bar.sync 4, %0;" ::"n"(NUM_EPI_WARPS * 32 + 64) : "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (kPair) mbar_arrive_cluster_relaxed(mapa_shared(tempty_bar(as), 0));
      else mbar_arrive_relaxed(tempty_bar(as));
    }
    if (kStats && P.stats) st_busy += clock64() - c_busy;
  }
  if (kStats && P.stats && lane == 0) {
    atomicAdd(P.stats + 0, st_wait);
    atomicAdd(P.stats + 1, st_busy);
    atomicAdd(P.stats + 7, st_tmem);
    atomicAdd(P.stats + 8, st_body);
  }
}

template <bool kTF32>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_kernel(const __grid_constant__ GemmParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base_u32;
  const uint32_t sB = sA + STAGES * A_STAGE_BYTES;
  const uint32_t sBar = sB + STAGES * B_STAGE_BYTES;
  // barrier layout: full[STAGES], empty[STAGES], tfull[2], tempty[2], tmem addr slot
  auto full_bar = [&](int s) { return sBar + 8u * s; };
  auto empty_bar = [&](int s) { return sBar + 8u * (STAGES + s); };
  auto tfull_bar = [&](int s) { return sBar + 8u * (2 * STAGES + s); };
  auto tempty_bar = [&](int s) { return sBar + 8u * (2 * STAGES + 2 + s); };
  const uint32_t tmem_slot = sBar + 8u * (2 * STAGES + 4);
  uint8_t* smem_gen = smem_raw + (base_u32 - smem_u32(smem_raw));
  volatile uint32_t* tmem_slot_ptr =
      reinterpret_cast<volatile uint32_t*>(smem_gen + (tmem_slot - base_u32));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t* epi_stage = reinterpret_cast<uint32_t*>(smem_gen + (sBar + 256 - base_u32));
  constexpr int ESIZE = kTF32 ? 4 : 2;
  constexpr int BK = ROW_BYTES / ESIZE;     // elements of K per stage
  constexpr int CH = ROW_BYTES / ESIZE;     // MN-major atom width in elements
  constexpr int KMMA = 32 / ESIZE;          // K per tcgen05.mma
  constexpr int NK = BK / KMMA;             // MMAs per stage (4)

  if (warp == W_TMA && lane == 0) {
    for (int i = 0; i < P.nmaps; ++i) prefetch_map(&P.maps[i]);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull_bar(s), 1);
      mbar_init(tempty_bar(s), NUM_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_ALLOC) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  // programmatic dependent launch: the prologue above (barrier init, TMEM alloc, tensor-map
  // prefetch) overlapped the previous kernel's tail; global memory is touched only once that
  // kernel has completed.  Our own dependents may start their prologue from here on.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int total = P.total_tiles;

  if (is_epi_warp(warp)) {
    reg_alloc_epilogue();
    epilogue_loop<BM, false>(P, tmem_base, tfull_bar(0), tempty_bar(0), blockIdx.x, gridDim.x, 0u, warp, lane,
                             epi_stage);
  } else {
  reg_dealloc_mainloop();
  if (warp >= W_PUB0) {
    publisher_loop<BM>(P, blockIdx.x, gridDim.x, 0u, warp, lane);
  } else if (warp == W_TMA) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        TileCoord tc = tile_coord<BM>(P, t);
        const Problem& pr = P.probs[tc.prob];
        const uint32_t bytes = (uint32_t)(BM + pr.BN) * ROW_BYTES;
        for (int sg = 0; sg < pr.nsegs; ++sg) {
          const Segment& seg = pr.segs[sg];
          const CUtensorMap* ma = &P.maps[seg.a.map];
          const CUtensorMap* mb = &P.maps[seg.b.map];
          for (int kt = 0; kt < seg.k_tiles; ++kt) {
            const int kblk = kt / seg.kpb;
            const int kin = (kt - kblk * seg.kpb) * BK;
            mbar_wait(empty_bar(stage), phase ^ 1u);
            mbar_expect_tx(full_bar(stage), bytes);
            const uint32_t da = sA + stage * A_STAGE_BYTES;
            const uint32_t db = sB + stage * B_STAGE_BYTES;
            const int slot_a = op_slot(seg.a, kblk, tc.qn);
            const int slot_b = op_slot(seg.b, kblk, tc.qn);
            if (!seg.a.mn) {
              tma_load_3d(ma, full_bar(stage), da, kin, tc.m0, slot_a);
            } else if (seg.a.atoms4d == 2) {
              tma_load_5d(ma, full_bar(stage), da, tc.m0 / CH, kin / 8, slot_a);
            } else if (seg.a.atoms4d) {
              tma_load_4d(ma, full_bar(stage), da, 0, kin, tc.m0 / CH, slot_a);
            } else {
#pragma unroll 1
              for (int c = 0; c < BM / CH; ++c)
                tma_load_3d(ma, full_bar(stage), da + c * (BK * ROW_BYTES), tc.m0 + c * CH, kin, slot_a);
            }
            if (!seg.b.mn) {
              tma_load_3d(mb, full_bar(stage), db, kin, tc.nin, slot_b);
            } else if (seg.b.atoms4d) {
              tma_load_4d(mb, full_bar(stage), db, 0, kin, tc.nin / CH, slot_b);
            } else {
#pragma unroll 1
              for (int c = 0; c < pr.BN / CH; ++c)
                tma_load_3d(mb, full_bar(stage), db + c * (BK * ROW_BYTES), tc.nin + c * CH, kin, slot_b);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == W_MMA) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++iter) {
        TileCoord tc = tile_coord<BM>(P, t);
        const Problem& pr = P.probs[tc.prob];
        const int as = iter & 1;
        const uint32_t aphase = (iter >> 1) & 1;
        mbar_wait(tempty_bar(as), aphase ^ 1u);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + as * BN_MAX;
        uint32_t accum = 0;
        for (int sg = 0; sg < pr.nsegs; ++sg) {
          const Segment& seg = pr.segs[sg];
          for (int kt = 0; kt < seg.k_tiles; ++kt) {
            if (!(P.dbg & 2)) mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            const uint32_t da = sA + stage * A_STAGE_BYTES;
            const uint32_t db = sB + stage * B_STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
              // MN-major A: atom-major tile (LBO = atom stride, SBO = 1024) or the interleaved
              // canonical tile (LBO = 1024 between MN atoms, SBO = 2 KB between 8-row K groups)
              // MN-major TF32 (atom-major tile only): 4-row K groups of the 32-byte-atom swizzle
              // (SBO = 512 B), one MMA = K 8 = two groups
              constexpr uint32_t MN_SBO = kTF32 ? 512u : 1024u, MN_LAYOUT = kTF32 ? 1u : 2u;
              uint64_t ad = !seg.a.mn ? sdesc(da + kk * 32, 16, 1024)
                            : (seg.a.atoms4d == 2 ? sdesc(da + kk * (KMMA / 8) * (BM / CH) * 1024, 1024, (BM / CH) * 1024)
                                                  : sdesc(da + kk * (KMMA * ROW_BYTES), BK * ROW_BYTES, MN_SBO, MN_LAYOUT));
              uint64_t bd = seg.b.mn ? sdesc(db + kk * (KMMA * ROW_BYTES), BK * ROW_BYTES, MN_SBO, MN_LAYOUT)
                                     : sdesc(db + kk * 32, 16, 1024);
              mma_issue<kTF32>(tmem_d, ad, bd, seg.idesc, accum);
              accum = 1;
            }
            mma_commit(empty_bar(stage));
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          }
        }
        mma_commit(tfull_bar(as));
      }
    }
    __syncwarp();
  }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_ALLOC) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace ppx
