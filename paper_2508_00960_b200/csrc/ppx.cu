// libppx.so — host side of the C ABI declared in include/ppx.h.
//
// Builds tensor maps and grouped-GEMM problem tables for the tcgen05 kernel in gemm_sm100.cuh,
// launches the small elementwise kernels in elementwise.cuh, and drives NCCL for the phantom
// all-gather / reduce-scatter.  No torch types cross this boundary.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ppx.h"
#include "elementwise.cuh"
#include "gemm_sm100.cuh"
#include "gemm_pair_sm100.cuh"

struct ppx_ctx {
  int world = 1, rank = 0, device = 0, num_sms = 148;
  int reserved_sms = 0;   // SMs GEMM grids leave free for a concurrent collective
  ncclComm_t comm = nullptr;
  std::string err;
  // FP32-tier hi/lo split workspace: a pool of chunks, bump-allocated per call and reused by the
  // next call (stream ordered: FP32-tier calls of one ctx must share a stream)
  std::vector<std::pair<char*, size_t>> ws;
  std::vector<void*> ipc_own;      // ppx_peer_alloc regions (cudaFree at destroy)
  std::vector<void*> ipc_mapped;   // ppx_peer_open mappings (cudaIpcCloseMemHandle at destroy)
  unsigned int* fuse_done = nullptr;     // fused launches' CTA exit counter (self-resetting)
  unsigned int* reduce_done = nullptr;   // ppx_reduce_received's block exit counter (self-resetting)
  // FP32-tier operand cache (ppx_tf32_scope): inside a scope, the 3xTF32 low part of every GEMM
  // operand read on `lo_stream` is split once and kept across calls until a ppx call writes an
  // overlapping range (then its buffer returns to the pool)
  struct LoEntry {
    int64_t bytes;
    char* lo;
    size_t cap;
  };
  long long launches = 0;   // kernels this context enqueued (ppx_kernel_launches)
  bool lo_scope = false;
  cudaStream_t lo_stream = nullptr;
  cudaEvent_t lo_done = nullptr;   // recorded when a scope ends: the next scope's stream waits on it
  bool lo_done_valid = false;
  std::map<std::pair<const char*, int64_t>, LoEntry> lo_live;   // (operand base, elements) -> low part
  std::multimap<size_t, char*> lo_pool;                         // free buffers by capacity
  std::vector<char*> lo_all;
};

namespace {
// a ppx call wrote [p, p + bytes): drop the cached low parts of every overlapping operand
void lo_invalidate(ppx_ctx* ctx, const void* p, int64_t bytes) {
  if (!ctx || ctx->lo_live.empty() || !p || bytes <= 0) return;
  const char* a = reinterpret_cast<const char*>(p);
  for (auto it = ctx->lo_live.begin(); it != ctx->lo_live.end();) {
    const char* b = it->first.first;
    if (b < a + bytes && a < b + it->second.bytes) {
      ctx->lo_pool.insert({it->second.cap, it->second.lo});
      it = ctx->lo_live.erase(it);
    } else {
      ++it;
    }
  }
}
void lo_clear(ppx_ctx* ctx) {
  if (!ctx) return;
  for (auto& kv : ctx->lo_live) ctx->lo_pool.insert({kv.second.cap, kv.second.lo});
  ctx->lo_live.clear();
}
}  // namespace

namespace {

using ppx::GemmParams;
using ppx::Problem;
using ppx::Segment;

ppx_status fail(ppx_ctx* ctx, ppx_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(ctx, PPX_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                        \
  do {                                                                                             \
    ncclResult_t r_ = (expr);                                                                      \
    if (r_ != ncclSuccess) return fail(ctx, PPX_E_PROTOCOL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

inline int64_t round8(int64_t x) { return (x + 7) / 8 * 8; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Flat {  // element offsets of the flat (rank, layer) parameter block
  int64_t lds, ldk, local, comp, dec, bias, total;
  Flat(int s, int k, int p) {
    lds = round8(s);
    ldk = round8(k);
    local = 0;
    comp = (int64_t)s * lds;
    dec = comp + (int64_t)k * lds;
    bias = dec + (int64_t)(p - 1) * s * ldk;
    total = bias + round8(s);
  }
};

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 3D row-major view, in elements: [slots][rows][cols] with leading dim / slot stride
struct View {
  const void* ptr;
  int64_t cols, rows, slots, ld, slot_stride;
};
inline View view2(const void* p, int64_t rows, int64_t cols, int64_t ld) { return {p, cols, rows, 1, ld, rows * ld}; }
inline View view3(const void* p, int64_t slots, int64_t rows, int64_t cols, int64_t ld, int64_t ss) {
  return {p, cols, rows, slots, ld, ss};
}

struct Opnd {
  View v;
  int mn = 0;         // 0 K-major (cols = K), 1 MN-major (cols = M or N)
  int slot_src = 0;   // 0 const, 1 K-block, 2 N-block
  int slot_base = 0;
  int slot_skip = INT_MAX;
};

inline ppx::Tensor2 t2(void* p, int64_t ld, int f32, int64_t ss = 0) {
  ppx::Tensor2 t;
  t.ptr = p;
  t.ld = ld;
  t.slot_stride = ss;
  t.f32 = f32;
  t.pad_ = 0;
  return t;
}

uint32_t make_idesc(bool tf32, int a_mn, int b_mn, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                    // D = F32
  d |= (tf32 ? 2u : 1u) << 7;      // A = TF32 / BF16
  d |= (tf32 ? 2u : 1u) << 10;     // B = TF32 / BF16
  d |= (uint32_t)(a_mn & 1) << 15;
  d |= (uint32_t)(b_mn & 1) << 16;
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(ppx::BM >> 4) << 24;
  return d;
}

struct Builder {
  ppx_ctx* ctx;
  cudaStream_t st;
  bool tf32;
  int esize, BK, CH;
  GemmParams P;
  std::map<std::pair<const void*, int64_t>, std::pair<void*, void*>> splits;  // tf32 hi/lo copies
  size_t ws_chunk = 0, ws_off = 0;
  ppx_status status = PPX_OK;

  void* ws_alloc(size_t bytes) {
    while (ws_chunk < ctx->ws.size() && ws_off + bytes > ctx->ws[ws_chunk].second) {
      ++ws_chunk;
      ws_off = 0;
    }
    if (ws_chunk == ctx->ws.size()) {
      size_t cap = bytes < ((size_t)64 << 20) ? ((size_t)64 << 20) : bytes;
      char* p = nullptr;
      if (cudaMalloc(&p, cap) != cudaSuccess) return nullptr;
      ctx->ws.push_back({p, cap});
      ws_off = 0;
    }
    void* r = ctx->ws[ws_chunk].first + ws_off;
    ws_off += bytes;
    return r;
  }

  bool use4d = getenv("PPX_NO_4D") == nullptr;
  // 2-SM (cta_group::2) kernel for bf16 launches whose operands tile into 64-wide atoms
  bool want_pair = false, use_pair = false;
  int BKf = 64;   // K per stage of the kernel actually launched
  int fuse_world = 0;          // > 0: a fused compress + exchange + forward launch over this many GPUs
  bool lpt = false;            // static longest-processing-time schedule of the tiles over the clusters
  int* fuse_epoch = nullptr;
  int* fuse_bad = nullptr;
  // MN-major A (activations / deltas of the weight-gradient GEMMs) as the interleaved 5D tile
  bool use5d = getenv("PPX_NO_5D") == nullptr;

  Builder(ppx_ctx* c, ppx_dtype dt, void* stream) : ctx(c), st((cudaStream_t)stream), tf32(dt == PPX_FP32) {
    esize = tf32 ? 4 : 2;
    want_pair = !tf32 && getenv("PPX_NO_PAIR") == nullptr;
    BK = ppx::ROW_BYTES / esize;
    CH = BK;
    memset(&P, 0, sizeof(P));
  }

  bool ok() const { return status == PPX_OK; }
  void error(ppx_status s, const char* msg) {
    if (status == PPX_OK) {
      status = s;
      fail(ctx, s, "%s", msg);
    }
  }

  struct MapKey {
    const void* ptr;
    int64_t cols, rows, slots, ld, ss;
    int bi, br, mn = 0;
    bool operator<(const MapKey& o) const {
      return std::tie(ptr, cols, rows, slots, ld, ss, bi, br, mn) <
             std::tie(o.ptr, o.cols, o.rows, o.slots, o.ld, o.ss, o.bi, o.br, o.mn);
    }
  };
  // MN-major 32-bit (TF32) operands need the 128B swizzle with 32-byte atoms (the UMMA
  // SWIZZLE_128B_BASE32B smem layout); everything else uses the 16-byte-atom 128B swizzle
  CUtensorMapSwizzle swizzle(bool mn) const {
    return tf32 && mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  }
  std::map<MapKey, int> map_cache;

  int add_map(const View& v, int box_inner, int box_rows, bool mn) {
    if (!ok()) return 0;
    MapKey key{v.ptr, v.cols, v.rows, v.slots, v.ld, v.slot_stride, box_inner, box_rows, mn ? 1 : 0};
    auto hit = map_cache.find(key);
    if (hit != map_cache.end()) return hit->second;
    if (P.nmaps >= ppx::MAX_MAPS) { error(PPX_E_CONFIG, "too many tensor maps in one launch"); return 0; }
    if (!get_encode()) { error(PPX_E_CUDA, "cuTensorMapEncodeTiled unavailable"); return 0; }
    if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) || (v.ld * esize) % 16 || (v.slot_stride * esize) % 16) {
      error(PPX_E_CONFIG, "tensor base must be 16B aligned and leading dims multiples of 16 bytes");
      return 0;
    }
    cuuint64_t dims[3] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows, (cuuint64_t)v.slots};
    cuuint64_t strides[2] = {(cuuint64_t)(v.ld * esize), (cuuint64_t)(v.slot_stride * esize)};
    cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(&P.maps[P.nmaps], tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          3, const_cast<void*>(v.ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle(mn), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      char msg[256];
      snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (%d): dims %llu,%llu,%llu box %d,%d", (int)r,
               (unsigned long long)v.cols, (unsigned long long)v.rows, (unsigned long long)v.slots, box_inner,
               box_rows);
      error(PPX_E_CUDA, msg);
      return 0;
    }
    map_cache[key] = P.nmaps;
    return P.nmaps++;
  }

  int add_map_nd(const View& v, int rank, const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                 int tag) {
    if (!ok()) return -1;
    MapKey key{v.ptr, v.cols, v.rows, v.slots, v.ld, v.slot_stride, tag, (int)(box[1] * 1000 + box[2])};
    auto hit = map_cache.find(key);
    if (hit != map_cache.end()) return hit->second;
    if (P.nmaps >= ppx::MAX_MAPS) { error(PPX_E_CONFIG, "too many tensor maps in one launch"); return -1; }
    if (!get_encode()) { error(PPX_E_CUDA, "cuTensorMapEncodeTiled unavailable"); return -1; }
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(&P.maps[P.nmaps], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(v.ptr), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      char msg[256];
      snprintf(msg, sizeof(msg), "cuTensorMapEncodeTiled failed (2-SM operand map, err %d, rank %d, dims %llu %llu %llu %llu, box %u %u %u %u, tag %d)",
               (int)r, rank, (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
               (unsigned long long)dims[3], box[0], box[1], box[2], box[3], tag);
      error(PPX_E_CUDA, msg);
      return -1;
    }
    map_cache[key] = P.nmaps;
    return P.nmaps++;
  }

  // 2-SM kernel operand map (gemm_pair_sm100.cuh): K-major -> [2 K-atoms][rows][128 B] per stage,
  // MN-major -> interleaved [16 K groups][atoms][8][128 B] (5D) or [atoms][128 K rows][128 B] (4D)
  int pair_map(const View& v, bool mn, int rows_or_atoms, bool interleaved, int& mode) {
    const cuuint64_t es = 2;
    if (!mn) {
      cuuint64_t dims[4] = {64, (cuuint64_t)v.rows, (cuuint64_t)(v.cols / 64), (cuuint64_t)v.slots};
      cuuint64_t strides[3] = {(cuuint64_t)v.ld * es, 128, (cuuint64_t)v.slot_stride * es};
      cuuint32_t box[4] = {64, (cuuint32_t)rows_or_atoms, (cuuint32_t)ppx::PKA, 1};
      mode = 0;
      return add_map_nd(v, 4, dims, strides, box, -100);
    }
    if (interleaved) {
      cuuint64_t dims[5] = {64, 8, (cuuint64_t)(v.cols / 64), (cuuint64_t)(v.rows / 8), (cuuint64_t)v.slots};
      cuuint64_t strides[4] = {(cuuint64_t)v.ld * es, 128, (cuuint64_t)(8 * v.ld) * es, (cuuint64_t)v.slot_stride * es};
      cuuint32_t box[5] = {64, 8, (cuuint32_t)rows_or_atoms, (cuuint32_t)(ppx::PBK / 8), 1};
      mode = 2;
      return add_map_nd(v, 5, dims, strides, box, -101);
    }
    cuuint64_t dims[4] = {64, (cuuint64_t)v.rows, (cuuint64_t)(v.cols / 64), (cuuint64_t)v.slots};
    cuuint64_t strides[3] = {(cuuint64_t)v.ld * es, 128, (cuuint64_t)v.slot_stride * es};
    cuuint32_t box[4] = {64, (cuuint32_t)ppx::PBK, (cuuint32_t)rows_or_atoms, 1};
    mode = 1;
    return add_map_nd(v, 4, dims, strides, box, -102);
  }

  void finalize_pair(Problem* pr, const Opnd& a, const Opnd& b, int k_tiles, int kpb) {
    if (pr->nsegs >= ppx::MAX_SEGS) { error(PPX_E_CONFIG, "too many K segments"); return; }
    Segment& s = pr->segs[pr->nsegs++];
    const int bnc = pr->BN / 2;
    int ma = 0, mb = 0;
    const int ia = pair_map(a.v, a.mn, a.mn ? ppx::BM / 64 : ppx::BM, a.mn && a.v.rows % 8 == 0 && use5d, ma);
    const int ib = pair_map(b.v, b.mn, b.mn ? bnc / 64 : bnc, false, mb);
    if (!ok()) return;
    s.a.map = (int8_t)ia;
    s.a.mn = (int8_t)a.mn;
    s.a.atoms4d = (int8_t)ma;
    s.a.slot_src = (int8_t)a.slot_src;
    s.a.slot_base = a.slot_base;
    s.a.slot_skip = a.slot_skip;
    s.b.map = (int8_t)ib;
    s.b.mn = (int8_t)b.mn;
    s.b.atoms4d = (int8_t)mb;
    s.b.slot_src = (int8_t)b.slot_src;
    s.b.slot_base = b.slot_base;
    s.b.slot_skip = b.slot_skip;
    s.k_tiles = k_tiles;
    s.kpb = kpb;
    uint32_t d = make_idesc(false, a.mn, b.mn, pr->BN);
    d = (d & ~(0x1Fu << 24)) | ((uint32_t)(2 * ppx::BM) >> 4) << 24;   // M = 256 (cta_group::2)
    s.idesc = d;
  }

  // every operand must tile into whole 64-wide atoms for the 2-SM kernel
  bool pair_shapes_ok() const {
    for (int i = 0; i < P.nprobs; ++i)
      for (const PendingSeg& ps : pend[i]) {
        if (ps.a.v.cols % 64 || ps.b.v.cols % 64) return false;
        if (ps.a.mn && ps.a.v.rows % 8) return false;
      }
    return true;
  }

  // MN-major operand as ONE 4D box per stage: {CH elements, BK rows, atoms, 1} over the view
  // re-indexed as [slots][atoms][rows][CH] (atom stride = CH elements). Needs cols % CH == 0.
  int add_map4(const View& v, int atoms) {
    if (!ok()) return 0;
    MapKey key{v.ptr, v.cols, v.rows, v.slots, v.ld, v.slot_stride, -CH, atoms};
    auto hit = map_cache.find(key);
    if (hit != map_cache.end()) return hit->second;
    if (P.nmaps >= ppx::MAX_MAPS) { error(PPX_E_CONFIG, "too many tensor maps in one launch"); return 0; }
    if (!get_encode()) { error(PPX_E_CUDA, "cuTensorMapEncodeTiled unavailable"); return 0; }
    cuuint64_t dims[4] = {(cuuint64_t)CH, (cuuint64_t)v.rows, (cuuint64_t)(v.cols / CH), (cuuint64_t)v.slots};
    cuuint64_t strides[3] = {(cuuint64_t)(v.ld * esize), (cuuint64_t)(CH * esize), (cuuint64_t)(v.slot_stride * esize)};
    cuuint32_t box[4] = {(cuuint32_t)CH, (cuuint32_t)BK, (cuuint32_t)atoms, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = g_encode(&P.maps[P.nmaps], tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          4, const_cast<void*>(v.ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle(true), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -1;  // caller falls back to per-atom 3D boxes
    map_cache[key] = P.nmaps;
    return P.nmaps++;
  }

  // MN-major A operand in the canonical interleaved SW128 order: ONE 5D box per stage,
  // {CH elements, 8 rows, atoms, BK/8 groups, 1} over [slots][K groups][8 rows][atoms][CH]
  int add_map5(const View& v, int atoms) {
    if (!ok()) return 0;
    MapKey key{v.ptr, v.cols, v.rows, v.slots, v.ld, v.slot_stride, -2 * CH, atoms};
    auto hit = map_cache.find(key);
    if (hit != map_cache.end()) return hit->second;
    if (v.rows % 8) return -1;
    if (P.nmaps >= ppx::MAX_MAPS) { error(PPX_E_CONFIG, "too many tensor maps in one launch"); return 0; }
    if (!get_encode()) { error(PPX_E_CUDA, "cuTensorMapEncodeTiled unavailable"); return 0; }
    cuuint64_t dims[5] = {(cuuint64_t)CH, 8, (cuuint64_t)(v.cols / CH), (cuuint64_t)(v.rows / 8), (cuuint64_t)v.slots};
    cuuint64_t strides[4] = {(cuuint64_t)(v.ld * esize), (cuuint64_t)(CH * esize), (cuuint64_t)(8 * v.ld * esize),
                             (cuuint64_t)(v.slot_stride * esize)};
    cuuint32_t box[5] = {(cuuint32_t)CH, 8, (cuuint32_t)atoms, (cuuint32_t)(BK / 8), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(&P.maps[P.nmaps], tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          5, const_cast<void*>(v.ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -1;
    map_cache[key] = P.nmaps;
    return P.nmaps++;
  }

  // the scope's cached low part of the operand [base, base + n) (split now on a miss), or null
  // when no pooled buffer fits and none may be allocated (stream capture): per-call path then
  char* scoped_lo(const char* base, int64_t n) {
    auto key = std::make_pair(base, n);
    auto it = ctx->lo_live.find(key);
    if (it != ctx->lo_live.end()) return it->second.lo;
    const size_t bytes = ((size_t)n * 4 + 255) / 256 * 256;
    char* l = nullptr;
    size_t cap = 0;
    auto pit = ctx->lo_pool.lower_bound(bytes);
    if (pit != ctx->lo_pool.end() && pit->first <= 2 * bytes) {
      cap = pit->first;
      l = pit->second;
      ctx->lo_pool.erase(pit);
    } else {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
      if (cudaMalloc(&l, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
      ctx->lo_all.push_back(l);
      cap = bytes;
    }
    ppx::launch_split_tf32(reinterpret_cast<const float*>(base), nullptr, reinterpret_cast<float*>(l), n, st);
    ++ctx->launches;
    ctx->lo_live[key] = {n * 4, l, cap};
    return l;
  }

  // FP32 tier (3xTF32): x = hi + lo with hi = x with its low 13 mantissa bits cleared and
  // lo = x - hi, each over the whole strided extent of the view and in the view's own layout
  // (MN-major views stay MN-major: kind::tf32 reads them through the 32-byte-atom swizzle).
  // kind::tf32 reads a 32-bit operand with the low 13 bits ignored (checked bit for bit by
  // tests/test_gemm_gpu.py::test_tf32_raw_hi), so x itself serves as hi and only lo is written;
  // PPX_AB_TF32_HI_COPY=1 writes the explicit hi copy instead (A/B and that test).
  std::pair<View, View> split(const View& v) {
    View hi = v, lo = v;
    const int64_t n = (v.slots - 1) * v.slot_stride + (v.rows - 1) * v.ld + v.cols;
    const char* ab = getenv("PPX_AB_TF32_HI_COPY");   // read per call: the raw-hi test flips it
    const bool hi_copy = ab && *ab && *ab != '0';
    if (ctx->lo_scope && st == ctx->lo_stream && !hi_copy) {
      char* l = scoped_lo(reinterpret_cast<const char*>(v.ptr), n);
      if (l) {
        lo.ptr = l;
        return {hi, lo};
      }
      if (!ok()) return {hi, lo};
    }
    auto key = std::make_pair(v.ptr, n);
    auto it = splits.find(key);
    void *h = nullptr, *l = nullptr;
    if (it != splits.end()) {
      h = it->second.first;
      l = it->second.second;
    } else {
      const size_t bytes = ((size_t)n * 4 + 255) / 256 * 256;
      h = hi_copy ? ws_alloc(bytes) : const_cast<void*>(v.ptr);
      l = ws_alloc(bytes);
      if (!h || !l) { error(PPX_E_CUDA, "workspace allocation failed"); return {hi, lo}; }
      ppx::launch_split_tf32(reinterpret_cast<const float*>(v.ptr), hi_copy ? (float*)h : nullptr, (float*)l, n, st);
      ++ctx->launches;
      splits[key] = {h, l};
    }
    hi.ptr = h;
    lo.ptr = l;
    return {hi, lo};
  }

  struct PendingSeg {
    Opnd a, b;
    int kext;    // K elements per block (rounded up to BK)
    int nkblk;   // number of K blocks (slots walked by a K-blocked segment; 1 otherwise)
  };
  std::vector<PendingSeg> pend[ppx::MAX_PROBS];
  bool prob_bmn[ppx::MAX_PROBS] = {};
  int prio[ppx::MAX_PROBS] = {};   // LPT schedule: higher priority tiles are scheduled first

  static int pick_bn(int nb_extent, int gran) {
    int ntiles = (int)cdiv(nb_extent, ppx::BN_MAX);
    int bn = (int)cdiv(cdiv(nb_extent, ntiles), gran) * gran;
    return bn > ppx::BN_MAX ? ppx::BN_MAX : bn;
  }

  Problem* new_problem(int M, int nb_extent, int nblk, bool b_mn) {
    if (!ok()) return nullptr;
    if (P.nprobs >= ppx::MAX_PROBS) { error(PPX_E_CONFIG, "too many problems in one launch"); return nullptr; }
    if (M <= 0 || nb_extent <= 0 || nblk <= 0) { error(PPX_E_CONFIG, "empty GEMM problem"); return nullptr; }
    const int idx = P.nprobs++;
    Problem* pr = &P.probs[idx];
    memset(pr, 0, sizeof(*pr));
    pend[idx].clear();
    prob_bmn[idx] = b_mn;
    prio[idx] = 0;
    pr->M = M;
    pr->nb_extent = nb_extent;
    pr->nblk = nblk;
    pr->BN = pick_bn(nb_extent, b_mn ? CH : 16);
    pr->m_tiles = (int)cdiv(M, ppx::BM);
    pr->npb = (int)cdiv(nb_extent, pr->BN);
    pr->epi.out_skip = INT_MAX;
    return pr;
  }

  // record a K segment; tensor maps are built in launch() once every problem's BN is final
  // callers pass k_tiles / kpb in units of BK; they are kept as (K extent per block, blocks) so
  // launch() can re-tile K for the 2-SM kernel's 128-wide stages
  void add_segment(Problem* pr, Opnd a, Opnd b, int k_tiles, int kpb) {
    if (!ok() || !pr) return;
    if (k_tiles <= 0 || kpb <= 0 || k_tiles % kpb) { error(PPX_E_CONFIG, "empty or ragged K segment"); return; }
    pend[pr - P.probs].push_back({a, b, kpb * BK, k_tiles / kpb});
  }

  void finalize(Problem* pr, const PendingSeg& ps) {
    Opnd a = ps.a, b = ps.b;
    const int kpb = (int)cdiv(ps.kext, BKf);
    const int k_tiles = kpb * ps.nkblk;
    if (use_pair) { finalize_pair(pr, a, b, k_tiles, kpb); return; }
    // an MN-major tile is loaded in whole 128-byte atoms: a partial atom would never complete
    // the stage's transaction count
    if (b.mn && pr->BN % CH) { error(PPX_E_CONFIG, "MN-major B tile width must be a multiple of one 128-byte atom"); return; }
    auto push = [&](const View& av, const View& bv) {
      if (pr->nsegs >= ppx::MAX_SEGS) { error(PPX_E_CONFIG, "too many K segments"); return; }
      Segment& s = pr->segs[pr->nsegs++];
      s.a.atoms4d = 0;
      s.b.atoms4d = 0;
      if (a.mn && use5d && !tf32 && av.cols % CH == 0) {   // 8-row K groups: 16-bit operands only
        int m = add_map5(av, ppx::BM / CH);
        if (m >= 0) { s.a.map = (int8_t)m; s.a.atoms4d = 2; }
      }
      if (a.mn && !s.a.atoms4d && use4d && av.cols % CH == 0) {
        int m = add_map4(av, ppx::BM / CH);
        if (m >= 0) { s.a.map = (int8_t)m; s.a.atoms4d = 1; }
      }
      if (!s.a.atoms4d) s.a.map = (int8_t)(a.mn ? add_map(av, CH, BK, true) : add_map(av, BK, ppx::BM, false));
      s.a.mn = (int8_t)a.mn;
      s.a.slot_src = (int8_t)a.slot_src;
      s.a.slot_base = a.slot_base;
      s.a.slot_skip = a.slot_skip;
      if (b.mn && use4d && bv.cols % CH == 0 && pr->BN % CH == 0) {
        int m = add_map4(bv, pr->BN / CH);
        if (m >= 0) { s.b.map = (int8_t)m; s.b.atoms4d = 1; }
      }
      if (!s.b.atoms4d) s.b.map = (int8_t)(b.mn ? add_map(bv, CH, BK, true) : add_map(bv, BK, pr->BN, false));
      s.b.mn = (int8_t)b.mn;
      s.b.slot_src = (int8_t)b.slot_src;
      s.b.slot_base = b.slot_base;
      s.b.slot_skip = b.slot_skip;
      s.k_tiles = k_tiles;
      s.kpb = kpb;
      s.idesc = make_idesc(tf32, a.mn, b.mn, pr->BN);
    };
    if (!tf32) {
      push(a.v, b.v);
    } else {
      auto as = split(a.v);
      auto bs = split(b.v);
      if (!ok()) return;
      push(as.second, bs.first);  // lo * hi
      push(as.first, bs.second);  // hi * lo
      push(as.first, bs.first);   // hi * hi
    }
  }

  static int ptiles(const Problem& pr) {
    const int span = pr.nspan > 1 ? pr.nspan : 1;
    return pr.m_tiles * (int)cdiv(pr.nblk, span) * pr.npb;
  }


  // 2-SM kernel: a problem whose N blocks (slots) are each at most half a tile wide runs tiles
  // that span two consecutive blocks, one per CTA (e.g. the 7 k-wide phantom slots of
  // ppx_error_phantoms / the decompressor gradient: 256 x 256 tiles instead of 256 x 128)
  void pick_span() {
    for (int i = 0; i < P.nprobs; ++i) {
      Problem& pr = P.probs[i];
      pr.nspan = 1;
      if (pr.nblk < 2 || pr.npb != 1 || (pr.epi.flags & (ppx::EP_COLSUM | ppx::EP_BIAS))) continue;
      bool slots_n = !pend[i].empty();
      for (const PendingSeg& ps : pend[i]) slots_n = slots_n && ps.b.slot_src == 2 && ps.a.slot_src != 2;
      if (!slots_n) continue;
      const int g = prob_bmn[i] ? 64 : 16;
      const int half = (int)cdiv(pr.nb_extent, g) * g;
      if (2 * half > ppx::BN_MAX) continue;
      pr.nspan = 2;
      pr.BN = 2 * half;
    }
  }

  // Wave-quantisation trim for the static tile schedule: when the last round of tiles would
  // occupy at most half of the clusters, the trailing M-tile rows of the last problem move into
  // a copy of that problem with half-width N tiles, so the last round runs twice as many
  // half-length tiles (e.g. 256 tiles on 74 clusters: 3.5 tile-times instead of 4).
  void split_tail(int clusters) {
    if (clusters < 2 || P.nprobs < 1 || P.nprobs >= ppx::MAX_PROBS) return;
    int T = 0;
    for (int i = 0; i < P.nprobs; ++i) T += ptiles(P.probs[i]);
    const int rounds = T / clusters, rem = T % clusters;
    if (rounds < 1 || rem == 0 || rem > clusters / 2) return;
    const int li = P.nprobs - 1;
    Problem& last = P.probs[li];
    const int gran = prob_bmn[li] ? 128 : 64;
    const int half = last.BN / 2;
    if (half < gran || half % gran || half % 16 || (last.nspan < 2 && last.nb_extent <= half)) return;
    const int ntn = ptiles(last) / last.m_tiles;
    const int rows = (int)cdiv(rem, ntn);
    if (rows >= last.m_tiles) return;
    const int ti = P.nprobs++;
    Problem& tail = P.probs[ti];
    tail = last;
    last.m_tiles -= rows;
    tail.m_base = last.m_base + last.m_tiles * 2 * ppx::BM;
    tail.m_tiles = rows;
    tail.BN = half;
    tail.nspan = 1;   // a spanning tile's half is one whole N block
    tail.npb = (int)cdiv(tail.nb_extent, half);
    pend[ti] = pend[li];
    prob_bmn[ti] = prob_bmn[li];
    prio[ti] = prio[li];
  }

  static void dbg_pending(const char* where) {
    static const bool on = getenv("PPX_DEBUG_ERRORS") != nullptr;
    if (!on) return;
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) fprintf(stderr, "[ppx debug] CUDA error %d pending at %s\n", (int)e, where);
  }

  ppx_status launch() {
    dbg_pending("launch entry");
    if (!ok()) return status;
    use_pair = want_pair && pair_shapes_ok();
    BKf = use_pair ? ppx::PBK : BK;
    if (use_pair) {
      for (int i = 0; i < P.nprobs; ++i) {
        Problem& pr = P.probs[i];
        pr.m_tiles = (int)cdiv(pr.M, 2 * ppx::BM);
        pr.BN = pick_bn(pr.nb_extent, prob_bmn[i] ? 128 : 32);
        pr.npb = (int)cdiv(pr.nb_extent, pr.BN);
      }
      if (!getenv("PPX_NO_SPAN")) pick_span();
    }
    auto count_tiles = [&]() {
      int t = 0;
      for (int i = 0; i < P.nprobs; ++i) t += ptiles(P.probs[i]);
      return t;
    };
    // small launches: trade N-tile width for more CTAs (tcgen05 throughput per SM is N-invariant)
    const int slots = use_pair ? ctx->num_sms / 2 : ctx->num_sms;
    for (int guard = 0; guard < 4 && count_tiles() * 4 < slots * 3; ++guard) {
      bool changed = false;
      for (int i = 0; i < P.nprobs; ++i) {
        Problem& pr = P.probs[i];
        const int gran = use_pair ? (prob_bmn[i] ? 128 : 64) : (prob_bmn[i] ? CH : 32);
        if (pr.nspan > 1) {
          if ((pr.BN / 2) % gran) continue;   // a half-width MN-major tile would split an atom per CTA
          pr.nspan = 1;
          pr.BN /= 2;
          changed = true;
          continue;
        }
        if (pr.BN / 2 >= gran && (pr.BN / 2) % gran == 0 && (pr.BN / 2) % 16 == 0 && pr.nb_extent > pr.BN / 2) {
          pr.BN /= 2;
          pr.npb = (int)cdiv(pr.nb_extent, pr.BN);
          changed = true;
        }
      }
      if (!changed) break;
    }
    // wave quantisation: halve the N tiles when the finer grid finishes sooner, modelling a
    // half-width tile as costing 0.5 / qbal of a full one (PPX_QBAL; 0 disables)
    {
      static const double qbal = getenv("PPX_QBAL") ? atof(getenv("PPX_QBAL")) : 0.0;
      const int C = slots - (use_pair ? ctx->reserved_sms / 2 : ctx->reserved_sms);
      for (int guard = 0; qbal > 0 && C > 0 && guard < 2; ++guard) {
        const int T1 = count_tiles();
        Problem save[ppx::MAX_PROBS];
        memcpy(save, P.probs, sizeof(Problem) * P.nprobs);
        bool changed = false;
        for (int i = 0; i < P.nprobs; ++i) {
          Problem& pr = P.probs[i];
          const int gran = use_pair ? (prob_bmn[i] ? 128 : 64) : (prob_bmn[i] ? CH : 32);
          if (pr.nspan > 1) {
            if ((pr.BN / 2) % gran) continue;
            pr.nspan = 1; pr.BN /= 2; changed = true; continue;
          }
          if (pr.BN / 2 >= gran && (pr.BN / 2) % gran == 0 && (pr.BN / 2) % 16 == 0 && pr.nb_extent > pr.BN / 2) {
            pr.BN /= 2;
            pr.npb = (int)cdiv(pr.nb_extent, pr.BN);
            changed = true;
          }
        }
        const int T2 = count_tiles();
        const double t1 = (double)((T1 + C - 1) / C), t2 = (double)((T2 + C - 1) / C) * 0.5 / qbal;
        if (!changed || t2 >= t1) { memcpy(P.probs, save, sizeof(Problem) * P.nprobs); break; }
      }
    }
    if (use_pair && !lpt && !getenv("PPX_NO_TAILSPLIT")) split_tail(ctx->num_sms / 2 - ctx->reserved_sms / 2);
    for (int i = 0; i < P.nprobs; ++i)
      if ((P.probs[i].epi.flags & (ppx::EP_BITS | ppx::EP_MASKBITS)) && (P.probs[i].BN % 32 || P.probs[i].nspan > 1))
        return fail(ctx, PPX_E_CONFIG, "bit-mask epilogues need 32-aligned, non-spanning tiles");
    for (int i = 0; i < P.nprobs && ok(); ++i)
      for (const PendingSeg& ps : pend[i]) finalize(&P.probs[i], ps);
    if (!ok()) return status;
    dbg_pending("after finalize");
    int tiles = 0;
    for (int i = 0; i < P.nprobs; ++i) {
      P.probs[i].tile_begin = tiles;
      tiles += ptiles(P.probs[i]);
    }
    P.total_tiles = tiles;
    P.nsched = 0;
    if (lpt && use_pair && !fuse_world && tiles <= ppx::MAX_SCHED && ctx->num_sms / 2 < 76) {
      // LPT: tiles in decreasing cost (K stages + epilogue, scaled by tile width) each go to the
      // least-loaded cluster; every role of a cluster walks the same list
      const int sms_avail = ctx->num_sms - ctx->reserved_sms;
      const int C = tiles < sms_avail / 2 ? tiles : sms_avail / 2;
      // assignment: plain LPT over all tiles (balance); order within each cluster: priority tiles
      // (prio[i] > 0, e.g. error compression whose outputs other GPUs wait for) first.  Putting
      // priority tiles first in the ASSIGNMENT instead would stack them on top of the clusters that
      // also draw two long tiles (R=1 fused error + weight-gradient launch: 148 vs 128 us)
      std::vector<std::pair<double, int>> cost(tiles);
      std::vector<int> tprio(tiles, 0);
      static const char* ab = getenv("PPX_AB_NO_PRIO");   // A/B of the priority classes only
      for (int i = 0; i < P.nprobs; ++i) {
        const Problem& pr = P.probs[i];
        int kst = 0;
        for (int g = 0; g < pr.nsegs; ++g) kst += pr.segs[g].k_tiles;
        const double c = (kst + 4.0) * pr.BN / 256.0;
        for (int t = pr.tile_begin; t < pr.tile_begin + ptiles(pr); ++t) {
          cost[t] = {-c, t};
          tprio[t] = (ab && *ab) ? 0 : prio[i];
        }
      }
      std::stable_sort(cost.begin(), cost.end());
      std::vector<double> load(C, 0.0);
      std::vector<std::vector<int>> lists(C);
      for (const auto& ct : cost) {
        int best = 0;
        for (int c = 1; c < C; ++c)
          if (load[c] < load[best]) best = c;
        load[best] -= ct.first;
        lists[best].push_back(ct.second);
      }
      for (auto& l : lists)
        std::stable_sort(l.begin(), l.end(), [&](int x, int y) { return tprio[x] > tprio[y]; });
      int o = 0;
      for (int c = 0; c < C; ++c) {
        P.sched_off[c] = (uint16_t)o;
        for (int t : lists[c]) P.sched[o++] = (uint16_t)t;
      }
      P.sched_off[C] = (uint16_t)o;
      P.nsched = tiles;
    }
    if (fuse_world) {   // fused compress + exchange + forward: arrivals per epoch on this GPU
      if (!use_pair) return fail(ctx, PPX_E_CONFIG, "fused forward needs the 2-SM kernel (bf16, 64-aligned shapes)");
      int ct = 0;
      for (int i = 0; i < P.nprobs; ++i)
        if (P.probs[i].epi.narrive) ct += ptiles(P.probs[i]);
      for (int i = 0; i < P.nprobs; ++i)
        if (P.probs[i].wait_ctr) P.probs[i].wait_per_epoch = fuse_world * 2 * ct;
      P.epoch = fuse_epoch;
      P.done = ctx->fuse_done;
      P.bad = fuse_bad;
    }
    {
      const char* ep = getenv("PPX_DEBUG_EPI");
      P.dbg = (getenv("PPX_DEBUG_NOEPI") ? 1 : 0) | (getenv("PPX_DEBUG_NOWAIT") ? 2 : 0) |
              (ep && strstr(ep, "mask") ? 4 : 0) | (ep && strstr(ep, "colsum") ? 8 : 0) |
              (ep && strstr(ep, "scatter") ? 16 : 0);
    }
    if (tiles == 0) return PPX_OK;
    cudaError_t e;
    const int sms = ctx->num_sms - ctx->reserved_sms;
    static unsigned long long* dstats = nullptr;
    const bool want_stats = getenv("PPX_DEBUG_STATS") != nullptr;
    if (want_stats && !dstats) cudaMalloc(&dstats, 16 * sizeof(unsigned long long));
    P.stats = want_stats ? dstats : nullptr;
    if (want_stats) cudaMemsetAsync(dstats, 0, 16 * sizeof(unsigned long long), st);
    if (use_pair) {
      const int clusters = tiles < sms / 2 ? tiles : sms / 2;
      e = ppx::launch_gemm_pair(P, 2 * clusters, st);
      if (want_stats) {
        unsigned long long h[16];
        cudaMemcpyAsync(h, dstats, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const double n = (double)(h[6] ? h[6] : 1), ne = 16.0 * n;   // MMA issuers; epilogue warps
        fprintf(stderr, "[ppx stats] tiles=%d clusters=%d  per-MMA-warp kcyc: total %.1f tempty-wait %.1f full-wait %.1f | "
                "producer empty-wait %.1f | per-epi-warp tfull-wait %.1f busy %.1f (tmem ld %.1f body %.1f)\n",
                tiles, clusters, h[5] / n / 1e3, h[3] / n / 1e3, h[4] / n / 1e3, h[2] / (2 * n) / 1e3, h[0] / ne / 1e3,
                h[1] / ne / 1e3, h[7] / ne / 1e3, h[8] / ne / 1e3);
      }
    } else {
      int grid = tiles < sms ? tiles : sms;
      e = tf32 ? ppx::launch_gemm<true>(P, grid, st) : ppx::launch_gemm<false>(P, grid, st);
    }
    if (e != cudaSuccess) return fail(ctx, PPX_E_CUDA, "gemm launch: %s", cudaGetErrorString(e));
    ++ctx->launches;
    dbg_pending("after gemm launch");
    invalidate_outputs();
    return PPX_OK;
  }

  // the FP32-tier operand cache forgets every operand this launch's epilogues write: the span
  // from row 0 to the last element of the problem's last row and slot (peer replicas included)
  void invalidate_outputs() {
    if (ctx->lo_live.empty()) return;
    for (int i = 0; i < P.nprobs; ++i) {
      const Problem& pr = P.probs[i];
      const ppx::Epilogue& E = pr.epi;
      const int64_t last_row = pr.m_base + pr.M - 1;
      const int64_t last_slot = pr.nblk - 1 + (E.out_skip != INT_MAX ? 1 : 0);
      for (const ppx::Tensor2* t : {&E.out, &E.aux, &E.preact, &E.master, &E.adam_m, &E.adam_v}) {
        if (!t->ptr) continue;
        const bool words = t == &E.preact && (E.flags & ppx::EP_BITS);   // 1-bit masks in uint32 words
        const int64_t es = words ? 4 : (t->f32 ? 4 : 2);
        const int64_t cols = words ? (pr.nb_extent + 31) / 32 : pr.nb_extent;
        const int64_t bytes = (last_row * t->ld + last_slot * t->slot_stride + cols) * es;
        lo_invalidate(ctx, t->ptr, bytes);
        if (t == &E.out)
          for (int r = 0; r < E.nrep; ++r) lo_invalidate(ctx, (const char*)t->ptr + E.rep_off[r], bytes);
      }
    }
  }
};

inline bool bad_layer(const ppx_layer* L) {
  return !L || L->s < 1 || L->k < 1 || L->k > L->s || L->p < 1 || L->rank < 0 || L->rank >= L->p || !L->w ||
         !L->master;
}

inline const char* elem(ppx_dtype dt, const void* base, int64_t off) {
  return reinterpret_cast<const char*>(base) + off * (dt == PPX_FP32 ? 4 : 2);
}

}  // namespace

namespace ppx {
template <bool kTF32>
cudaError_t launch_gemm(const GemmParams& P, int grid, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<kTF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  static const bool pdl = getenv("PPX_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemm_kernel<kTF32>, P);
}
cudaError_t launch_gemm_pair(const GemmParams& P, int grid, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PSMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = PSMEM_BYTES;
  cfg.stream = st;
  static const bool pdl = getenv("PPX_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddepcontrol in the kernel
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, gemm_pair_kernel, P);
}
template cudaError_t launch_gemm<true>(const GemmParams&, int, cudaStream_t);
template cudaError_t launch_gemm<false>(const GemmParams&, int, cudaStream_t);
}  // namespace ppx

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

int ppx_abi_version(void) { return PPX_ABI_VERSION; }

int32_t ppx_peek_error(void) { return (int32_t)cudaPeekAtLastError(); }

int64_t ppx_layer_elems(int32_t s, int32_t k, int32_t p) { return Flat(s, k, p).total; }

ppx_status ppx_get_unique_id(uint8_t uid[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PPX_E_PROTOCOL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(uid, &id, 128);
  return PPX_OK;
}

ppx_status ppx_create(int32_t world, int32_t rank, int32_t device, const uint8_t* uid, ppx_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return PPX_E_CONFIG;
  ppx_ctx* ctx = new ppx_ctx();
  ctx->world = world;
  ctx->rank = rank;
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return PPX_E_CUDA; }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) ctx->num_sms = sms;
  if (cudaMalloc(&ctx->fuse_done, sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(ctx->fuse_done, 0, sizeof(unsigned int)) != cudaSuccess) { delete ctx; return PPX_E_CUDA; }
  if (world > 1) {
    if (!uid) { delete ctx; return PPX_E_CONFIG; }
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) { delete ctx; return PPX_E_PROTOCOL; }
  }
  *out = ctx;
  return PPX_OK;
}

ppx_status ppx_destroy(ppx_ctx* ctx) {
  if (!ctx) return PPX_OK;
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (auto& c : ctx->ws) cudaFree(c.first);
  for (char* m : ctx->lo_all) cudaFree(m);
  if (ctx->lo_done) cudaEventDestroy(ctx->lo_done);
  for (void* m : ctx->ipc_mapped) cudaIpcCloseMemHandle(m);
  if (ctx->fuse_done) cudaFree(ctx->fuse_done);
  if (ctx->reduce_done) cudaFree(ctx->reduce_done);
  for (void* m : ctx->ipc_own) cudaFree(m);
  delete ctx;
  return PPX_OK;
}

const char* ppx_last_error(const ppx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int32_t ppx_num_sms(const ppx_ctx* ctx) { return ctx ? ctx->num_sms : 0; }
int64_t ppx_kernel_launches(const ppx_ctx* ctx) { return ctx ? ctx->launches : 0; }

ppx_status ppx_set_reserved_sms(ppx_ctx* ctx, int32_t n) {
  if (!ctx || n < 0 || n > ctx->num_sms - 2) return PPX_E_CONFIG;
  ctx->reserved_sms = n;
  return PPX_OK;
}

ppx_status ppx_reserve_workspace(ppx_ctx* ctx, int64_t bytes) {
  if (!ctx || bytes < 0) return PPX_E_CONFIG;
  if (!ctx->ws.empty() && (int64_t)ctx->ws.front().second >= bytes) return PPX_OK;
  for (auto& c : ctx->ws) cudaFree(c.first);
  ctx->ws.clear();
  if (bytes == 0) return PPX_OK;
  char* p = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&p, (size_t)bytes));
  ctx->ws.push_back({p, (size_t)bytes});
  return PPX_OK;
}

// ---------------------------------------------------------------------------------------------
static ppx_status add_compress(ppx_ctx* ctx, ppx_dtype dt, Builder& b, const ppx_rank_io& io, int32_t B,
                               void* phantoms) {
  const ppx_layer* L = io.layer;
  if (bad_layer(L) || B < 1 || !io.x || !phantoms) return fail(ctx, PPX_E_CONFIG, "compress: bad arguments");
  Flat f(L->s, L->k, L->p);
  Problem* pr = b.new_problem(B, L->k, 1, false);
  Opnd a{view2(io.x, B, L->s, io.ld_x)};
  Opnd w{view2(elem(dt, L->w, f.comp), L->k, L->s, f.lds)};
  b.add_segment(pr, a, w, (int)cdiv(L->s, b.BK), (int)cdiv(L->s, b.BK));
  if (pr) pr->epi.out = t2((char*)phantoms + (int64_t)L->rank * B * f.ldk * b.esize, f.ldk, dt == PPX_FP32);
  return b.ok() ? PPX_OK : b.status;
}

ppx_status ppx_compress_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B, void* phantoms,
                          void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io) return fail(ctx, PPX_E_CONFIG, "ppx_compress_n: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < n; ++i) {
    ppx_status s = add_compress(ctx, dt, b, io[i], B, phantoms);
    if (s != PPX_OK) return s;
  }
  return b.launch();
}

ppx_status ppx_compress(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, const void* y_prev, int64_t ld_y,
                        void* phantoms, void* stream) {
  ppx_rank_io io{};
  io.layer = L;
  io.x = y_prev;
  io.ld_x = ld_y;
  return ppx_compress_n(ctx, dt, 1, &io, B, phantoms, stream);
}

static ppx_status add_forward(ppx_ctx* ctx, ppx_dtype dt, Builder& b, const ppx_rank_io& io, int32_t B, ppx_act act,
                              const void* phantoms, int output_layer, float delta_scale, float loss_scale,
                              float* loss) {
  const ppx_layer* L = io.layer;
  // the output layer may skip storing y (training needs only the delta and the loss)
  if (bad_layer(L) || B < 1 || !io.x || (!io.out && !output_layer))
    return fail(ctx, PPX_E_CONFIG, "forward: bad arguments");
  if (output_layer && (!io.target || !io.aux || !loss)) return fail(ctx, PPX_E_CONFIG, "forward output: bad arguments");
  Flat f(L->s, L->k, L->p);
  Problem* pr = b.new_problem(B, L->s, 1, false);
  Opnd a{view2(io.x, B, L->s, io.ld_x)};
  Opnd w{view2(elem(dt, L->w, f.local), L->s, L->s, f.lds)};
  b.add_segment(pr, a, w, (int)cdiv(L->s, b.BK), (int)cdiv(L->s, b.BK));
  if (L->p > 1) {
    if (!phantoms) return fail(ctx, PPX_E_SEQUENCING, "forward: phantom buffer missing");
    Opnd g{view3(phantoms, L->p, B, L->k, f.ldk, (int64_t)B * f.ldk)};
    g.slot_src = 1;
    g.slot_skip = L->rank;
    Opnd d{view3(elem(dt, L->w, f.dec), L->p - 1, L->s, L->k, f.ldk, (int64_t)L->s * f.ldk)};
    d.slot_src = 1;
    int kpb = (int)cdiv(L->k, b.BK);
    b.add_segment(pr, g, d, kpb * (L->p - 1), kpb);
  }
  if (!pr) return b.status;
  const int f32 = dt == PPX_FP32;
  pr->epi.bias = L->bias ? L->bias : L->master + f.bias;
  pr->epi.flags = ppx::EP_BIAS | (act == PPX_RELU ? ppx::EP_RELU : 0u);
  pr->epi.out = t2(io.out, io.ld_out, f32);
  if (!output_layer) {
    if (io.aux && io.bits) return fail(ctx, PPX_E_CONFIG, "forward: pre-activation and bit mask are exclusive");
    if (io.aux) {
      pr->epi.flags |= ppx::EP_PREACT;
      pr->epi.preact = t2(io.aux, io.ld_aux, f32);
    }
    if (io.bits) {   // the recurrence's ReLU' mask, 1 bit per element (the preact slot carries it)
      if (f32 || L->s % 32 || act != PPX_RELU || io.ld_bits < L->s / 32)
        return fail(ctx, PPX_E_CONFIG, "forward: bit masks need bf16, ReLU and s % 32 == 0");
      pr->epi.flags |= ppx::EP_BITS;
      pr->epi.preact = t2(io.bits, io.ld_bits, 0);
    }
  } else {
    pr->epi.flags |= ppx::EP_LOSS | (io.colsum ? ppx::EP_COLSUM : 0u);
    pr->epi.aux = t2(io.aux, io.ld_aux, f32);
    pr->epi.target = t2(const_cast<void*>(io.target), io.ld_t, f32);
    pr->epi.scale = delta_scale;
    pr->epi.loss_scale = loss_scale;
    pr->epi.loss = loss;
    pr->epi.colsum = io.colsum;
  }
  return b.ok() ? PPX_OK : b.status;
}

ppx_status ppx_forward_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B, ppx_act act,
                         const void* phantoms, int32_t output_layer, float delta_scale, float loss_scale, float* loss,
                         void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io) return fail(ctx, PPX_E_CONFIG, "ppx_forward_n: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < n; ++i) {
    ppx_status s = add_forward(ctx, dt, b, io[i], B, act, phantoms, output_layer, delta_scale, loss_scale, loss);
    if (s != PPX_OK) return s;
  }
  return b.launch();
}

// phantom.py:135-166 for the n local ranks as ONE launch: compression tiles (first in the tile
// order) store their phantoms locally and into every peer's buffer (NVLink) and bump every GPU's
// arrival counter; the forward tiles run their local-block K segment, then spin (producer warp)
// until all GPUs' compression tiles of this layer have arrived, then the decompression segment.
ppx_status ppx_forward_fused(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B, ppx_act act,
                             void* phantoms, int32_t output_layer, float delta_scale, float loss_scale, float* loss,
                             const ppx_exchange* ex, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io || !phantoms || !ex || !ex->arrive || !ex->wait_counter || !ex->epoch || ex->n_peers < 0 ||
      ex->n_peers > ppx::MAX_REP || (ex->n_peers && !ex->peer_phantoms) || dt != PPX_BF16)
    return fail(ctx, PPX_E_CONFIG, "ppx_forward_fused: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < n; ++i) {
    ppx_status st = add_compress(ctx, dt, b, io[i], B, phantoms);
    if (st != PPX_OK) return st;
    ppx::Epilogue& E = b.P.probs[b.P.nprobs - 1].epi;
    E.nrep = ex->n_peers;
    for (int r = 0; r < ex->n_peers; ++r)
      E.rep_off[r] = (long long)((const char*)ex->peer_phantoms[r] - (const char*)phantoms);
    E.narrive = ex->n_peers + 1;
    for (int r = 0; r <= ex->n_peers; ++r) E.arrive[r] = ex->arrive[r];
  }
  for (int i = 0; i < n; ++i) {
    ppx_status st = add_forward(ctx, dt, b, io[i], B, act, phantoms, output_layer, delta_scale, loss_scale, loss);
    if (st != PPX_OK) return st;
    Problem& pr = b.P.probs[b.P.nprobs - 1];
    if (io[i].layer->p > 1) {
      pr.wait_ctr = ex->wait_counter;
      pr.wait_seg = 1;   // segment 0 = local block, 1 = the gathered phantoms
    }
  }
  b.fuse_world = ex->n_peers + 1;
  b.fuse_epoch = ex->epoch;
  b.fuse_bad = ex->bad;
  return b.launch();
}

ppx_status ppx_forward_update(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act,
                              const void* y_prev, int64_t ld_y, const void* phantoms, void* y_out, int64_t ld_out,
                              void* preact, int64_t ld_pre, void* stream) {
  ppx_rank_io io{};
  io.layer = L;
  io.x = y_prev;
  io.ld_x = ld_y;
  io.out = y_out;
  io.ld_out = ld_out;
  io.aux = preact;
  io.ld_aux = ld_pre;
  return ppx_forward_n(ctx, dt, 1, &io, B, act, phantoms, 0, 1.f, 0.f, nullptr, stream);
}

ppx_status ppx_forward_output(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act,
                              const void* y_prev, int64_t ld_y, const void* phantoms, void* y_out, int64_t ld_out,
                              const void* target, int64_t ld_t, void* delta, int64_t ld_d, float delta_scale,
                              float loss_scale, float* loss, float* bias_grad, void* stream) {
  ppx_rank_io io{};
  io.layer = L;
  io.x = y_prev;
  io.ld_x = ld_y;
  io.out = y_out;
  io.ld_out = ld_out;
  io.aux = delta;
  io.ld_aux = ld_d;
  io.target = target;
  io.ld_t = ld_t;
  io.colsum = bias_grad;
  return ppx_forward_n(ctx, dt, 1, &io, B, act, phantoms, 1, delta_scale, loss_scale, loss, stream);
}

ppx_status ppx_output_delta(ppx_ctx* ctx, ppx_dtype dt, int32_t B, int32_t s, ppx_act act, const void* y_out,
                            int64_t ld_y, const void* target, int64_t ld_t, const void* pre, int64_t ld_p, void* delta,
                            int64_t ld_d, float delta_scale, float loss_scale, float* loss, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (B < 1 || s < 1 || !y_out || !target || !delta || (act == PPX_RELU && !pre))
    return fail(ctx, PPX_E_CONFIG, "ppx_output_delta: bad arguments");
  lo_invalidate(ctx, delta, (int64_t)B * ld_d * (dt == PPX_FP32 ? 4 : 2));
  ++ctx->launches;
  cudaError_t e = ppx::launch_output_delta(dt == PPX_FP32, B, s, act == PPX_RELU, y_out, ld_y, target, ld_t, pre, ld_p,
                                           delta, ld_d, delta_scale, loss_scale, loss, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "output_delta: %s", cudaGetErrorString(e));
}

ppx_status ppx_error_phantoms(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, const void* delta,
                              int64_t ld_d, void* contrib, int32_t accumulate, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (bad_layer(L) || B < 1 || !delta || !contrib) return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms: bad arguments");
  if (L->p < 2) return PPX_OK;  // no peers: every slot but the (unwritten) own one is absent
  Flat f(L->s, L->k, L->p);
  Builder b(ctx, dt, stream);
  Problem* pr = b.new_problem(B, L->k, L->p - 1, true);
  Opnd a{view2(delta, B, L->s, ld_d)};
  Opnd d{view3(elem(dt, L->w, f.dec), L->p - 1, L->s, L->k, f.ldk, (int64_t)L->s * f.ldk)};
  d.mn = 1;
  d.slot_src = 2;
  int kt = (int)cdiv(L->s, b.BK);
  b.add_segment(pr, a, d, kt, kt);
  if (pr) {
    pr->epi.out = t2(contrib, f.ldk, dt == PPX_FP32, (int64_t)B * f.ldk);
    pr->epi.out_skip = L->rank;
    pr->epi.flags = accumulate ? ppx::EP_ACCUM : 0u;
  }
  return b.launch();
}

// One error-compression problem over `nslots` (1 or 2) consecutive output slots i0.. of the
// [p][B, ldk] contribution buffer: segment j (every local rank contributing to one of the slots)
// reads rank j's decompressor stack in stack mode, so with two slots each CTA of a pair tile takes
// one slot and rank j's own slot (absent from its stack) loads as TMA zeros.  Two slots make
// 256-wide tiles (one 128-wide slot per CTA) instead of L2-bandwidth-bound 128-wide ones.
// Peer-owned slots are also copied to their owner's staging area (sc) — both slots of a pair
// belong to the same owner when R is even — or accumulate into `contrib`.
static Problem* error_slot_problem(Builder& b, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                   void* contrib, int i0, int nslots, const ppx_scatter* sc, int accumulate) {
  const int p = io[0].layer->p, s = io[0].layer->s, k = io[0].layer->k;
  Flat f(s, k, p);
  const int es = dt == PPX_FP32 ? 4 : 2;
  const int64_t slot_bytes = (int64_t)B * f.ldk * es;
  const int kt = (int)cdiv(s, b.BK);
  int nseg = 0;
  for (int j = 0; j < n; ++j) {
    const int r = io[j].layer->rank;
    nseg += nslots == 2 ? 1 : (r != i0);
  }
  if (!nseg) return nullptr;
  Problem* pr = b.new_problem(B, k, nslots, true);
  if (!pr) return nullptr;
  for (int j = 0; j < n; ++j) {
    const ppx_layer* L = io[j].layer;
    if (nslots == 1 && L->rank == i0) continue;
    Opnd a{view2(io[j].x, B, s, io[j].ld_x)};
    Opnd d{view3(elem(dt, L->w, f.dec), p - 1, s, k, f.ldk, (int64_t)s * f.ldk)};
    d.mn = 1;
    if (nslots == 2) {
      d.slot_src = 2;
      d.slot_base = i0;
      d.slot_skip = -(L->rank + 1);
    } else {
      d.slot_base = i0 - (i0 > L->rank ? 1 : 0);
    }
    b.add_segment(pr, a, d, kt, kt);
  }
  char* local = (char*)contrib + (int64_t)i0 * slot_bytes;
  pr->epi.out = t2(local, f.ldk, dt == PPX_FP32, (int64_t)B * f.ldk);
  if (accumulate) pr->epi.flags |= ppx::EP_ACCUM;
  if (sc && nslots == 2 && i0 / n != (i0 + 1) / n) {
    // one logical rank per GPU: the two slots of a pair belong to different owners
    pr->epi.rep_per_half = 1;
    pr->epi.arrive_units = 1;
    for (int h = 0; h < 2; ++h) {
      const int g = (i0 + h) / n;
      if (g == sc->rank) continue;          // own slot: stays in contrib (reduced in place)
      char* dst = (char*)sc->stage[g] + ((int64_t)sc->rank * n + (i0 + h - g * n)) * slot_bytes;
      pr->epi.rep_off[h] = (long long)(dst - (local + h * slot_bytes));
      pr->epi.arrive[h] = sc->arrive[g];
    }
    pr->epi.nrep = 2;
    pr->epi.narrive = 2;
  } else if (sc) {
    const int g = i0 / n;
    if (g != sc->rank) {
      char* dst = (char*)sc->stage[g] + ((int64_t)sc->rank * n + (i0 - g * n)) * slot_bytes;
      pr->epi.nrep = 1;
      pr->epi.rep_off[0] = (long long)(dst - local);
      pr->epi.narrive = 1;
      pr->epi.arrive_units = 1;
      pr->epi.arrive[0] = sc->arrive[g];
    }
  }
  return pr;
}

// slot pairs need bf16 (2-SM tiles), k a multiple of 64 (each half one whole 64-atom block per CTA)
// and an even number of local ranks (both slots of a pair then share an owner) or exactly one (each
// half then publishes to its own owner)
static bool error_pairs(ppx_dtype dt, int n, int p, int k) {
  static const char* ab = getenv("PPX_AB_NO_ERROR_PAIRS");   // A/B of this planner choice only
  static const bool off = ab && *ab;
  return !off && dt == PPX_BF16 && (n % 2 == 0 || n == 1) && p % 2 == 0 && k % 64 == 0;
}

// Grouped error compression for the n logical ranks one GPU owns (phantom.py:199-205): output
// slot i = sum over contributing ranks j != i (ascending) of delta_j . D_{i->j}, as ONE
// K-concatenated problem per slot (segment j reads D_{i->j} = slot i - (i > j) of rank j's
// decompressor stack), so the ranks' contributions are summed in the fp32 accumulator instead
// of n accumulate launches.  Slots without a contributor are not written.  Falls back to the
// per-rank accumulate launches when a slot would need more than MAX_SEGS segments (3 per
// contributing rank in the 3xTF32 tier).
ppx_status ppx_error_phantoms_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                void* contrib, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io || B < 1 || !contrib) return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms_n: bad arguments");
  for (int j = 0; j < n; ++j) {
    const ppx_layer* L = io[j].layer;
    if (bad_layer(L) || !io[j].x || L->s != io[0].layer->s || L->k != io[0].layer->k || L->p != io[0].layer->p ||
        (j && L->rank <= io[j - 1].layer->rank))
      return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms_n: ranks must share (s, k, p) and ascend");
  }
  const int p = io[0].layer->p, s = io[0].layer->s, k = io[0].layer->k;
  if (p < 2) return PPX_OK;
  Flat f(s, k, p);
  const int es = dt == PPX_FP32 ? 4 : 2;
  if (n == 1 || n * (dt == PPX_FP32 ? 3 : 1) > ppx::MAX_SEGS) {
    if (n > 1) {
      cudaError_t e = cudaMemsetAsync(contrib, 0, (size_t)p * B * f.ldk * es, (cudaStream_t)stream);
      if (e != cudaSuccess) return fail(ctx, PPX_E_CUDA, "error_phantoms_n: %s", cudaGetErrorString(e));
    }
    for (int j = 0; j < n; ++j) {
      ppx_status st = ppx_error_phantoms(ctx, dt, io[j].layer, B, io[j].x, io[j].ld_x, contrib, n > 1, stream);
      if (st != PPX_OK) return st;
    }
    return PPX_OK;
  }
  const int step = error_pairs(dt, n, p, k) ? 2 : 1;
  int i = 0;
  while (i < p) {
    Builder b(ctx, dt, stream);
    for (; i < p && b.P.nprobs < ppx::MAX_PROBS - 1; i += step) error_slot_problem(b, dt, n, io, B, contrib, i, step, nullptr, 0);
    ppx_status st = b.launch();
    if (st != PPX_OK) return st;
  }
  (void)es;
  (void)f;
  return PPX_OK;
}

// ---- NVLink peer memory: the phantom all-gather as NVLink stores from the compression GEMM ----
ppx_status ppx_peer_alloc(ppx_ctx* ctx, int64_t bytes, void** ptr, uint8_t* handle) {
  if (!ctx || bytes <= 0 || !ptr || !handle) return PPX_E_CONFIG;
  if (!ctx->reduce_done) {   // reduce exit counter (allocated here: never during capture)
    CUDA_TRY(ctx, cudaMalloc(&ctx->reduce_done, sizeof(unsigned int)));
    CUDA_TRY(ctx, cudaMemset(ctx->reduce_done, 0, sizeof(unsigned int)));
  }
  void* p = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&p, (size_t)bytes));
  ctx->ipc_own.push_back(p);
  CUDA_TRY(ctx, cudaMemset(p, 0, (size_t)bytes));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, p));
  memcpy(handle, &h, 64);
  *ptr = p;
  return PPX_OK;
}

ppx_status ppx_peer_open(ppx_ctx* ctx, const uint8_t* handle, void** peer_ptr) {
  if (!ctx || !handle || !peer_ptr) return PPX_E_CONFIG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* p = nullptr;
  CUDA_TRY(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ctx->ipc_mapped.push_back(p);
  *peer_ptr = p;
  return PPX_OK;
}

// NVLink reduce-scatter, sender side (phantom.py:199-205 + collectives.py:345-357): one problem per
// phantom slot i over this GPU's contributing ranks (as ppx_error_phantoms_n, also for n = 1); the
// slots this GPU owns stay in `contrib`, every other slot is computed into `contrib` and copied by
// the epilogue into its owner's staging area (sc->stage[g] + (rank * R + i - g * R) * slot) with
// the owner's arrival counter bumped by rows * cols / 8 per CTA part.
ppx_status ppx_error_phantoms_scatter(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                      void* contrib, const ppx_scatter* sc, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io || B < 1 || !contrib || !sc || !sc->stage || !sc->arrive || sc->world < 1 || sc->rank < 0 ||
      sc->rank >= sc->world || dt != PPX_BF16 || n > ppx::MAX_SEGS)
    return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms_scatter: bad arguments");
  const int p = io[0].layer->p, s = io[0].layer->s, k = io[0].layer->k;
  for (int j = 0; j < n; ++j) {
    const ppx_layer* L = io[j].layer;
    if (bad_layer(L) || !io[j].x || L->s != s || L->k != k || L->p != p || (j && L->rank <= io[j - 1].layer->rank))
      return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms_scatter: ranks must share (s, k, p) and ascend");
  }
  if (p < 2) return PPX_OK;
  if (p % sc->world || p / sc->world != n) return fail(ctx, PPX_E_CONFIG, "ppx_error_phantoms_scatter: R != p / world");
  Flat f(s, k, p);
  const int R = n, es = 2;
  const int64_t slot_bytes = (int64_t)B * f.ldk * es;
  const int step = error_pairs(dt, R, p, k) ? 2 : 1;
  int i = 0;
  while (i < p) {
    Builder b(ctx, dt, stream);
    for (; i < p && b.P.nprobs < ppx::MAX_PROBS - 1; i += step) error_slot_problem(b, dt, R, io, B, contrib, i, step, sc, 0);
    ppx_status st = b.launch();
    if (st != PPX_OK) return st;
  }
  (void)slot_bytes;
  (void)f;
  return PPX_OK;
}

ppx_status ppx_reduce_received(ppx_ctx* ctx, ppx_dtype dt, int32_t R, int64_t slot_elems, int32_t world, int32_t rank,
                               const void* stage, const void* own, void* out, const int32_t* counter, int32_t* epoch,
                               int32_t* bad, void* stream) {
  if (!ctx || !stage || !own || !out || !counter || !epoch || R < 1 || world < 1 || rank < 0 || rank >= world ||
      slot_elems % 8 || dt != PPX_BF16)
    return fail(ctx, PPX_E_CONFIG, "ppx_reduce_received: bad arguments");
  if (!ctx->reduce_done) return fail(ctx, PPX_E_SEQUENCING, "ppx_reduce_received before ppx_peer_alloc");
  lo_invalidate(ctx, out, (int64_t)R * slot_elems * 2);
  ppx::ReduceArgs a;
  a.stage = (const __nv_bfloat16*)stage;
  a.own = (const __nv_bfloat16*)own;
  a.out = (__nv_bfloat16*)out;
  a.slot_x8 = R * slot_elems / 8;
  a.src_stride_x8 = R * slot_elems / 8;
  a.world = world;
  a.me = rank;
  a.counter = counter;
  a.epoch = epoch;
  a.per_epoch = 0;   // set below: (world - 1) sources x R slots x slot elements / 8
  a.per_epoch = (int)((int64_t)(world - 1) * R * slot_elems / 8);
  a.bad = bad;
  a.done = ctx->reduce_done;
  ++ctx->launches;
  CUDA_TRY(ctx, ppx::launch_reduce_received(a, (cudaStream_t)stream));
  return PPX_OK;
}

static ncclDataType_t nccl_type(ppx_dtype dt) { return dt == PPX_FP32 ? ncclFloat32 : ncclBfloat16; }

ppx_status ppx_all_gather(ppx_ctx* ctx, ppx_dtype dt, void* phantoms, int64_t slot_elems, int32_t local_ranks,
                          void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (ctx->world == 1) return PPX_OK;
  const int64_t chunk = slot_elems * local_ranks;
  char* base = (char*)phantoms;
  const int es = dt == PPX_FP32 ? 4 : 2;
  lo_invalidate(ctx, base, chunk * ctx->world * es);
  NCCL_TRY(ctx, ncclAllGather(base + (int64_t)ctx->rank * chunk * es, base, (size_t)chunk, nccl_type(dt), ctx->comm,
                              (cudaStream_t)stream));
  return PPX_OK;
}

ppx_status ppx_reduce_scatter(ppx_ctx* ctx, ppx_dtype dt, void* contrib, int64_t slot_elems, int32_t local_ranks,
                              void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (ctx->world == 1) return PPX_OK;
  const int64_t chunk = slot_elems * local_ranks;
  char* base = (char*)contrib;
  const int es = dt == PPX_FP32 ? 4 : 2;
  lo_invalidate(ctx, base, chunk * ctx->world * es);
  NCCL_TRY(ctx, ncclReduceScatter(base, base + (int64_t)ctx->rank * chunk * es, (size_t)chunk, nccl_type(dt), ncclSum,
                                  ctx->comm, (cudaStream_t)stream));
  return PPX_OK;
}

ppx_status ppx_reduce_scatter_to(ppx_ctx* ctx, ppx_dtype dt, const void* contrib, void* recv, int64_t slot_elems,
                                 int32_t local_ranks, void* stream) {
  if (!ctx || !contrib || !recv) return PPX_E_CONFIG;
  const int64_t chunk = slot_elems * local_ranks;
  const int es = dt == PPX_FP32 ? 4 : 2;
  lo_invalidate(ctx, recv, chunk * es);
  if (ctx->world == 1) {
    CUDA_TRY(ctx, cudaMemcpyAsync(recv, contrib, (size_t)(chunk * es), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return PPX_OK;
  }
  NCCL_TRY(ctx, ncclReduceScatter(contrib, recv, (size_t)chunk, nccl_type(dt), ncclSum, ctx->comm, (cudaStream_t)stream));
  return PPX_OK;
}

ppx_status ppx_all_reduce_f32(ppx_ctx* ctx, float* buf, int64_t count, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  lo_invalidate(ctx, buf, count * 4);
  if (ctx->world == 1) return PPX_OK;
  NCCL_TRY(ctx, ncclAllReduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, ctx->comm, (cudaStream_t)stream));
  return PPX_OK;
}

ppx_status ppx_all_reduce(ppx_ctx* ctx, ppx_dtype dt, void* buf, int64_t count, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  lo_invalidate(ctx, buf, count * (dt == PPX_FP32 ? 4 : 2));
  if (ctx->world == 1) return PPX_OK;
  NCCL_TRY(ctx, ncclAllReduce(buf, buf, (size_t)count, nccl_type(dt), ncclSum, ctx->comm, (cudaStream_t)stream));
  return PPX_OK;
}

static void set_update(ppx::Epilogue& E, const ppx_update* upd, ppx_dtype dt, int64_t off, int64_t ld, int64_t ss) {
  const int es = dt == PPX_FP32 ? 4 : 2;
  E.flags = (upd->kind == PPX_UPDATE_ADAM ? ppx::EP_ADAM : ppx::EP_SGD) | (upd->bad ? ppx::EP_FINITE : 0u);
  E.hyper = upd->hyper;
  E.master = t2(upd->master + off, ld, 1, ss);
  if (upd->kind == PPX_UPDATE_ADAM) {
    E.adam_m = t2(upd->adam_m + off, ld, 1, ss);
    E.adam_v = t2(upd->adam_v + off, ld, 1, ss);
  }
  E.out = t2(upd->w_next ? (char*)upd->w_next + off * es : nullptr, ld, dt == PPX_FP32, ss);
  if (upd->grad) {
    E.flags |= ppx::EP_GRAD;
    E.aux = t2(upd->grad + off, ld, 1, ss);
  }
  E.bad = upd->bad;
}

static ppx_status wgrad_add(ppx_ctx* ctx, ppx_dtype dt, Builder& b, const ppx_wgrad_item& it) {
  const ppx_layer* L = it.layer;
  const ppx_update* upd = it.upd;
  const int32_t B = it.B;
  const bool update = upd && upd->kind != PPX_UPDATE_NONE;
  float* grad = it.grad;
  if (bad_layer(L) || B < 1 || !it.delta || !it.y_prev || (!grad && !update))
    return fail(ctx, PPX_E_CONFIG, "param grads: bad arguments");
  if (update && (!upd->master || !upd->hyper || (upd->kind == PPX_UPDATE_ADAM && (!upd->adam_m || !upd->adam_v))))
    return fail(ctx, PPX_E_CONFIG, "param grads: incomplete update");
  const bool need_r = L->p > 1 && (it.parts & PPX_GRAD_COMP);
  const bool need_g = L->p > 1 && (it.parts & PPX_GRAD_DEC);
  if ((need_r && !it.received) || (need_g && !it.phantoms))
    return fail(ctx, PPX_E_SEQUENCING, "param grads: phantom tape or received gradient missing");
  Flat f(L->s, L->k, L->p);
  const int kt = (int)cdiv(B, b.BK);
  if (it.parts & PPX_GRAD_LOCAL) {  // d local = delta^T y_prev   [s, s]
    Problem* pr = b.new_problem(L->s, L->s, 1, true);
    Opnd a{view2(it.delta, B, L->s, it.ld_d)};
    a.mn = 1;
    Opnd y{view2(it.y_prev, B, L->s, it.ld_y)};
    y.mn = 1;
    b.add_segment(pr, a, y, kt, kt);
    if (pr) {
      if (update) set_update(pr->epi, upd, dt, f.local, f.lds, 0);
      else pr->epi.out = t2(grad + f.local, f.lds, 1);
    }
  }
  if (need_r) {  // d compressor = r^T y_prev   [k, s]
    Problem* pr = b.new_problem(L->k, L->s, 1, true);
    Opnd r{view2(it.received, B, L->k, f.ldk)};
    r.mn = 1;
    Opnd y{view2(it.y_prev, B, L->s, it.ld_y)};
    y.mn = 1;
    b.add_segment(pr, r, y, kt, kt);
    if (pr) {
      if (update) set_update(pr->epi, upd, dt, f.comp, f.lds, 0);
      else pr->epi.out = t2(grad + f.comp, f.lds, 1);
    }
  } else if ((it.parts & PPX_GRAD_COMP) && grad) {  // p == 1: no peers, zero gradient
    cudaMemsetAsync(grad + f.comp, 0, sizeof(float) * L->k * f.lds, b.st);
  }
  if (need_g) {  // d decompressor_q = delta^T g_{src(q)}   [p-1][s, k]
    Problem* pd = b.new_problem(L->s, L->k, L->p - 1, true);
    const int H = it.phantom_halves == 2 ? 2 : 1;
    if (B % H) return fail(ctx, PPX_E_CONFIG, "param grads: batch not divisible into phantom halves");
    const int Bh = B / H;
    const int es = dt == PPX_FP32 ? 4 : 2;
    for (int h = 0; h < H; ++h) {   // the batch (K) splits into one segment per gathered half
      Opnd a{view2(elem(dt, it.delta, (int64_t)h * Bh * it.ld_d), Bh, L->s, it.ld_d)};
      a.mn = 1;
      Opnd g{view3((const char*)it.phantoms + (int64_t)h * L->p * Bh * f.ldk * es, L->p, Bh, L->k, f.ldk,
                   (int64_t)Bh * f.ldk)};
      g.mn = 1;
      g.slot_src = 2;
      g.slot_skip = L->rank;
      const int kth = (int)cdiv(Bh, b.BK);
      b.add_segment(pd, a, g, kth, kth);
    }
    if (pd) {
      if (update) set_update(pd->epi, upd, dt, f.dec, f.ldk, (int64_t)L->s * f.ldk);
      else pd->epi.out = t2(grad + f.dec, f.ldk, 1, (int64_t)L->s * f.ldk);
    }
  }
  return b.ok() ? PPX_OK : b.status;
}

static ppx_status wgrad_bias(ppx_ctx* ctx, ppx_dtype dt, const ppx_wgrad_item& it, cudaStream_t st) {
  if (!(it.parts & PPX_GRAD_BIAS) || !it.grad) return PPX_OK;
  Flat f(it.layer->s, it.layer->k, it.layer->p);
  ++ctx->launches;
  cudaError_t e = ppx::launch_colsum(dt == PPX_FP32, it.B, it.layer->s, it.delta, it.ld_d, it.grad + f.bias, 0, st);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "colsum: %s", cudaGetErrorString(e));
}

ppx_status ppx_param_grads(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, const void* delta,
                           int64_t ld_d, const void* y_prev, int64_t ld_y, const void* phantoms,
                           const void* received, float* grad, const ppx_update* upd, int32_t parts,
                           void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  ppx_wgrad_item it{L, parts, B, delta, ld_d, y_prev, ld_y, phantoms, received, grad, upd, 1};
  return ppx_wgrad(ctx, dt, 1, &it, stream);
}

ppx_status ppx_wgrad(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (nitems < 0 || (nitems > 0 && !items)) return fail(ctx, PPX_E_CONFIG, "ppx_wgrad: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < nitems; ++i) {
    ppx_status s = wgrad_add(ctx, dt, b, items[i]);
    if (s != PPX_OK) return s;
  }
  ppx_status s = b.launch();
  if (s != PPX_OK) return s;
  for (int i = 0; i < nitems; ++i) {
    s = wgrad_bias(ctx, dt, items[i], (cudaStream_t)stream);
    if (s != PPX_OK) return s;
  }
  return PPX_OK;
}

// Compressor gradients with the batch (K) split into nsplit chunks (phantom.py:247-249, the
// layer-0 compressor gradient: the step's exposed tail, k rows x s columns over K = B is a handful
// of long tiles): grouped launches of nitems x nsplit problems storing fp32 partial sums into
// partials[item][chunk][k, lds], then per item ONE elementwise pass that sums the chunks in order
// and applies the fused update (and/or stores the raw gradient).
ppx_status ppx_wgrad_splitk(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items, int32_t nsplit,
                            float* partials, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (nitems < 1 || nitems > 16 || !items || nsplit < 1 || nsplit > ppx::MAX_PROBS || !partials)
    return fail(ctx, PPX_E_CONFIG, "ppx_wgrad_splitk: bad arguments (1..16 items)");
  for (int i = 0; i < nitems; ++i) {
    const ppx_wgrad_item& it = items[i];
    const ppx_layer* L = it.layer;
    const bool update = it.upd && it.upd->kind != PPX_UPDATE_NONE;
    if (bad_layer(L) || it.parts != PPX_GRAD_COMP || L->p < 2 || !it.received || !it.y_prev || it.B < nsplit ||
        it.B % nsplit || (!it.grad && !update))
      return fail(ctx, PPX_E_CONFIG, "ppx_wgrad_splitk: compressor gradients (p > 1) with B %% nsplit == 0 only");
    if (update && (!it.upd->master || !it.upd->hyper ||
                   (it.upd->kind == PPX_UPDATE_ADAM && (!it.upd->adam_m || !it.upd->adam_v))))
      return fail(ctx, PPX_E_CONFIG, "ppx_wgrad_splitk: incomplete update");
  }
  const cudaStream_t st = (cudaStream_t)stream;
  int q = 0;
  const int total = nitems * nsplit;
  int kmax = 0;
  for (int i = 0; i < nitems; ++i) kmax = items[i].layer->k > kmax ? items[i].layer->k : kmax;
  while (q < total) {
    Builder b(ctx, dt, stream);
    // k <= 128 rows fit the 1-SM kernel's tile exactly: a 2-SM pair tile would leave its second
    // CTA's 128 rows empty, and 148 single SMs take the chunk tiles in one round
    if (kmax <= ppx::BM) b.want_pair = false;
    for (; q < total && b.P.nprobs < ppx::MAX_PROBS; ++q) {
      const ppx_wgrad_item& it = items[q / nsplit];
      const int c = q % nsplit;
      const ppx_layer* L = it.layer;
      Flat f(L->s, L->k, L->p);
      const int Bc = it.B / nsplit;
      Problem* pr = b.new_problem(L->k, L->s, 1, true);
      // the chunks as slots of one view per operand: every chunk problem shares its tensor maps
      Opnd r{view3(it.received, nsplit, Bc, L->k, f.ldk, (int64_t)Bc * f.ldk)};
      r.mn = 1;
      r.slot_base = c;
      Opnd y{view3(it.y_prev, nsplit, Bc, L->s, it.ld_y, (int64_t)Bc * it.ld_y)};
      y.mn = 1;
      y.slot_base = c;
      const int kt = (int)cdiv(Bc, b.BK);
      b.add_segment(pr, r, y, kt, kt);
      if (pr) pr->epi.out = t2(partials + (int64_t)q * L->k * f.lds, f.lds, 1);
    }
    ppx_status s = b.launch();
    if (s != PPX_OK) return s;
  }
  // one summing + update launch for all items (they share k, s, the update kind and hyper)
  const ppx_wgrad_item& i0 = items[0];
  const bool update = i0.upd && i0.upd->kind != PPX_UPDATE_NONE;
  const int mode = update ? (i0.upd->kind == PPX_UPDATE_ADAM ? 2 : 1) : 0;
  Flat f0(i0.layer->s, i0.layer->k, i0.layer->p);
  const int64_t n = (int64_t)i0.layer->k * f0.lds;
  const int es = dt == PPX_FP32 ? 4 : 2;
  ppx::SplitkItems si;
  memset(&si, 0, sizeof(si));
  for (int i = 0; i < nitems; ++i) {
    const ppx_wgrad_item& it = items[i];
    const ppx_update* u = it.upd;
    const bool upd_i = u && u->kind != PPX_UPDATE_NONE;
    if (upd_i != update || (update && (u->kind != i0.upd->kind || u->hyper != i0.upd->hyper || u->bad != i0.upd->bad)) ||
        it.layer->k != i0.layer->k || it.layer->s != i0.layer->s || it.layer->p != i0.layer->p)
      return fail(ctx, PPX_E_CONFIG, "ppx_wgrad_splitk: items must share the shapes and the update");
    if (update) {
      si.w[i] = u->master + f0.comp;
      si.m[i] = u->adam_m ? u->adam_m + f0.comp : nullptr;
      si.v[i] = u->adam_v ? u->adam_v + f0.comp : nullptr;
      si.copy[i] = u->w_next ? (char*)u->w_next + f0.comp * es : nullptr;
      si.g_out[i] = u->grad ? u->grad + f0.comp : nullptr;
      lo_invalidate(ctx, si.w[i], n * 4);
      if (si.copy[i]) lo_invalidate(ctx, si.copy[i], n * es);
    } else {
      si.g_out[i] = it.grad + f0.comp;
    }
  }
  ++ctx->launches;
  cudaError_t e = ppx::launch_splitk_update(mode, update ? i0.upd->hyper : nullptr, partials, nsplit, n, n, nitems, si,
                                            dt == PPX_FP32, update ? i0.upd->bad : nullptr, st);
  if (e != cudaSuccess) return fail(ctx, PPX_E_CUDA, "splitk update: %s", cudaGetErrorString(e));
  return PPX_OK;
}

static ppx_status add_backward(ppx_ctx* ctx, ppx_dtype dt, Builder& b, const ppx_rank_io& io, int32_t B,
                               ppx_act act_prev) {
  const ppx_layer* L = io.layer;
  if (bad_layer(L) || B < 1 || !io.x || !io.out || (act_prev == PPX_RELU && !io.mask && !io.bits))
    return fail(ctx, PPX_E_CONFIG, "backward_delta: bad arguments");
  if (L->p > 1 && !io.received) return fail(ctx, PPX_E_SEQUENCING, "backward_delta: received gradient missing");
  Flat f(L->s, L->k, L->p);
  Problem* pr = b.new_problem(B, L->s, 1, true);
  Opnd a{view2(io.x, B, L->s, io.ld_x)};
  Opnd w{view2(elem(dt, L->w, f.local), L->s, L->s, f.lds)};
  w.mn = 1;
  b.add_segment(pr, a, w, (int)cdiv(L->s, b.BK), (int)cdiv(L->s, b.BK));
  if (L->p > 1) {
    Opnd r{view2(io.received, B, L->k, f.ldk)};
    Opnd c{view2(elem(dt, L->w, f.comp), L->k, L->s, f.lds)};
    c.mn = 1;
    b.add_segment(pr, r, c, (int)cdiv(L->k, b.BK), (int)cdiv(L->k, b.BK));
  }
  if (!pr) return b.status;
  const int f32 = dt == PPX_FP32;
  pr->epi.out = t2(io.out, io.ld_out, f32);
  if (act_prev == PPX_RELU && io.bits) {
    if (f32 || L->s % 32 || io.ld_bits < L->s / 32)
      return fail(ctx, PPX_E_CONFIG, "backward_delta: bit masks need bf16 and s % 32 == 0");
    pr->epi.flags |= ppx::EP_MASK | ppx::EP_MASKBITS;
    pr->epi.mask = t2(io.bits, io.ld_bits, 0);
  } else if (act_prev == PPX_RELU) {
    pr->epi.flags |= ppx::EP_MASK;
    pr->epi.mask = t2(const_cast<void*>(io.mask), io.ld_m, f32);
  }
  if (io.colsum) {
    pr->epi.flags |= ppx::EP_COLSUM;
    pr->epi.colsum = io.colsum;
  }
  return b.ok() ? PPX_OK : b.status;
}

ppx_status ppx_backward_delta_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                ppx_act act_prev, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 1 || !io) return fail(ctx, PPX_E_CONFIG, "ppx_backward_delta_n: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < n; ++i) {
    ppx_status s = add_backward(ctx, dt, b, io[i], B, act_prev);
    if (s != PPX_OK) return s;
  }
  return b.launch();
}

// Weight gradients (+ fused optimizer) of `nitems` items and the error recurrence of the n ranks as
// ONE launch with a static LPT tile schedule: the long weight-gradient tiles and the short
// recurrence tiles share the rounds (one logical rank per GPU leaves either launch alone at ~1.4
// rounds of tiles).  Needs the reduced phantom gradient (r) of the layer already in place.
ppx_status ppx_backward_fused(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items, int32_t n,
                              const ppx_rank_io* io, int32_t B, ppx_act act_prev, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (nitems < 0 || (nitems > 0 && !items) || n < 0 || (n > 0 && !io))
    return fail(ctx, PPX_E_CONFIG, "ppx_backward_fused: bad arguments");
  Builder b(ctx, dt, stream);
  for (int i = 0; i < nitems; ++i) {
    ppx_status st = wgrad_add(ctx, dt, b, items[i]);
    if (st != PPX_OK) return st;
  }
  for (int i = 0; i < n; ++i) {
    ppx_status st = add_backward(ctx, dt, b, io[i], B, act_prev);
    if (st != PPX_OK) return st;
  }
  b.lpt = getenv("PPX_NO_LPT") == nullptr;
  ppx_status st = b.launch();
  if (st != PPX_OK) return st;
  for (int i = 0; i < nitems; ++i) {
    st = wgrad_bias(ctx, dt, items[i], (cudaStream_t)stream);
    if (st != PPX_OK) return st;
  }
  return PPX_OK;
}

// Error-compression problems (phantom.py:199-205) of the n local ranks io[] into `contrib` ([p]
// slots of [B, ldk]): one K-concatenated problem per slot i that has a contributor (segment j reads
// D_{i->j}); peer-owned slots are also copied to their owner's staging area over NVLink with the
// owner's arrival counter bumped (sc, as ppx_error_phantoms_scatter), or the slots accumulate
// into what `contrib` holds (accumulate: one GPU running its logical ranks one launch at a time).
static ppx_status add_error_problems(ppx_ctx* ctx, ppx_dtype dt, Builder& b, int32_t n, const ppx_rank_io* io,
                                     int32_t B, void* contrib, const ppx_scatter* sc, int accumulate, int prio) {
  const int p = io[0].layer->p, k = io[0].layer->k;
  const int step = error_pairs(dt, n, p, k) ? 2 : 1;
  for (int i = 0; i < p; i += step) {
    Problem* pr = error_slot_problem(b, dt, n, io, B, contrib, i, step, sc, accumulate);
    if (pr) b.prio[pr - b.P.probs] = prio;
    if (!b.ok()) return b.status;
  }
  (void)ctx;
  return PPX_OK;
}

// Error compression of layer l + the weight gradients that do not need r_l as ONE LPT-scheduled
// launch, the error-compression tiles first (their outputs are what the reduce-scatter moves, so
// with sc the NVLink scatter overlaps the weight-gradient tiles); the recurrence follows after
// the received error phantoms are reduced (ppx_reduce_received / the caller's reduce-scatter).
ppx_status ppx_backward_wgrad_errors(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items,
                                     int32_t n, const ppx_rank_io* io, int32_t B, void* contrib,
                                     const ppx_scatter* sc, int32_t accumulate, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (nitems < 0 || (nitems > 0 && !items) || n < 1 || !io || B < 1 || !contrib || dt != PPX_BF16 ||
      n > ppx::MAX_SEGS || (sc && (accumulate || !sc->stage || !sc->arrive || sc->rank < 0 || sc->rank >= sc->world)))
    return fail(ctx, PPX_E_CONFIG, "ppx_backward_wgrad_errors: bad arguments");
  const int p = io[0].layer->p, s = io[0].layer->s, k = io[0].layer->k;
  for (int j = 0; j < n; ++j) {
    const ppx_layer* L = io[j].layer;
    if (bad_layer(L) || !io[j].x || L->s != s || L->k != k || L->p != p || (j && L->rank <= io[j - 1].layer->rank))
      return fail(ctx, PPX_E_CONFIG, "ppx_backward_wgrad_errors: ranks must share (s, k, p) and ascend");
  }
  if (sc && (p % sc->world || p / sc->world != n))
    return fail(ctx, PPX_E_CONFIG, "ppx_backward_wgrad_errors: scatter needs all p / world local ranks");
  Builder b(ctx, dt, stream);
  if (p > 1) {
    ppx_status st = add_error_problems(ctx, dt, b, n, io, B, contrib, sc, accumulate, 1);
    if (st != PPX_OK) return st;
  }
  for (int i = 0; i < nitems; ++i) {
    ppx_status st = wgrad_add(ctx, dt, b, items[i]);
    if (st != PPX_OK) return st;
  }
  b.lpt = true;
  ppx_status st = b.launch();
  if (st != PPX_OK) return st;
  for (int i = 0; i < nitems; ++i) {
    st = wgrad_bias(ctx, dt, items[i], (cudaStream_t)stream);
    if (st != PPX_OK) return st;
  }
  return PPX_OK;
}

ppx_status ppx_backward_delta(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act_prev,
                              const void* delta, int64_t ld_d, const void* received, const void* mask_src,
                              int64_t ld_m, void* delta_prev, int64_t ld_dp, float* bias_grad_prev, void* stream) {
  ppx_rank_io io{};
  io.layer = L;
  io.x = delta;
  io.ld_x = ld_d;
  io.out = delta_prev;
  io.ld_out = ld_dp;
  io.mask = mask_src;
  io.ld_m = ld_m;
  io.received = received;
  io.colsum = bias_grad_prev;
  return ppx_backward_delta_n(ctx, dt, 1, &io, B, act_prev, stream);
}

ppx_status ppx_colsum(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, const void* x, int64_t ld, float* out,
                      int32_t accumulate, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (rows < 1 || cols < 1 || !x || !out) return fail(ctx, PPX_E_CONFIG, "ppx_colsum: bad arguments");
  lo_invalidate(ctx, out, (int64_t)cols * 4);
  ++ctx->launches;
  cudaError_t e = ppx::launch_colsum(dt == PPX_FP32, rows, cols, x, ld, out, accumulate, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "colsum: %s", cudaGetErrorString(e));
}

ppx_status ppx_optimizer_step(ppx_ctx* ctx, int32_t kind, const float* hyper, float* params, const float* grad,
                              float* adam_m, float* adam_v, int64_t n, ppx_dtype dt, void* w_copy, int* bad,
                              void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 0 || !hyper || (n > 0 && (!params || !grad)) ||
      (kind == PPX_UPDATE_ADAM && n > 0 && (!adam_m || !adam_v)) ||
      (kind != PPX_UPDATE_SGD && kind != PPX_UPDATE_ADAM))
    return fail(ctx, PPX_E_CONFIG, "ppx_optimizer_step: bad arguments");
  if (n == 0) return PPX_OK;
  lo_clear(ctx);
  ++ctx->launches;
  cudaError_t e = ppx::launch_optimizer(kind == PPX_UPDATE_ADAM, hyper, params, grad, adam_m, adam_v, n,
                                        dt == PPX_FP32, w_copy, bad, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "optimizer: %s", cudaGetErrorString(e));
}

ppx_status ppx_hyper_advance(ppx_ctx* ctx, float* hyper, int32_t* step, double beta1, double beta2, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (!hyper || !step) return fail(ctx, PPX_E_CONFIG, "ppx_hyper_advance: bad arguments");
  lo_invalidate(ctx, hyper, 6 * 4);
  lo_invalidate(ctx, step, 4);
  ++ctx->launches;
  cudaError_t e = ppx::launch_hyper_advance(hyper, step, beta1, beta2, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "hyper_advance: %s", cudaGetErrorString(e));
}

ppx_status ppx_gemm(ppx_ctx* ctx, ppx_dtype dt, int32_t M, int32_t N, int32_t K, const void* a, int64_t lda,
                    int32_t trans_a, const void* bm, int64_t ldb, int32_t trans_b, void* c, int64_t ldc,
                    ppx_dtype out_dt, const ppx_epilogue* epi, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (M < 1 || N < 1 || K < 1 || !a || !bm || !c) return fail(ctx, PPX_E_CONFIG, "ppx_gemm: bad arguments");
  Builder b(ctx, dt, stream);
  const bool b_mn = !trans_b;
  Problem* pr = b.new_problem(M, N, 1, b_mn);
  Opnd A{trans_a ? view2(a, K, M, lda) : view2(a, M, K, lda)};
  A.mn = trans_a ? 1 : 0;
  Opnd Bo{trans_b ? view2(bm, N, K, ldb) : view2(bm, K, N, ldb)};
  Bo.mn = b_mn ? 1 : 0;
  int kt = (int)cdiv(K, b.BK);
  b.add_segment(pr, A, Bo, kt, kt);
  if (pr) {
    const int f32 = out_dt == PPX_FP32;
    pr->epi.out = t2(c, ldc, f32);
    if (epi) {
      if (epi->bias) { pr->epi.flags |= ppx::EP_BIAS; pr->epi.bias = epi->bias; }
      if (epi->act == PPX_RELU) pr->epi.flags |= ppx::EP_RELU;
      if (epi->accumulate) pr->epi.flags |= ppx::EP_ACCUM;
      if (epi->mask) { pr->epi.flags |= ppx::EP_MASK; pr->epi.mask = t2(const_cast<void*>(epi->mask), epi->ld_mask, f32); }
      if (epi->colsum) { pr->epi.flags |= ppx::EP_COLSUM; pr->epi.colsum = epi->colsum; }
    }
  }
  return b.launch();
}

ppx_status ppx_gemm_update(ppx_ctx* ctx, ppx_dtype dt, int32_t M, int32_t N, int32_t K, const void* a, int64_t lda,
                           int32_t trans_a, const void* bm, int64_t ldb, int32_t trans_b, const ppx_update* upd,
                           int64_t ld_w, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (M < 1 || N < 1 || K < 1 || !a || !bm || !upd || upd->kind == PPX_UPDATE_NONE || !upd->master || !upd->hyper ||
      (upd->kind == PPX_UPDATE_ADAM && (!upd->adam_m || !upd->adam_v)))
    return fail(ctx, PPX_E_CONFIG, "ppx_gemm_update: bad arguments");
  Builder b(ctx, dt, stream);
  const bool b_mn = !trans_b;
  Problem* pr = b.new_problem(M, N, 1, b_mn);
  Opnd A{trans_a ? view2(a, K, M, lda) : view2(a, M, K, lda)};
  A.mn = trans_a ? 1 : 0;
  Opnd Bo{trans_b ? view2(bm, N, K, ldb) : view2(bm, K, N, ldb)};
  Bo.mn = b_mn ? 1 : 0;
  int kt = (int)cdiv(K, b.BK);
  b.add_segment(pr, A, Bo, kt, kt);
  if (pr) set_update(pr->epi, upd, dt, 0, ld_w, 0);
  return b.launch();
}

ppx_status ppx_tf32_scope(ppx_ctx* ctx, int32_t on, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  const cudaStream_t st = (cudaStream_t)stream;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
  if (on && !ctx->lo_pool.empty() && ctx->lo_done_valid && st != ctx->lo_stream && !capturing) {
    // the pooled buffers were last used on another stream: order this scope after that one
    // (a capture is preceded by a device synchronisation in the engine)
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->lo_done, 0));
  }
  lo_clear(ctx);
  if (!on && ctx->lo_scope && !capturing && ctx->lo_stream == st) {
    if (!ctx->lo_done) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->lo_done, cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventRecord(ctx->lo_done, st));
    ctx->lo_done_valid = true;
  }
  ctx->lo_scope = on != 0;
  ctx->lo_stream = st;
  return PPX_OK;
}

ppx_status ppx_zero(ppx_ctx* ctx, void* ptr, int64_t bytes, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (bytes < 0 || (bytes > 0 && !ptr)) return fail(ctx, PPX_E_CONFIG, "ppx_zero: bad arguments");
  if (bytes == 0) return PPX_OK;
  lo_invalidate(ctx, ptr, bytes);
  CUDA_TRY(ctx, cudaMemsetAsync(ptr, 0, (size_t)bytes, (cudaStream_t)stream));
  return PPX_OK;
}

ppx_status ppx_cast(ppx_ctx* ctx, ppx_dtype src_dt, const void* src, ppx_dtype dst_dt, void* dst, int64_t n,
                    void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (n < 0 || (n > 0 && (!src || !dst))) return fail(ctx, PPX_E_CONFIG, "ppx_cast: bad arguments");
  if (n == 0) return PPX_OK;
  lo_invalidate(ctx, dst, n * (dst_dt == PPX_FP32 ? 4 : 2));
  ++ctx->launches;
  cudaError_t e = ppx::launch_cast(src_dt == PPX_FP32, src, dst_dt == PPX_FP32, dst, n, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "cast: %s", cudaGetErrorString(e));
}

ppx_status ppx_bias_act(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, const void* x, int64_t ldx,
                        const float* bias, ppx_act act, void* y, int64_t ldy, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (rows < 1 || cols < 1 || !x || !y) return fail(ctx, PPX_E_CONFIG, "ppx_bias_act: bad arguments");
  lo_clear(ctx);
  ++ctx->launches;
  cudaError_t e = ppx::launch_bias_act(dt == PPX_FP32, rows, cols, x, ldx, bias, act == PPX_RELU, y, ldy,
                                       (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "bias_act: %s", cudaGetErrorString(e));
}

ppx_status ppx_relu_mask(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, void* x, int64_t ldx,
                         const void* mask_src, int64_t ldm, void* stream) {
  if (!ctx) return PPX_E_CONFIG;
  if (rows < 1 || cols < 1 || !x || !mask_src) return fail(ctx, PPX_E_CONFIG, "ppx_relu_mask: bad arguments");
  lo_clear(ctx);
  ++ctx->launches;
  cudaError_t e = ppx::launch_relu_mask(dt == PPX_FP32, rows, cols, x, ldx, mask_src, ldm, (cudaStream_t)stream);
  return e == cudaSuccess ? PPX_OK : fail(ctx, PPX_E_CUDA, "relu_mask: %s", cudaGetErrorString(e));
}

}  // extern "C"
