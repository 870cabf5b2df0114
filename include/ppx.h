/* ppx.h — C ABI of libppx.so, the B200 (sm_100a) phantom-parallel FFN engine.
 *
 * Drop-in boundary for the hot path of arXiv 2508.00960's reference simulator `phantomsim`
 * (/root/reference/pkg/src/phantomsim).  The reference is pure Python/numpy; its "FFI" for this
 * path is the Python function surface exported by phantomsim/__init__.py:5-33.  Every entry point
 * below replaces one of those functions (or the device half of one), cited per declaration; the
 * Python package paper_2508_00960_b200 binds them with ctypes (INTEGRATION.md shows the stub a
 * phantomsim maintainer would add).
 *
 * Conventions
 *  - All matrices are row-major on the device with an explicit leading dimension in elements
 *    (a multiple of 8).  The reference stores (features x batch) with batch as columns
 *    (core.py:3-4); this ABI stores (batch x features), i.e. the transpose, so activations are
 *    [B, s] and weights keep the reference's (out x in) orientation.
 *  - dtype PPX_BF16: bf16 operands, fp32 accumulation (tcgen05 kind::f16).
 *    dtype PPX_FP32: fp32 operands through 3xTF32 on tcgen05 kind::tf32 (hi*hi + hi*lo + lo*hi).
 *  - Calls are asynchronous on `stream` (a cudaStream_t); the caller owns every buffer.
 *    A ctx is not re-entrant; collectives must be issued in the same order on every GPU
 *    (the Communicator contract, collectives.py:88-94).
 *  - Status codes map onto phantomsim.errors (errors.py:4-29):
 *    PPX_E_CONFIG -> ConfigurationError, PPX_E_PROTOCOL -> ProtocolError,
 *    PPX_E_SEQUENCING -> SequencingError, PPX_E_NONFINITE -> TrainingError.
 *
 * Per-(rank, layer) parameter block ("flat layout").  One contiguous buffer in the PSHARD01
 * record order of checkpoint.py:57-64 (local, compressor, decompressors ascending source rank
 * with self skipped, bias), with lds = round8(s), ldk = round8(k):
 *    local        [s, lds]            at 0
 *    compressor   [k, lds]            at s*lds
 *    decompressor [p-1][s, ldk]       at (s+k)*lds          (block q <-> source rank q + (q >= rank))
 *    bias         [s]                 at (s+k)*lds + (p-1)*s*ldk
 *    total        ppx_layer_elems(s, k, p)
 * When s and k are multiples of 8 this is byte-for-byte the PSHARD01 record (in the element
 * type of the buffer).  Gradients, fp32 master weights and Adam moments use the same layout.
 *
 * Phantom buffers ("slots"): [p][B, ldk] with slot stride B*ldk; slot i holds rank i's k-wide
 * block (collectives.py:337-339 all-gather order; phantom.py:155 dict view).
 */
#ifndef PPX_H_
#define PPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPX_ABI_VERSION 1

typedef struct ppx_ctx ppx_ctx;

typedef enum {
  PPX_OK = 0,
  PPX_E_CONFIG = 1,
  PPX_E_PROTOCOL = 2,
  PPX_E_SEQUENCING = 3,
  PPX_E_NONFINITE = 4,
  PPX_E_CUDA = 5
} ppx_status;

typedef enum { PPX_BF16 = 0, PPX_FP32 = 1 } ppx_dtype;
typedef enum { PPX_RELU = 0, PPX_IDENTITY = 1 } ppx_act; /* core.py:64-82 Activation */

typedef enum { PPX_UPDATE_NONE = 0, PPX_UPDATE_SGD = 1, PPX_UPDATE_ADAM = 2 } ppx_update_kind;

/* One logical rank's shard of one layer (phantom.py:23-54 PhantomLayer). */
typedef struct {
  int32_t s, k, p, rank;
  const void* w;        /* flat parameter block in the call's dtype (what the GEMMs read) */
  const float* master;  /* flat fp32 block (may equal w for FP32) */
  const float* bias;    /* [s] fp32 bias; NULL = the bias slot of `master` */
} ppx_layer;

/* parts of a layer's gradient (ppx_param_grads / ppx_wgrad) */
enum { PPX_GRAD_LOCAL = 1, PPX_GRAD_COMP = 2, PPX_GRAD_DEC = 4, PPX_GRAD_BIAS = 8, PPX_GRAD_ALL = 15 };

/* Optimizer fused into the weight-gradient epilogue (training.py:74-105). */
typedef struct {
  int32_t kind;          /* ppx_update_kind */
  const float* hyper;    /* device: [lr, beta1, beta2, eps, 1-beta1^t, 1-beta2^t] */
  float* master;         /* flat fp32 master, updated in place */
  void* w_next;          /* flat copy in the compute dtype written from the new master (NULL: none) */
  float* adam_m;         /* flat fp32 first moment (Adam) */
  float* adam_v;         /* flat fp32 second moment (Adam) */
  float* grad;           /* optional flat fp32 raw-gradient output (NULL: not stored) */
  int* bad;              /* device flag set to 1 on a non-finite gradient (NULL: unchecked) */
} ppx_update;

/* Generic epilogue for ppx_gemm (the Megatron TP comparison pipeline reuses it). */
typedef struct {
  int32_t act;           /* ppx_act applied after bias */
  const float* bias;     /* [N] or NULL */
  int32_t accumulate;    /* C += result */
  const void* mask;      /* multiply by (mask[m, n] > 0), same dtype as C, or NULL */
  int64_t ld_mask;
  float* colsum;         /* += column sums of the stored result, or NULL */
} ppx_epilogue;

/* ---- context / communicator (collectives.py:87-194 Communicator -> NCCL over NVLink) ---- */
int ppx_abi_version(void);
/* debugging: the calling thread's pending CUDA runtime error (cudaPeekAtLastError), 0 = none */
int32_t ppx_peek_error(void);
int64_t ppx_layer_elems(int32_t s, int32_t k, int32_t p);
ppx_status ppx_get_unique_id(uint8_t uid[128]);
/* world GPUs, this process drives GPU `rank` on CUDA device `device`; uid from rank 0
   (ignored when world == 1). */
ppx_status ppx_create(int32_t world, int32_t rank, int32_t device, const uint8_t* uid, ppx_ctx** out);
ppx_status ppx_destroy(ppx_ctx* ctx);
const char* ppx_last_error(const ppx_ctx* ctx);
int32_t ppx_num_sms(const ppx_ctx* ctx);
/* Kernels this context has enqueued so far (GEMMs, TF32 splits, elementwise helpers; not NCCL,
   not memsets): the engine's per-step launch count (bench.py `gpu_launches`). */
int64_t ppx_kernel_launches(const ppx_ctx* ctx);
/* GEMM launches issued while this is non-zero leave `n` SMs free, so a collective running on
   another stream (NCCL needs SMs of its own) can progress under the GEMM. */
ppx_status ppx_set_reserved_sms(ppx_ctx* ctx, int32_t n);
/* Pre-allocate the FP32-tier split workspace (needed before CUDA-graph capture of FP32 calls). */
ppx_status ppx_reserve_workspace(ppx_ctx* ctx, int64_t bytes);
/* FP32 tier (3xTF32): between on = 1 and on = 0, the low part (x - tf32(x)) of every GEMM operand
   read on `stream` is split once and reused by later calls until a ppx call writes an
   overlapping range.  The caller guarantees that nothing but ppx calls writes those operands
   inside the scope (the engine brackets one training / inference step).  A scope on another
   stream than the previous one waits for it (event) before reusing the pooled buffers, except
   under stream capture (the engine synchronises the device before capturing).  No kernel
   launch.  Engine-internal: the reference splits nothing (numpy float64). */
ppx_status ppx_tf32_scope(ppx_ctx* ctx, int32_t on, void* stream);

/* ---- phantom-parallel layer ops -------------------------------------------------------- */

/* phantom.py:153 — own phantom block g = C . y_prev, written to phantoms slot `rank`. */
ppx_status ppx_compress(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B,
                        const void* y_prev, int64_t ld_y, void* phantoms, void* stream);

/* collectives.py:115-120 / 337-339 — in-place all-gather of the phantom slots.  This GPU owns
   `local_ranks` consecutive logical ranks starting at rank*local_ranks; slot_elems = B*ldk. */
ppx_status ppx_all_gather(ppx_ctx* ctx, ppx_dtype dt, void* phantoms, int64_t slot_elems,
                          int32_t local_ranks, void* stream);

/* phantom.py:152-163 — y = act(L.y_prev + sum_{i != rank asc} D_i.g_i + b), ONE K-concatenated
   tcgen05 contraction over [y_prev | g_peers]; optional pre-activation output. */
ppx_status ppx_forward_update(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act,
                              const void* y_prev, int64_t ld_y, const void* phantoms,
                              void* y_out, int64_t ld_out, void* preact, int64_t ld_pre, void* stream);

/* phantom.py:152-182 + training.py:59-71,195-199 — the output layer's update fused with the
   output delta, the half-squared loss partial and the output bias gradient:
     y = act(pre); delta = (y - t) * act'(pre) * delta_scale; *loss += loss_scale * sum (y-t)^2;
     bias_grad += sum_batch delta (if non-NULL). */
ppx_status ppx_forward_output(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act,
                              const void* y_prev, int64_t ld_y, const void* phantoms,
                              void* y_out, int64_t ld_out, const void* target, int64_t ld_t,
                              void* delta, int64_t ld_d, float delta_scale, float loss_scale,
                              float* loss, float* bias_grad, void* stream);

/* ---- grouped (multi-rank) launches: the logical ranks one GPU owns share ONE kernel launch,
   so n small per-rank grids become one grid with n times the tiles (no wave-quantisation tail
   per rank).  Each entry names one rank's operands; unused fields are NULL / 0. ------------- */
typedef struct {
  const ppx_layer* layer;
  const void* x;       int64_t ld_x;    /* y_prev (compress / forward) or delta (backward) */
  void* out;           int64_t ld_out;  /* y (forward) or delta_prev (backward) */
  void* aux;           int64_t ld_aux;  /* forward: pre-activation (NULL: none); output layer: delta */
  const void* target;  int64_t ld_t;    /* output layer: target */
  const void* mask;    int64_t ld_m;    /* backward: ReLU' source (pre_prev or y_prev) */
  const void* received;                 /* backward: [B, ldk] reduced phantom gradient */
  float* colsum;                        /* output layer / backward: += batch sums of the delta */
  void* bits;          int64_t ld_bits; /* optional, bf16 2-SM launches, s % 32 == 0: forward — also
                                           store ReLU'(pre) as a bit mask (bit i of uint32 word
                                           [row, col / 32] = y > 0, ld_bits words per row);
                                           backward — read the ReLU' mask from such bits instead of
                                           `mask` (1/16 of the bytes) */
} ppx_rank_io;

/* n x ppx_compress in one launch */
ppx_status ppx_compress_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                          void* phantoms, void* stream);
/* n x ppx_forward_update (output_layer = 0) or n x ppx_forward_output (output_layer = 1; io.out
   may then be NULL: the training step needs only the delta, the loss and the bias gradient) */
ppx_status ppx_forward_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B, ppx_act act,
                         const void* phantoms, int32_t output_layer, float delta_scale, float loss_scale,
                         float* loss, void* stream);
/* n x ppx_backward_delta */
ppx_status ppx_backward_delta_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                ppx_act act_prev, void* stream);

/* ---- NVLink peer memory (IPC regions every GPU maps): the fused forward's in-kernel phantom
   all-gather (collectives.py:115-120, 337-339) and the NVLink reduce-scatter store straight into
   them.  Regions come from ppx_peer_alloc (cudaMalloc + IPC handle, zero-filled, freed by
   ppx_destroy); the 64-byte handles are exchanged by the caller (any channel) and mapped with
   ppx_peer_open (closed by ppx_destroy). -------------------------------------------------------- */
ppx_status ppx_peer_alloc(ppx_ctx* ctx, int64_t bytes, void** ptr, uint8_t handle[64]);
ppx_status ppx_peer_open(ppx_ctx* ctx, const uint8_t handle[64], void** peer_ptr);
/* Fused compression + phantom all-gather + forward of one layer for the n local ranks, ONE
   launch of the 2-SM kernel (bf16): the compression tiles store their phantoms into `phantoms`
   and into every peer's copy (NVLink), then add 1 to every arrive[i] (own counter first); the
   forward tiles (io as for ppx_forward_n) compute the local block, wait in-kernel until
   *wait_counter reached this launch's epoch target (all GPUs' compression tiles), then add the
   decompressed phantoms.  *epoch (per layer, local) is bumped by the launch itself.  Counters
   start at 0 on every GPU; every GPU must issue the same fused launches in the same order. */
typedef struct {
  int32_t n_peers;
  void* const* peer_phantoms;    /* [n_peers] peer mappings of `phantoms` (same layout) */
  int32_t* const* arrive;        /* [n_peers + 1] arrival counters of this layer: own, then peers' */
  const int32_t* wait_counter;   /* this GPU's arrival counter of the layer (== arrive[0]) */
  int32_t* epoch;                /* this GPU's launch counter of the layer */
  int32_t* bad;                  /* optional: |= 2 if a wait gave up after ~20 s (lost peer) */
} ppx_exchange;
ppx_status ppx_forward_fused(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B, ppx_act act,
                             void* phantoms, int32_t output_layer, float delta_scale, float loss_scale,
                             float* loss, const ppx_exchange* ex, void* stream);
/* The phantom reduce-scatter over NVLink (collectives.py:122-127, 345-357) without NCCL.
   Sender: ppx_error_phantoms_scatter computes every slot i = sum_{local j != i} delta_j . D_{i->j}
   (one launch, R = n = p / world local ranks); slots owned by this GPU stay in `contrib`, every
   other slot is also copied from the epilogue into its owner g's staging area
   stage[g] + (rank * R + i - g * R) * slot bytes, adding rows * cols / 8 per CTA part to
   *arrive[g].  Receiver: ppx_reduce_received waits (in the kernel) until its counter reached
   (epoch + 1) * (world - 1) * R * slot / 8, then out[j] = sum over source GPUs in ascending rank
   order (its own contribution from `own`), and bumps *epoch.  bf16 tier. */
typedef struct {
  int32_t world, rank;
  void* const* stage;       /* [world] each GPU's staging area of this layer ([world][R][B, ldk]) */
  int32_t* const* arrive;   /* [world] each GPU's arrival counter of this layer */
} ppx_scatter;
ppx_status ppx_error_phantoms_scatter(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                      void* contrib, const ppx_scatter* sc, void* stream);
ppx_status ppx_reduce_received(ppx_ctx* ctx, ppx_dtype dt, int32_t R, int64_t slot_elems, int32_t world,
                               int32_t rank, const void* stage, const void* own, void* out,
                               const int32_t* counter, int32_t* epoch, int32_t* bad, void* stream);
/* phantom.py:169-182 (+ training.py:66-69 scaling) — standalone output delta and loss partial.
   `pre` is the pre-activation (or the layer output: ReLU'(pre) == (y > 0)). */
ppx_status ppx_output_delta(ppx_ctx* ctx, ppx_dtype dt, int32_t B, int32_t s, ppx_act act,
                            const void* y_out, int64_t ld_y, const void* target, int64_t ld_t,
                            const void* pre, int64_t ld_p, void* delta, int64_t ld_d,
                            float delta_scale, float loss_scale, float* loss, void* stream);

/* phantom.py:199-205 — slot i (i != rank) of contrib = D_i^T . delta, i.e. [B, k] = delta . D_i.
   accumulate != 0 adds into contrib (several logical ranks on one GPU sum their slots in
   ascending rank order before the cross-GPU reduce-scatter). The own slot is not written. */
ppx_status ppx_error_phantoms(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B,
                              const void* delta, int64_t ld_d, void* contrib, int32_t accumulate,
                              void* stream);
/* phantom.py:199-205 for the n logical ranks one GPU owns (io[j].layer ascending, io[j].x =
   delta_j): slot i of contrib = sum_{j != i} delta_j . D_{i->j}, summed in the fp32 accumulator
   in ascending rank order, every slot with at least one contributor OVERWRITTEN (no zeroing
   pass, no accumulate launches); slots without a contributor are left untouched. */
ppx_status ppx_error_phantoms_n(ppx_ctx* ctx, ppx_dtype dt, int32_t n, const ppx_rank_io* io, int32_t B,
                                void* contrib, void* stream);

/* collectives.py:122-127 / 345-357 — in-place reduce-scatter of the contribution slots: after
   it, slot j of `contrib` (for this GPU's local ranks) is the sum over all GPUs. */
ppx_status ppx_reduce_scatter(ppx_ctx* ctx, ppx_dtype dt, void* contrib, int64_t slot_elems,
                              int32_t local_ranks, void* stream);

/* out-of-place reduce-scatter: recv [local_ranks, slot] = this GPU's slots of the sum over GPUs of
   contrib [p, slot] (collectives.py:122-127, 345-357); contrib is not modified, so slots no
   local rank writes (the own slot when one logical rank per GPU) stay zero across steps. */
ppx_status ppx_reduce_scatter_to(ppx_ctx* ctx, ppx_dtype dt, const void* contrib, void* recv,
                                 int64_t slot_elems, int32_t local_ranks, void* stream);

/* collectives.py:138-142 — elementwise fp32 sum over GPUs, in place (the scalar loss,
   training.py:70). */
ppx_status ppx_all_reduce_f32(ppx_ctx* ctx, float* buf, int64_t count, void* stream);
/* same, in the compute dtype (Megatron TP all-reduce of activations / input gradients) */
ppx_status ppx_all_reduce(ppx_ctx* ctx, ppx_dtype dt, void* buf, int64_t count, void* stream);

/* phantom.py:239-267 — parameter gradients of one layer (fp32, flat layout `grad`):
     local = delta^T y_prev, compressor = r^T y_prev, decompressor_i = delta^T g_i,
     bias = sum_batch delta.   received r is [B, ldk] (slot `rank` of the reduced buffer).
   `parts` (PPX_GRAD_*) selects which gradients are formed.  With upd != NULL and upd->kind !=
   NONE the optimizer is applied in the same epilogue (the bias part is never fused: use
   ppx_optimizer_step on the bias gradient); grad may then be NULL. */
ppx_status ppx_param_grads(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B,
                           const void* delta, int64_t ld_d, const void* y_prev, int64_t ld_y,
                           const void* phantoms, const void* received, float* grad,
                           const ppx_update* upd, int32_t parts, void* stream);

/* Several layers' / ranks' weight gradients in ONE grouped tcgen05 launch (up to 8 problems):
   the engine overlaps the reduce-scatter of layer l with {d local_l, d decompressor_l,
   d compressor_{l+1}} this way. */
typedef struct {
  const ppx_layer* layer;
  int32_t parts;
  int32_t B;
  const void* delta;
  int64_t ld_d;
  const void* y_prev;
  int64_t ld_y;
  const void* phantoms;
  const void* received;
  float* grad;
  const ppx_update* upd;
  int32_t phantom_halves;   /* 0/1: phantoms is [p][B, ldk]; 2: two batch halves [2][p][B/2, ldk]
                               (the engine all-gathers each half separately to overlap it) */
} ppx_wgrad_item;
ppx_status ppx_wgrad(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items, void* stream);
/* phantom.py:247-249 — compressor gradients only (parts == PPX_GRAD_COMP, p > 1) with the batch
   (K) split into nsplit chunks: grouped launches of nitems x nsplit problems store fp32 partial
   sums in partials[item][chunk][k, lds] (caller's buffer, nitems * nsplit * k * lds floats, padding
   columns zero), then ONE elementwise launch sums each item's chunks in chunk order
   (deterministic) and applies upd (SGD / Adam, w_next copy, upd->grad) or stores the raw gradient
   to grad.  1..16 items sharing (s, k, p) and the update kind / hyper / bad flag.  The
   engine uses it for the layer-0 compressor gradient: k x s over K = B is only a few long tiles,
   the step's exposed tail. */
ppx_status ppx_wgrad_splitk(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items,
                            int32_t nsplit, float* partials, void* stream);

/* phantom.py:199-207 + 239-267 in ONE LPT-scheduled launch of the 2-SM kernel (bf16): the error
   compression of the n local ranks io[] (as ppx_error_phantoms_n, into contrib [p][B, ldk]; with
   sc the peer-owned slots are also stored into their owner's staging area over NVLink and counted,
   as ppx_error_phantoms_scatter; with accumulate the slots add to contrib instead) scheduled
   FIRST on every cluster, followed by the weight-gradient requests items[] (as ppx_wgrad).  The
   engine uses it when a GPU owns one or two logical ranks: the reduce-scatter then overlaps the
   weight gradients, and the recurrence (ppx_backward_delta_n) follows ppx_reduce_received. */
ppx_status ppx_backward_wgrad_errors(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items,
                                     int32_t n, const ppx_rank_io* io, int32_t B, void* contrib,
                                     const ppx_scatter* sc, int32_t accumulate, void* stream);
/* phantom.py:210-267 as one launch: the weight gradients (+ fused update) of `nitems` items and the
   error recurrence of the n ranks (io as for ppx_backward_delta_n), tiles scheduled longest-first
   over the clusters.  The layer's reduced phantom gradient must already be in place. */
ppx_status ppx_backward_fused(ppx_ctx* ctx, ppx_dtype dt, int32_t nitems, const ppx_wgrad_item* items, int32_t n,
                              const ppx_rank_io* io, int32_t B, ppx_act act_prev, void* stream);

/* phantom.py:210-236 — delta_prev = (local^T delta + compressor^T r) * act'(pre_prev): ONE
   K-concatenated contraction [delta | r] . [L ; C]; `mask_src` is pre_prev or y_prev (only its
   sign is read; NULL for IDENTITY).  bias_grad_prev += sum_batch delta_prev if non-NULL. */
ppx_status ppx_backward_delta(ppx_ctx* ctx, ppx_dtype dt, const ppx_layer* L, int32_t B, ppx_act act_prev,
                              const void* delta, int64_t ld_d, const void* received,
                              const void* mask_src, int64_t ld_m, void* delta_prev, int64_t ld_dp,
                              float* bias_grad_prev, void* stream);

/* phantom.py:253 — bias gradient alone: out[j] (+)= sum_b x[b, j]. */
ppx_status ppx_colsum(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, const void* x, int64_t ld,
                      float* out, int32_t accumulate, void* stream);

/* training.py:74-82 / 92-105 — elementwise SGD / Adam over one fp32 array (params -= ...),
   non-finite gradients flag *bad.  w_copy (optional) receives the new params in `dt`. */
ppx_status ppx_optimizer_step(ppx_ctx* ctx, int32_t kind, const float* hyper, float* params,
                              const float* grad, float* adam_m, float* adam_v, int64_t n,
                              ppx_dtype dt, void* w_copy, int* bad, void* stream);

/* training.py:92-105 (t incremented per step, training.py:297-300) — advances the device step
   counter *step and writes the Adam bias corrections hyper[4] = 1 - beta1^t, hyper[5] = 1 - beta2^t
   on `stream`.  hyper = [lr, beta1, beta2, eps, 1 - beta1^t, 1 - beta2^t] (fp32, device).  The
   engine issues it first in every step, so graph replays and back-to-back steps need no host
   write. */
ppx_status ppx_hyper_advance(ppx_ctx* ctx, float* hyper, int32_t* step, double beta1, double beta2,
                             void* stream);

/* core.py:39-61 gemm: C[M,N] = op(a) . op(b), op(a) = a [M,K] or a^T (a stored [K,M]),
   op(b) = b [K,N] or b^T (b stored [N,K]).  out_dt selects C's element type. */
ppx_status ppx_gemm(ppx_ctx* ctx, ppx_dtype dt, int32_t M, int32_t N, int32_t K,
                    const void* a, int64_t lda, int32_t trans_a, const void* b, int64_t ldb,
                    int32_t trans_b, void* c, int64_t ldc, ppx_dtype out_dt,
                    const ppx_epilogue* epi, void* stream);

/* Weight-gradient GEMM with the optimizer fused into its epilogue (the Megatron TP comparison
   pipeline): G = op(a) . op(b) [M, N] is applied to the fp32 master (leading dim ld_w) by
   SGD / Adam and the new weights are written to upd->w_next in `dt`. */
ppx_status ppx_gemm_update(ppx_ctx* ctx, ppx_dtype dt, int32_t M, int32_t N, int32_t K,
                           const void* a, int64_t lda, int32_t trans_a, const void* b, int64_t ldb,
                           int32_t trans_b, const ppx_update* upd, int64_t ld_w, void* stream);

/* elementwise helpers used by the host engine */
ppx_status ppx_zero(ppx_ctx* ctx, void* ptr, int64_t bytes, void* stream); /* cudaMemsetAsync */
ppx_status ppx_cast(ppx_ctx* ctx, ppx_dtype src_dt, const void* src, ppx_dtype dst_dt, void* dst,
                    int64_t n, void* stream);
/* y = act(x + bias) over [rows, cols] (TP row-parallel epilogue after the all-reduce);
   y may alias x */
ppx_status ppx_bias_act(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, const void* x,
                        int64_t ldx, const float* bias, ppx_act act, void* y, int64_t ldy, void* stream);
/* out[i] = mask ? (x[i] if mask_src[i] > 0 else 0) : x  — ReLU' applied in place */
ppx_status ppx_relu_mask(ppx_ctx* ctx, ppx_dtype dt, int32_t rows, int32_t cols, void* x, int64_t ldx,
                         const void* mask_src, int64_t ldm, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PPX_H_ */
