// Bandwidth-bound helper kernels of the phantom-parallel engine (everything that is not a
// tensor-core contraction).  All are grid-stride / 2D-tiled, vector-friendly and launched on the
// caller's stream.  References: phantom.py:169-182 (output delta), phantom.py:253 (bias grad),
// training.py:74-105 (SGD / Adam), core.py:64-98 (activations).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ppx {

struct GemmParams;
template <bool kTF32>
cudaError_t launch_gemm(const GemmParams& P, int grid, cudaStream_t st);
cudaError_t launch_gemm_pair(const GemmParams& P, int grid, cudaStream_t st);

__device__ __forceinline__ float ld_elem(const void* p, int64_t i, bool f32) {
  return f32 ? reinterpret_cast<const float*>(p)[i] : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ void st_elem(void* p, int64_t i, bool f32, float v) {
  if (f32) reinterpret_cast<float*>(p)[i] = v;
  else reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

inline int ew_grid(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

// ---- 3xTF32 operand split: hi = x with the low 13 mantissa bits cleared, lo = x - hi ----------
__global__ void split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(lo) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(hi) & 15) == 0) {
    const int64_t n4 = n / 4;
    for (int64_t i = t0; i < n4; i += stride) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
      float4 h, l;
      h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
      h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
      h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
      h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
      l.x = v.x - h.x;
      l.y = v.y - h.y;
      l.z = v.z - h.z;
      l.w = v.w - h.w;
      reinterpret_cast<float4*>(lo)[i] = l;
      if (hi) reinterpret_cast<float4*>(hi)[i] = h;
    }
    for (int64_t i = n4 * 4 + t0; i < n; i += stride) {
      const float v = x[i], h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      lo[i] = v - h;
      if (hi) hi[i] = h;
    }
    return;
  }
  for (int64_t i = t0; i < n; i += stride) {
    const float v = x[i], h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    lo[i] = v - h;
    if (hi) hi[i] = h;
  }
}
// FP32 tier operand split: lo = x - tf32(x) (and, when `hi` is given, hi = tf32(x) explicitly)
inline void launch_split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t st) {
  split_tf32_kernel<<<ew_grid((n + 3) / 4), 256, 0, st>>>(x, hi, lo, n);
}

// ---- output delta + half-squared loss (phantom.py:169-182, training.py:59-71, 196-199) --------
__global__ void output_delta_kernel(bool f32, int rows, int cols, bool relu, const void* y, int64_t ldy,
                                    const void* t, int64_t ldt, const void* pre, int64_t ldp, void* d, int64_t ldd,
                                    float scale, float loss_scale, float* loss) {
  float acc = 0.f;
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float diff = ld_elem(y, r * ldy + c, f32) - ld_elem(t, r * ldt + c, f32);
    acc += diff * diff;
    const float g = relu ? (ld_elem(pre, r * ldp + c, f32) > 0.f ? 1.f : 0.f) : 1.f;
    st_elem(d, r * ldd + c, f32, diff * g * scale);
  }
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && loss) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    atomicAdd(loss, s * loss_scale);
  }
}
inline cudaError_t launch_output_delta(bool f32, int rows, int cols, bool relu, const void* y, int64_t ldy,
                                       const void* t, int64_t ldt, const void* pre, int64_t ldp, void* d,
                                       int64_t ldd, float scale, float loss_scale, float* loss, cudaStream_t st) {
  output_delta_kernel<<<ew_grid((int64_t)rows * cols), 256, 0, st>>>(f32, rows, cols, relu, y, ldy, t, ldt, pre, ldp,
                                                                      d, ldd, scale, loss_scale, loss);
  return cudaGetLastError();
}

// ---- column sums (bias gradient, phantom.py:253): out[c] += sum_r x[r, c] --------------------
__global__ void colsum_kernel(bool f32, int rows, int cols, const void* x, int64_t ld, float* out) {
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ty = threadIdx.x >> 5;  // 8 row lanes
  float acc = 0.f;
  if (c < cols)
    for (int r = blockIdx.y * 8 + ty; r < rows; r += gridDim.y * 8) acc += ld_elem(x, (int64_t)r * ld + c, f32);
  __shared__ float red[8][33];
  red[ty][threadIdx.x & 31] = acc;
  __syncthreads();
  if (ty == 0 && c < cols) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += red[i][threadIdx.x & 31];
    atomicAdd(out + c, s);
  }
}
inline cudaError_t launch_colsum(bool f32, int rows, int cols, const void* x, int64_t ld, float* out, int accumulate,
                                 cudaStream_t st) {
  if (!accumulate) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float) * cols, st);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((cols + 31) / 32, 1);
  int ry = (rows + 255) / 256;
  int maxy = (148 * 8 + (int)grid.x - 1) / (int)grid.x;
  grid.y = ry < 1 ? 1 : (ry > maxy ? (maxy < 1 ? 1 : maxy) : ry);
  colsum_kernel<<<grid, 256, 0, st>>>(f32, rows, cols, x, ld, out);
  return cudaGetLastError();
}

// ---- SGD / Adam (training.py:74-82, 92-105) with non-finite detection -------------------------
// hyper = [lr, beta1, beta2, eps, 1 - beta1^t, 1 - beta2^t]
__device__ __forceinline__ float opt_apply(bool adam, const float* __restrict__ hyper, float gi, float wi,
                                           float* __restrict__ m, float* __restrict__ v, int64_t i) {
  const float lr = hyper[0];
  if (adam) {
    const float b1 = hyper[1], b2 = hyper[2], eps = hyper[3], bc1 = hyper[4], bc2 = hyper[5];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    return wi - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
  return wi - lr * gi;
}

__global__ void optimizer_kernel(bool adam, const float* __restrict__ hyper, float* __restrict__ w,
                                 const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v, int64_t n,
                                 bool copy_f32, void* copy, int* bad) {
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    nonfinite |= !isfinite(gi);
    const float wi = opt_apply(adam, hyper, gi, w[i], m, v, i);
    w[i] = wi;
    if (copy) st_elem(copy, i, copy_f32, wi);
  }
  if (bad && __any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}
inline cudaError_t launch_optimizer(bool adam, const float* hyper, float* w, const float* g, float* m, float* v,
                                    int64_t n, bool copy_f32, void* copy, int* bad, cudaStream_t st) {
  optimizer_kernel<<<ew_grid(n), 256, 0, st>>>(adam, hyper, w, g, m, v, n, copy_f32, copy, bad);
  return cudaGetLastError();
}

// Split-K weight gradient, second half, for up to 16 items (blockIdx.y): g = sum of `nparts` fp32
// partial sums (in chunk order, so deterministic), optionally stored to g_out, then SGD / Adam
// (mode 1 / 2; 0 = none) on w with the new weights also written to `copy` in the compute dtype
struct SplitkItems {
  float* w[16];
  float* m[16];
  float* v[16];
  void* copy[16];
  float* g_out[16];
};
__global__ void splitk_update_kernel(int mode, const float* __restrict__ hyper, const float* __restrict__ parts,
                                     int nparts, int64_t part_stride, int64_t n, const __grid_constant__ SplitkItems it,
                                     bool copy_f32, int* bad) {
  const int q = blockIdx.y;
  const float* pq = parts + (int64_t)q * nparts * part_stride;
  float* w = it.w[q];
  float* g_out = it.g_out[q];
  void* copy = it.copy[q];
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // eight loads in flight per thread, summed in chunk order
    float gi = 0.f;
    int c = 0;
    for (; c + 8 <= nparts; c += 8) {
      float a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldg(pq + (c + u) * part_stride + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) gi += a[u];
    }
    for (; c < nparts; ++c) gi += __ldg(pq + c * part_stride + i);
    nonfinite |= !isfinite(gi);
    if (g_out) g_out[i] = gi;
    if (mode) {
      const float wi = opt_apply(mode == 2, hyper, gi, w[i], it.m[q], it.v[q], i);
      w[i] = wi;
      if (copy) st_elem(copy, i, copy_f32, wi);
    }
  }
  if (bad && __any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}
inline cudaError_t launch_splitk_update(int mode, const float* hyper, const float* parts, int nparts,
                                        int64_t part_stride, int64_t n, int nitems, const SplitkItems& it,
                                        bool copy_f32, int* bad, cudaStream_t st) {
  int gx = ew_grid(n);
  const int cap = 148 * 16 / nitems;
  gx = gx > cap ? (cap < 1 ? 1 : cap) : gx;
  splitk_update_kernel<<<dim3(gx, nitems), 256, 0, st>>>(mode, hyper, parts, nparts, part_stride, n, it, copy_f32,
                                                         bad);
  return cudaGetLastError();
}

// Adam step counter advanced on the device (training.py:95: t += 1 before the bias corrections):
// hyper[4] = 1 - beta1^t, hyper[5] = 1 - beta2^t in double, so CUDA-graph replays never need a
// host write and steps may be issued back to back.
__global__ void hyper_advance_kernel(float* hyper, int* step, double beta1, double beta2) {
  const int t = *step + 1;
  *step = t;
  hyper[4] = (float)(1.0 - pow(beta1, (double)t));
  hyper[5] = (float)(1.0 - pow(beta2, (double)t));
}
inline cudaError_t launch_hyper_advance(float* hyper, int* step, double b1, double b2, cudaStream_t st) {
  hyper_advance_kernel<<<1, 1, 0, st>>>(hyper, step, b1, b2);
  return cudaGetLastError();
}

// ---- casts and activations ------------------------------------------------------------------
__global__ void cast_kernel(bool src_f32, const void* src, bool dst_f32, void* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    st_elem(dst, i, dst_f32, ld_elem(src, i, src_f32));
}
inline cudaError_t launch_cast(bool src_f32, const void* src, bool dst_f32, void* dst, int64_t n, cudaStream_t st) {
  cast_kernel<<<ew_grid(n), 256, 0, st>>>(src_f32, src, dst_f32, dst, n);
  return cudaGetLastError();
}

__global__ void bias_act_kernel(bool f32, int rows, int cols, const void* x, int64_t ldx, const float* bias,
                                bool relu, void* y, int64_t ldy) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    float v = ld_elem(x, r * ldx + c, f32) + (bias ? bias[c] : 0.f);
    if (relu) v = fmaxf(v, 0.f);
    st_elem(y, r * ldy + c, f32, v);
  }
}
inline cudaError_t launch_bias_act(bool f32, int rows, int cols, const void* x, int64_t ldx, const float* bias,
                                   bool relu, void* y, int64_t ldy, cudaStream_t st) {
  bias_act_kernel<<<ew_grid((int64_t)rows * cols), 256, 0, st>>>(f32, rows, cols, x, ldx, bias, relu, y, ldy);
  return cudaGetLastError();
}

__global__ void relu_mask_kernel(bool f32, int rows, int cols, void* x, int64_t ldx, const void* m, int64_t ldm) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    if (!(ld_elem(m, r * ldm + c, f32) > 0.f)) st_elem(x, r * ldx + c, f32, 0.f);
  }
}
inline cudaError_t launch_relu_mask(bool f32, int rows, int cols, void* x, int64_t ldx, const void* m, int64_t ldm,
                                    cudaStream_t st) {
  relu_mask_kernel<<<ew_grid((int64_t)rows * cols), 256, 0, st>>>(f32, rows, cols, x, ldx, m, ldm);
  return cudaGetLastError();
}



// Owner side of the NVLink reduce-scatter: wait until every source GPU's error-compression tiles
// for this GPU's slots have arrived (wrap-safe counter >= (epoch+1) * per_epoch), then
// out[j] = sum over source GPUs in ascending rank order of their contribution to local slot j
// (this GPU's own contribution read from `own`, the peers' from stage[g]), fp32 sum, one rounding.
struct ReduceArgs {
  const __nv_bfloat16* stage;   // [world][R][slot] bf16, indexed by source GPU
  const __nv_bfloat16* own;     // [R][slot] this GPU's contribution to its own slots
  __nv_bfloat16* out;           // [R][slot]
  long long slot_x8;            // R * slot elements / 8
  long long src_stride_x8;      // R * slot / 8 (stage stride between source GPUs)
  int world, me;
  const int* counter;
  int* epoch;
  int per_epoch;
  int* bad;
  unsigned int* done;
};
__global__ void reduce_received_kernel(ReduceArgs a) {
  if (threadIdx.x == 0) {
    const int target = (int)((unsigned)(*(volatile int*)a.epoch + 1) * (unsigned)a.per_epoch);
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int x;
    for (;;) {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(x) : "l"(a.counter) : "memory");
      if ((int)((unsigned)x - (unsigned)target) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {
        if (a.bad) atomicOr(a.bad, 2);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.slot_x8; i += stride) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int g = 0; g < a.world; ++g) {
      const uint4 q = g == a.me ? reinterpret_cast<const uint4*>(a.own)[i]
                                : reinterpret_cast<const uint4*>(a.stage)[g * a.src_stride_x8 + i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    }
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    reinterpret_cast<uint4*>(a.out)[i] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      *a.done = 0u;
      atomicAdd(a.epoch, 1);
    }
  }
}
inline cudaError_t launch_reduce_received(const ReduceArgs& a, cudaStream_t st) {
  long long blocks = (a.slot_x8 + 255) / 256;
  if (blocks > 148) blocks = 148;   // all resident: every block reads the epoch before the last bumps it
  if (blocks < 1) blocks = 1;
  reduce_received_kernel<<<(int)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ppx
