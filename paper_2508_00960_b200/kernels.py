"""Torch-facing wrappers over the C ABI: tensor -> (pointer, leading dim, dtype, stream).

Every function here launches sm_100a code from libppx.so on the current CUDA stream; they raise
ConfigurationError for non-CUDA or wrongly laid-out tensors instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ConfigurationError

_DT = {torch.bfloat16: _lib.PPX_BF16, torch.float32: _lib.PPX_FP32}


def ppx_dtype(t: torch.dtype) -> int:
    try:
        return _DT[t]
    except KeyError:
        raise ConfigurationError(f"unsupported dtype {t}; use bfloat16 or float32") from None


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ConfigurationError("tensor must live on a CUDA device (no CPU fallback)")
    return t.data_ptr()


def ld(t: torch.Tensor) -> int:
    """Leading dimension (elements) of a row-major 2-d view."""
    if t.dim() != 2 or t.stride(1) != 1:
        raise ConfigurationError(f"expected a row-major 2-d tensor, got shape {tuple(t.shape)} "
                                 f"strides {t.stride()}")
    return t.stride(0)


def ctx_for(t: torch.Tensor) -> _lib.Context:
    return _lib.default_context(t.device.index or 0)


def gemm(a: torch.Tensor, b: torch.Tensor, transpose_a: bool = False, transpose_b: bool = False,
         out_dtype: torch.dtype | None = None, *, bias: torch.Tensor | None = None,
         relu: bool = False, out: torch.Tensor | None = None, accumulate: bool = False,
         mask: torch.Tensor | None = None, colsum: torch.Tensor | None = None,
         ctx: _lib.Context | None = None) -> torch.Tensor:
    """op(a) @ op(b) on the tensor cores (reference core.py:39-61 semantics).

    a: [M, K] (or [K, M] with transpose_a); b: [K, N] (or [N, K] with transpose_b).
    bf16 inputs run tcgen05 kind::f16; fp32 inputs run 3xTF32 on kind::tf32.
    """
    if a.dtype != b.dtype:
        raise ConfigurationError("gemm operands must share a dtype")
    dt = ppx_dtype(a.dtype)
    M, K = (a.shape[1], a.shape[0]) if transpose_a else (a.shape[0], a.shape[1])
    Kb, N = (b.shape[1], b.shape[0]) if transpose_b else (b.shape[0], b.shape[1])
    if K != Kb:
        raise ConfigurationError(f"gemm dimension mismatch: ({M}x{K}) x ({Kb}x{N})")
    out_dtype = out_dtype or (out.dtype if out is not None else a.dtype)
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=a.device)
    epi = None
    if bias is not None or relu or accumulate or mask is not None or colsum is not None:
        epi = _lib.Epilogue(_lib.PPX_RELU if relu else _lib.PPX_IDENTITY, ptr(bias), int(accumulate),
                            ptr(mask), ld(mask) if mask is not None else 0, ptr(colsum))
    ctx = ctx or ctx_for(a)
    ctx.call("ppx_gemm", dt, M, N, K, ptr(a), ld(a), int(transpose_a), ptr(b), ld(b),
             int(transpose_b), ptr(out), ld(out), ppx_dtype(out_dtype),
             ctypes.byref(epi) if epi is not None else None, stream_handle())
    return out
