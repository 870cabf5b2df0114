"""Numerics core mirroring phantomsim.core (reference core.py:18-125) on the GPU.

* Activation keeps the reference's enum values and derivative convention (ReLU'(0) = 0).
* gemm() runs op(a) @ op(b) on the sm_100a tensor cores (kernels.gemm); non-finite results raise
  ConfigurationError exactly like core.py:59-60.
* flat_offsets() is the per-(rank, layer) parameter layout of include/ppx.h (PSHARD01 order).
"""

from __future__ import annotations

import math
import zlib
from enum import Enum

import numpy as np
import torch

from . import _lib, kernels
from .errors import ConfigurationError


def _key_word(part) -> int:
    """One spawn-key word: strings hash through CRC-32, integers keep their low 32 bits."""
    return zlib.crc32(part.encode("utf-8")) if isinstance(part, str) else int(part) & 0xFFFFFFFF


def substream(seed: int, *key) -> np.random.Generator:
    """core.py:101-114 — an independent Philox stream per (seed, *key): SeedSequence(seed) with
    the key as spawn key, two 64-bit words of its state as the Philox key.  Host-side: model
    construction must reproduce the reference's draws bit for bit."""
    seq = np.random.SeedSequence(entropy=int(seed) & (2**63 - 1), spawn_key=tuple(_key_word(x) for x in key))
    return np.random.Generator(np.random.Philox(key=seq.generate_state(2, dtype=np.uint64)))


def uniform_init(rng: np.random.Generator, rows: int, cols: int, fan_in: int, fan_out: int) -> np.ndarray:
    """core.py:117-125 — Glorot-uniform U[-a, a], a = sqrt(6 / (fan_in + fan_out)), float64."""
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-bound, bound, size=(rows, cols))


class FlopCounter:
    """core.py:18-36 — running count of floating point operations (2mnk per product)."""

    __slots__ = ("total",)

    def __init__(self) -> None:
        self.total = 0

    def add(self, flops: int) -> None:
        self.total += int(flops)

    def reset(self) -> None:
        self.total = 0


class Activation(Enum):
    """core.py:64-82 — elementwise nonlinearity; ReLU uses grad(0) = 0."""

    RELU = "relu"
    IDENTITY = "identity"

    @property
    def code(self) -> int:
        return _lib.PPX_RELU if self is Activation.RELU else _lib.PPX_IDENTITY

    def apply(self, z: torch.Tensor) -> torch.Tensor:
        return apply_activation(z, self)

    def grad(self, pre: torch.Tensor) -> torch.Tensor:
        return activation_grad(pre, self)


def as_activation(a) -> Activation:
    if isinstance(a, Activation):
        return a
    return Activation(getattr(a, "value", a))


def round8(x: int) -> int:
    return (x + 7) // 8 * 8


def flat_offsets(s: int, k: int, p: int) -> dict:
    """Element offsets of the flat parameter block (include/ppx.h; checkpoint.py:57-64 order)."""
    lds, ldk = round8(s), round8(k)
    comp = s * lds
    dec = comp + k * lds
    bias = dec + (p - 1) * s * ldk
    return {"lds": lds, "ldk": ldk, "local": 0, "comp": comp, "dec": dec, "bias": bias,
            "total": bias + round8(s)}


def gemm(a: torch.Tensor, b: torch.Tensor, transpose_a: bool = False, transpose_b: bool = False,
         counter: FlopCounter | None = None) -> torch.Tensor:
    """core.py:39-61 — (a or a^T) @ (b or b^T) in fp32 output on the tensor cores."""
    if a.dim() != 2 or b.dim() != 2:
        raise ConfigurationError("gemm expects 2-d operands")
    left = (a.shape[1], a.shape[0]) if transpose_a else tuple(a.shape)
    right = (b.shape[1], b.shape[0]) if transpose_b else tuple(b.shape)
    if left[1] != right[0]:
        raise ConfigurationError(f"gemm dimension mismatch: {left} x {right}")
    dt = a.dtype if a.dtype in (torch.bfloat16, torch.float32) else torch.float32
    a = row_major(a.to(dt))
    b = row_major(b.to(dt))
    out = kernels.gemm(a, b, transpose_a, transpose_b, out_dtype=torch.float32)
    if counter is not None:
        counter.add(2 * left[0] * left[1] * right[1])
    if not bool(torch.isfinite(out).all()):
        raise ConfigurationError("gemm produced non-finite values")
    return out


def row_major(t: torch.Tensor) -> torch.Tensor:
    """2-d tensor with unit column stride and a leading dim that is a multiple of 8."""
    if t.dim() != 2:
        raise ConfigurationError("expected a 2-d tensor")
    if t.stride(1) == 1 and t.stride(0) % 8 == 0 and t.stride(0) >= t.shape[1] and t.data_ptr() % 16 == 0:
        return t
    r, c = t.shape
    buf = torch.empty((r, round8(max(c, 1))), dtype=t.dtype, device=t.device)
    buf[:, :c].copy_(t)
    return buf[:, :c]


def apply_activation(z: torch.Tensor, act: Activation, counter: FlopCounter | None = None) -> torch.Tensor:
    """core.py:85-90 on the device (ppx_bias_act)."""
    act = as_activation(act)
    z2 = row_major(z)
    out = torch.empty_like(z2)
    out = row_major(out) if out.stride(0) % 8 else out
    dt = kernels.ppx_dtype(z2.dtype)
    kernels.ctx_for(z2).call("ppx_bias_act", dt, z2.shape[0], z2.shape[1], kernels.ptr(z2), kernels.ld(z2),
                             None, act.code, kernels.ptr(out), kernels.ld(out), kernels.stream_handle())
    if counter is not None:
        counter.add(out.numel())
    return out


def activation_grad(pre: torch.Tensor, act: Activation, counter: FlopCounter | None = None) -> torch.Tensor:
    """core.py:93-98 on the device: 1 where pre > 0 (ReLU) else 0; ones for identity."""
    act = as_activation(act)
    pre2 = row_major(pre)
    out = row_major(torch.ones(pre2.shape, dtype=pre2.dtype, device=pre2.device))
    if act is Activation.RELU:
        dt = kernels.ppx_dtype(pre2.dtype)
        kernels.ctx_for(pre2).call("ppx_relu_mask", dt, pre2.shape[0], pre2.shape[1], kernels.ptr(out),
                                   kernels.ld(out), kernels.ptr(pre2), kernels.ld(pre2), kernels.stream_handle())
    if counter is not None:
        counter.add(out.numel())
    return out
