"""ctypes binding of libppx.so (include/ppx.h) — the only way this package reaches the GPU.

There is no CPU fallback: importing the binding on a machine without the built library raises
DeviceError, and every compute entry point requires CUDA tensors.  The same stub is what a
phantomsim maintainer would drop into the reference to call the engine.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (ConfigurationError, DeviceError, ProtocolError,
                     SequencingError, TrainingError)

LIB_PATH = os.environ.get("PPX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libppx.so")

PPX_OK, PPX_E_CONFIG, PPX_E_PROTOCOL, PPX_E_SEQUENCING, PPX_E_NONFINITE, PPX_E_CUDA = range(6)
PPX_BF16, PPX_FP32 = 0, 1
PPX_RELU, PPX_IDENTITY = 0, 1
PPX_UPDATE_NONE, PPX_UPDATE_SGD, PPX_UPDATE_ADAM = 0, 1, 2

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_fp = ctypes.c_void_p  # float*


class Layer(ctypes.Structure):
    """ppx_layer: one logical rank's shard of one layer."""
    _fields_ = [("s", _i32), ("k", _i32), ("p", _i32), ("rank", _i32), ("w", _vp), ("master", _vp),
                ("bias", _vp)]


class Update(ctypes.Structure):
    """ppx_update: optimizer fused into the weight-gradient epilogue."""
    _fields_ = [("kind", _i32), ("hyper", _vp), ("master", _vp), ("w_next", _vp),
                ("adam_m", _vp), ("adam_v", _vp), ("grad", _vp), ("bad", _vp)]


class WgradItem(ctypes.Structure):
    """ppx_wgrad_item: one layer's weight-gradient request in a grouped launch."""
    _fields_ = [("layer", ctypes.POINTER(Layer)), ("parts", _i32), ("B", _i32), ("delta", _vp), ("ld_d", _i64),
                ("y_prev", _vp), ("ld_y", _i64), ("phantoms", _vp), ("received", _vp), ("grad", _vp),
                ("upd", ctypes.POINTER(Update)), ("phantom_halves", _i32)]


class Exchange(ctypes.Structure):
    """ppx_exchange: NVLink peers and counters of one layer's fused forward launch."""
    _fields_ = [("n_peers", _i32), ("peer_phantoms", ctypes.POINTER(_vp)), ("arrive", ctypes.POINTER(_vp)),
                ("wait_counter", _vp), ("epoch", _vp), ("bad", _vp)]


class Scatter(ctypes.Structure):
    """ppx_scatter: owners' staging areas and arrival counters of one layer (NVLink reduce-scatter)."""
    _fields_ = [("world", _i32), ("rank", _i32), ("stage", ctypes.POINTER(_vp)), ("arrive", ctypes.POINTER(_vp))]


class RankIO(ctypes.Structure):
    """ppx_rank_io: one logical rank's operands in a grouped launch."""
    _fields_ = [("layer", ctypes.POINTER(Layer)), ("x", _vp), ("ld_x", _i64), ("out", _vp), ("ld_out", _i64),
                ("aux", _vp), ("ld_aux", _i64), ("target", _vp), ("ld_t", _i64), ("mask", _vp), ("ld_m", _i64),
                ("received", _vp), ("colsum", _vp), ("bits", _vp), ("ld_bits", _i64)]


GRAD_LOCAL, GRAD_COMP, GRAD_DEC, GRAD_BIAS, GRAD_ALL = 1, 2, 4, 8, 15


class Epilogue(ctypes.Structure):
    """ppx_epilogue: generic GEMM epilogue."""
    _fields_ = [("act", _i32), ("bias", _vp), ("accumulate", _i32), ("mask", _vp),
                ("ld_mask", _i64), ("colsum", _vp)]


_SIGS = {
    "ppx_abi_version": (_i32, []),
    "ppx_layer_elems": (_i64, [_i32, _i32, _i32]),
    "ppx_get_unique_id": (_i32, [ctypes.c_char_p]),
    "ppx_create": (_i32, [_i32, _i32, _i32, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "ppx_destroy": (_i32, [_vp]),
    "ppx_last_error": (ctypes.c_char_p, [_vp]),
    "ppx_num_sms": (_i32, [_vp]),
    "ppx_kernel_launches": (_i64, [_vp]),
    "ppx_reserve_workspace": (_i32, [_vp, _i64]),
    "ppx_tf32_scope": (_i32, [_vp, _i32, _vp]),
    "ppx_set_reserved_sms": (_i32, [_vp, _i32]),
    "ppx_compress": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _vp, _i64, _vp, _vp]),
    "ppx_compress_n": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _vp, _vp]),
    "ppx_forward_n": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _i32, _vp, _i32, _f32, _f32, _fp, _vp]),
    "ppx_backward_delta_n": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _i32, _vp]),
    "ppx_all_gather": (_i32, [_vp, _i32, _vp, _i64, _i32, _vp]),
    "ppx_forward_update": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _i32, _vp, _i64, _vp,
                                  _vp, _i64, _vp, _i64, _vp]),
    "ppx_forward_output": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _i32, _vp, _i64, _vp,
                                  _vp, _i64, _vp, _i64, _vp, _i64, _f32, _f32, _fp, _fp, _vp]),
    "ppx_output_delta": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64,
                                _vp, _i64, _f32, _f32, _fp, _vp]),
    "ppx_error_phantoms": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _vp, _i64, _vp, _i32, _vp]),
    "ppx_error_phantoms_n": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _vp, _vp]),
    "ppx_reduce_scatter_to": (_i32, [_vp, _i32, _vp, _vp, _i64, _i32, _vp]),
    "ppx_peek_error": (_i32, []),
    "ppx_peer_alloc": (_i32, [_vp, _i64, ctypes.POINTER(_vp), ctypes.c_char_p]),
    "ppx_peer_open": (_i32, [_vp, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "ppx_forward_fused": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _i32, _vp, _i32, _f32, _f32, _fp,
                                   ctypes.POINTER(Exchange), _vp]),
    "ppx_error_phantoms_scatter": (_i32, [_vp, _i32, _i32, ctypes.POINTER(RankIO), _i32, _vp, ctypes.POINTER(Scatter),
                                           _vp]),
    "ppx_reduce_received": (_i32, [_vp, _i32, _i32, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ppx_backward_fused": (_i32, [_vp, _i32, _i32, ctypes.POINTER(WgradItem), _i32, ctypes.POINTER(RankIO), _i32, _i32,
                                   _vp]),
    "ppx_reduce_scatter": (_i32, [_vp, _i32, _vp, _i64, _i32, _vp]),
    "ppx_all_reduce_f32": (_i32, [_vp, _fp, _i64, _vp]),
    "ppx_all_reduce": (_i32, [_vp, _i32, _vp, _i64, _vp]),
    "ppx_param_grads": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _vp, _i64, _vp, _i64, _vp,
                               _vp, _fp, ctypes.POINTER(Update), _i32, _vp]),
    "ppx_wgrad": (_i32, [_vp, _i32, _i32, ctypes.POINTER(WgradItem), _vp]),
    "ppx_wgrad_splitk": (_i32, [_vp, _i32, _i32, ctypes.POINTER(WgradItem), _i32, _fp, _vp]),
    "ppx_backward_delta": (_i32, [_vp, _i32, ctypes.POINTER(Layer), _i32, _i32, _vp, _i64, _vp,
                                  _vp, _i64, _vp, _i64, _fp, _vp]),
    "ppx_colsum": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _fp, _i32, _vp]),
    "ppx_optimizer_step": (_i32, [_vp, _i32, _fp, _fp, _fp, _fp, _fp, _i64, _i32, _vp, _vp, _vp]),
    "ppx_backward_wgrad_errors": (_i32, [_vp, _i32, _i32, ctypes.POINTER(WgradItem), _i32, ctypes.POINTER(RankIO), _i32,
                                          _vp, ctypes.POINTER(Scatter), _i32, _vp]),
    "ppx_hyper_advance": (_i32, [_vp, _vp, _vp, ctypes.c_double, ctypes.c_double, _vp]),
    "ppx_gemm": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _i64,
                        _i32, ctypes.POINTER(Epilogue), _vp]),
    "ppx_gemm_update": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _i64, _i32,
                               ctypes.POINTER(Update), _i64, _vp]),
    "ppx_zero": (_i32, [_vp, _vp, _i64, _vp]),
    "ppx_cast": (_i32, [_vp, _i32, _vp, _i32, _vp, _i64, _vp]),
    "ppx_bias_act": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _fp, _i32, _vp, _i64, _vp]),
    "ppx_relu_mask": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _i64, _vp]),
}

EXPORTS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()
_DEBUG_ERRORS = bool(os.environ.get("PPX_DEBUG_ERRORS"))


def load():
    """Load libppx.so (once). Raises DeviceError when it was never built: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("PPX_LIB") and not hasattr(lib, name):
                    continue   # A/B runs against an older build (PPX_LIB): bind what it exports
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.ppx_abi_version() != 1:
                raise DeviceError("libppx.so ABI version mismatch")
            _lib = lib
    return _lib


_ERRORS = {
    PPX_E_CONFIG: ConfigurationError,
    PPX_E_PROTOCOL: ProtocolError,
    PPX_E_SEQUENCING: SequencingError,
    PPX_E_NONFINITE: TrainingError,
    PPX_E_CUDA: DeviceError,
}


def check(status: int, ctx=None, what: str = "") -> None:
    if status == PPX_OK:
        return
    msg = ""
    if ctx is not None:
        raw = load().ppx_last_error(ctx)
        msg = raw.decode() if raw else ""
    raise _ERRORS.get(status, DeviceError)(f"{what}: {msg}" if what else msg)


class Context:
    """One ppx_ctx: this process's handle on one GPU (+ its NCCL communicator when world > 1)."""

    def __init__(self, world: int = 1, rank: int = 0, device: int = 0, uid: bytes | None = None):
        lib = load()
        self.world, self.rank, self.device = world, rank, device
        h = _vp()
        check(lib.ppx_create(world, rank, device, uid, ctypes.byref(h)), None, "ppx_create")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(load().ppx_get_unique_id(buf), None, "ppx_get_unique_id")
        return buf.raw

    def call(self, name: str, *args):
        check(getattr(load(), name)(self.handle, *args), self.handle, name)
        if _DEBUG_ERRORS:
            e = load().ppx_peek_error()
            if e:
                raise DeviceError(f"{name} left CUDA runtime error {e} pending")

    @property
    def num_sms(self) -> int:
        return load().ppx_num_sms(self.handle)

    @property
    def kernel_launches(self) -> int:
        """Kernels this context has enqueued (GEMMs, TF32 splits, elementwise helpers)."""
        return int(load().ppx_kernel_launches(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            load().ppx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    """Single-GPU context (world = 1) for the in-process API on `device`.

    A ppx_ctx is not re-entrant (it owns the FP32-tier workspace and the last-error string), and
    the in-process Communicator runs one host thread per logical rank, so contexts are per
    (thread, device)."""
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(1, 0, device)
    return ctx
