"""Phantom-parallel layers on B200 — the drop-in for phantomsim.phantom (reference phantom.py).

Same names, argument meaning and error behaviour as the reference; tensors are CUDA tensors.
Activations at this API keep the reference orientation (features x batch, core.py:3-4); they
are transposed *views* of the engine's native [batch, features] row-major buffers, so the
kernels never see a layout copy on the common path.

Parameters of one (rank, layer) live in ONE flat fp32 master buffer laid out in PSHARD01 order
(include/ppx.h); `local`, `compressor`, `decompressors[i]` and `bias` are views into it, and
the compute copy (bf16, or the master itself for the fp32 tier) is refreshed by `sync()`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, kernels
from .collectives import Communicator, Direction
from .core import (Activation, FlopCounter, as_activation, flat_offsets, round8, row_major, substream,
                   uniform_init)
from .errors import ConfigurationError, SequencingError

DEFAULT_DTYPE = torch.bfloat16


def _to_device(a, device, dtype=torch.float32) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=device).to(dtype)


class PhantomLayer:
    """phantom.py:23-54 — one rank's shard of one layer (square local, k x s compressor,
    per-peer s x k decompressors keyed by source rank, s bias)."""

    def __init__(self, local, compressor, decompressors: dict, bias, *, rank: int | None = None,
                 p: int | None = None, dtype: torch.dtype = DEFAULT_DTYPE, device=None, _flat=None):
        if _flat is not None:
            self.s, self.k, self.p, self.rank, self.master, self.dtype = _flat
            self._views()
            self.w = self.master if self.dtype == torch.float32 else None
            self.sync()
            return
        device = torch.device(device or "cuda")
        local = _to_device(local, device)
        compressor = _to_device(compressor, device)
        bias = _to_device(bias, device)
        s = local.shape[0]
        if local.dim() != 2 or tuple(local.shape) != (s, s):
            raise ConfigurationError(f"local block must be square, got {tuple(local.shape)}")
        k = compressor.shape[0]
        if not 1 <= k <= s:
            raise ConfigurationError(f"need 1 <= k <= n/p, got k={k}, n/p={s}")
        if tuple(compressor.shape) != (k, s):
            raise ConfigurationError(f"compressor must be (k, n/p), got {tuple(compressor.shape)}")
        decs = {int(i): _to_device(d, device) for i, d in decompressors.items()}
        for i, d in decs.items():
            if tuple(d.shape) != (s, k):
                raise ConfigurationError(f"decompressor for rank {i} must be (n/p, k), got {tuple(d.shape)}")
        if tuple(bias.shape) != (s,):
            raise ConfigurationError(f"bias must be (n/p,), got {tuple(bias.shape)}")
        p = p if p is not None else len(decs) + 1
        if rank is None:
            missing = [r for r in range(p) if r not in decs]
            if len(missing) != 1:
                raise ConfigurationError("cannot infer the layer's rank from its decompressor keys")
            rank = missing[0]
        if set(decs) != {i for i in range(p) if i != rank}:
            raise ConfigurationError("decompressors must be keyed by every peer rank (self excluded)")
        self.s, self.k, self.p, self.rank, self.dtype = s, k, p, rank, dtype
        off = flat_offsets(s, k, p)
        self.master = torch.zeros(off["total"], dtype=torch.float32, device=device)
        self._views()
        self.local.copy_(local)
        self.compressor.copy_(compressor)
        for i, d in decs.items():
            self.decompressors[i].copy_(d)
        self.bias.copy_(bias)
        self.w = self.master if dtype == torch.float32 else None
        self.sync()

    def _views(self):
        s, k, p = self.s, self.k, self.p
        off = flat_offsets(s, k, p)
        self.off = off
        m = self.master
        lds, ldk = off["lds"], off["ldk"]
        self.local = m[0:s * lds].view(s, lds)[:, :s]
        self.compressor = m[off["comp"]:off["comp"] + k * lds].view(k, lds)[:, :s]
        self.decompressors = {}
        for q in range(p - 1):
            i = q + (1 if q >= self.rank else 0)
            base = off["dec"] + q * s * ldk
            self.decompressors[i] = m[base:base + s * ldk].view(s, ldk)[:, :k]
        self.bias = m[off["bias"]:off["bias"] + s]

    @classmethod
    def from_flat(cls, master: torch.Tensor, s: int, k: int, p: int, rank: int, dtype=DEFAULT_DTYPE):
        return cls(None, None, {}, None, _flat=(s, k, p, rank, master, dtype))

    def sync(self):
        """Refresh the compute copy from the fp32 master (after editing the views)."""
        if self.dtype == torch.float32:
            self.w = self.master
            return
        if self.w is None:
            self.w = torch.empty(self.master.numel(), dtype=self.dtype, device=self.master.device)
        ctx = kernels.ctx_for(self.master)
        ctx.call("ppx_cast", _lib.PPX_FP32, self.master.data_ptr(), kernels.ppx_dtype(self.dtype),
                 self.w.data_ptr(), self.master.numel(), kernels.stream_handle())

    def abi(self) -> _lib.Layer:
        return _lib.Layer(self.s, self.k, self.p, self.rank, self.w.data_ptr(), self.master.data_ptr(), None)

    @property
    def shard_width(self) -> int:
        return self.s

    def to_numpy(self) -> dict:
        return {"local": self.local.double().cpu().numpy(), "compressor": self.compressor.double().cpu().numpy(),
                "decompressors": {i: d.double().cpu().numpy() for i, d in self.decompressors.items()},
                "bias": self.bias.double().cpu().numpy()}


@dataclass
class LayerTape:
    """phantom.py:57-64 — per-layer forward state kept for the backward pass."""

    inputs: torch.Tensor                 # (n/p, batch) view
    preact: torch.Tensor                 # (n/p, batch) view
    phantoms: dict                       # source rank -> (k, batch), own block included
    phantom_grad: torch.Tensor | None = None
    # native buffers the kernels read (batch-major); not part of the reference surface
    _y: torch.Tensor | None = field(default=None, repr=False)
    _pre: torch.Tensor | None = field(default=None, repr=False)
    _ph: torch.Tensor | None = field(default=None, repr=False)


@dataclass
class PhantomGradients:
    """phantom.py:67-74 — views into one flat fp32 gradient block (same layout as the params)."""

    bias: torch.Tensor
    local: torch.Tensor
    compressor: torch.Tensor
    decompressors: dict
    flat: torch.Tensor | None = field(default=None, repr=False)


@dataclass
class PhantomModel:
    """phantom.py:77-99."""

    n: int
    p: int
    k: int
    activations: list
    rank_layers: list
    seed: int = 0

    @property
    def layer_count(self) -> int:
        return len(self.activations)

    @property
    def shard_width(self) -> int:
        return self.n // self.p


# ----------------------------------------------------------------------------------------------
# model construction
# ----------------------------------------------------------------------------------------------
def _reference_init_arrays(n, p, k, layers, seed, j, l):
    """The reference's seeded Glorot-uniform draws (phantom.py:126-129), bit-for-bit on the host."""
    s = n // p
    local = uniform_init(substream(seed, "pp", l, j, "local"), s, s, s, s)
    comp = uniform_init(substream(seed, "pp", l, j, "compressor"), k, s, s, k)
    decs = {i: uniform_init(substream(seed, "pp", l, j, "decompressor", i), s, k, k, s) for i in range(p) if i != j}
    return local, comp, decs


def init_phantom_model(n: int, p: int, k: int, layers: int, activation=Activation.RELU, seed: int = 0, *,
                       dtype: torch.dtype = DEFAULT_DTYPE, device=None, init: str = "reference",
                       ranks=None) -> PhantomModel:
    """phantom.py:102-132.  init="reference" reproduces the reference's Philox draws exactly
    (weights identical to phantomsim for the same seed); init="device" draws the same Glorot
    bounds with torch's device generator (fast, for throughput runs).  `ranks` restricts
    materialisation to the logical ranks this process owns (others are None)."""
    if p < 1:
        raise ConfigurationError("p must be >= 1")
    if n % p != 0:
        raise ConfigurationError(f"n={n} not divisible by p={p}")
    s = n // p
    if not 1 <= k <= s:
        raise ConfigurationError(f"need 1 <= k <= n/p, got k={k}, n/p={s}")
    acts = list(activation) if isinstance(activation, (list, tuple)) else [activation] * layers
    if len(acts) != layers:
        raise ConfigurationError("need one activation per layer")
    acts = [as_activation(a) for a in acts]
    device = torch.device(device or "cuda")
    own = set(range(p)) if ranks is None else set(ranks)
    rank_layers = []
    gen = None
    for j in range(p):
        if j not in own:
            rank_layers.append(None)
            continue
        row = []
        for l in range(layers):
            off = flat_offsets(s, k, p)
            master = torch.zeros(off["total"], dtype=torch.float32, device=device)
            layer = PhantomLayer.from_flat(master, s, k, p, j, dtype)
            if init == "reference":
                local, comp, decs = _reference_init_arrays(n, p, k, layers, seed, j, l)
                layer.local.copy_(torch.from_numpy(local))
                layer.compressor.copy_(torch.from_numpy(comp))
                for i, d in decs.items():
                    layer.decompressors[i].copy_(torch.from_numpy(d))
            elif init == "device":
                if gen is None:
                    gen = torch.Generator(device=device)
                gen.manual_seed(hash((seed, j, l)) & 0x7FFFFFFF)
                a = (6.0 / (s + s)) ** 0.5
                layer.local.uniform_(-a, a, generator=gen)
                a = (6.0 / (s + k)) ** 0.5
                layer.compressor.uniform_(-a, a, generator=gen)
                for d in layer.decompressors.values():
                    d.uniform_(-a, a, generator=gen)
            else:
                raise ConfigurationError(f"unknown init {init!r}")
            layer.sync()
            row.append(layer)
        rank_layers.append(row)
    return PhantomModel(n, p, k, acts, rank_layers, seed)


def model_from_numpy(rank_layers_np, n, p, k, activations, seed=0, dtype=DEFAULT_DTYPE, device=None):
    """Build a device model from reference-format arrays (dicts or phantomsim PhantomLayers)."""
    rows = []
    for j, row in enumerate(rank_layers_np):
        out = []
        for lay in row:
            get = (lambda name: lay[name]) if isinstance(lay, dict) else (lambda name: getattr(lay, name))
            out.append(PhantomLayer(get("local"), get("compressor"), get("decompressors"), get("bias"),
                                    rank=j, p=p, dtype=dtype, device=device))
        rows.append(out)
    return PhantomModel(n, p, k, [as_activation(a) for a in activations], rows, seed)


# ----------------------------------------------------------------------------------------------
# layout helpers: reference (features x batch) <-> native [batch, features]
# ----------------------------------------------------------------------------------------------
def _native(t: torch.Tensor, dtype) -> torch.Tensor:
    """A (features x batch) tensor as a row-major [batch, features] buffer (view when possible)."""
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t, dtype=np.float64), device="cuda")
    if not t.is_cuda:
        raise ConfigurationError("activations must be CUDA tensors (no CPU fallback)")
    return row_major(t.t().to(dtype))


def _empty_native(B, cols, dtype, device):
    return torch.empty((B, round8(cols)), dtype=dtype, device=device)[:, :cols]


def _ph_buffer(p, B, k, dtype, device):
    return torch.zeros((p, B, round8(k)), dtype=dtype, device=device)


def _received_native(received, k, dtype) -> torch.Tensor:
    """(k, batch) phantom gradient -> [batch, round8(k)] buffer (the ABI's received layout)."""
    r = _native(received, dtype)
    if r.stride(0) == round8(k):
        return r
    buf = _ph_buffer(1, r.shape[0], k, dtype, r.device)[0]
    buf[:, :k].copy_(r)
    return buf[:, :k]


# ----------------------------------------------------------------------------------------------
# the five layer operations (phantom.py:135-267)
# ----------------------------------------------------------------------------------------------
def pp_forward_layer(layer: PhantomLayer, y_prev, comm: Communicator, rank: int, tape: list | None = None, *,
                     activation=Activation.RELU, layer_index: int = 0,
                     counter: FlopCounter | None = None) -> torch.Tensor:
    """phantom.py:135-166: compress, all-gather, ONE K-concatenated local+decompress GEMM with the
    bias+activation epilogue. Returns the (n/p, batch) output; appends a LayerTape."""
    act = as_activation(activation)
    s, k, p = layer.s, layer.k, layer.p
    if not isinstance(y_prev, torch.Tensor) or y_prev.dim() != 2 or y_prev.shape[0] != s:
        shape = tuple(getattr(y_prev, "shape", ()))
        raise ConfigurationError(f"layer input must be (n/p, batch) = ({s}, *), got {shape}")
    dt = layer.dtype
    pdt = kernels.ppx_dtype(dt)
    y = _native(y_prev, dt)
    B = y.shape[0]
    dev = y.device
    ctx = kernels.ctx_for(y)
    st = kernels.stream_handle()
    L = layer.abi()
    ph = _ph_buffer(p, B, k, dt, dev)
    ctx.call("ppx_compress", pdt, ctypes.byref(L), B, y.data_ptr(), kernels.ld(y), ph.data_ptr(), st)
    own = ph[rank, :, :k].t()                                   # (k, batch) view
    gathered = comm.all_gather(rank, own, direction=Direction.FORWARD, layer=layer_index)
    if gathered.shape != (p * k, B):
        raise ConfigurationError("phantom all-gather returned an unexpected shape")
    for i in range(p):
        if i != rank:
            ph[i, :, :k].copy_(gathered[i * k:(i + 1) * k].t())
    out = _empty_native(B, s, dt, dev)
    pre = _empty_native(B, s, dt, dev)
    ctx.call("ppx_forward_update", pdt, ctypes.byref(L), B, act.code, y.data_ptr(), kernels.ld(y), ph.data_ptr(),
             out.data_ptr(), kernels.ld(out), pre.data_ptr(), kernels.ld(pre), st)
    if counter is not None:
        counter.add(2 * s * s * B + 2 * k * s * B + (p - 1) * (2 * s * k * B + s * B) + 2 * s * B)
    if tape is not None:
        phantoms = {i: gathered[i * k:(i + 1) * k] for i in range(p)}
        tape.append(LayerTape(inputs=y.t(), preact=pre.t(), phantoms=phantoms, _y=y, _pre=pre, _ph=ph))
    return out.t()


def pp_output_delta(y_out, y_true, preact, act, counter: FlopCounter | None = None) -> torch.Tensor:
    """phantom.py:169-182 — (y_out - y_true) * act'(preact)."""
    act = as_activation(act)
    if tuple(y_out.shape) != tuple(y_true.shape) or tuple(y_out.shape) != tuple(preact.shape):
        raise ConfigurationError("output delta operands must share one shape")
    dt = y_out.dtype if y_out.dtype in (torch.bfloat16, torch.float32) else torch.float32
    y, t, pre = _native(y_out, dt), _native(y_true, dt), _native(preact, dt)
    B, s = y.shape
    d = _empty_native(B, s, dt, y.device)
    kernels.ctx_for(y).call("ppx_output_delta", kernels.ppx_dtype(dt), B, s, act.code, y.data_ptr(), kernels.ld(y),
                            t.data_ptr(), kernels.ld(t), pre.data_ptr(), kernels.ld(pre), d.data_ptr(), kernels.ld(d),
                            1.0, 0.0, None, kernels.stream_handle())
    if counter is not None:
        counter.add(3 * y.numel())
    return d.t()


def pp_exchange_error_phantoms(layer: PhantomLayer, delta, comm: Communicator, rank: int, *, layer_index: int = 0,
                               counter: FlopCounter | None = None) -> torch.Tensor:
    """phantom.py:185-207 — slot i = D_i^T delta (own slot zero), then ONE reduce-scatter."""
    s, k, p = layer.s, layer.k, layer.p
    dt = layer.dtype
    d = _native(delta, dt)
    B = d.shape[0]
    contrib = _ph_buffer(p, B, k, dt, d.device)
    L = layer.abi()
    kernels.ctx_for(d).call("ppx_error_phantoms", kernels.ppx_dtype(dt), ctypes.byref(L), B, d.data_ptr(),
                            kernels.ld(d), contrib.data_ptr(), 0, kernels.stream_handle())
    if counter is not None:
        counter.add((p - 1) * 2 * s * k * B)
    contributions = contrib[:, :, :k].transpose(1, 2).reshape(p * k, B)
    return comm.reduce_scatter(rank, contributions, direction=Direction.BACKWARD, layer=layer_index)


def pp_backward_layer(layer_next: PhantomLayer, delta_next, preact, act, comm: Communicator, rank: int, *,
                      layer_index: int = 0, received=None, counter: FlopCounter | None = None) -> torch.Tensor:
    """phantom.py:210-236 — (local^T delta + compressor^T r) * act'(preact), one K-concatenated
    [delta | r] . [L ; C] contraction with the ReLU'-mask epilogue."""
    act = as_activation(act)
    if received is None:
        received = pp_exchange_error_phantoms(layer_next, delta_next, comm, rank, layer_index=layer_index,
                                              counter=counter)
    dt = layer_next.dtype
    d = _native(delta_next, dt)
    B, s = d.shape
    r = _received_native(received, layer_next.k, dt)
    mask = _native(preact, dt) if act is Activation.RELU else None
    out = _empty_native(B, s, dt, d.device)
    L = layer_next.abi()
    kernels.ctx_for(d).call("ppx_backward_delta", kernels.ppx_dtype(dt), ctypes.byref(L), B, act.code,
                            d.data_ptr(), kernels.ld(d), r.data_ptr(),
                            mask.data_ptr() if mask is not None else None, kernels.ld(mask) if mask is not None else 0,
                            out.data_ptr(), kernels.ld(out), None, kernels.stream_handle())
    if counter is not None:
        counter.add(2 * s * s * B + 2 * layer_next.k * s * B + 2 * s * B)
    return out.t()


def grads_from_flat(flat: torch.Tensor, s: int, k: int, p: int, rank: int) -> PhantomGradients:
    off = flat_offsets(s, k, p)
    lds, ldk = off["lds"], off["ldk"]
    decs = {}
    for q in range(p - 1):
        i = q + (1 if q >= rank else 0)
        base = off["dec"] + q * s * ldk
        decs[i] = flat[base:base + s * ldk].view(s, ldk)[:, :k]
    return PhantomGradients(bias=flat[off["bias"]:off["bias"] + s],
                            local=flat[0:s * lds].view(s, lds)[:, :s],
                            compressor=flat[off["comp"]:off["comp"] + k * lds].view(k, lds)[:, :s],
                            decompressors=decs, flat=flat)


def pp_param_grads(layer: PhantomLayer, delta, tape_entry: LayerTape, received_phantom_grads, *,
                   counter: FlopCounter | None = None) -> PhantomGradients:
    """phantom.py:239-267 — bias = batch sum of delta; local = delta y^T; compressor = r y^T;
    decompressor_i = delta g_i^T, as ONE grouped tcgen05 launch (fp32 gradients)."""
    if tape_entry is None:
        raise SequencingError("backward requires the layer's forward tape entry")
    if tuple(delta.shape) != tuple(tape_entry.preact.shape):
        raise ConfigurationError(f"delta shape {tuple(delta.shape)} does not match tape "
                                 f"{tuple(tape_entry.preact.shape)}")
    s, k, p = layer.s, layer.k, layer.p
    dt = layer.dtype
    d = _native(delta, dt)
    B = d.shape[0]
    y = tape_entry._y if tape_entry._y is not None else _native(tape_entry.inputs, dt)
    ph = tape_entry._ph
    if ph is None:
        ph = _ph_buffer(p, B, k, dt, d.device)
        for i in range(p):
            if i not in tape_entry.phantoms:
                raise SequencingError(f"tape holds no phantom block from rank {i}")
            ph[i, :, :k].copy_(tape_entry.phantoms[i].t())
    for i in layer.decompressors:
        if i not in tape_entry.phantoms:
            raise SequencingError(f"tape holds no phantom block from rank {i}")
    r = _received_native(received_phantom_grads, k, dt)
    off = flat_offsets(s, k, p)
    flat = torch.zeros(off["total"], dtype=torch.float32, device=d.device)
    L = layer.abi()
    kernels.ctx_for(d).call("ppx_param_grads", kernels.ppx_dtype(dt), ctypes.byref(L), B, d.data_ptr(),
                            kernels.ld(d), y.data_ptr(), kernels.ld(y), ph.data_ptr(), r.data_ptr(), flat.data_ptr(),
                            None, _lib.GRAD_ALL, kernels.stream_handle())
    if counter is not None:
        counter.add(2 * s * s * B + 2 * k * s * B + (p - 1) * 2 * s * k * B + s * B)
    return grads_from_flat(flat, s, k, p, layer.rank)


def effective_weight(model: PhantomModel, layer_index: int) -> torch.Tensor:
    """reference.py:143-157 — the dense n x n matrix a phantom layer applies: diagonal block j is
    local_j, block (row j, col i) is decompressor_{i->j} . compressor_i (rank <= k), built on the
    model's device in fp32 (a verification helper for the layout invariant of SURVEY §8e, not on
    the training path)."""
    if not 0 <= layer_index < model.layer_count:
        raise ConfigurationError(f"layer {layer_index} out of range")
    s, p = model.shard_width, model.p
    first = model.rank_layers[0][layer_index].local
    W = torch.zeros((model.n, model.n), dtype=torch.float32, device=first.device)
    for j in range(p):
        lay = model.rank_layers[j][layer_index]
        W[j * s:(j + 1) * s, j * s:(j + 1) * s] = lay.local.float()
        for i, dec in lay.decompressors.items():
            comp = model.rank_layers[i][layer_index].compressor
            W[j * s:(j + 1) * s, i * s:(i + 1) * s] = dec.float() @ comp.float()
    return W


def pp_model_size(n: int, p: int, k: int, layers: int) -> int:
    """phantom.py:270-280."""
    if p < 2:
        raise ConfigurationError("p must be >= 2")
    if n % p != 0:
        raise ConfigurationError(f"n={n} not divisible by p={p}")
    if not 1 <= k <= n // p:
        raise ConfigurationError(f"need 1 <= k <= n/p, got k={k}")
    return layers * (n * n // p + p * k * n)


def valid_k(n: int, p: int) -> tuple[int, float]:
    """phantom.py:283-296."""
    if p < 2:
        raise ConfigurationError("p must be >= 2")
    if n % p != 0:
        raise ConfigurationError(f"n={n} not divisible by p={p}")
    s = n // p
    return s, s * (p - 1) / p
