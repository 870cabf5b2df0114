"""Tensor-parallel comparison pipeline (reference tensor_parallel.py, training.py:216-244).

Two layers of the same engine live here:

* The drop-in API — TPLayer / TPModel / init_tp_model (p-independent full weights, row blocks,
  tensor_parallel.py:23-92), tp_forward_layer / tp_backward_layer with the reference's row-block
  schedule over the in-process Communicator (all-gather + redundant broadcast forward,
  all-reduce + redundant reduce-scatter backward, tensor_parallel.py:95-153), and tp_iteration.
  It is an exact reparameterisation of the dense FFN (the TP parity oracle is dense training).

* TPEngine — the throughput comparison on B200 that north_star asks for: a Megatron-style FFN
  (column-parallel layer 2m, row-parallel layer 2m+1, ONE all-reduce of batch x n per pair in
  each direction) built on the same tcgen05 kernel and C ABI as the phantom engine, with bias /
  ReLU / ReLU'-mask / bias-gradient epilogues and SGD fused into the weight-gradient GEMMs.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .collectives import Communicator, Direction
from .core import Activation, FlopCounter, as_activation, gemm, row_major
from .errors import ConfigurationError, SequencingError, TrainingError
from .schedule import tp_comm_bytes_per_step  # noqa: F401  (re-export for bench/docs)


# ----------------------------------------------------------------------------------------------
# drop-in API (reference tensor_parallel.py)
# ----------------------------------------------------------------------------------------------
@dataclass
class TPLayer:
    """tensor_parallel.py:23-35 — one rank's row block (n/p, n) and bias (n/p,)."""

    weight: torch.Tensor
    bias: torch.Tensor

    def __post_init__(self):
        if self.weight.dim() != 2:
            raise ConfigurationError("weight must be 2-d")
        if tuple(self.bias.shape) != (self.weight.shape[0],):
            raise ConfigurationError(f"bias shape {tuple(self.bias.shape)} does not match weight rows")


@dataclass
class TPLayerTape:
    y_full: torch.Tensor
    preact: torch.Tensor


@dataclass
class TPGradients:
    weight: torch.Tensor
    bias: torch.Tensor


@dataclass
class TPModel:
    n: int
    p: int
    activations: list
    rank_layers: list
    seed: int = 0

    @property
    def layer_count(self) -> int:
        return len(self.activations)

    @property
    def shard_width(self) -> int:
        return self.n // self.p


def full_layer_weight(n: int, layer: int, seed: int) -> np.ndarray:
    """tensor_parallel.py:67-73 — the reference's Philox draw of one full weight (host numpy)."""
    import zlib
    ss = np.random.SeedSequence(entropy=int(seed) & (2**63 - 1),
                                spawn_key=(zlib.crc32(b"tp"), int(layer) & 0xFFFFFFFF, zlib.crc32(b"weight")))
    rng = np.random.Generator(np.random.Philox(key=ss.generate_state(2, dtype=np.uint64)))
    a = math.sqrt(6.0 / (n + n))
    return rng.uniform(-a, a, size=(n, n))


def init_tp_model(n: int, p: int, layers: int, activation=Activation.RELU, seed: int = 0, *,
                  dtype: torch.dtype = torch.float32, device=None) -> TPModel:
    """tensor_parallel.py:76-92 (weights identical to the reference for the same seed)."""
    if p < 1:
        raise ConfigurationError("p must be >= 1")
    if n % p != 0:
        raise ConfigurationError(f"n={n} not divisible by p={p}")
    acts = list(activation) if isinstance(activation, (list, tuple)) else [activation] * layers
    if len(acts) != layers:
        raise ConfigurationError("need one activation per layer")
    device = torch.device(device or "cuda")
    s = n // p
    rank_layers = [[] for _ in range(p)]
    for l in range(layers):
        full = torch.from_numpy(full_layer_weight(n, l, seed)).to(device=device, dtype=dtype)
        for j in range(p):
            rank_layers[j].append(TPLayer(full[j * s:(j + 1) * s].clone(), torch.zeros(s, dtype=dtype, device=device)))
    return TPModel(n, p, [as_activation(a) for a in acts], rank_layers, seed)


def tp_model_size(n: int, layers: int) -> int:
    """tensor_parallel.py:156-158."""
    return layers * n * n


def tp_forward_layer(layer: TPLayer, y_prev_shard, comm: Communicator, rank: int, tape: list | None = None, *,
                     activation=Activation.RELU, layer_index: int = 0, counter: FlopCounter | None = None):
    """tensor_parallel.py:95-122 — all-gather + scheduled broadcast, then act(W y_full + b)."""
    act = as_activation(activation)
    s, n = layer.weight.shape
    if y_prev_shard.dim() != 2 or y_prev_shard.shape[0] != s:
        raise ConfigurationError(f"layer input must be (n/p, batch) = ({s}, *), got {tuple(y_prev_shard.shape)}")
    gathered = comm.all_gather(rank, y_prev_shard, direction=Direction.FORWARD, layer=layer_index)
    y_full = comm.broadcast(rank, 0, gathered if rank == 0 else None, direction=Direction.FORWARD, layer=layer_index)
    dt = layer.weight.dtype
    # preact^T (batch, s) = y_full^T . W^T on the tensor cores, bias added in the epilogue
    pre_t = kernels.gemm(row_major(y_full.to(dt)), row_major(layer.weight), transpose_a=True, transpose_b=True,
                         out_dtype=dt, bias=layer.bias.float().contiguous())
    pre = pre_t.t()
    if counter is not None:
        counter.add(2 * s * n * y_full.shape[1] + pre.numel())
    out = act.apply(pre)
    if tape is not None:
        tape.append(TPLayerTape(y_full=y_full, preact=pre))
    return out


def tp_backward_layer(layer: TPLayer, delta_shard, tape_entry: TPLayerTape, comm: Communicator, rank: int, *,
                      layer_index: int = 0, counter: FlopCounter | None = None):
    """tensor_parallel.py:125-153 — grads, then all-reduce (+ scheduled reduce-scatter) of W^T delta."""
    if tape_entry is None:
        raise SequencingError("backward requires the layer's forward tape entry")
    s, n = layer.weight.shape
    dt = layer.weight.dtype
    d = row_major(delta_shard.to(dt))
    grad_w = kernels.gemm(d, row_major(tape_entry.y_full.to(dt)), transpose_b=True, out_dtype=torch.float32)
    grad_b = _rowsum(d)
    grad_full = kernels.gemm(row_major(layer.weight), d, transpose_a=True, out_dtype=dt)
    summed = comm.all_reduce(rank, grad_full, direction=Direction.BACKWARD, layer=layer_index)
    scattered = comm.reduce_scatter(rank, grad_full, direction=Direction.BACKWARD, layer=layer_index)
    del scattered
    if counter is not None:
        counter.add(2 * s * n * d.shape[1] * 2 + d.numel())
    return summed[rank * s:(rank + 1) * s].clone(), TPGradients(grad_w, grad_b)


def _rowsum(x: torch.Tensor) -> torch.Tensor:
    """sum over the batch (columns) of a (features, batch) matrix with the colsum kernel."""
    xt = row_major(x.t())                       # (batch, features)
    out = torch.empty(xt.shape[1], dtype=torch.float32, device=x.device)
    kernels.ctx_for(xt).call("ppx_colsum", kernels.ppx_dtype(xt.dtype), xt.shape[0], xt.shape[1], xt.data_ptr(),
                             kernels.ld(xt), out.data_ptr(), 0, kernels.stream_handle())
    return out


# ----------------------------------------------------------------------------------------------
# TPEngine: Megatron column/row pairs over NCCL
# ----------------------------------------------------------------------------------------------
def tp_step_flops(n: int, world: int, layers: int, batch: int) -> int:
    """GEMM FLOPs per GPU per Megatron training step: 6 L B s n - 2 B s n (no input grad of layer 0)."""
    s = n // world
    return 6 * layers * batch * s * n - 2 * batch * s * n


class TPEngine:
    def __init__(self, n: int, layers: int, batch: int, *, world: int = 1, rank: int = 0, device: int = 0,
                 uid: bytes | None = None, lr: float = 3e-6, dtype: torch.dtype = torch.bfloat16, seed: int = 0,
                 reduction: str = "mean", ctx: _lib.Context | None = None):
        if layers % 2:
            raise ConfigurationError("the Megatron pipeline pairs layers: layers must be even")
        if n % world:
            raise ConfigurationError(f"n={n} not divisible by {world} GPUs")
        self.n, self.L, self.B, self.world, self.rank = n, layers, batch, world, rank
        self.s = s = n // world
        self.P = layers // 2
        self.dtype, self.pdt = dtype, kernels.ppx_dtype(dtype)
        self.lr, self.reduction = lr, reduction
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        self.ctx = ctx or _lib.Context(world, rank, device, uid)
        f32, P, B = torch.float32, self.P, batch
        # masters: Wa[m] rows [s, n] of layer 2m; Wb[m] column block [n, s] of layer 2m+1
        self.Wa = torch.empty((P, s, n), dtype=f32, device=self.dev)
        self.Wb = torch.empty((P, n, s), dtype=f32, device=self.dev)
        g = torch.Generator(device=self.dev)
        a = math.sqrt(6.0 / (2 * n))
        for m in range(P):
            g.manual_seed(seed * 7 + 2 * m * 1009 + rank)
            self.Wa[m].uniform_(-a, a, generator=g)
            g.manual_seed(seed * 7 + (2 * m + 1) * 1009 + rank)
            self.Wb[m].uniform_(-a, a, generator=g)
        self.wa = [torch.empty((P, s, n), dtype=dtype, device=self.dev) for _ in range(2)]
        self.wb = [torch.empty((P, n, s), dtype=dtype, device=self.dev) for _ in range(2)]
        st = torch.cuda.current_stream().cuda_stream
        for par in range(2):
            self.ctx.call("ppx_cast", _lib.PPX_FP32, self.Wa.data_ptr(), self.pdt, self.wa[par].data_ptr(),
                          self.Wa.numel(), st)
            self.ctx.call("ppx_cast", _lib.PPX_FP32, self.Wb.data_ptr(), self.pdt, self.wb[par].data_ptr(),
                          self.Wb.numel(), st)
        self.bias = torch.zeros(P * (s + n), dtype=f32, device=self.dev)     # [ba (P*s) | bb (P*n)]
        self.gbias = torch.zeros_like(self.bias)
        self.X = [[torch.empty((B, n), dtype=dtype, device=self.dev) for _ in range(P + 1)] for _ in range(2)]
        for m in range(1, P + 1):
            self.X[1][m] = self.X[0][m]
        self.Tgt = [torch.empty((B, n), dtype=dtype, device=self.dev) for _ in range(2)]
        self.Ya = [torch.empty((B, s), dtype=dtype, device=self.dev) for _ in range(P)]
        self.Dfull = [torch.empty((B, n), dtype=dtype, device=self.dev) for _ in range(2)]
        self.Dya = torch.empty((B, s), dtype=dtype, device=self.dev)
        self.loss = torch.zeros(1, dtype=f32, device=self.dev)
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.hyper = torch.tensor([lr, 0.9, 0.999, 1e-8, 0.1, 0.001], dtype=f32, device=self.dev)
        self.graphs = [None, None]
        self.parity = 0
        self._keep = []
        self.launch_count = 0

    def load_full_weights(self, weights, biases=None):
        """weights[l]: full (n, n) matrices (numpy or torch); GPU g keeps rows g*s.. of layer 2m
        and columns g*s.. of layer 2m+1 (Megatron split of the same dense model)."""
        s, r = self.s, self.rank
        for m in range(self.P):
            wa = torch.as_tensor(weights[2 * m], dtype=torch.float64)
            wb = torch.as_tensor(weights[2 * m + 1], dtype=torch.float64)
            self.Wa[m].copy_(wa[r * s:(r + 1) * s, :])
            self.Wb[m].copy_(wb[:, r * s:(r + 1) * s])
            if biases is not None:
                self._ba(m).copy_(torch.as_tensor(biases[2 * m], dtype=torch.float64)[r * s:(r + 1) * s])
                self._bb(m).copy_(torch.as_tensor(biases[2 * m + 1], dtype=torch.float64))
        st = torch.cuda.current_stream().cuda_stream
        for par in range(2):
            self.ctx.call("ppx_cast", _lib.PPX_FP32, self.Wa.data_ptr(), self.pdt, self.wa[par].data_ptr(),
                          self.Wa.numel(), st)
            self.ctx.call("ppx_cast", _lib.PPX_FP32, self.Wb.data_ptr(), self.pdt, self.wb[par].data_ptr(),
                          self.Wb.numel(), st)

    def _ba(self, m):
        return self.bias[m * self.s:(m + 1) * self.s]

    def _bb(self, m):
        o = self.P * self.s
        return self.bias[o + m * self.n:o + (m + 1) * self.n]

    def _gba(self, m):
        return self.gbias[m * self.s:(m + 1) * self.s]

    def _gbb(self, m):
        o = self.P * self.s
        return self.gbias[o + m * self.n:o + (m + 1) * self.n]

    def _gemm(self, M, N, K, a, lda, ta, b, ldb, tb, c, ldc, st, act=_lib.PPX_IDENTITY, bias=None, mask=None,
              ld_mask=0, colsum=None):
        epi = _lib.Epilogue(act, bias, 0, mask, ld_mask, colsum)
        self._keep.append(epi)
        self.ctx.call("ppx_gemm", self.pdt, M, N, K, a, lda, ta, b, ldb, tb, c, ldc, self.pdt, ctypes.byref(epi), st)

    def _gemm_update(self, M, N, K, a, lda, ta, b, ldb, tb, master, w_next, ld_w, st):
        u = _lib.Update(_lib.PPX_UPDATE_SGD, self.hyper.data_ptr(), master, w_next, None, None, None,
                        self.bad.data_ptr())
        self._keep.append(u)
        self.ctx.call("ppx_gemm_update", self.pdt, M, N, K, a, lda, ta, b, ldb, tb, ctypes.byref(u), ld_w, st)

    def _step_body(self, par, S):
        self._keep.clear()
        c, st = self.ctx, S.cuda_stream
        k0 = c.kernel_launches
        n, s, B, P, pdt = self.n, self.s, self.B, self.P, self.pdt
        X, Ya = self.X[par], self.Ya
        c.call("ppx_zero", self.loss.data_ptr(), 4, st)
        c.call("ppx_zero", self.gbias.data_ptr(), self.gbias.numel() * 4, st)
        # ---- forward: column-parallel (bias+ReLU epilogue) then row-parallel partial + all-reduce
        for m in range(P):
            self._gemm(B, s, n, X[m].data_ptr(), n, 0, self.wa[par][m].data_ptr(), n, 1, Ya[m].data_ptr(), s, st,
                       act=_lib.PPX_RELU, bias=self._ba(m).data_ptr())
            self._gemm(B, n, s, Ya[m].data_ptr(), s, 0, self.wb[par][m].data_ptr(), s, 1, X[m + 1].data_ptr(), n, st)
            c.call("ppx_all_reduce", pdt, X[m + 1].data_ptr(), B * n, st)
            c.call("ppx_bias_act", pdt, B, n, X[m + 1].data_ptr(), n, self._bb(m).data_ptr(), _lib.PPX_RELU,
                   X[m + 1].data_ptr(), n, st)
        mean = self.reduction == "mean"
        cur = 0
        c.call("ppx_output_delta", pdt, B, n, _lib.PPX_RELU, X[P].data_ptr(), n, self.Tgt[par].data_ptr(), n,
               X[P].data_ptr(), n, self.Dfull[cur].data_ptr(), n, 1.0 / B if mean else 1.0,
               0.5 / B if mean else 0.5, self.loss.data_ptr(), st)
        # ---- backward
        for m in range(P - 1, -1, -1):
            D = self.Dfull[cur]
            c.call("ppx_colsum", pdt, B, n, D.data_ptr(), n, self._gbb(m).data_ptr(), 0, st)
            # d Wb = D^T Ya  [n, s]  (+SGD)
            self._gemm_update(n, s, B, D.data_ptr(), n, 1, Ya[m].data_ptr(), s, 0, self.Wb[m].data_ptr(),
                              self.wb[1 - par][m].data_ptr(), s, st)
            # d Ya = (D Wb) * relu'(Ya)   [B, s], bias grad of layer 2m fused
            self._gemm(B, s, n, D.data_ptr(), n, 0, self.wb[par][m].data_ptr(), s, 0, self.Dya.data_ptr(), s, st,
                       mask=Ya[m].data_ptr(), ld_mask=s, colsum=self._gba(m).data_ptr())
            # d Wa = Dya^T X[m]  [s, n]  (+SGD)
            self._gemm_update(s, n, B, self.Dya.data_ptr(), s, 1, X[m].data_ptr(), n, 0, self.Wa[m].data_ptr(),
                              self.wa[1 - par][m].data_ptr(), n, st)
            if m > 0:
                Dn = self.Dfull[1 - cur]
                self._gemm(B, n, s, self.Dya.data_ptr(), s, 0, self.wa[par][m].data_ptr(), n, 0, Dn.data_ptr(), n,
                           st)
                c.call("ppx_all_reduce", pdt, Dn.data_ptr(), B * n, st)
                c.call("ppx_relu_mask", pdt, B, n, Dn.data_ptr(), n, X[m].data_ptr(), n, st)
                cur = 1 - cur
        c.call("ppx_optimizer_step", _lib.PPX_UPDATE_SGD, self.hyper.data_ptr(), self.bias.data_ptr(),
               self.gbias.data_ptr(), None, None, self.bias.numel(), _lib.PPX_FP32, None, self.bad.data_ptr(), st)
        self.launch_count = c.kernel_launches - k0   # kernels enqueued by this step (GEMMs + helpers)

    def step(self, graph: bool = True):
        par = self.parity
        if graph and self.graphs[par] is not None:
            self.graphs[par].replay()
        else:
            self._step_body(par, torch.cuda.current_stream())
        self.parity = 1 - par

    def capture(self):
        torch.cuda.synchronize()
        for par in (0, 1):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(self.dev)
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cs):
                self._step_body(par, torch.cuda.current_stream())
            self.graphs[par] = g
        torch.cuda.synchronize()

    def set_batch(self, x_full, t_full, par=None):
        par = self.parity if par is None else par
        self.X[par][0].copy_(x_full)
        self.Tgt[par].copy_(t_full)

    def read_loss(self) -> float:
        torch.cuda.current_stream().synchronize()
        if int(self.bad.item()):
            raise TrainingError("non-finite gradient detected on the device")
        return float(self.loss.item())

    def close(self):
        if self.ctx.handle is None:
            return
        torch.cuda.synchronize()
        for g in self.graphs:
            if g is not None:
                g.reset()
        self.graphs = [None, None]
        torch.cuda.synchronize()
        self.ctx.close()


def tp_iteration(comm: Communicator, rank: int, layers, activations, x_shard, y_shard, reduction: str = "sum",
                 counter: FlopCounter | None = None):
    """training.py:216-244 — one tensor-parallel forward/backward pass on one rank."""
    from .training import IterationOutput, _output_delta, mse_loss_sharded
    tape = []
    out = x_shard
    for l, layer in enumerate(layers):
        out = tp_forward_layer(layer, out, comm, rank, tape, activation=activations[l], layer_index=l, counter=counter)
    local, global_loss = mse_loss_sharded(out, y_shard, comm, rank, reduction)
    delta = _output_delta(out, y_shard.to(out.dtype), tape[-1].preact, activations[-1],
                          1.0 / x_shard.shape[1] if reduction == "mean" else 1.0)
    count = len(layers)
    grads = [None] * count
    deltas = [None] * count
    for l in range(count - 1, -1, -1):
        deltas[l] = delta
        shard, grads[l] = tp_backward_layer(layers[l], delta, tape[l], comm, rank, layer_index=l, counter=counter)
        if l > 0:
            mask = tape[l - 1].preact
            d2 = row_major(shard)
            if as_activation(activations[l - 1]) is Activation.RELU:
                m2 = row_major(mask)
                kernels.ctx_for(d2).call("ppx_relu_mask", kernels.ppx_dtype(d2.dtype), d2.shape[0], d2.shape[1],
                                         d2.data_ptr(), kernels.ld(d2), m2.data_ptr(), kernels.ld(m2),
                                         kernels.stream_handle())
            delta = d2
    return IterationOutput(out, local, global_loss, grads, deltas, tape)


def train_tp(config, data):
    """training.py:312-378 for mode "tp" on the in-process Communicator (p logical ranks, 1 GPU)."""
    import time
    from .training import TrainResult, sgd_step, adam_step, AdamState
    model = init_tp_model(config.n, config.p, config.layers, config.activation, config.seed, dtype=config.dtype)
    samples = data.sample_count
    batch = config.batch or samples
    if batch > samples or samples % batch:
        raise ConfigurationError(f"batch={batch} must divide the sample count {samples}")
    iters = samples // batch
    s = config.n // config.p
    comm = Communicator(config.p, mode=config.scheduler)
    x = data.inputs.to(config.dtype)
    y = data.targets.to(config.dtype)

    def worker(c, r):
        layers = model.rank_layers[r]
        hist, conv, state = [], False, None
        for epoch in range(config.max_epochs):
            losses = []
            for it in range(iters):
                sl = slice(it * batch, (it + 1) * batch)
                out = tp_iteration(c, r, layers, model.activations, x[r * s:(r + 1) * s, sl], y[r * s:(r + 1) * s, sl],
                                   config.loss_reduction)
                if not math.isfinite(out.global_loss):
                    raise TrainingError(f"loss diverged to {out.global_loss} at epoch {epoch}")
                params = [t for lay in layers for t in (lay.weight, lay.bias)]
                grads = [t for g in out.grads for t in (g.weight, g.bias)]
                if config.optimizer == "adam":
                    state = state or AdamState(m=[torch.zeros_like(p_) for p_ in params],
                                               v=[torch.zeros_like(p_) for p_ in params])
                    adam_step(params, grads, state, config.lr)
                else:
                    sgd_step(params, grads, config.lr)
                losses.append(out.global_loss)
            hist.append(float(np.mean(losses)))
            if config.target_loss is not None and hist[-1] <= config.target_loss:
                conv = True
                break
        return hist, conv

    t0 = time.perf_counter()
    history, converged = comm.run(worker)[0] if config.max_epochs else ([], False)
    torch.cuda.synchronize()
    return TrainResult(len(history), len(history) * iters, converged, history[-1] if history else float("inf"),
                       history, {"seconds": time.perf_counter() - t0, "records": len(comm.records)})
