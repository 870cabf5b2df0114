"""Iteration, loss, optimizers and the training loop — drop-in for phantomsim.training
(reference training.py:28-378) on the in-process Communicator.

The schedule is the reference's: per layer one all-gather forward and one reduce-scatter
backward shared by the parameter gradients and the error recurrence, plus one scalar loss
all-reduce per iteration (training.py:181-213).  The throughput path with NCCL, fused
optimizer epilogues and CUDA graphs is engine.PhantomEngine; both call the same kernels.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .collectives import Communicator, Direction
from .core import Activation, FlopCounter, as_activation, gemm
from .errors import ConfigurationError, TrainingError
from .phantom import (_empty_native, _native, init_phantom_model, pp_backward_layer,
                      pp_exchange_error_phantoms, pp_forward_layer, pp_param_grads, valid_k)


@dataclass
class Dataset:
    """training.py:28-40 — teacher-generated samples (features x samples), device tensors."""

    inputs: torch.Tensor
    targets: torch.Tensor
    teacher: torch.Tensor
    seed: int

    @property
    def sample_count(self) -> int:
        return self.inputs.shape[1]


def teacher_targets(teacher: torch.Tensor, inputs: torch.Tensor) -> torch.Tensor:
    """training.py:43-45 — relu(teacher @ relu(inputs)), on the tensor cores (fp32 3xTF32)."""
    hidden = torch.clamp_min(inputs.float(), 0.0)
    return torch.clamp_min(gemm(teacher.float(), hidden), 0.0)


def gen_dataset(n: int, samples: int, seed: int, device=None) -> Dataset:
    """training.py:48-56 — the reference's Philox draws (bit-identical inputs and teacher),
    targets computed on the GPU."""
    if n < 1 or samples < 1:
        raise ConfigurationError("n and samples must be >= 1")
    from .phantom import _reference_init_arrays  # noqa: F401  (same keyed-stream construction)
    import zlib
    ss = np.random.SeedSequence(entropy=int(seed) & (2**63 - 1), spawn_key=(zlib.crc32(b"dataset"),))
    rng = np.random.Generator(np.random.Philox(key=ss.generate_state(2, dtype=np.uint64)))
    teacher = rng.standard_normal((n, n))
    inputs = rng.standard_normal((n, samples))
    device = torch.device(device or "cuda")
    t = torch.from_numpy(teacher).to(device=device, dtype=torch.float32)
    x = torch.from_numpy(inputs).to(device=device, dtype=torch.float32)
    return Dataset(x, teacher_targets(t, x), t, seed)


def mse_loss_sharded(y_out, y_true, comm: Communicator, rank: int, reduction: str = "sum") -> tuple[float, float]:
    """training.py:59-71 — local half-squared error of this shard and its all-reduced sum."""
    if tuple(y_out.shape) != tuple(y_true.shape):
        raise ConfigurationError("loss operands must share one shape")
    dt = y_out.dtype if y_out.dtype in (torch.bfloat16, torch.float32) else torch.float32
    y, t = _native(y_out, dt), _native(y_true, dt)
    B, s = y.shape
    scratch = _empty_native(B, s, dt, y.device)
    acc = torch.zeros(1, dtype=torch.float32, device=y.device)
    scale = 0.5 / B if reduction == "mean" else 0.5
    kernels.ctx_for(y).call("ppx_output_delta", kernels.ppx_dtype(dt), B, s, _lib.PPX_IDENTITY, y.data_ptr(),
                            kernels.ld(y), t.data_ptr(), kernels.ld(t), None, 0, scratch.data_ptr(),
                            kernels.ld(scratch), 1.0, scale, acc.data_ptr(), kernels.stream_handle())
    total = comm.all_reduce(rank, acc.view(1, 1), direction=Direction.LOSS)
    return float(acc.item()), float(total.view(-1)[0].item())


def _hyper(lr, betas=(0.9, 0.999), eps=1e-8, t=1, device=None) -> torch.Tensor:
    b1, b2 = betas
    return torch.tensor([lr, b1, b2, eps, 1 - b1 ** t, 1 - b2 ** t], dtype=torch.float32, device=device)


def _flat_step(kind, params, grads, hyper, states=None, names=None):
    bad = torch.zeros(1, dtype=torch.int32, device=hyper.device)
    flags = []
    for i, (theta, g) in enumerate(zip(params, grads)):
        if theta.numel() == 0:
            continue
        work = theta if theta.is_contiguous() else theta.contiguous()
        gw = g.to(torch.float32).contiguous()
        m = v = None
        if kind == _lib.PPX_UPDATE_ADAM:
            m, v = states[0][i], states[1][i]
        kernels.ctx_for(work).call("ppx_optimizer_step", kind, hyper.data_ptr(), work.data_ptr(), gw.data_ptr(),
                                   m.data_ptr() if m is not None else None, v.data_ptr() if v is not None else None,
                                   work.numel(), _lib.PPX_FP32, None, bad.data_ptr(), kernels.stream_handle())
        if work is not theta:
            theta.copy_(work)
        flags.append(i)
    if int(bad.item()):
        # locate the first offending parameter for the reference's message (training.py:79-81)
        for i in flags:
            if not bool(torch.isfinite(grads[i]).all()):
                label = names[i] if names else f"parameter {i}"
                raise TrainingError(f"non-finite gradient for {label} (shape {tuple(grads[i].shape)})")
        raise TrainingError("non-finite gradient")


def sgd_step(params, grads, lr: float, names=None) -> None:
    """training.py:74-82 — in-place theta -= lr * grad on the device; non-finite -> TrainingError."""
    if lr <= 0:
        raise ConfigurationError("learning rate must be positive")
    if not params:
        return
    _flat_step(_lib.PPX_UPDATE_SGD, params, grads, _hyper(lr, device=params[0].device), names=names)


@dataclass
class AdamState:
    """training.py:85-89."""

    m: list
    v: list
    t: int = 0


def adam_step(params, grads, state: AdamState, lr: float, betas=(0.9, 0.999), eps: float = 1e-8,
              names=None) -> None:
    """training.py:92-105 — bias-corrected Adam, in place, on the device."""
    state.t += 1
    if not params:
        return
    state.m = [m if (isinstance(m, torch.Tensor) and m.is_contiguous()) else torch.zeros_like(p).contiguous()
               for m, p in zip(state.m, params)]
    state.v = [v if (isinstance(v, torch.Tensor) and v.is_contiguous()) else torch.zeros_like(p).contiguous()
               for v, p in zip(state.v, params)]
    _flat_step(_lib.PPX_UPDATE_ADAM, params, grads, _hyper(lr, betas, eps, state.t, params[0].device),
               (state.m, state.v), names)


@dataclass
class TrainConfig:
    """training.py:108-154 (same fields and validation)."""

    mode: str
    n: int
    p: int
    layers: int
    k: int = 0
    batch: int = 0
    lr: float = 0.01
    optimizer: str = "sgd"
    target_loss: float | None = None
    max_epochs: int = 100
    seed: int = 0
    loss_reduction: str = "sum"
    activation: Activation = Activation.RELU
    scheduler: str = "lockstep"
    include_loss_comm_in_beta: bool = False
    dtype: torch.dtype = torch.bfloat16

    def validate(self) -> None:
        if self.mode not in ("pp", "tp"):
            raise ConfigurationError(f"mode must be pp or tp, got {self.mode!r}")
        if self.n < 1 or self.p < 1 or self.layers < 1:
            raise ConfigurationError("n, p and layers must be >= 1")
        if self.n % self.p != 0:
            raise ConfigurationError(f"n={self.n} not divisible by p={self.p}")
        if self.mode == "pp":
            if self.p < 2:
                raise ConfigurationError("pp mode needs p >= 2")
            comm_bound, _ = valid_k(self.n, self.p)
            if not 1 <= self.k < comm_bound:
                raise ConfigurationError(f"k={self.k} outside valid_k range [1, {comm_bound}) for "
                                         f"n={self.n}, p={self.p}")
        if self.batch < 0:
            raise ConfigurationError("batch must be >= 0 (0 = full batch)")
        if self.lr <= 0:
            raise ConfigurationError("lr must be positive")
        if self.optimizer not in ("sgd", "adam"):
            raise ConfigurationError(f"optimizer must be sgd or adam, got {self.optimizer!r}")
        if self.target_loss is not None and self.target_loss <= 0:
            raise ConfigurationError("target_loss must be positive")
        if self.max_epochs < 0:
            raise ConfigurationError("max_epochs must be >= 0")
        if self.loss_reduction not in ("sum", "mean"):
            raise ConfigurationError("loss_reduction must be sum or mean")
        if self.scheduler not in ("lockstep", "threads"):
            raise ConfigurationError("scheduler must be lockstep or threads")


@dataclass
class TrainResult:
    """training.py:157-164; `cost` carries measured seconds/joules instead of the modeled report."""

    epochs_run: int
    iterations_run: int
    converged: bool
    final_loss: float
    loss_history: list
    cost: dict | None = None


@dataclass
class IterationOutput:
    """training.py:171-178."""

    y_out: torch.Tensor
    local_loss: float
    global_loss: float
    grads: list
    deltas: list
    tape: list


def pp_iteration(comm: Communicator, rank: int, layers, activations, x_shard, y_shard, reduction: str = "sum",
                 counter: FlopCounter | None = None) -> IterationOutput:
    """training.py:181-213 — one phantom-parallel forward/backward pass on one rank."""
    tape = []
    out = x_shard
    for l, layer in enumerate(layers):
        out = pp_forward_layer(layer, out, comm, rank, tape, activation=activations[l], layer_index=l,
                               counter=counter)
    local, global_loss = mse_loss_sharded(out, y_shard, comm, rank, reduction)
    delta = _output_delta(out, y_shard, tape[-1].preact, activations[-1],
                          1.0 / x_shard.shape[1] if reduction == "mean" else 1.0)
    if counter is not None:
        counter.add(3 * out.numel() + (out.numel() if reduction == "mean" else 0))
    count = len(layers)
    grads = [None] * count
    deltas = [None] * count
    for l in range(count - 1, -1, -1):
        deltas[l] = delta
        received = pp_exchange_error_phantoms(layers[l], delta, comm, rank, layer_index=l, counter=counter)
        tape[l].phantom_grad = received
        grads[l] = pp_param_grads(layers[l], delta, tape[l], received, counter=counter)
        if l > 0:
            delta = pp_backward_layer(layers[l], delta, tape[l - 1].preact, activations[l - 1], comm, rank,
                                      layer_index=l, received=received, counter=counter)
    return IterationOutput(out, local, global_loss, grads, deltas, tape)


def _output_delta(y_out, y_true, preact, act, scale):
    """pp_output_delta (phantom.py:169-182) with the mean-reduction 1/B folded in
    (training.py:196-199), one elementwise kernel."""
    act = as_activation(act)
    dt = y_out.dtype
    y, t, pre = _native(y_out, dt), _native(y_true, dt), _native(preact, dt)
    B, s = y.shape
    d = _empty_native(B, s, dt, y.device)
    kernels.ctx_for(y).call("ppx_output_delta", kernels.ppx_dtype(dt), B, s, act.code, y.data_ptr(), kernels.ld(y),
                            t.data_ptr(), kernels.ld(t), pre.data_ptr(), kernels.ld(pre), d.data_ptr(), kernels.ld(d),
                            float(scale), 0.0, None, kernels.stream_handle())
    return d.t()


def _pp_param_lists(layers, grads):
    """training.py:251-264 order; here one flat (master, grad) pair per layer covers it."""
    params, gradients, names = [], [], []
    for l, (layer, grad) in enumerate(zip(layers, grads)):
        params.append(layer.master)
        gradients.append(grad.flat)
        names.append(f"layer{l}")
    return params, gradients, names


def _rank_train_loop(comm, rank, config, model, x_shard, y_shard, batch, iters_per_epoch):
    """training.py:276-309."""
    layers = model.rank_layers[rank]
    acts = model.activations
    adam_state = None
    history = []
    converged = False
    for epoch in range(config.max_epochs):
        epoch_losses = []
        for it in range(iters_per_epoch):
            sl = slice(it * batch, (it + 1) * batch)
            out = pp_iteration(comm, rank, layers, acts, x_shard[:, sl], y_shard[:, sl], config.loss_reduction)
            if not math.isfinite(out.global_loss):
                raise TrainingError(f"loss diverged to {out.global_loss} at epoch {epoch}")
            params, grads, names = _pp_param_lists(layers, out.grads)
            if config.optimizer == "adam":
                if adam_state is None:
                    adam_state = AdamState(m=[torch.zeros_like(g) for g in grads],
                                           v=[torch.zeros_like(g) for g in grads])
                adam_step(params, grads, adam_state, config.lr, names=names)
            else:
                sgd_step(params, grads, config.lr, names=names)
            for layer in layers:
                layer.sync()
            epoch_losses.append(out.global_loss)
        epoch_loss = float(np.mean(epoch_losses))
        history.append(epoch_loss)
        if config.target_loss is not None and epoch_loss <= config.target_loss:
            converged = True
            break
    return history, converged


def train(config: TrainConfig, data: Dataset, comm_model=None, rates=None) -> TrainResult:
    """training.py:312-378 — the configured loop on one GPU with p logical ranks (PP mode)."""
    config.validate()
    if config.mode != "pp":
        from .tensor_parallel import train_tp
        return train_tp(config, data)
    if data.inputs.shape[0] != config.n:
        raise ConfigurationError(f"dataset width {data.inputs.shape[0]} does not match n={config.n}")
    samples = data.sample_count
    batch = config.batch or samples
    if batch > samples or samples % batch != 0:
        raise ConfigurationError(f"batch={batch} must divide the sample count {samples}")
    iters_per_epoch = samples // batch
    model = init_phantom_model(config.n, config.p, config.k, config.layers, config.activation, config.seed,
                               dtype=config.dtype)
    s = config.n // config.p
    comm = Communicator(config.p, mode=config.scheduler)
    x = data.inputs.to(config.dtype)
    y = data.targets.to(config.dtype)
    t0 = time.perf_counter()
    if config.max_epochs == 0:
        history, converged = [], False
    else:
        outputs = comm.run(lambda c, r: _rank_train_loop(c, r, config, model, x[r * s:(r + 1) * s],
                                                         y[r * s:(r + 1) * s], batch, iters_per_epoch))
        history, converged = outputs[0]
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    epochs_run = len(history)
    return TrainResult(epochs_run=epochs_run, iterations_run=epochs_run * iters_per_epoch, converged=converged,
                       final_loss=history[-1] if history else float("inf"), loss_history=history,
                       cost={"seconds": elapsed, "records": len(comm.records)})


# ----------------------------------------------------------------------------------------------
# on-device training loops: the fused engine runs the reference's TrainConfig
# semantics — contiguous mini-batches in order, pre-update iteration losses, epoch loss = mean
# of iteration losses, stop at target (training.py:276-309) — with measured time and NVML energy
# ----------------------------------------------------------------------------------------------
def _shard_batches(data: Dataset, s: int, ranks, dtype):
    """Per logical rank, the (samples, s) row-major view of its feature rows."""
    x = data.inputs.to(dtype)
    y = data.targets.to(dtype)
    return ([x[j * s:(j + 1) * s].t() for j in ranks], [y[j * s:(j + 1) * s].t() for j in ranks])


def _reference_rows(config: TrainConfig, ranks):
    from .phantom import _reference_init_arrays
    s = config.n // config.p
    rows = {}
    for j in ranks:
        row = []
        for l in range(config.layers):
            local, comp, decs = _reference_init_arrays(config.n, config.p, config.k, config.layers, config.seed, j, l)
            row.append({"local": local, "compressor": comp, "decompressors": decs, "bias": np.zeros(s)})
        rows[j] = row
    return rows


def train_engine(config: TrainConfig, data: Dataset, *, world: int = 1, rank: int = 0, device: int = 0,
                 uid: bytes | None = None, init: str = "reference", graphs: bool = True) -> TrainResult:
    """training.py:312-378 (PP mode) on the fused engine: this process owns p/world logical ranks.
    cost = {seconds, joules (this GPU), samples_per_s, iterations}."""
    from .energy import EnergyMeter
    from .engine import PhantomEngine
    config.validate()
    if config.mode != "pp":
        return train_tp_engine(config, data, world=world, rank=rank, device=device, uid=uid, graphs=graphs)
    if data.inputs.shape[0] != config.n:
        raise ConfigurationError(f"dataset width {data.inputs.shape[0]} does not match n={config.n}")
    samples = data.sample_count
    batch = config.batch or samples
    if batch > samples or samples % batch != 0:
        raise ConfigurationError(f"batch={batch} must divide the sample count {samples}")
    iters = samples // batch
    eng = PhantomEngine(config.n, config.p, config.k, config.layers, batch, world=world, rank=rank, device=device,
                        uid=uid, activation=config.activation, reduction=config.loss_reduction,
                        optimizer=config.optimizer, lr=config.lr, dtype=config.dtype, seed=config.seed)
    try:
        if init == "reference":
            eng.load_params(_reference_rows(config, eng.local))
        xs, ys = _shard_batches(data, config.n // config.p, eng.local, config.dtype)
        history, converged, it_done, it_losses = [], False, 0, []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with EnergyMeter(device) as meter:
            for epoch in range(config.max_epochs):
                losses = []
                for it in range(iters):
                    sl = slice(it * batch, (it + 1) * batch)
                    eng.set_batch([x[sl] for x in xs], [y[sl] for y in ys])
                    use_graph = graphs and it_done > 0
                    if use_graph and eng.graphs[0] is None:
                        eng.capture()
                    eng.step(graph=use_graph)
                    loss = eng.read_loss()
                    if not math.isfinite(loss):
                        raise TrainingError(f"loss diverged to {loss} at epoch {epoch}")
                    losses.append(loss)
                    it_losses.append(loss)
                    it_done += 1
                epoch_loss = float(np.mean(losses))
                history.append(epoch_loss)
                if config.target_loss is not None and epoch_loss <= config.target_loss:
                    converged = True
                    break
            torch.cuda.synchronize()
        elapsed = time.perf_counter() - t0
    finally:
        eng.close()
    return TrainResult(epochs_run=len(history), iterations_run=it_done, converged=converged,
                       final_loss=history[-1] if history else float("inf"), loss_history=history,
                       cost={"seconds": elapsed, "joules": meter.joules, "iterations": it_done,
                             "samples_per_s": it_done * batch / elapsed if elapsed > 0 else None,
                             "iteration_losses": it_losses})


def train_tp_engine(config: TrainConfig, data: Dataset, *, world: int = 1, rank: int = 0, device: int = 0,
                    uid: bytes | None = None, graphs: bool = True) -> TrainResult:
    """The Megatron comparison pipeline under the same loop (SGD, mean or sum reduction): the
    dense model of tensor_parallel.full_layer_weight (the reference's TP init), p = world GPUs."""
    from .energy import EnergyMeter
    from .tensor_parallel import TPEngine, full_layer_weight
    config.validate()
    if config.optimizer != "sgd":
        raise ConfigurationError("the TP engine trains with SGD")
    samples = data.sample_count
    batch = config.batch or samples
    if batch > samples or samples % batch != 0:
        raise ConfigurationError(f"batch={batch} must divide the sample count {samples}")
    iters = samples // batch
    eng = TPEngine(config.n, config.layers, batch, world=world, rank=rank, device=device, uid=uid, lr=config.lr,
                   dtype=config.dtype, seed=config.seed, reduction=config.loss_reduction)
    try:
        eng.load_full_weights([full_layer_weight(config.n, l, config.seed) for l in range(config.layers)])
        x = data.inputs.to(config.dtype).t()
        y = data.targets.to(config.dtype).t()
        history, converged, it_done, it_losses = [], False, 0, []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with EnergyMeter(device) as meter:
            for epoch in range(config.max_epochs):
                losses = []
                for it in range(iters):
                    sl = slice(it * batch, (it + 1) * batch)
                    eng.set_batch(x[sl], y[sl])
                    use_graph = graphs and it_done > 0
                    if use_graph and eng.graphs[0] is None:
                        eng.capture()
                    eng.step(graph=use_graph)
                    loss = eng.read_loss()
                    if not math.isfinite(loss):
                        raise TrainingError(f"loss diverged to {loss} at epoch {epoch}")
                    losses.append(loss)
                    it_losses.append(loss)
                    it_done += 1
                epoch_loss = float(np.mean(losses))
                history.append(epoch_loss)
                if config.target_loss is not None and epoch_loss <= config.target_loss:
                    converged = True
                    break
            torch.cuda.synchronize()
        elapsed = time.perf_counter() - t0
    finally:
        eng.close()
    return TrainResult(epochs_run=len(history), iterations_run=it_done, converged=converged,
                       final_loss=history[-1] if history else float("inf"), loss_history=history,
                       cost={"seconds": elapsed, "joules": meter.joules, "iterations": it_done,
                             "samples_per_s": it_done * batch / elapsed if elapsed > 0 else None,
                             "iteration_losses": it_losses})


def gen_dataset_device(n: int, samples: int, seed: int, device=None, dtype=torch.bfloat16) -> Dataset:
    """gen_dataset's teacher task drawn with the device generator (N(0,1) teacher and inputs,
    targets relu(teacher . relu(x)) on the tensor cores) for widths where the reference's host
    Philox draws are too slow; same distribution, not the same bits."""
    if n < 1 or samples < 1:
        raise ConfigurationError("n and samples must be >= 1")
    dev = torch.device(device or "cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed) & 0x7FFFFFFF)
    teacher = torch.randn((n, n), generator=g, device=dev).to(dtype)
    x = torch.randn((n, samples), generator=g, device=dev).to(dtype)
    hidden = torch.clamp_min(x, 0)
    t = torch.empty((samples, n), dtype=dtype, device=dev)
    for c in range(0, samples, 8192):
        e = min(samples, c + 8192)
        t[c:e] = kernels.gemm(hidden[:, c:e], teacher, transpose_a=True, transpose_b=True, out_dtype=dtype,
                              relu=True)
    return Dataset(x, t.t(), teacher, seed)
