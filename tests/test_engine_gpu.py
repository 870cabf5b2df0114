"""PhantomEngine (fused epilogues, grouped wgrad with in-place SGD/Adam, CUDA graphs) against
the pinned CPU oracle: one and several training steps with p logical ranks on one GPU.

Every test compares the losses and the weight UPDATES W_T - W_0 of every tensor (local,
compressor, each decompressor, bias) with the oracle's: a zero, dropped or misplaced gradient moves
its update by ~100%.  fp32 tier 1e-4 (normwise).  bf16 tier: losses 2e-2; SGD updates 1e-1 and
Adam updates 2.5e-1 — against the float64 oracle the bf16 activations perturb every gradient by a
few 1e-2 over three ReLU layers at width 512 (the per-kernel bf16 arithmetic itself is checked
teacher-forced at 5e-3 in test_parity_scale_gpu.py), and Adam's m / sqrt(v) turns the relative
noise of near-zero gradient entries into O(1) noise of their updates.
"""
import copy

import numpy as np
import pytest
import torch

from oracle import phantom_oracle as po

pytestmark = pytest.mark.gpu


def nerr(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def _setup(n, p, k, L, B, dtype, optimizer, lr, seed=3, act="relu", **kw):
    from paper_2508_00960_b200.engine import PhantomEngine
    model = po.init_phantom_model(n, p, k, L, seed)
    rng = np.random.default_rng(seed)
    for row in model:       # non-zero biases so the bias path is exercised
        for lay in row:
            lay["bias"] = 0.1 * rng.standard_normal(lay["bias"].shape)
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = PhantomEngine(n, p, k, L, B, optimizer=optimizer, lr=lr, dtype=dtype, activation=act, **kw)
    eng.load_params(model)
    s = n // p
    xs = [torch.from_numpy(x[j * s:(j + 1) * s].T.copy()).cuda() for j in range(p)]
    ys = [torch.from_numpy(y[j * s:(j + 1) * s].T.copy()).cuda() for j in range(p)]
    for par in (0, 1):
        eng.set_batch(xs, ys, par)
    return eng, model, x, y


def _check_updates(eng, model0, model, tol):
    """normwise error of the engine's update of every parameter tensor vs the oracle's update."""
    worst = 0.0
    for jj, j in enumerate(eng.local):
        for l in range(eng.L):
            v = eng.layer_views(jj, l)
            pairs = [(v[nm], model0[j][l][nm], model[j][l][nm]) for nm in ("local", "compressor", "bias")]
            pairs += [(d, model0[j][l]["decompressors"][i], model[j][l]["decompressors"][i])
                      for i, d in v["decompressors"].items()]
            for got, w0, w1 in pairs:
                e = nerr(got.double().cpu().numpy() - w0, w1 - w0)
                worst = max(worst, e)
    assert worst <= tol, worst
    return worst


def _oracle_steps(model, x, y, L, steps, optimizer, lr, act="relu"):
    p = len(model)
    s = x.shape[0] // p
    losses = []
    state = [None] * p
    for _ in range(steps):
        out = po.pp_iteration(model, [act] * L, [x[j * s:(j + 1) * s] for j in range(p)],
                              [y[j * s:(j + 1) * s] for j in range(p)], "mean")
        losses.append(out["global_loss"])
        for j in range(p):
            params, gs = po.pp_param_list(model[j], out["grads"][j])
            if optimizer == "adam":
                if state[j] is None:
                    state[j] = {"m": [np.zeros_like(g) for g in gs], "v": [np.zeros_like(g) for g in gs], "t": 0}
                po.adam_step(params, gs, state[j], lr)
            else:
                po.sgd_step(params, gs, lr)
    return losses


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
@pytest.mark.parametrize("graph", [False, True])
def test_engine_steps_match_oracle(dtype, tol, optimizer, graph):
    n, p, k, L, B = 512, 4, 32, 3, 64
    lr = 3e-3 if optimizer == "sgd" else 1e-3
    eng, model, x, y = _setup(n, p, k, L, B, dtype, optimizer, lr)
    model0 = copy.deepcopy(model)
    steps = 3
    if graph:
        eng.capture()
    losses = []
    for _ in range(steps):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, steps, optimizer, lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= tol * abs(b), (losses, ref)
    _check_updates(eng, model0, model, tol if dtype == torch.float32 else (1e-1 if optimizer == "sgd" else 2.5e-1))


@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
@pytest.mark.parametrize("group", [None, 1])
def test_engine_layer0_splitk_matches_oracle(optimizer, group):
    """B = 512 splits the layer-0 compressor gradient over the batch (ppx_wgrad_splitk: 4 chunks
    of fp32 partial sums, then the summing SGD / Adam pass): fp32 tier vs the oracle over 3 graph
    steps, and the plan really took the split.  SGD 1e-4; Adam 1e-3: at this shape Adam's
    m / sqrt(v) turns the fp32 rounding of near-zero gradient entries into up to 6.8e-4 normwise
    update error in the layer-0 tensors — identical with the split off (PPX_NO_SPLITK=1), so it
    is the tier's arithmetic, not the split."""
    n, p, k, L, B = 512, 4, 32, 2, 512
    lr = 3e-3 if optimizer == "sgd" else 1e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.float32, optimizer, lr, group=group)
    assert eng._layer0_split(eng.group) > 1
    model0 = copy.deepcopy(model)
    eng.step(graph=False)
    assert "ppx_wgrad_splitk" in eng.trace
    eng.capture()
    for _ in range(2):
        eng.step()
    loss = eng.read_loss()
    ref = _oracle_steps(model, x, y, L, 3, optimizer, lr)
    assert abs(loss - ref[-1]) <= 1e-4 * abs(ref[-1]), (loss, ref)
    _check_updates(eng, model0, model, 1e-4 if optimizer == "sgd" else 1e-3)


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_engine_unsynchronised_graph_replays(optimizer):
    """Five CUDA-graph steps issued back to back with no host synchronisation in between (the
    bench's timing loop): the Adam bias corrections 1 - beta^t are advanced on the device, so
    every step uses its own t (training.py:92-105) — fp32 tier vs the oracle at 1e-4."""
    n, p, k, L, B = 512, 4, 32, 3, 64
    lr = 1e-3 if optimizer == "adam" else 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.float32, optimizer, lr)
    model0 = copy.deepcopy(model)
    eng.capture()
    for _ in range(5):
        eng.step()
    loss = eng.read_loss()
    ref = _oracle_steps(model, x, y, L, 5, optimizer, lr)
    assert abs(loss - ref[-1]) <= 1e-4 * abs(ref[-1]), (loss, ref)
    _check_updates(eng, model0, model, 1e-4)


def test_engine_forward_only_matches_oracle():
    n, p, k, L, B = 1024, 2, 16, 4, 64
    eng, model, x, y = _setup(n, p, k, L, B, torch.float32, "sgd", 1e-4)
    outs = eng.forward_only()
    torch.cuda.synchronize()
    s = n // p
    ref = po.pp_forward(model, ["relu"] * L, [x[j * s:(j + 1) * s] for j in range(p)])
    for j in range(p):
        assert nerr(outs[j].t(), ref[j]) <= 1e-4


@pytest.mark.parametrize("graph", [False, True])
def test_engine_fused_forward_matches_oracle(graph):
    """fused=True: compression + (in-kernel) phantom exchange + forward of each layer as ONE
    2-SM launch (forward tiles wait on the compression tiles' arrival counter) — bf16 steps
    against the float64 oracle."""
    n, p, k, L, B, lr = 512, 4, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr, fused=True)
    model0 = copy.deepcopy(model)
    assert eng.fused
    if graph:
        eng.capture()
    losses = []
    for _ in range(3):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, 3, "sgd", lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref)
    _check_updates(eng, model0, model, 1e-1)


@pytest.mark.parametrize("graph", [False, True])
def test_engine_pair_kernel_matches_oracle(graph):
    """64-aligned s and k: every contraction runs on the 2-SM kernel (spanning phantom-slot tiles,
    M < 256 weight-gradient problems) — bf16 steps against the float64 oracle."""
    n, p, k, L, B, lr = 512, 4, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr, fused=False)
    model0 = copy.deepcopy(model)
    if graph:
        eng.capture()
    losses = []
    for _ in range(3):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, 3, "sgd", lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref)
    _check_updates(eng, model0, model, 1e-1)


@pytest.mark.parametrize("k3", [False, True])
@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("graph", [False, True])
def test_engine_backward_fused_matches_oracle(graph, p, k3):
    """group=1 (one logical rank per launch): k3=False — weight gradients (+ fused SGD) and the error
    recurrence of each layer as ONE launch with a static longest-first tile schedule; k3=True —
    error compression + weight gradients as one such launch (error tiles first), then the
    recurrence — bf16 steps against the float64 oracle."""
    n, k, L, B, lr = 128 * p, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr, group=1, k3_fused=k3)
    model0 = copy.deepcopy(model)
    assert (eng.k3_fused, eng.bwd_fused) == (k3, not k3)
    if graph:
        eng.capture()
    losses = []
    for _ in range(3):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, 3, "sgd", lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref)
    _check_updates(eng, model0, model, 1e-1)
