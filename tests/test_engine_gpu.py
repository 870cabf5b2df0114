"""PhantomEngine (fused epilogues, grouped wgrad with in-place SGD/Adam, CUDA graphs) against
the pinned CPU oracle: one and several training steps with p logical ranks on one GPU.

fp32 tier tolerance 1e-4 (normwise); bf16 tier: loss 2e-2, weights after the step 2e-2.
"""
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


def _setup(n, p, k, L, B, dtype, optimizer, lr, seed=3, act="relu"):
    from paper_2508_00960_b200.engine import PhantomEngine
    model = po.init_phantom_model(n, p, k, L, seed)
    rng = np.random.default_rng(seed)
    for row in model:       # non-zero biases so the bias path is exercised
        for lay in row:
            lay["bias"] = 0.1 * rng.standard_normal(lay["bias"].shape)
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = PhantomEngine(n, p, k, L, B, optimizer=optimizer, lr=lr, dtype=dtype, activation=act)
    eng.load_params(model)
    s = n // p
    xs = [torch.from_numpy(x[j * s:(j + 1) * s].T.copy()).cuda() for j in range(p)]
    ys = [torch.from_numpy(y[j * s:(j + 1) * s].T.copy()).cuda() for j in range(p)]
    for par in (0, 1):
        eng.set_batch(xs, ys, par)
    return eng, model, x, y


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
    for jj in range(p):
        for l in range(L):
            v = eng.layer_views(jj, l)
            assert nerr(v["local"], model[jj][l]["local"]) <= tol
            assert nerr(v["compressor"], model[jj][l]["compressor"]) <= tol
            assert nerr(v["bias"], model[jj][l]["bias"]) <= tol
            for i, d in v["decompressors"].items():
                assert nerr(d, model[jj][l]["decompressors"][i]) <= tol


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
def test_engine_fused_forward_matches_oracle(graph, monkeypatch):
    """PPX_FUSED=1: compression + (in-kernel) phantom exchange + forward of each layer as ONE
    2-SM launch (forward tiles wait on the compression tiles' arrival counter) — bf16 steps
    against the float64 oracle."""
    monkeypatch.setenv("PPX_FUSED", "1")
    n, p, k, L, B, lr = 512, 4, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr)
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
    for jj in range(p):
        for l in range(L):
            v = eng.layer_views(jj, l)
            assert nerr(v["local"], model[jj][l]["local"]) <= 2e-2
            assert nerr(v["compressor"], model[jj][l]["compressor"]) <= 2e-2


@pytest.mark.parametrize("graph", [False, True])
def test_engine_pair_kernel_matches_oracle(graph):
    """64-aligned s and k: every contraction runs on the 2-SM kernel (spanning phantom-slot tiles,
    M < 256 weight-gradient problems) — bf16 steps against the float64 oracle."""
    n, p, k, L, B, lr = 512, 4, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr)
    if graph:
        eng.capture()
    losses = []
    for _ in range(3):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, 3, "sgd", lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref)


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("graph", [False, True])
def test_engine_backward_fused_matches_oracle(graph, p, monkeypatch):
    """PPX_BWD_FUSED=1: weight gradients (+ fused SGD) and the error recurrence of each layer as ONE
    launch with a static longest-first tile schedule — bf16 steps against the float64 oracle."""
    monkeypatch.setenv("PPX_BWD_FUSED", "1")
    n, k, L, B, lr = 128 * p, 64, 3, 256, 3e-3
    eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr)
    assert eng.bwd_fused
    if graph:
        eng.capture()
    losses = []
    for _ in range(3):
        eng.step(graph=graph)
        losses.append(eng.read_loss())
    ref = _oracle_steps(model, x, y, L, 3, "sgd", lr)
    for a, b in zip(losses, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref)
    for jj in range(p):
        for l in range(L):
            v = eng.layer_views(jj, l)
            assert nerr(v["local"], model[jj][l]["local"]) <= 2e-2
            for i, d in v["decompressors"].items():
                assert nerr(d, model[jj][l]["decompressors"][i]) <= 2e-2
