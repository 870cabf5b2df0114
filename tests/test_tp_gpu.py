"""Tensor-parallel comparison pipeline on B200: the reference-API row-block TP iteration against the
reference's golden vectors, and the Megatron TPEngine (fused epilogues, SGD in the wgrad
epilogue, CUDA graphs) against the dense oracle (TP is an exact reparameterisation of dense)."""
import os

import numpy as np
import pytest
import torch

from oracle import phantom_oracle as po

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def nerr(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def test_tp_iteration_fp32_matches_reference():
    from paper_2508_00960_b200.collectives import Communicator
    from paper_2508_00960_b200.tensor_parallel import init_tp_model, tp_iteration
    z = np.load(os.path.join(GOLD, "tiny.npz"))
    n, p, L, B, seed = (int(v) for v in z["tp_cfg"])
    s = n // p
    model = init_tp_model(n, p, L, seed=seed, dtype=torch.float32)
    x = torch.from_numpy(z["tp_x"]).cuda().float()
    y = torch.from_numpy(z["tp_y"]).cuda().float()
    comm = Communicator(p)
    outs = comm.run(lambda c, r: tp_iteration(c, r, model.rank_layers[r], model.activations,
                                              x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], "sum"))
    assert abs(outs[0].global_loss - float(z["tp_global_loss"])) <= 1e-4 * abs(float(z["tp_global_loss"]))
    for r in range(p):
        assert nerr(outs[r].y_out, z[f"tp_r{r}_y_out"]) <= 1e-4
        for l in range(L):
            assert nerr(outs[r].grads[l].weight, z[f"tp_r{r}_l{l}_g_weight"]) <= 1e-4
            assert nerr(outs[r].grads[l].bias, z[f"tp_r{r}_l{l}_g_bias"]) <= 1e-4
            assert nerr(outs[r].deltas[l], z[f"tp_r{r}_l{l}_delta"]) <= 1e-4


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 3e-2)])
@pytest.mark.parametrize("graph", [False, True])
def test_tp_engine_matches_dense_oracle(dtype, tol, graph):
    from paper_2508_00960_b200.tensor_parallel import TPEngine
    n, L, B, lr = 512, 4, 64, 3e-3
    rng = np.random.default_rng(5)
    a = np.sqrt(6.0 / (2 * n))
    W = [rng.uniform(-a, a, (n, n)) for _ in range(L)]
    b = [0.1 * rng.standard_normal(n) for _ in range(L)]
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = TPEngine(n, L, B, lr=lr, dtype=dtype)
    eng.load_full_weights(W, b)
    for par in (0, 1):
        eng.set_batch(torch.from_numpy(x.T.copy()).cuda(), torch.from_numpy(y.T.copy()).cuda(), par)
    if graph:
        eng.step(graph=False)
        eng.read_loss()
        eng.capture()
    steps = 3
    losses = [None] * steps
    for t in range(steps):
        eng.step(graph=graph)
        losses[t] = eng.read_loss()
    # dense oracle: full-batch SGD on the same weights (mean loss), one step per engine step
    Wd = [w.copy() for w in W]
    bd = [v.copy() for v in b]
    total = steps + (1 if graph else 0)
    ref = []
    for _ in range(total):
        out = po.tp_iteration([[{"weight": Wd[l], "bias": bd[l]} for l in range(L)]], ["relu"] * L, [x], [y], "mean")
        ref.append(out["global_loss"])
        for l in range(L):
            Wd[l] -= lr * out["grads"][0][l]["weight"]
            bd[l] -= lr * out["grads"][0][l]["bias"]
    ref = ref[-steps:]
    for g, r in zip(losses, ref):
        assert abs(g - r) <= tol * abs(r), (losses, ref)
    assert nerr(eng.Wa[0], Wd[0]) <= tol
    assert nerr(eng.Wb[1].t(), Wd[3].T) <= tol
