"""Pins oracle/teacher.py (the torch restatement the GPU parity tests use at benchmarked sizes)
against the float64 oracle (itself pinned to the reference's golden vectors, test_oracle.py):
every per-layer function, fed the oracle's own tape, in float64 on the CPU, to 1e-12."""
import numpy as np
import pytest
import torch

from oracle import phantom_oracle as po
from oracle import teacher as tc


def _t(a):
    """oracle (features x batch) -> teacher [batch, features] float64 tensor."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T))


def _W(lay, j, p):
    return {"local": torch.from_numpy(lay["local"]), "compressor": torch.from_numpy(lay["compressor"]),
            "dec": torch.stack([torch.from_numpy(lay["decompressors"][i]) for i in range(p) if i != j]),
            "bias": torch.from_numpy(lay["bias"])}


@pytest.mark.parametrize("n,p,k,L,B", [(64, 4, 4, 3, 5), (48, 2, 3, 2, 7), (96, 8, 2, 2, 3)])
def test_teacher_matches_oracle(n, p, k, L, B):
    model = po.init_phantom_model(n, p, k, L, seed=11)
    rng = np.random.default_rng(5)
    for row in model:
        for lay in row:
            lay["bias"] = 0.1 * rng.standard_normal(lay["bias"].shape)
    s = n // p
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    xs = [x[j * s:(j + 1) * s] for j in range(p)]
    ys = [y[j * s:(j + 1) * s] for j in range(p)]
    ref = po.pp_iteration(model, ["relu"] * L, xs, ys, "mean")
    tol = 1e-12
    total = 0.0
    for l in range(L):
        Ws = [_W(model[j][l], j, p) for j in range(p)]
        Y = [_t(ref["tapes"][j][l]["inputs"]) for j in range(p)]
        G = [tc.compress(Ws[j], Y[j]) for j in range(p)]
        for j in range(p):
            assert tc.nerr(G[j], _t(ref["tapes"][j][l]["phantoms"][j])) < tol
            pre, out = tc.forward_layer(Ws[j], j, Y[j], G)
            assert tc.nerr(pre, _t(ref["tapes"][j][l]["preact"])) < tol
            nxt = ref["tapes"][j][l + 1]["inputs"] if l + 1 < L else ref["y_out"][j]
            assert tc.nerr(out, _t(nxt)) < tol
            if l == L - 1:
                loss, d = tc.loss_and_delta(out, pre, _t(ys[j]), "mean")
                total += loss
                assert abs(loss - ref["local_loss"][j]) <= tol * abs(ref["local_loss"][j])
                assert tc.nerr(d, _t(ref["deltas"][j][l])) < tol
        D = [_t(ref["deltas"][j][l]) for j in range(p)]
        R = tc.error_phantoms(Ws, D)
        for j in range(p):
            assert tc.nerr(R[j], _t(ref["received"][j][l])) < tol
            g = tc.param_grads(j, D[j], Y[j], G, R[j])
            want = ref["grads"][j][l]
            assert tc.nerr(g["local"], torch.from_numpy(want["local"])) < tol
            assert tc.nerr(g["compressor"], torch.from_numpy(want["compressor"])) < tol
            assert tc.nerr(g["bias"], torch.from_numpy(want["bias"])) < tol
            for q, i in enumerate(i for i in range(p) if i != j):
                assert tc.nerr(g["dec"][q], torch.from_numpy(want["decompressors"][i])) < tol
            if l > 0:
                d_prev = tc.backward_delta(Ws[j], D[j], R[j], Y[j])
                assert tc.nerr(d_prev, _t(ref["deltas"][j][l - 1])) < tol
    assert abs(total - ref["global_loss"]) <= tol * abs(ref["global_loss"])
