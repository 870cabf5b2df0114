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


def test_fp32_arithmetic_drift_on_c1_training():
    """Why the fp32 tier's C1 training curves are held to 5e-3 per epoch (tests/
    test_train_engine_gpu.py), not 1e-4: the same training loop in EXACT fp32 arithmetic on the
    CPU (this restatement, no tensor cores) already drifts from float64 by more than 1e-4 by the
    second epoch — the reference problem amplifies rounding — while staying inside 5e-3.  The
    float64 run itself reproduces the reference's golden curve (tests/golden/c1.npz)."""
    import os
    from paper_2508_00960_b200.phantom import _reference_init_arrays
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1.npz"))
    n, p, k, L, B, seed = (int(v) for v in gold["cfg"])
    s = n // p
    model = []
    for j in range(p):
        row = []
        for l in range(L):
            loc, comp, decs = _reference_init_arrays(n, p, k, L, seed, j, l)
            row.append({"local": loc, "compressor": comp, "decompressors": decs, "bias": np.zeros(s)})
        model.append(row)
    x, y, _ = po.gen_dataset(n, 1024, seed)
    h64 = tc.train_sgd_curve(model, x, y, L, B, 1e-4, 3, torch.float64)
    h32 = tc.train_sgd_curve(model, x, y, L, B, 1e-4, 3, torch.float32)
    np.testing.assert_allclose(h64, gold["train_sgd_hist"], rtol=1e-10)
    drift = [abs(a - b) / b for a, b in zip(h32, h64)]
    print("fp32 vs fp64 epoch drift:", drift)
    assert max(drift) > 1e-4          # 1e-4 per epoch is out of reach of fp32 arithmetic itself
    assert max(drift) < 5e-3
