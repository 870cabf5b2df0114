"""Pin the CPU oracle (oracle/phantom_oracle.py) against the reference's own outputs.

Golden vectors in tests/golden/*.npz were produced by the unmodified reference
(tests/golden/make_golden.py); the hand-worked cases restate the reference tests' known answers
(test_phantom.py:13-36, 106-121, 144-149, 185-198; test_collectives.py:22-60).
"""
import os

import numpy as np
import pytest

from oracle import phantom_oracle as po

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _tiny():
    return np.load(os.path.join(GOLD, "tiny.npz"))


def _tiny_cases(z):
    i = 0
    while f"c{i}_cfg" in z:
        yield i
        i += 1


def _model_from(z, pre, p, L, s, k):
    model = []
    for r in range(p):
        own = []
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            dec = z[q + "w_dec"]
            peers = [i for i in range(p) if i != r]
            own.append({"local": z[q + "w_local"].copy(), "compressor": z[q + "w_comp"].copy(),
                        "decompressors": {i: dec[qi].copy() for qi, i in enumerate(peers)},
                        "bias": np.zeros(s)})
        model.append(own)
    return model


def test_init_matches_reference_tiny():
    z = _tiny()
    for ci in _tiny_cases(z):
        n, p, k, L, B, seed = (int(v) for v in z[f"c{ci}_cfg"])
        model = po.init_phantom_model(n, p, k, L, seed)
        for r in range(p):
            for l in range(L):
                q = f"c{ci}_r{r}_l{l}_"
                assert np.array_equal(model[r][l]["local"], z[q + "w_local"])
                assert np.array_equal(model[r][l]["compressor"], z[q + "w_comp"])
                dec = model[r][l]["decompressors"]
                got = np.stack([dec[i] for i in sorted(dec)]) if dec else np.zeros((0, n // p, k))
                assert np.array_equal(got, z[q + "w_dec"])


@pytest.mark.parametrize("ci", range(9))
def test_pp_iteration_matches_reference(ci):
    z = _tiny()
    n, p, k, L, B, seed = (int(v) for v in z[f"c{ci}_cfg"])
    act = str(z[f"c{ci}_act"])
    red = str(z[f"c{ci}_red"])
    s = n // p
    pre = f"c{ci}_"
    model = _model_from(z, pre, p, L, s, k)
    x, y = z[pre + "x"], z[pre + "y"]
    res = po.pp_iteration(model, [act] * L, [x[r * s:(r + 1) * s] for r in range(p)],
                          [y[r * s:(r + 1) * s] for r in range(p)], red)
    tol = dict(rtol=1e-12, atol=1e-13)
    assert res["global_loss"] == pytest.approx(float(z[pre + "global_loss"]), rel=1e-13)
    for r in range(p):
        np.testing.assert_allclose(res["y_out"][r], z[f"{pre}r{r}_y_out"], **tol)
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            g = res["grads"][r][l]
            np.testing.assert_allclose(g["local"], z[q + "g_local"], **tol)
            np.testing.assert_allclose(g["compressor"], z[q + "g_comp"], **tol)
            np.testing.assert_allclose(g["bias"], z[q + "g_bias"], **tol)
            dec = g["decompressors"]
            got = np.stack([dec[i] for i in sorted(dec)]) if dec else np.zeros((0, s, k))
            np.testing.assert_allclose(got, z[q + "g_dec"], **tol)
            np.testing.assert_allclose(res["deltas"][r][l], z[q + "delta"], **tol)
            np.testing.assert_allclose(res["tapes"][r][l]["preact"], z[q + "preact"], **tol)
            np.testing.assert_allclose(np.stack([res["tapes"][r][l]["phantoms"][i] for i in range(p)]),
                                       z[q + "phantoms"], **tol)
            np.testing.assert_allclose(res["received"][r][l], z[q + "received"], **tol)
    # forward equals the dense twin (test_acceptance.py:30-61 criterion)
    dense = po.dense_forward([po.effective_weight(model, l) for l in range(L)],
                             [np.zeros(n)] * L, [act] * L, x)
    np.testing.assert_allclose(dense, z[pre + "dense_out"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(np.concatenate(res["y_out"]), dense, rtol=1e-10, atol=1e-10)


def test_tp_iteration_matches_reference():
    z = _tiny()
    n, p, L, B, seed = (int(v) for v in z["tp_cfg"])
    s = n // p
    model = po.init_tp_model(n, p, L, seed)
    x, y = z["tp_x"], z["tp_y"]
    res = po.tp_iteration(model, ["relu"] * L, [x[r * s:(r + 1) * s] for r in range(p)],
                          [y[r * s:(r + 1) * s] for r in range(p)])
    assert res["global_loss"] == pytest.approx(float(z["tp_global_loss"]), rel=1e-13)
    for r in range(p):
        np.testing.assert_allclose(res["y_out"][r], z[f"tp_r{r}_y_out"], rtol=1e-12, atol=1e-13)
        for l in range(L):
            np.testing.assert_allclose(res["grads"][r][l]["weight"], z[f"tp_r{r}_l{l}_g_weight"],
                                       rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(res["deltas"][r][l], z[f"tp_r{r}_l{l}_delta"], rtol=1e-12, atol=1e-13)


def test_model_sizes():
    z = _tiny()
    for case, val in zip(z["size_cases"], z["size_values"]):
        assert po.pp_model_size(*(int(c) for c in case)) == int(val)
    assert po.valid_k(16384, 8) == (2048, 1792.0)


def test_c1_iteration_matches_reference():
    c1 = np.load(os.path.join(GOLD, "c1.npz"))
    n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
    s = n // p
    inputs, targets, teacher = po.gen_dataset(n, 1024, seed)
    assert float(teacher.sum()) == pytest.approx(float(c1["teacher_sum"]), rel=1e-12)
    x, y = inputs[:, :B], targets[:, :B]
    assert float(x.sum()) == pytest.approx(float(c1["x_sum"]), rel=1e-12)
    assert float((y * y).sum()) == pytest.approx(float(c1["y_sq"]), rel=1e-12)
    model = po.init_phantom_model(n, p, k, L, seed)
    res = po.pp_iteration(model, ["relu"] * L, [x[r * s:(r + 1) * s] for r in range(p)],
                          [y[r * s:(r + 1) * s] for r in range(p)], "mean")
    assert res["global_loss"] == pytest.approx(float(c1["global_loss"]), rel=1e-11)
    for r in range(p):
        np.testing.assert_allclose(res["y_out"][r].ravel()[c1[f"r{r}_y_idx"]], c1[f"r{r}_y_val"], rtol=1e-10)
        for l in range(L):
            q = f"r{r}_l{l}_"
            lay, g = model[r][l], res["grads"][r][l]
            arrs = {"w_local": lay["local"], "w_comp": lay["compressor"],
                    "w_dec": np.stack([lay["decompressors"][i] for i in sorted(lay["decompressors"])]),
                    "g_local": g["local"], "g_comp": g["compressor"],
                    "g_dec": np.stack([g["decompressors"][i] for i in sorted(g["decompressors"])]),
                    "g_bias": g["bias"], "delta": res["deltas"][r][l], "received": res["received"][r][l],
                    "preact": res["tapes"][r][l]["preact"]}
            for name, a in arrs.items():
                np.testing.assert_allclose(a.ravel()[c1[q + name + "_idx"]], c1[q + name + "_val"],
                                           rtol=1e-9, atol=1e-12, err_msg=q + name)
                assert np.linalg.norm(a) == pytest.approx(float(c1[q + name + "_norm"]), rel=1e-10)


def test_c1_training_curve_matches_reference():
    c1 = np.load(os.path.join(GOLD, "c1.npz"))
    n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
    inputs, targets, _ = po.gen_dataset(n, 1024, seed)
    model = po.init_phantom_model(n, p, k, L, seed)
    hist = po.train_pp(model, ["relu"] * L, inputs, targets, B, 1e-4, 3, "mean", "sgd")
    np.testing.assert_allclose(hist, c1["train_sgd_hist"], rtol=1e-10)
    model = po.init_phantom_model(n, p, k, L, seed)
    hist = po.train_pp(model, ["relu"] * L, inputs, targets, B, 1e-4, 2, "mean", "adam")
    np.testing.assert_allclose(hist, c1["train_adam_hist"], rtol=1e-10)


# ---- hand-worked known answers from the reference tests -----------------------------------
def worked_example():
    """test_phantom.py:13-20 — p=2, k=1, n=4, identity."""
    r0 = {"local": np.eye(2), "compressor": np.array([[0.5, 0.5]]),
          "decompressors": {1: np.array([[1.0], [2.0]])}, "bias": np.zeros(2)}
    r1 = {"local": np.eye(2), "compressor": np.array([[1.0, 0.0]]),
          "decompressors": {0: np.array([[0.0], [0.0]])}, "bias": np.zeros(2)}
    return [[r0], [r1]]


def test_worked_forward_example():
    m = worked_example()
    outs, tapes = po.pp_forward_layer([m[0][0], m[1][0]], [np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])],
                                      po.IDENTITY)
    np.testing.assert_array_equal(outs[0], [[4.0], [8.0]])
    np.testing.assert_array_equal(outs[1], [[3.0], [4.0]])
    np.testing.assert_array_equal(tapes[0]["phantoms"][0], [[1.5]])
    np.testing.assert_array_equal(tapes[0]["phantoms"][1], [[3.0]])


def test_output_delta_hand_cases():
    y = np.array([[1.0, 2.0]])
    assert not po.pp_output_delta(y, y, y, po.IDENTITY).any()
    out = po.pp_output_delta(np.array([[5.0], [5.0]]), np.zeros((2, 1)), np.array([[-1.0], [3.0]]), po.RELU)
    np.testing.assert_array_equal(out, [[0.0], [5.0]])
    # ReLU'(0) = 0 (core.py:79-81)
    assert po.pp_output_delta(np.array([[1.0]]), np.zeros((1, 1)), np.zeros((1, 1)), po.RELU)[0, 0] == 0.0


def test_param_grads_outer_product_hand_case():
    """test_phantom.py:185-198."""
    layer = {"local": np.zeros((2, 2)), "compressor": np.zeros((1, 2)),
             "decompressors": {1: np.zeros((2, 1))}, "bias": np.zeros(2)}
    tape = {"inputs": np.array([[2.0], [3.0]]), "preact": np.zeros((2, 1)),
            "phantoms": {0: np.zeros((1, 1)), 1: np.array([[4.0]])}}
    g = po.pp_param_grads(layer, np.array([[1.0], [0.0]]), tape, np.array([[7.0]]))
    np.testing.assert_array_equal(g["local"], [[2.0, 3.0], [0.0, 0.0]])
    np.testing.assert_array_equal(g["bias"], [1.0, 0.0])
    np.testing.assert_array_equal(g["compressor"], [[14.0, 21.0]])
    np.testing.assert_array_equal(g["decompressors"][1], [[4.0], [0.0]])


def test_single_rank_backward_hand_case():
    """test_phantom.py:144-149."""
    layer = {"local": np.array([[2.0]]), "compressor": np.array([[1.0]]), "decompressors": {}, "bias": np.zeros(1)}
    out = po.pp_backward_layer(layer, np.array([[3.0]]), np.array([[1.0]]), po.IDENTITY, np.zeros((1, 1)))
    np.testing.assert_array_equal(out, [[6.0]])


def test_reduce_scatter_semantics():
    """test_collectives.py:50-60: rank j receives the ascending sum of slot j."""
    layers = [{"decompressors": {1: np.array([[1.0]])}, "compressor": np.zeros((1, 1))},
              {"decompressors": {0: np.array([[10.0]])}, "compressor": np.zeros((1, 1))}]
    rec = po.pp_exchange_error_phantoms(layers, [np.array([[2.0]]), np.array([[3.0]])])
    np.testing.assert_array_equal(rec[0], [[30.0]])   # rank 1's D_0^T delta_1 = 10 * 3
    np.testing.assert_array_equal(rec[1], [[2.0]])    # rank 0's D_1^T delta_0 = 1 * 2


def test_flop_formula_matches_closed_form():
    # 6 L B s (s + p k) - 2 B s (s + k) at C3 (2.401 TFLOP per rank per step)
    f = po.pp_gemm_flops_per_rank(16384, 8, 128, 8, 8192)
    assert f == pytest.approx(2.401e12, rel=1e-3)
