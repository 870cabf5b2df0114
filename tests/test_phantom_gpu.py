"""GPU parity of the drop-in API (phantom.py / training.py) against the reference's golden
vectors (tests/golden, produced by phantomsim itself) and the pinned CPU oracle.

Tolerances (normwise ||gpu - ref|| / ||ref|| per tensor, SURVEY §7 "hard parts"):
  * fp32 tier (3xTF32 tcgen05):  1e-4 for activations, deltas, gradients and losses (north_star).
  * bf16 tier: 5e-2 forward activations / losses; 5e-2 gradients on identity-activation
    stacks (ReLU mask flips near preact = 0 make elementwise gradient parity ill-posed in bf16).
"""
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
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def _tiny():
    return np.load(os.path.join(GOLD, "tiny.npz"))


def _model_np(z, pre, p, L, s):
    rows = []
    for r in range(p):
        own = []
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            dec = z[q + "w_dec"]
            peers = [i for i in range(p) if i != r]
            own.append({"local": z[q + "w_local"], "compressor": z[q + "w_comp"],
                        "decompressors": {i: dec[qi] for qi, i in enumerate(peers)}, "bias": np.zeros(s)})
        rows.append(own)
    return rows


def run_api_iteration(z, ci, dtype):
    from paper_2508_00960_b200.collectives import Communicator
    from paper_2508_00960_b200.phantom import model_from_numpy
    from paper_2508_00960_b200.training import pp_iteration
    n, p, k, L, B, seed = (int(v) for v in z[f"c{ci}_cfg"])
    act = str(z[f"c{ci}_act"])
    red = str(z[f"c{ci}_red"])
    s = n // p
    pre = f"c{ci}_"
    model = model_from_numpy(_model_np(z, pre, p, L, s), n, p, k, [act] * L, dtype=dtype)
    x = torch.from_numpy(z[pre + "x"]).cuda().to(dtype)
    y = torch.from_numpy(z[pre + "y"]).cuda().to(dtype)
    comm = Communicator(p)
    outs = comm.run(lambda c, r: pp_iteration(c, r, model.rank_layers[r], model.activations,
                                              x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], red))
    torch.cuda.synchronize()
    return outs, comm, (n, p, k, L, B, act)


@pytest.mark.parametrize("ci", range(9))
def test_pp_iteration_fp32_tier_matches_reference(ci):
    z = _tiny()
    outs, comm, (n, p, k, L, B, act) = run_api_iteration(z, ci, torch.float32)
    pre = f"c{ci}_"
    tol = 1e-4
    assert abs(outs[0].global_loss - float(z[pre + "global_loss"])) <= tol * max(1.0, abs(float(z[pre + "global_loss"])))
    for r in range(p):
        assert nerr(outs[r].y_out, z[f"{pre}r{r}_y_out"]) <= tol
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            g = outs[r].grads[l]
            assert nerr(g.local, z[q + "g_local"]) <= tol, (r, l, "local")
            assert nerr(g.compressor, z[q + "g_comp"]) <= tol, (r, l, "comp")
            assert nerr(g.bias, z[q + "g_bias"]) <= tol, (r, l, "bias")
            if p > 1:
                dec = torch.stack([g.decompressors[i] for i in sorted(g.decompressors)])
                assert nerr(dec, z[q + "g_dec"]) <= tol, (r, l, "dec")
            assert nerr(outs[r].deltas[l], z[q + "delta"]) <= tol, (r, l, "delta")
            assert nerr(outs[r].tape[l].preact, z[q + "preact"]) <= tol
            assert nerr(outs[r].tape[l].phantom_grad, z[q + "received"]) <= tol
    # Table I schedule (test_acceptance.py:189-223): L all-gathers, 1 loss all-reduce, L reduce-scatters
    kinds = [rec.collective.value for rec in comm.records]
    assert kinds == ["all_gather"] * L + ["all_reduce"] + ["reduce_scatter"] * L
    assert all(rec.message_size == k * B for rec in comm.records if rec.collective.value != "all_reduce")


@pytest.mark.parametrize("ci", [0, 1, 7])   # identity-activation stacks
def test_pp_iteration_bf16_tier_identity(ci):
    z = _tiny()
    outs, _, (n, p, k, L, B, act) = run_api_iteration(z, ci, torch.bfloat16)
    pre = f"c{ci}_"
    for r in range(p):
        assert nerr(outs[r].y_out, z[f"{pre}r{r}_y_out"]) <= 5e-2
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            assert nerr(outs[r].grads[l].local, z[q + "g_local"]) <= 5e-2
            assert nerr(outs[r].deltas[l], z[q + "delta"]) <= 5e-2


@pytest.mark.parametrize("ci", [3, 5, 6])   # relu stacks: forward + loss
def test_pp_forward_bf16_tier_relu(ci):
    z = _tiny()
    outs, _, (n, p, k, L, B, act) = run_api_iteration(z, ci, torch.bfloat16)
    pre = f"c{ci}_"
    assert abs(outs[0].global_loss - float(z[pre + "global_loss"])) <= 5e-2 * abs(float(z[pre + "global_loss"]))
    for r in range(p):
        assert nerr(outs[r].y_out, z[f"{pre}r{r}_y_out"]) <= 5e-2


def test_worked_example_exact():
    """test_phantom.py:13-36 hand case, fp32 tier."""
    from paper_2508_00960_b200.collectives import Communicator
    from paper_2508_00960_b200.core import Activation
    from paper_2508_00960_b200.phantom import PhantomLayer, pp_forward_layer
    r0 = PhantomLayer(np.eye(2), np.array([[0.5, 0.5]]), {1: np.array([[1.0], [2.0]])}, np.zeros(2),
                      dtype=torch.float32)
    r1 = PhantomLayer(np.eye(2), np.array([[1.0, 0.0]]), {0: np.array([[0.0], [0.0]])}, np.zeros(2),
                      dtype=torch.float32)
    layers = [r0, r1]
    inputs = [torch.tensor([[1.0], [2.0]], device="cuda"), torch.tensor([[3.0], [4.0]], device="cuda")]
    tapes = [[], []]
    comm = Communicator(2)
    outs = comm.run(lambda c, r: pp_forward_layer(layers[r], inputs[r], c, r, tapes[r],
                                                  activation=Activation.IDENTITY))
    assert outs[0].cpu().tolist() == [[4.0], [8.0]]
    assert outs[1].cpu().tolist() == [[3.0], [4.0]]
    assert tapes[0][0].phantoms[0].cpu().tolist() == [[1.5]]
    assert tapes[0][0].phantoms[1].cpu().tolist() == [[3.0]]


def test_c1_iteration_fp32_tier_vs_oracle():
    """Config C1 (n=1024, p=2, k=16, L=4, B=64, mean): reference init and data."""
    from paper_2508_00960_b200.collectives import Communicator
    from paper_2508_00960_b200.phantom import init_phantom_model
    from paper_2508_00960_b200.training import pp_iteration
    c1 = np.load(os.path.join(GOLD, "c1.npz"))
    n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
    s = n // p
    inputs, targets, _ = po.gen_dataset(n, 1024, seed)
    x, y = inputs[:, :B], targets[:, :B]
    ref = po.pp_iteration(po.init_phantom_model(n, p, k, L, seed), ["relu"] * L,
                          [x[r * s:(r + 1) * s] for r in range(p)], [y[r * s:(r + 1) * s] for r in range(p)], "mean")
    model = init_phantom_model(n, p, k, L, seed=seed, dtype=torch.float32)
    xd = torch.from_numpy(x).cuda().float()
    yd = torch.from_numpy(y).cuda().float()
    outs = Communicator(p).run(lambda c, r: pp_iteration(c, r, model.rank_layers[r], model.activations,
                                                         xd[r * s:(r + 1) * s], yd[r * s:(r + 1) * s], "mean"))
    assert abs(outs[0].global_loss - ref["global_loss"]) <= 1e-4 * ref["global_loss"]
    assert outs[0].global_loss == pytest.approx(float(c1["global_loss"]), rel=1e-4)
    for r in range(p):
        assert nerr(outs[r].y_out, ref["y_out"][r]) <= 1e-4
        for l in range(L):
            g, gr = outs[r].grads[l], ref["grads"][r][l]
            assert nerr(g.local, gr["local"]) <= 1e-4
            assert nerr(g.compressor, gr["compressor"]) <= 1e-4
            assert nerr(g.bias, gr["bias"]) <= 1e-4
            for i in gr["decompressors"]:
                assert nerr(g.decompressors[i], gr["decompressors"][i]) <= 1e-4
            assert nerr(outs[r].deltas[l], ref["deltas"][r][l]) <= 1e-4


@pytest.mark.parametrize("mode", ["lockstep", "threads"])
def test_effective_weight_and_schedulers(mode):
    """reference.py:143-157 effective weight (block (j, i) = D_{i->j} . C_i) of the reference-init
    model vs the oracle, and one pp_iteration under both schedulers of the Communicator (the
    reference default is lockstep): identical results and record streams."""
    import paper_2508_00960_b200 as ps
    n, p, k, L, B = 64, 4, 3, 2, 5
    model = ps.init_phantom_model(n, p, k, L, seed=4, dtype=torch.float32)
    ref_model = po.init_phantom_model(n, p, k, L, 4)
    for l in range(L):
        assert nerr(ps.effective_weight(model, l), po.effective_weight(ref_model, l)) <= 1e-6
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, B))).cuda().float()
    y = torch.from_numpy(np.maximum(rng.standard_normal((n, B)), 0)).cuda().float()
    s = n // p
    comm = ps.Communicator(p, mode=mode)
    outs = comm.run(lambda c, r: ps.pp_iteration(c, r, model.rank_layers[r], model.activations,
                                                 x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], "mean"))
    ref = po.pp_iteration(ref_model, ["relu"] * L, [x[r * s:(r + 1) * s].double().cpu().numpy() for r in range(p)],
                          [y[r * s:(r + 1) * s].double().cpu().numpy() for r in range(p)], "mean")
    assert outs[0].global_loss == pytest.approx(ref["global_loss"], rel=1e-4)
    kinds = [(r.collective.value, r.message_size) for r in comm.records]
    assert kinds == [("all_gather", k * B)] * L + [("all_reduce", 1)] + [("reduce_scatter", k * B)] * L
