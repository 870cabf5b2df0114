"""The on-device training loop (training.train_engine) against the reference's own
C1 training curves (tests/golden/c1.npz: phantomsim.train, 1024 samples, B=64, lr=1e-4, mean):
fp32 tier within 1e-4 per iteration (while trajectories are close) and 5e-3 per epoch, bf16
tier within 2e-2; TrainConfig semantics (stop at target,
iteration counts) and the TP comparison loop."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _c1():
    return np.load(os.path.join(GOLD, "c1.npz"))


def _cfg(optimizer, epochs, dtype, target=None):
    from paper_2508_00960_b200.training import TrainConfig
    c1 = _c1()
    n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
    return TrainConfig(mode="pp", n=n, p=p, layers=L, k=k, batch=B, lr=1e-4, optimizer=optimizer, max_epochs=epochs,
                       seed=seed, loss_reduction="mean", dtype=dtype, target_loss=target)


def _ref_iters():
    return np.load(os.path.join(GOLD, "c1_train.npz"))


@pytest.mark.parametrize("optimizer, epochs, key", [("sgd", 3, "train_sgd_hist"), ("adam", 2, "train_adam_hist")])
def test_c1_curve_fp32_tier(optimizer, epochs, key):
    """Iteration losses match the reference within 1e-4 while the trajectories are still close;
    this training problem amplifies ~1e-6 per-step rounding differences ~10x every few steps
    (the f64 reference itself moves 4e-5 by step 16 under a 1e-7 weight perturbation), so the
    later epoch means are held to 5e-3."""
    from paper_2508_00960_b200.training import gen_dataset, train_engine
    cfg = _cfg(optimizer, epochs, torch.float32)
    data = gen_dataset(cfg.n, 1024, cfg.seed)
    res = train_engine(cfg, data)
    assert res.epochs_run == epochs and res.iterations_run == epochs * (1024 // cfg.batch)
    it_ref = _ref_iters()[f"{optimizer}_iter_losses"]
    got = np.array(res.cost["iteration_losses"][:6])
    assert np.all(np.abs(got - it_ref[:6]) <= 1e-4 * it_ref[:6]), (got, it_ref[:6])
    ref = _c1()[key]
    for e, (g, w) in enumerate(zip(res.loss_history, ref)):
        assert abs(g - w) <= 5e-3 * w, (e, res.loss_history, ref)
    assert res.cost["seconds"] > 0 and res.cost["samples_per_s"] > 0


def test_c1_curve_bf16_tier():
    from paper_2508_00960_b200.training import gen_dataset, train_engine
    cfg = _cfg("sgd", 3, torch.bfloat16)
    res = train_engine(cfg, gen_dataset(cfg.n, 1024, cfg.seed))
    it_ref = _ref_iters()["sgd_iter_losses"]
    got = np.array(res.cost["iteration_losses"][:6])
    assert np.all(np.abs(got - it_ref[:6]) <= 2e-2 * it_ref[:6]), (got, it_ref[:6])
    for got, want in zip(res.loss_history, _c1()["train_sgd_hist"]):
        assert abs(got - want) <= 2e-2 * want


def test_stop_at_target():
    from paper_2508_00960_b200.training import gen_dataset, train_engine
    ref = _c1()["train_sgd_hist"]
    cfg = _cfg("sgd", 10, torch.float32, target=float(ref[1]) * 1.01)
    res = train_engine(cfg, gen_dataset(cfg.n, 1024, cfg.seed))
    assert res.converged and res.epochs_run == 2


def test_tp_loop_trains():
    from paper_2508_00960_b200.training import TrainConfig, gen_dataset, train_engine
    cfg = TrainConfig(mode="tp", n=256, p=1, layers=2, batch=64, lr=1e-3, max_epochs=3, seed=0,
                      loss_reduction="mean", dtype=torch.float32)
    res = train_engine(cfg, gen_dataset(256, 256, 0))
    assert res.epochs_run == 3 and res.loss_history[-1] < res.loss_history[0]
