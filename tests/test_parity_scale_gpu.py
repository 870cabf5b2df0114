"""Gradient-level bf16 parity at the BENCHMARKED shapes, teacher-forced (oracle/teacher.py, pinned
to the float64 oracle by tests/test_teacher.py).

One eager training step of the default launch plan is captured (every layer's delta, the raw fp32
weight gradients from the optimizer epilogue, the received error phantoms, the gathered phantoms
and the activations) and each layer's kernels are checked against an fp32 torch restatement of
phantom.py fed the engine's own inputs of that layer:

  * C3 (n=16384, L=8, p=8, k=128, B=8192) with all 8 logical ranks grouped per launch — exactly
    what bench.py times on one GPU (fused compression+forward launches, grouped error compression,
    grouped weight gradients with the SGD epilogue, grouped recurrence);
  * C3 with one logical rank per launch (group=1) — the per-GPU launch shapes of the 8-GPU run
    (per-rank forward, per-rank weight-gradient + recurrence LPT launches at s=2048);
  * a C4 slice (n=65536, p=8, k=256, s=8192: L=2, B=1024);
  * C5 inference (fused train=False forward and the unfused path for k not a multiple of 64).

Stated bf16-tier tolerances (normwise relative, per layer and rank): tensors the engine stores in
bf16 (phantoms, activations, deltas, received error phantoms) <= 5e-3 (= 2.5 bf16 ulps; rounding
alone gives ~1.1e-3); raw fp32 weight gradients and the loss <= 1e-4 (fp32 accumulation order
only); bias gradients (column sums of the fp32 delta before its bf16 store) <= 5e-3.  Each test
also asserts that the phantom terms are large enough for a single dropped slot to exceed the
tolerance by 4x, so a lost all-gather slot, a wrong reduce-scatter slot or a zero gradient fails.
"""
import pytest
import torch

from oracle import teacher as tc

pytestmark = pytest.mark.gpu

TOL_BF16 = 5e-3
TOL_FP32 = 1e-4
BF16_KEYS = ("phantoms", "activations", "output", "delta_out", "received", "delta", "grad_bias")
FP32_KEYS = ("grad_local", "grad_compressor", "grad_decompressor", "loss")


def _engine(n, p, k, L, B, **kw):
    from paper_2508_00960_b200.engine import PhantomEngine
    torch.backends.cuda.matmul.allow_tf32 = False
    eng = PhantomEngine(n, p, k, L, B, lr=1e-3, capture=True, store_output=True, **kw)
    g = torch.Generator(device="cuda").manual_seed(7)
    eng.bias.copy_(0.05 * torch.randn(eng.bias.shape, generator=g, device="cuda"))
    xs = [torch.randn((B, eng.s), generator=g, device="cuda").bfloat16() for _ in range(p)]
    ts = [torch.randn((B, eng.s), generator=g, device="cuda").clamp_min(0).bfloat16() for _ in range(p)]
    for par in (0, 1):
        eng.set_batch(xs, ts, par)
    return eng, ts


def _step_and_check(eng, ts, steps=2, sensitivity=True):
    for _ in range(steps - 1):      # a warm step first: the checked step reads updated weights
        eng.step(graph=False)
    par = eng.parity
    bias0 = eng.bias.clone()
    eng.step(graph=False)
    loss = eng.read_loss()
    worst, share = tc.check_engine_step(eng, par, bias0, ts, loss)
    print({k: f"{v:.2e}" for k, v in worst.items()}, share)
    for key in BF16_KEYS:
        assert worst[key] <= TOL_BF16, (key, worst)
    for key in FP32_KEYS:
        assert worst[key] <= TOL_FP32, (key, worst)
    # sensitivity: one dropped phantom slot (1/(p-1) of the phantom term) must exceed 4x tolerance
    if sensitivity:
        for key in ("forward", "backward"):
            assert share[key] / (eng.p - 1) > 4 * TOL_BF16, (key, share)
    return worst


@pytest.mark.parametrize("n,p,k,L,B,kw", [
    (512, 4, 32, 3, 64, {}),            # 1-SM kernel (k not a multiple of 64), grouped launches
    (1024, 2, 16, 4, 64, {}),           # C1 shapes in bf16
    (512, 4, 64, 3, 256, {"group": 1}),  # per-rank launches, [error compression + wgrad] fused, small
    (512, 4, 64, 3, 256, {"group": 1, "k3_fused": False}),  # per-rank, [wgrad + recurrence] fused
    (768, 4, 24, 2, 96, {"fused": False}),   # ragged k / batch tiles
    (512, 4, 64, 3, 256, {"mask_bits": False}),   # ReLU' mask from the bf16 activations
    (512, 4, 64, 2, 512, {"group": 1}),  # layer-0 compressor gradient split over the batch
])
def test_small_shapes_teacher_forced(n, p, k, L, B, kw):
    """The small engine-test shapes, checked kernel by kernel (what the float64 step comparisons
    in test_engine_gpu.py can only bound loosely in bf16)."""
    eng, ts = _engine(n, p, k, L, B, **kw)
    w = _step_and_check(eng, ts, sensitivity=False)
    assert w["grad_local"] <= TOL_FP32
    eng.close()


def test_c3_grouped_default_plan():
    eng, ts = _engine(16384, 8, 128, 8, 8192)
    assert eng.fused and eng.group == 8 and not eng.bwd_fused
    _step_and_check(eng, ts)
    eng.close()


@pytest.mark.parametrize("plan", ["k3_fused", "bwd_fused"])
def test_c3_one_rank_per_launch(plan):
    """k3_fused (default): [error compression + weight gradients] LPT launch per rank, then the
    recurrence; bwd_fused: error compression, then [weight gradients + recurrence] per rank."""
    eng, ts = _engine(16384, 8, 128, 8, 8192, group=1, k3_fused=plan == "k3_fused")
    assert eng.group == 1 and not eng.fused
    assert (eng.k3_fused, eng.bwd_fused) == ((True, False) if plan == "k3_fused" else (False, True))
    _step_and_check(eng, ts)
    eng.close()


def test_c4_slice():
    eng, ts = _engine(65536, 8, 256, 2, 1024)
    assert eng.fused
    _step_and_check(eng, ts)
    eng.close()


@pytest.mark.parametrize("k", [32, 128, 512])
def test_c5_inference(k):
    """forward_only (config C5: n=16384, B=8192) against the teacher, layer by layer."""
    from paper_2508_00960_b200.engine import PhantomEngine
    torch.backends.cuda.matmul.allow_tf32 = False
    n, p, L, B = 16384, 8, 3, 8192
    eng = PhantomEngine(n, p, k, L, B, lr=1e-3)
    assert eng.fused == (k % 64 == 0)
    g = torch.Generator(device="cuda").manual_seed(3)
    eng.bias.copy_(0.05 * torch.randn(eng.bias.shape, generator=g, device="cuda"))
    xs = [torch.randn((B, eng.s), generator=g, device="cuda").bfloat16() for _ in range(p)]
    eng.set_batch(xs, xs, 0)
    outs = eng.forward_only(0)
    torch.cuda.synchronize()
    worst = {"phantoms": 0.0, "activations": 0.0}
    for l in range(L):
        Ws = [tc.engine_weights(eng, j, l, 0) for j in range(p)]
        G = [eng.phantoms_view(l)[i].float() for i in range(p)]
        for j in range(p):
            Y = eng.Y[0][j][l].float()
            worst["phantoms"] = max(worst["phantoms"], tc.nerr(G[j], tc.compress(Ws[j], Y)))
            _, out = tc.forward_layer(Ws[j], j, Y, G)
            got = outs[j] if l == L - 1 else eng.Y[0][j][l + 1]
            worst["activations"] = max(worst["activations"], tc.nerr(got, out))
    print(worst)
    assert max(worst.values()) <= TOL_BF16, worst
    eng.close()
