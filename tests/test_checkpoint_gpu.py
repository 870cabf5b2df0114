"""PSHARD01 interop on the GPU: reference-written checkpoints load into the
device models and the training engine and are written back byte for byte; an engine resumed
from save_state continues exactly like the uninterrupted run."""
import os

import numpy as np
import pytest
import torch

from paper_2508_00960_b200 import checkpoint as ck

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["pp_small.pshard", "pp_mixed.pshard", "tp_small.pshard"])
def test_model_round_trip_bytes(tmp_path, name):
    src = os.path.join(GOLD, name)
    model = ck.load_model(src)
    out = tmp_path / name
    ck.save_model(out, model)
    assert out.read_bytes() == open(src, "rb").read()


def _engine(optimizer="sgd", dtype=torch.float32, B=32):
    from paper_2508_00960_b200.engine import PhantomEngine
    return PhantomEngine(16, 4, 2, 2, B, optimizer=optimizer, lr=1e-2, dtype=dtype)


def test_engine_round_trip_bytes(tmp_path):
    src = os.path.join(GOLD, "pp_small.pshard")
    eng = _engine()
    seed = eng.load_checkpoint(src)
    assert seed == 3
    out = tmp_path / "eng.pshard"
    eng.save_checkpoint(out, seed)
    assert out.read_bytes() == open(src, "rb").read()
    eng.close()


def test_engine_checkpoint_matches_reference_model_views():
    eng = _engine()
    eng.load_checkpoint(os.path.join(GOLD, "pp_small.pshard"))
    arr = np.load(os.path.join(GOLD, "checkpoints.npz"))
    for jj, j in enumerate(eng.local):
        for l in range(eng.L):
            v = eng.layer_views(jj, l)
            assert np.array_equal(v["local"].double().cpu().numpy(), arr[f"pp_{j}_{l}_local"])
            assert np.array_equal(v["bias"].double().cpu().numpy(), arr[f"pp_{j}_{l}_bias"])
            for i, d in v["decompressors"].items():
                assert np.array_equal(d.double().cpu().numpy(), arr[f"pp_{j}_{l}_dec{i}"])
    eng.close()


def test_mismatched_engine_is_rejected():
    from paper_2508_00960_b200.engine import PhantomEngine
    from paper_2508_00960_b200.errors import ConfigurationError
    eng = PhantomEngine(16, 4, 1, 2, 16, dtype=torch.float32)
    with pytest.raises(ConfigurationError, match="does not match the engine"):
        eng.load_checkpoint(os.path.join(GOLD, "pp_small.pshard"))
    eng.close()


@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
def test_resume_continues_exactly(tmp_path, optimizer):
    B = 32
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn((B, 4), device="cuda", generator=g) for _ in range(4)]
    ts = [torch.randn((B, 4), device="cuda", generator=g).clamp_min(0) for _ in range(4)]
    a = _engine(optimizer, B=B)
    a.load_checkpoint(os.path.join(GOLD, "pp_small.pshard"))
    for par in (0, 1):
        a.set_batch(xs, ts, par)
    for _ in range(2):
        a.step(graph=False)
    path = tmp_path / "state.pshard"
    a.save_checkpoint(path, 3, optimizer_state=True)
    b = _engine(optimizer, B=B)
    b.load_checkpoint(path, optimizer_state=True)
    b.parity = a.parity
    for par in (0, 1):
        b.set_batch(xs, ts, par)
    assert b.t == a.t
    a.step(graph=False)
    b.step(graph=False)
    la, lb = a.read_loss(), b.read_loss()
    assert abs(la - lb) <= 1e-6 * max(1.0, abs(la))
    d = (a.master - b.master).abs().max().item()
    assert d <= 1e-6 * max(1.0, a.master.abs().max().item()), d
    a.close()
    b.close()
