"""Collective timing model (reference collectives.py:380-535): evaluation, file round trip,
least-squares fit with nonnegative c1/c2, and the fit's input checks."""
import math

import pytest

from paper_2508_00960_b200.collectives import Collective
from paper_2508_00960_b200.commmodel import (CollectiveCost, CommCostModel, FitError, comm_time, fit_comm_model,
                                             load_comm_model, load_measurements, save_comm_model, save_measurements)


def _synthetic(c1, c2, c3, kinds=tuple(Collective)):
    return [(k, m, p, c1 * math.log2(p) + c2 * m + c3) for k in kinds for p in (2, 4, 8) for m in (16, 4096, 1 << 20)]


def test_fit_recovers_exact_coefficients():
    model = fit_comm_model(_synthetic(7.5, 3e-4, 2.0))
    for c in model.costs.values():
        assert c.c1 == pytest.approx(7.5, rel=1e-9) and c.c2 == pytest.approx(3e-4, rel=1e-9)
        assert c.c3 == pytest.approx(2.0, abs=1e-6)


def test_fit_clamps_negative_latency():
    # times that fall with log2 p: the unconstrained c1 is negative -> pinned at zero
    s = [(Collective.ALL_GATHER, m, p, 5.0 + 1e-3 * m - 0.5 * math.log2(p)) for p in (2, 4, 8) for m in (1, 100, 10000)]
    c = fit_comm_model(s).costs[Collective.ALL_GATHER]
    assert c.c1 == 0.0 and c.c2 > 0


def test_round_trip_files(tmp_path):
    model = fit_comm_model(_synthetic(1.0, 2e-5, 3.0))
    save_comm_model(model, tmp_path / "m.ini")
    back = load_comm_model(tmp_path / "m.ini")
    for k in Collective:
        assert back.costs[k] == model.costs[k]
    samples = _synthetic(1.0, 2e-5, 3.0)
    save_measurements(samples, tmp_path / "s.csv")
    got = load_measurements(tmp_path / "s.csv")
    assert [(a, int(b), c) for a, b, c, _ in got] == [(a, int(b), c) for a, b, c, _ in samples]


def test_time_and_errors():
    m = CommCostModel({Collective.ALL_GATHER: CollectiveCost(2.0, 1e-3, 1.0)})
    assert comm_time(m, "all_gather", 1000, 4) == pytest.approx(2.0 * 2 + 1.0 + 1.0)
    with pytest.raises(Exception):
        comm_time(m, "reduce_scatter", 1, 2)
    with pytest.raises(FitError):
        fit_comm_model([(Collective.ALL_GATHER, 1, 2, 1.0), (Collective.ALL_GATHER, 2, 2, 2.0),
                        (Collective.ALL_GATHER, 3, 2, 3.0)])


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference tree not present")
@pytest.mark.parametrize("seed", range(4))
def test_fit_matches_reference_fitter(seed):
    """Same coefficients as phantomsim's fit_comm_model (lstsq, then scipy lsq_linear with the
    bounds when c1 or c2 come out negative) on noisy samples, some with a falling latency term."""
    import sys
    import numpy as np
    sys.path.insert(0, REF_SRC)
    from phantomsim import collectives as ref
    rng = np.random.default_rng(seed)
    samples = []
    for kind in Collective:
        c1 = rng.uniform(-5.0, 20.0) if seed % 2 else rng.uniform(0.0, 20.0)
        for p in (2, 4, 8):
            for m in (4, 1 << 10, 1 << 16, 1 << 22):
                samples.append((kind, m, p, max(0.5, c1 * math.log2(p) + 2e-5 * m + 8.0 + rng.normal(0, 2.0))))
    ours = fit_comm_model(samples)
    theirs = ref.fit_comm_model([(k.value, m, p, t) for k, m, p, t in samples])
    for kind in Collective:
        a, b = ours.costs[kind], theirs.costs[ref.Collective(kind.value)]
        assert (a.c1, a.c2, a.c3) == pytest.approx((b.c1, b.c2, b.c3), rel=1e-6, abs=1e-9)
        assert ours.rmse_log2_us[kind] == pytest.approx(theirs.rmse_log2_us[ref.Collective(kind.value)], abs=1e-9)


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference tree not present")
def test_reads_reference_default_model(tmp_path):
    """The reference's shipped Frontier constants (data/default_comm_model.ini) load unchanged and
    survive a save/load round trip."""
    m = load_comm_model(REF_SRC + "/phantomsim/data/default_comm_model.ini")
    assert m.costs[Collective.ALL_GATHER].c1 == 149.94 and m.rmse_log2_us[Collective.REDUCE_SCATTER] == 3.91
    save_comm_model(m, tmp_path / "x.ini")
    assert load_comm_model(tmp_path / "x.ini").costs == m.costs
