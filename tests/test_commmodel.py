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
