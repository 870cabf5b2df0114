"""Collective timing model (reference collectives.py:380-535, paper Appendix / Table II):
time_us = c1 * log2(p) + c2 * m + c3 per collective (m = message elements per rank), the same
cost-model file format, and the least-squares fit used to publish measured B200 (NVLink 5 /
NVSwitch, NCCL) constants next to the paper's Frontier table (tools/comm_fit.py).
"""

from __future__ import annotations

import configparser
import csv
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .collectives import Collective
from .errors import ConfigurationError


class FitError(ConfigurationError):
    """The measurement set cannot determine the three coefficients."""


@dataclass(frozen=True)
class CollectiveCost:
    c1: float          # microseconds per log2(p)
    c2: float          # microseconds per element
    c3: float = 0.0    # microseconds

    def __post_init__(self):
        if self.c1 < 0 or self.c2 < 0:
            raise ConfigurationError("c1 and c2 must be nonnegative")


@dataclass
class CommCostModel:
    costs: dict
    rmse_log2_us: dict = field(default_factory=dict)

    def time_us(self, collective, m: int, p: int) -> float:
        return comm_time(self, collective, m, p)


def comm_time(model: CommCostModel, collective, m: int, p: int) -> float:
    if p < 1:
        raise ConfigurationError("p must be >= 1")
    if m < 0:
        raise ConfigurationError("message size must be >= 0")
    kind = Collective(collective)
    if kind not in model.costs:
        raise ConfigurationError(f"no timing constants for collective {kind.value}")
    c = model.costs[kind]
    return c.c1 * math.log2(p) + c.c2 * m + c.c3


def save_comm_model(model: CommCostModel, path) -> None:
    out = ["# Collective timing constants, microseconds.",
           "# time_us = c1 * log2(p) + c2 * m + c3   (m = message elements per rank)", ""]
    for kind in Collective:
        if kind not in model.costs:
            continue
        c = model.costs[kind]
        out += [f"[{kind.value}]", f"c1 = {c.c1!r}", f"c2 = {c.c2!r}", f"c3 = {c.c3!r}"]
        if kind in model.rmse_log2_us:
            out.append(f"rmse_log2_us = {model.rmse_log2_us[kind]!r}")
        out.append("")
    Path(path).write_text("\n".join(out), encoding="utf-8")


def load_comm_model(path, *, require_all: bool = True) -> CommCostModel:
    parser = configparser.ConfigParser()
    if not parser.read(path):
        raise ConfigurationError(f"cost-model file not found: {path}")
    costs, rmse = {}, {}
    for section in parser.sections():
        try:
            kind = Collective(section)
        except ValueError:
            raise ConfigurationError(f"{path}: unknown collective section [{section}]") from None
        try:
            costs[kind] = CollectiveCost(parser.getfloat(section, "c1"), parser.getfloat(section, "c2"),
                                         parser.getfloat(section, "c3", fallback=0.0))
            if parser.has_option(section, "rmse_log2_us"):
                rmse[kind] = parser.getfloat(section, "rmse_log2_us")
        except ValueError as exc:
            raise ConfigurationError(f"{path}: bad value in [{section}]: {exc}") from None
    missing = [k.value for k in Collective if k not in costs]
    if require_all and missing:
        raise ConfigurationError(f"{path}: missing sections for {missing}")
    return CommCostModel(costs, rmse)


def _nonneg_lstsq(X: np.ndarray, y: np.ndarray) -> np.ndarray:
    """min ||X b - y|| with b[0], b[1] >= 0 (b[2] free): the unconstrained solution, else the
    best of the fits with the violating coefficient(s) pinned at zero."""
    b, *_ = np.linalg.lstsq(X, y, rcond=None)
    if b[0] >= 0 and b[1] >= 0:
        return b
    best, best_err = None, math.inf
    for fixed in ((0,), (1,), (0, 1)):
        keep = [i for i in range(3) if i not in fixed]
        sub, *_ = np.linalg.lstsq(X[:, keep], y, rcond=None)
        cand = np.zeros(3)
        cand[keep] = sub
        if cand[0] < 0 or cand[1] < 0:
            continue
        err = float(np.linalg.norm(X @ cand - y))
        if err < best_err:
            best, best_err = cand, err
    return best


def fit_comm_model(samples) -> CommCostModel:
    """Per collective, least squares on regressors (log2 p, m, 1) in microseconds with c1, c2
    clamped nonnegative; needs >= 3 samples over >= 2 distinct p and >= 2 distinct m. The
    fit's RMSE is kept as log2(microseconds)."""
    groups = {}
    for coll, m, p, t in samples:
        groups.setdefault(Collective(coll), []).append((float(m), float(p), float(t)))
    if not groups:
        raise FitError("no samples supplied")
    costs, rmse = {}, {}
    for kind, rows in groups.items():
        n_p = len({p for _, p, _ in rows})
        n_m = len({m for m, _, _ in rows})
        if len(rows) < 3 or n_p < 2 or n_m < 2:
            raise FitError(f"{kind.value}: need >= 3 samples spanning >= 2 distinct p and 2 distinct m "
                           f"(got {len(rows)} samples, {n_p} p, {n_m} m)")
        X = np.array([[math.log2(p), m, 1.0] for m, p, _ in rows])
        y = np.array([t for _, _, t in rows])
        if np.linalg.matrix_rank(X) < 3:
            raise FitError(f"{kind.value}: rank-deficient regressor set")
        b = _nonneg_lstsq(X, y)
        r = float(np.sqrt(np.mean((X @ b - y) ** 2)))
        costs[kind] = CollectiveCost(max(float(b[0]), 0.0), max(float(b[1]), 0.0), float(b[2]))
        rmse[kind] = math.log2(r) if r > 0 else float("-inf")
    return CommCostModel(costs, rmse)


def load_measurements(path) -> list:
    """CSV with header collective,m,p,time_us -> [(Collective, m, p, time_us)]."""
    out = []
    with open(path, newline="", encoding="utf-8") as fh:
        rd = csv.reader(fh)
        head = next(rd, None)
        if head is None or [h.strip().lower() for h in head] != ["collective", "m", "p", "time_us"]:
            raise ConfigurationError(f"{path}:1: expected header collective,m,p,time_us")
        for lineno, row in enumerate(rd, start=2):
            if not row or (len(row) == 1 and not row[0].strip()):
                continue
            try:
                out.append((Collective(row[0].strip()), float(row[1]), int(row[2]), float(row[3])))
            except (ValueError, IndexError) as exc:
                raise ConfigurationError(f"{path}:{lineno}: malformed row: {exc}") from None
    return out


def save_measurements(samples, path) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["collective", "m", "p", "time_us"])
        for coll, m, p, t in samples:
            w.writerow([Collective(coll).value, int(m), int(p), f"{t:.4f}"])
