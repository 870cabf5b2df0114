"""Collective timing model: time_us(m, p) = c1 * log2(p) + c2 * m + c3 (m = elements per rank),
the paper's Table II form (PAPER.md Appendix), with the reference's public names and file format
(collectives.py:365-535) so phantomsim cost-model files and measurement CSVs load unchanged.

The B200 use is the other direction from the reference's: tools/comm_fit.py measures NCCL over
NVLink 5 / NVSwitch on the box and this module fits and publishes the constants
(profiles/*_comm_b200.ini) next to the Frontier defaults.

Implementation notes (this module's own design): the four collectives' constants live in one
[4, 3] coefficient table; evaluation is a dot product with the regressor (log2 p, m, 1); the fit
solves the 3-variable least-squares problem with c1, c2 >= 0 exactly by scanning the 4 active
sets of the two bounds (the objective is convex, so the feasible stationary point with the lowest
residual is the bounded optimum the reference obtains from scipy's lsq_linear).
"""

from __future__ import annotations

import csv
import itertools
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .collectives import Collective
from .errors import ConfigurationError, FitError

_ORDER = tuple(Collective)                 # row order of the coefficient table
_HEADER = ("collective", "m", "p", "time_us")


@dataclass(frozen=True)
class CollectiveCost:
    """(c1 per log2 p, c2 per element, c3 constant) in microseconds for one collective."""

    c1: float
    c2: float
    c3: float = 0.0

    def __post_init__(self):
        if min(self.c1, self.c2) < 0:
            raise ConfigurationError(f"latency and bandwidth terms must be >= 0 (c1={self.c1}, c2={self.c2})")


@dataclass
class CommCostModel:
    """Timing constants per collective (+ log2 RMSE of the fit that produced them)."""

    costs: dict
    rmse_log2_us: dict = field(default_factory=dict)

    def table(self) -> np.ndarray:
        """[4, 3] coefficients in Collective order (NaN rows for collectives without constants)."""
        t = np.full((len(_ORDER), 3), np.nan)
        for i, kind in enumerate(_ORDER):
            c = self.costs.get(kind)
            if c is not None:
                t[i] = (c.c1, c.c2, c.c3)
        return t

    def time_us(self, collective, m: int, p: int) -> float:
        return comm_time(self, collective, m, p)


def _regressor(m, p):
    return np.array([math.log2(p), float(m), 1.0])


def comm_time(model: CommCostModel, collective, m: int, p: int) -> float:
    """Modelled microseconds of one collective of m elements per rank over p ranks."""
    if p < 1 or m < 0:
        raise ConfigurationError(f"need p >= 1 and m >= 0 (got p={p}, m={m})")
    kind = Collective(collective)
    if kind not in model.costs:
        raise ConfigurationError(f"the model has no constants for {kind.value}")
    c = model.costs[kind]
    return float(np.dot((c.c1, c.c2, c.c3), _regressor(m, p)))


# ---------------------------------------------------------------------------------------------
# files: INI-style sections [collective] with c1, c2, c3 (, rmse_log2_us)
# ---------------------------------------------------------------------------------------------
def _parse_ini(text: str, path) -> dict:
    sections, cur = {}, None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].split(";", 1)[0].strip()
        if not line:
            continue
        if line.startswith("[") and line.endswith("]"):
            cur = sections.setdefault(line[1:-1].strip(), {})
            continue
        if cur is None or "=" not in line:
            raise ConfigurationError(f"{path}:{lineno}: expected '[collective]' or 'key = value'")
        key, val = (x.strip() for x in line.split("=", 1))
        cur[key.lower()] = val
    return sections


def load_comm_model(path, *, require_all: bool = True) -> CommCostModel:
    """Read a cost-model file (the reference's format); every collective must have a section
    unless require_all=False."""
    p = Path(path)
    if not p.is_file():
        raise ConfigurationError(f"cost-model file not found: {path}")
    costs, rmse = {}, {}
    for name, kv in _parse_ini(p.read_text(encoding="utf-8"), path).items():
        try:
            kind = Collective(name)
        except ValueError:
            raise ConfigurationError(f"{path}: [{name}] is not a collective") from None
        try:
            costs[kind] = CollectiveCost(float(kv["c1"]), float(kv["c2"]), float(kv.get("c3", 0.0)))
            if "rmse_log2_us" in kv:
                rmse[kind] = float(kv["rmse_log2_us"])
        except (KeyError, ValueError) as exc:
            raise ConfigurationError(f"{path}: [{name}] has a missing or bad value ({exc})") from None
    absent = [k.value for k in _ORDER if k not in costs]
    if require_all and absent:
        raise ConfigurationError(f"{path}: no section for {absent}")
    return CommCostModel(costs, rmse)


def save_comm_model(model: CommCostModel, path, note: str = "") -> None:
    """Write the model in the format load_comm_model (and the reference) reads."""
    out = ["# time_us = c1 * log2(p) + c2 * m + c3 per collective (m = elements per rank)"]
    if note:
        out += [f"# {ln}" for ln in note.splitlines()]
    for kind in _ORDER:
        c = model.costs.get(kind)
        if c is None:
            continue
        out += ["", f"[{kind.value}]"] + [f"{nm} = {v!r}" for nm, v in zip(("c1", "c2", "c3"), (c.c1, c.c2, c.c3))]
        if kind in model.rmse_log2_us:
            out.append(f"rmse_log2_us = {model.rmse_log2_us[kind]!r}")
    Path(path).write_text("\n".join(out) + "\n", encoding="utf-8")


# ---------------------------------------------------------------------------------------------
# fit
# ---------------------------------------------------------------------------------------------
def _bounded_lstsq(X: np.ndarray, y: np.ndarray) -> np.ndarray:
    """argmin ||X b - y||, b[0] >= 0, b[1] >= 0, b[2] free: try every subset of the two bounds as
    active (coefficient pinned at 0), keep the feasible candidate with the smallest residual."""
    best, best_r = None, math.inf
    for pinned in itertools.chain.from_iterable(itertools.combinations((0, 1), r) for r in range(3)):
        free = [i for i in range(3) if i not in pinned]
        b = np.zeros(3)
        b[free] = np.linalg.lstsq(X[:, free], y, rcond=None)[0]
        if b[0] < 0 or b[1] < 0:
            continue
        r = float(np.sum((X @ b - y) ** 2))
        if best is None or r < best_r - 1e-12 * max(1.0, best_r):
            best, best_r = b, r
    return best


def fit_comm_model(samples) -> CommCostModel:
    """Fit (c1, c2, c3) per collective to samples [(collective, m, p, time_us)] by least squares
    in microseconds with c1, c2 >= 0.  Each collective needs >= 3 samples over >= 2 distinct p and
    >= 2 distinct m (otherwise the regressors (log2 p, m, 1) are rank deficient -> FitError).
    The fit's RMSE is stored as log2(microseconds)."""
    by_kind: dict = {}
    for coll, m, p, t in samples:
        by_kind.setdefault(Collective(coll), []).append((math.log2(float(p)), float(m), 1.0, float(t)))
    if not by_kind:
        raise FitError("no samples supplied")
    costs, rmse = {}, {}
    for kind, rows in by_kind.items():
        A = np.array(rows)
        X, y = A[:, :3], A[:, 3]
        n_p, n_m = len(set(A[:, 0])), len(set(A[:, 1]))
        if len(A) < 3 or n_p < 2 or n_m < 2:
            raise FitError(f"{kind.value}: {len(A)} samples over {n_p} distinct p and {n_m} distinct m "
                           f"cannot fit 3 coefficients (need >= 3 samples, >= 2 p, >= 2 m)")
        if np.linalg.matrix_rank(X) < 3:
            raise FitError(f"{kind.value}: the regressors (log2 p, m, 1) are rank deficient")
        b = _bounded_lstsq(X, y)
        res = float(np.sqrt(np.mean((X @ b - y) ** 2)))
        costs[kind] = CollectiveCost(max(float(b[0]), 0.0), max(float(b[1]), 0.0), float(b[2]))
        rmse[kind] = math.log2(res) if res > 0 else float("-inf")
    return CommCostModel(costs, rmse)


# ---------------------------------------------------------------------------------------------
# measurement CSVs: header collective,m,p,time_us
# ---------------------------------------------------------------------------------------------
def load_measurements(path) -> list:
    """[(Collective, m, p, time_us)] from a CSV with header collective,m,p,time_us; a malformed
    row reports `path:line:`."""
    with open(path, newline="", encoding="utf-8") as fh:
        rows = list(csv.reader(fh))
    if not rows or tuple(h.strip().lower() for h in rows[0]) != _HEADER:
        raise ConfigurationError(f"{path}:1: header must be {','.join(_HEADER)}")
    out = []
    for lineno, row in enumerate(rows[1:], start=2):
        if not any(c.strip() for c in row):
            continue
        try:
            out.append((Collective(row[0].strip()), float(row[1]), int(row[2]), float(row[3])))
        except (ValueError, IndexError) as exc:
            raise ConfigurationError(f"{path}:{lineno}: cannot parse {row!r} ({exc})") from None
    return out


def save_measurements(samples, path) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(_HEADER)
        for coll, m, p, t in samples:
            w.writerow([Collective(coll).value, int(m), int(p), f"{t:.4f}"])
