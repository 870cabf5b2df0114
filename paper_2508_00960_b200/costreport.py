"""The paper's cost model (§III-C, Eq. alpha/beta/energy; reference energy.py:1-238) next
to what the B200 engine MEASURES.

The reference predicts one iteration's cost from closed-form FLOP counts (alpha = FLOPs per rank /
device rate), the Table-II collective timing model (beta) and a busy/idle power model
(E = busy_watts * alpha + idle_watts * beta).  This module keeps those modelled quantities with
the reference's names, formulas and file formats (so `costmodel`, `train` and `compare` reports
line up with phantomsim's), and adds the measured columns the B200 run produces: seconds per
iteration from CUDA events, NVML joules, and B200-calibrated alpha (measured sustained bf16
TF/s, MEASURED_PEAKS.json) and beta (the B200 NCCL fit, profiles/*_comm_b200.ini).

FLOP accounting (energy.py:63-89, 92-110): per rank and layer with s = n/p, b = batch
  forward   2 s^2 b + 2 k s b + 2 (p-1) k s b + (p-1) s b + 2 s b
  backward  2 (p-1) k s b + s b + 2 s^2 b + 2 k s b + 2 (p-1) k s b
  recurrence (L-1) b (2 s^2 + 2 k s + 3 s), output error 3 s b once; summed over p ranks.
TP (row blocks): per layer 2 s n b + 2 s b forward, 2 s n b + s b + 2 n s b backward, 2 s b per
recurrence transition, 3 s b output error.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

from .collectives import Collective, CommRecord, Direction
from .commmodel import CommCostModel, comm_time
from .errors import ConfigurationError


@dataclass(frozen=True)
class EnergyRates:
    """Busy / idle watts of one device and its compute rate (FLOP/s) — the model's inputs."""

    busy_watts: float = 560.0
    idle_watts: float = 90.0
    device_flops: float = 1e12

    def __post_init__(self):
        if not self.busy_watts > self.idle_watts > 0:
            raise ConfigurationError("need busy_watts > idle_watts > 0")
        if self.device_flops <= 0:
            raise ConfigurationError("device_flops must be positive")


@dataclass
class CostReport:
    """Per-iteration and whole-run modelled costs (+ measured columns when a GPU run produced
    them: None otherwise)."""

    mode: str
    flops_per_iteration_rank: int
    flops_per_iteration_total: int
    alpha_s: float
    beta_s: float
    e_per_iteration_j: float
    nu: int
    energy_total_j: float
    bytes_communicated: int
    measured_s_per_iteration: float | None = None
    measured_j_per_iteration: float | None = None
    measured_energy_total_j: float | None = None


def _shape(n, p, layers, batch):
    if min(n, p, layers, batch) < 1:
        raise ConfigurationError("n, p, layers and batch must be positive")
    if n % p:
        raise ConfigurationError(f"n={n} not divisible by p={p}")
    return n // p


def flops_pp_iteration(n: int, p: int, k: int, layers: int, batch: int) -> int:
    s = _shape(n, p, layers, batch)
    if not 1 <= k <= s:
        raise ConfigurationError(f"need 1 <= k <= n/p, got k={k}")
    per_layer = (2 * s * s + 2 * k * s + 2 * (p - 1) * k * s + (p - 1) * s + 2 * s) \
        + (2 * (p - 1) * k * s + s + 2 * s * s + 2 * k * s + 2 * (p - 1) * k * s)
    per_rank = batch * (layers * per_layer + (layers - 1) * (2 * s * s + 2 * k * s + 3 * s) + 3 * s)
    return p * per_rank


def flops_tp_iteration(n: int, p: int, layers: int, batch: int) -> int:
    s = _shape(n, p, layers, batch)
    per_layer = (2 * s * n + 2 * s) + (2 * s * n + s + 2 * n * s)
    return p * batch * (layers * per_layer + (layers - 1) * 2 * s + 3 * s)


def alpha_seconds(flops_total: int, p: int, rates: EnergyRates) -> float:
    if p < 1:
        raise ConfigurationError("p must be >= 1")
    return flops_total / p / rates.device_flops


def comm_time_iteration(records, model: CommCostModel, p: int, *, include_loss: bool = False) -> float:
    """Modelled seconds of an iteration's collective record stream (loss all-reduce excluded
    unless include_loss)."""
    us = sum(comm_time(model, r.collective, r.message_size, p) for r in records
             if include_loss or r.direction is not Direction.LOSS)
    return us * 1e-6


def pp_schedule_beta(k: int, p: int, layers: int, batch: int, model: CommCostModel, *,
                     include_loss: bool = False) -> float:
    """One all-gather + one reduce-scatter of k * batch elements per layer."""
    m = k * batch
    us = layers * (comm_time(model, Collective.ALL_GATHER, m, p) + comm_time(model, Collective.REDUCE_SCATTER, m, p))
    if include_loss:
        us += comm_time(model, Collective.ALL_REDUCE, 1, p)
    return us * 1e-6


def tp_schedule_beta(n: int, p: int, layers: int, batch: int, model: CommCostModel, *,
                     include_loss: bool = False) -> float:
    """Row-block TP: broadcast (n b) + all-gather (s b) forward, all-reduce (n b) +
    reduce-scatter (s b) backward, per layer."""
    s = _shape(n, p, layers, batch)
    us = layers * (comm_time(model, Collective.BROADCAST, n * batch, p)
                   + comm_time(model, Collective.ALL_GATHER, s * batch, p)
                   + comm_time(model, Collective.ALL_REDUCE, n * batch, p)
                   + comm_time(model, Collective.REDUCE_SCATTER, s * batch, p))
    if include_loss:
        us += comm_time(model, Collective.ALL_REDUCE, 1, p)
    return us * 1e-6


def energy_per_iteration(rates: EnergyRates, alpha_s: float, beta_s: float) -> float:
    if alpha_s < 0 or beta_s < 0:
        raise ConfigurationError("alpha and beta must be nonnegative")
    return rates.busy_watts * alpha_s + rates.idle_watts * beta_s


def total_energy(e_per_iteration: float, nu: int) -> float:
    if nu < 0:
        raise ConfigurationError("nu must be >= 0")
    return nu * e_per_iteration


def records_bytes(records) -> int:
    """Per-rank payload bytes of a record stream in the reference's float64 accounting."""
    return 8 * sum(r.message_size for r in records)


def iteration_records(mode: str, n: int, p: int, k: int, layers: int, batch: int) -> list:
    """The collective record stream of one iteration (what the reference's Communicator logs,
    training.py:181-244): PP — per layer an all-gather of k*B forward, the loss all-reduce, per
    layer a reduce-scatter of k*B backward; TP — per layer broadcast (n B) + all-gather (s B)
    forward, the loss all-reduce, per layer all-reduce (n B) + reduce-scatter (s B) backward."""
    s = _shape(n, p, layers, batch)
    recs = []
    if mode == "pp":
        recs += [CommRecord(0, Collective.ALL_GATHER, k * batch, Direction.FORWARD, l) for l in range(layers)]
        recs.append(CommRecord(0, Collective.ALL_REDUCE, 1, Direction.LOSS, None))
        recs += [CommRecord(0, Collective.REDUCE_SCATTER, k * batch, Direction.BACKWARD, l)
                 for l in range(layers - 1, -1, -1)]
    else:
        for l in range(layers):
            recs += [CommRecord(0, Collective.BROADCAST, n * batch, Direction.FORWARD, l),
                     CommRecord(0, Collective.ALL_GATHER, s * batch, Direction.FORWARD, l)]
        recs.append(CommRecord(0, Collective.ALL_REDUCE, 1, Direction.LOSS, None))
        for l in range(layers - 1, -1, -1):
            recs += [CommRecord(0, Collective.ALL_REDUCE, n * batch, Direction.BACKWARD, l),
                     CommRecord(0, Collective.REDUCE_SCATTER, s * batch, Direction.BACKWARD, l)]
    return [CommRecord(i, r.collective, r.message_size, r.direction, r.layer) for i, r in enumerate(recs)]


def build_cost_report(mode: str, n: int, p: int, k: int, layers: int, batch: int, nu: int, rates: EnergyRates,
                      model: CommCostModel, *, iteration_records=None, include_loss: bool = False,
                      total_records=None, measured: dict | None = None) -> CostReport:
    """Modelled report (records when a run produced them, else the analytic schedule) plus the
    measured seconds / joules per iteration of a GPU run (measured = {seconds, joules,
    iterations}, joules summed over the GPUs)."""
    if mode == "pp":
        flops = flops_pp_iteration(n, p, k, layers, batch)
    elif mode == "tp":
        flops = flops_tp_iteration(n, p, layers, batch)
    else:
        raise ConfigurationError(f"unknown mode {mode!r}")
    alpha = alpha_seconds(flops, p, rates)
    if iteration_records:
        beta = comm_time_iteration(iteration_records, model, p, include_loss=include_loss)
    elif mode == "pp":
        beta = pp_schedule_beta(k, p, layers, batch, model, include_loss=include_loss)
    else:
        beta = tp_schedule_beta(n, p, layers, batch, model, include_loss=include_loss)
    e = energy_per_iteration(rates, alpha, beta)
    rep = CostReport(mode, flops // p, flops, alpha, beta, e, nu, total_energy(e, nu),
                     records_bytes(total_records) if total_records is not None else 0)
    if measured and measured.get("iterations"):
        it = measured["iterations"]
        rep.measured_s_per_iteration = measured["seconds"] / it
        if measured.get("joules") is not None:
            rep.measured_j_per_iteration = measured["joules"] / it
            rep.measured_energy_total_j = rep.measured_j_per_iteration * nu
    return rep


def _fmt(v):
    return "" if v is None else (repr(v) if isinstance(v, float) else str(v))


def cost_report_text(report: CostReport) -> str:
    """[cost_report] key = value lines (the reference's names first, measured keys after)."""
    return "\n".join(["[cost_report]"] + [f"{f.name} = {_fmt(getattr(report, f.name))}"
                                          for f in fields(report)]) + "\n"


def cost_report_csv(report: CostReport) -> str:
    names = [f.name for f in fields(report)]
    return ",".join(names) + "\n" + ",".join(_fmt(getattr(report, nm)) for nm in names) + "\n"
