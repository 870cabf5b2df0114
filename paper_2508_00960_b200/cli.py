"""Command line of the B200 engine, with phantomsim's subcommands and output files
(reference cli.py:1-402):

    python -m paper_2508_00960_b200 train     --mode pp|tp --n N --p P --layers L [--k K] ... --out DIR
    python -m paper_2508_00960_b200 compare   --n N --p P --k K --layers L --target-loss T ... --out DIR
    python -m paper_2508_00960_b200 costmodel [--n 256,1024 --p 2,4,8 --k 4,16 --layers 2 --batch B] --out DIR
    python -m paper_2508_00960_b200 fit-comm  --measurements samples.csv --out DIR

Same flags, config-file sections ([train] / [compare] / [costmodel], flags win over the file),
manifest.ini (resolved configuration + git-blob hash of the cost-model file), loss_history.csv,
cost_report.ini/.csv, comparison.csv and costmodel.csv as the reference writes them — plus the
measured columns of the B200 run beside the modelled ones: seconds and NVML joules per
iteration (train / compare, on one GPU: p logical ranks in the phantom engine, the dense Megatron
pipeline for tp), and B200-calibrated alpha / beta / energy in the cost-model table (measured
sustained bf16 TF/s from MEASURED_PEAKS.json, the B200 NCCL fit, power from --b200-watts).
Exit codes: 0 ok, 1 usage / configuration error, 3 runtime or training failure.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
from pathlib import Path

from . import __version__
from .commmodel import fit_comm_model, load_comm_model, load_measurements, save_comm_model
from .costreport import (EnergyRates, alpha_seconds, build_cost_report, cost_report_csv, cost_report_text,
                         energy_per_iteration, flops_pp_iteration, flops_tp_iteration, iteration_records,
                         pp_schedule_beta, tp_schedule_beta)
from .errors import ConfigurationError, PhantomsimError

EXIT_OK, EXIT_USAGE, EXIT_RUNTIME = 0, 1, 3
DATA = Path(__file__).resolve().parent / "data"
ROOT = Path(__file__).resolve().parent.parent


def default_model_path() -> Path:
    """The paper's Table-II constants (the reference's default cost model)."""
    return DATA / "frontier_comm_model.ini"


def b200_model_path() -> Path | None:
    """The newest B200 NCCL fit committed under profiles/ (tools/comm_fit.py), if any."""
    cands = sorted((ROOT / "profiles").glob("*_comm_b200.ini"))
    return cands[-1] if cands else None


class _Parser(argparse.ArgumentParser):
    def error(self, message):          # usage errors exit 1 (2 is the reference's verification code)
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def blob_hash(path) -> str:
    data = Path(path).read_bytes()
    return hashlib.sha1(b"blob %d\x00" % len(data) + data).hexdigest()


def _section(path, name) -> dict:
    if not path:
        return {}
    from .commmodel import _parse_ini
    p = Path(path)
    if not p.is_file():
        raise ConfigurationError(f"config file not found: {path}")
    return _parse_ini(p.read_text(encoding="utf-8"), path).get(name, {})


class _Resolver:
    """flag > config-file value > default."""

    def __init__(self, args, section):
        self.args, self.file = args, _section(getattr(args, "config", None), section)

    def __call__(self, key, cast, default=None):
        v = getattr(self.args, key.replace("-", "_"), None)
        if v is not None:
            return v
        if key in self.file:
            raw = self.file[key]
            try:
                return raw.strip().lower() in ("1", "true", "yes", "on") if cast is bool else cast(raw)
            except ValueError:
                raise ConfigurationError(f"config key {key!r}: cannot parse {raw!r}") from None
        return default


def _rates(text) -> EnergyRates:
    if not text:
        return EnergyRates()
    parts = text.split(",")
    if len(parts) != 3:
        raise ConfigurationError("--rates expects busy_watts,idle_watts,device_flops")
    try:
        return EnergyRates(*(float(x) for x in parts))
    except ValueError:
        raise ConfigurationError(f"--rates: cannot parse {text!r}") from None


def _ints(text) -> list:
    try:
        return [int(x) for x in str(text).split(",") if x.strip()]
    except ValueError:
        raise ConfigurationError(f"cannot parse integer list {text!r}") from None


def write_manifest(path: Path, command: str, resolved: dict, comm_model_file: Path) -> None:
    lines = ["[manifest]", f"command = {command}", f"package_version = {__version__}",
             f"comm_model_file = {comm_model_file}", f"comm_model_hash = {blob_hash(comm_model_file)}"]
    lines += [f"{k} = {repr(v) if isinstance(v, float) else v}" for k, v in sorted(resolved.items())]
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")


# ---------------------------------------------------------------------------------------------
# train / compare (GPU)
# ---------------------------------------------------------------------------------------------
def _train_config(args):
    import torch
    from .core import Activation
    from .phantom import valid_k
    from .training import TrainConfig
    r = _Resolver(args, "train")
    mode, n, p, layers = r("mode", str), r("n", int), r("p", int), r("layers", int)
    for key, v in (("mode", mode), ("n", n), ("p", p), ("layers", layers)):
        if v is None:
            raise ConfigurationError(f"missing required key: {key}")
    k = r("k", int, 0)
    if mode == "pp":
        bound, _ = valid_k(n, p)
        if not 1 <= k < bound:
            raise ConfigurationError(f"key k: k={k} violates valid_k(n={n}, p={p}) = [1, {bound})")
    cfg = TrainConfig(mode=mode, n=n, p=p, layers=layers, k=k, batch=r("batch", int, 0), lr=r("lr", float, 0.01),
                      optimizer=r("optimizer", str, "sgd"), target_loss=r("target-loss", float, None),
                      max_epochs=r("max-epochs", int, 100), seed=r("seed", int, 0),
                      loss_reduction=r("loss-reduction", str, "sum"),
                      activation=Activation(r("activation", str, "relu")),
                      scheduler="threads" if r("threads", bool, False) else "lockstep",
                      include_loss_comm_in_beta=r("beta-includes-loss", bool, False),
                      dtype=torch.float32 if r("dtype", str, "fp32") == "fp32" else torch.bfloat16)
    cfg.validate()
    samples = r("samples", int, cfg.batch or 32)
    comm_file = Path(r("comm-model", str, str(default_model_path())))
    return cfg, samples, comm_file


def _run(cfg, samples):
    """One training run on this GPU (measured seconds and NVML joules in result.cost)."""
    from .training import gen_dataset, train_engine
    data = gen_dataset(cfg.n, samples, cfg.seed)
    return train_engine(cfg, data)


def _resolved(cfg, samples, rates) -> dict:
    return {"mode": cfg.mode, "n": cfg.n, "p": cfg.p, "k": cfg.k, "layers": cfg.layers, "batch": cfg.batch or samples,
            "samples": samples, "lr": cfg.lr, "optimizer": cfg.optimizer,
            "target_loss": "" if cfg.target_loss is None else cfg.target_loss, "max_epochs": cfg.max_epochs,
            "seed": cfg.seed, "loss_reduction": cfg.loss_reduction, "activation": cfg.activation.value,
            "scheduler": cfg.scheduler, "beta_includes_loss": cfg.include_loss_comm_in_beta,
            "busy_watts": rates.busy_watts, "idle_watts": rates.idle_watts, "device_flops": rates.device_flops,
            "dtype": "fp32" if str(cfg.dtype).endswith("float32") else "bf16", "device": _device_name()}


def _device_name() -> str:
    try:
        import torch
        return torch.cuda.get_device_name(0).replace(" ", "_")
    except Exception:
        return "unknown"


def _report(cfg, samples, rates, model, result):
    """The reference's report of the run (records of one iteration -> beta, the whole run's
    records -> bytes) + the measured seconds / joules."""
    batch = cfg.batch or samples
    recs = iteration_records(cfg.mode, cfg.n, cfg.p, cfg.k, cfg.layers, batch)
    return build_cost_report(cfg.mode, cfg.n, cfg.p, cfg.k, cfg.layers, batch, result.iterations_run, rates, model,
                             iteration_records=recs, include_loss=cfg.include_loss_comm_in_beta,
                             total_records=recs * result.iterations_run, measured=result.cost)


def cmd_train(args) -> int:
    cfg, samples, comm_file = _train_config(args)
    rates = _rates(args.rates)
    model = load_comm_model(comm_file)
    out = Path(args.out or "runs/train")
    out.mkdir(parents=True, exist_ok=True)
    result = _run(cfg, samples)
    rep = _report(cfg, samples, rates, model, result)
    write_manifest(out / "manifest.ini", "train", _resolved(cfg, samples, rates), comm_file)
    ipe = samples // (cfg.batch or samples)
    rows = ["epoch,global_loss,alpha_s,beta_s,energy_j,measured_s,measured_j"]
    ms = (rep.measured_s_per_iteration or 0.0) * ipe
    mj = (rep.measured_j_per_iteration or 0.0) * ipe if rep.measured_j_per_iteration is not None else None
    for e, loss in enumerate(result.loss_history):
        rows.append(",".join([str(e), repr(float(loss)), repr(rep.alpha_s * ipe), repr(rep.beta_s * ipe),
                              repr(rep.e_per_iteration_j * ipe), repr(ms), "" if mj is None else repr(mj)]))
    (out / "loss_history.csv").write_text("\n".join(rows) + "\n", encoding="utf-8")
    (out / "cost_report.ini").write_text(cost_report_text(rep), encoding="utf-8")
    (out / "cost_report.csv").write_text(cost_report_csv(rep), encoding="utf-8")
    if args.save_model:
        from .checkpoint import save_model
        from .phantom import init_phantom_model
        from .tensor_parallel import init_tp_model
        m = (init_phantom_model(cfg.n, cfg.p, cfg.k, cfg.layers, cfg.activation, cfg.seed) if cfg.mode == "pp"
             else init_tp_model(cfg.n, cfg.p, cfg.layers, cfg.activation, cfg.seed))
        save_model(args.save_model, m)
    status = "converged" if result.converged else "not-converged"
    print(f"{cfg.mode} n={cfg.n} p={cfg.p} k={cfg.k} epochs={result.epochs_run} "
          f"final_loss={result.final_loss:.6g} {status}")
    print(f"wrote {out}/manifest.ini, loss_history.csv, cost_report.ini")
    if cfg.target_loss is not None and not result.converged:
        print("warning: target loss not reached", file=sys.stderr)
    return EXIT_OK


def cmd_compare(args) -> int:
    import torch
    from .core import Activation
    from .phantom import pp_model_size
    from .tensor_parallel import tp_model_size
    from .training import TrainConfig
    r = _Resolver(args, "compare")
    n, p, k, layers, target = r("n", int), r("p", int), r("k", int), r("layers", int), r("target-loss", float)
    for key, v in (("n", n), ("p", p), ("k", k), ("layers", layers), ("target-loss", target)):
        if v is None:
            raise ConfigurationError(f"missing required key: {key}")
    seed, samples, batch = r("seed", int, 0), r("samples", int, 32), r("batch", int, 0)
    lr, max_epochs = r("lr", float, 0.01), r("max-epochs", int, 1000)
    reduction, optimizer = r("loss-reduction", str, "sum"), r("optimizer", str, "sgd")
    activation = Activation(r("activation", str, "relu"))
    scheduler = "threads" if r("threads", bool, False) else "lockstep"
    dtype = torch.float32 if r("dtype", str, "fp32") == "fp32" else torch.bfloat16
    rates = _rates(args.rates)
    comm_file = Path(r("comm-model", str, str(default_model_path())))
    model = load_comm_model(comm_file)
    res = {}
    for mode in ("pp", "tp"):
        cfg = TrainConfig(mode=mode, n=n, p=p, layers=layers, k=k if mode == "pp" else 0, batch=batch, lr=lr,
                          optimizer=optimizer, target_loss=target, max_epochs=max_epochs, seed=seed,
                          loss_reduction=reduction, activation=activation, scheduler=scheduler, dtype=dtype)
        cfg.validate()
        result = _run(cfg, samples)
        res[mode] = (cfg, result, _report(cfg, samples, rates, model, result))
    lines = ["mode,p,k,model_size,converged,epochs,final_loss,e_per_iteration_j,energy_total_j,"
             "measured_s_per_iteration,measured_j_per_iteration,measured_energy_total_j"]
    for mode in sorted(res):
        cfg, result, rep = res[mode]
        size = pp_model_size(n, p, k, layers) if mode == "pp" else tp_model_size(n, layers)
        vals = [mode, p, cfg.k, size, result.converged, result.epochs_run, repr(float(result.final_loss)),
                repr(rep.e_per_iteration_j), repr(rep.energy_total_j), repr(rep.measured_s_per_iteration),
                "" if rep.measured_j_per_iteration is None else repr(rep.measured_j_per_iteration),
                "" if rep.measured_energy_total_j is None else repr(rep.measured_energy_total_j)]
        lines.append(",".join(map(str, vals)))
    if all(res[m][1].converged for m in res):
        lines.append(f"# energy_ratio_pp_over_tp = {res['pp'][2].energy_total_j / res['tp'][2].energy_total_j!r}")
        mp, mt = res["pp"][2].measured_energy_total_j, res["tp"][2].measured_energy_total_j
        if mp and mt:
            lines.append(f"# measured_energy_ratio_pp_over_tp = {mp / mt!r}")
    else:
        lines.append("# not all runs converged; energy ratio omitted")
    table = "\n".join(lines) + "\n"
    print(table, end="")
    out = Path(args.out or "runs/compare")
    out.mkdir(parents=True, exist_ok=True)
    (out / "comparison.csv").write_text(table, encoding="utf-8")
    write_manifest(out / "manifest.ini", "compare",
                   {"n": n, "p": p, "k": k, "layers": layers, "target_loss": target, "seed": seed,
                    "samples": samples, "batch": batch or samples, "lr": lr, "max_epochs": max_epochs,
                    "loss_reduction": reduction, "optimizer": optimizer, "activation": activation.value,
                    "scheduler": scheduler, "busy_watts": rates.busy_watts, "idle_watts": rates.idle_watts,
                    "device_flops": rates.device_flops, "dtype": "fp32" if dtype == torch.float32 else "bf16",
                    "device": _device_name()}, comm_file)
    return EXIT_OK


# ---------------------------------------------------------------------------------------------
# costmodel / fit-comm (CPU)
# ---------------------------------------------------------------------------------------------
def _b200_rates(watts: str | None):
    """B200 calibration: sustained bf16 TF/s from MEASURED_PEAKS.json (fallback 1400 TF/s) and the
    busy/idle watts given (default 1000 W / 200 W, the B200 TDP envelope)."""
    tf = 1400.0
    try:
        tf = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("bf16_tflops_sustained", tf))
    except Exception:
        pass
    busy, idle = (float(x) for x in (watts or "1000,200").split(","))
    return EnergyRates(busy, idle, tf * 1e12)


def cmd_costmodel(args) -> int:
    from .phantom import valid_k
    r = _Resolver(args, "costmodel")
    ns, ps_, ks = _ints(r("n", str, "256,1024")), _ints(r("p", str, "2,4,8")), _ints(r("k", str, "4,16"))
    grid_l = _ints(r("layers", str, "2"))
    batch = r("batch", int, 1)
    rates = _rates(args.rates)
    comm_file = Path(r("comm-model", str, str(default_model_path())))
    model = load_comm_model(comm_file)
    b200_file = b200_model_path()
    b200 = load_comm_model(b200_file) if b200_file else None
    b200_rates = _b200_rates(args.b200_watts)
    head = ("n,p,k,layers,batch,flops_pp,flops_tp,beta_pp_s,beta_tp_s,e_pp_j,e_tp_j,alpha_dominates,"
            "beta_dominates,energy_dominates,k_below_compute_bound,k_below_comm_bound,skip_reason,"
            "b200_alpha_pp_s,b200_alpha_tp_s,b200_beta_pp_s,b200_beta_tp_s,b200_e_pp_j,b200_e_tp_j")
    empty_ref, empty_b = "," * 11, "," * 6
    rows = []
    for n in ns:
        for p in ps_:
            for k in ks:
                for layers in grid_l:
                    key = (n, p, k, layers)
                    if n % p:
                        rows.append((key, f"{n},{p},{k},{layers},{batch}{empty_ref},n not divisible by p{empty_b}"))
                        continue
                    bound, compute_bound = valid_k(n, p)
                    if not 1 <= k <= bound:
                        rows.append((key, f"{n},{p},{k},{layers},{batch}{empty_ref},k outside [1, n/p]{empty_b}"))
                        continue
                    fpp, ftp = flops_pp_iteration(n, p, k, layers, batch), flops_tp_iteration(n, p, layers, batch)
                    bpp, btp = pp_schedule_beta(k, p, layers, batch, model), tp_schedule_beta(n, p, layers, batch,
                                                                                             model)
                    epp = energy_per_iteration(rates, alpha_seconds(fpp, p, rates), bpp)
                    etp = energy_per_iteration(rates, alpha_seconds(ftp, p, rates), btp)
                    vals = [n, p, k, layers, batch, fpp, ftp, repr(bpp), repr(btp), repr(epp), repr(etp),
                            fpp < ftp, bpp < btp, epp < etp, k < compute_bound, k < bound, ""]
                    apb, atb = alpha_seconds(fpp, p, b200_rates), alpha_seconds(ftp, p, b200_rates)
                    if b200 is not None:
                        bpb = pp_schedule_beta(k, p, layers, batch, b200)
                        btb = tp_schedule_beta(n, p, layers, batch, b200)
                        vals += [repr(apb), repr(atb), repr(bpb), repr(btb),
                                 repr(energy_per_iteration(b200_rates, apb, bpb)),
                                 repr(energy_per_iteration(b200_rates, atb, btb))]
                    else:
                        vals += [repr(apb), repr(atb), "", "", "", ""]
                    rows.append((key, ",".join(map(str, vals))))
    rows.sort(key=lambda t: t[0])
    table = head + "\n" + "\n".join(t for _, t in rows) + "\n"
    print(table, end="")
    if args.out:
        out = Path(args.out)
        out.mkdir(parents=True, exist_ok=True)
        (out / "costmodel.csv").write_text(table, encoding="utf-8")
        write_manifest(out / "manifest.ini", "costmodel",
                       {"n": ",".join(map(str, ns)), "p": ",".join(map(str, ps_)), "k": ",".join(map(str, ks)),
                        "layers": ",".join(map(str, grid_l)), "batch": batch, "busy_watts": rates.busy_watts,
                        "idle_watts": rates.idle_watts, "device_flops": rates.device_flops,
                        "b200_comm_model": str(b200_file or ""), "b200_device_flops": b200_rates.device_flops,
                        "b200_busy_watts": b200_rates.busy_watts, "b200_idle_watts": b200_rates.idle_watts},
                       comm_file)
    return EXIT_OK


def cmd_fit_comm(args) -> int:
    samples = load_measurements(args.measurements)
    model = fit_comm_model(samples)
    out = Path(args.out or "runs/fit_comm")
    out.mkdir(parents=True, exist_ok=True)
    f = out / "comm_model.ini"
    save_comm_model(model, f)
    write_manifest(out / "manifest.ini", "fit-comm", {"measurements": args.measurements,
                                                      "measurements_hash": blob_hash(args.measurements),
                                                      "samples": len(samples)}, f)
    for kind, c in model.costs.items():
        print(f"{kind.value:15s} c1={c.c1:.6g} c2={c.c2:.6g} c3={c.c3:.3g} "
              f"rmse_log2_us={model.rmse_log2_us.get(kind, float('nan')):.3f}")
    print(f"wrote {f}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="python -m paper_2508_00960_b200", description=__doc__.split("\n\n")[0])
    ap.add_argument("--version", action="version", version=__version__)
    sub = ap.add_subparsers(dest="command", required=True, parser_class=_Parser)

    def common(sp, section_flags):
        sp.add_argument("--config")
        sp.add_argument("--out")
        sp.add_argument("--rates")
        sp.add_argument("--comm-model")
        for flag, typ in section_flags:
            if typ is bool:
                sp.add_argument(f"--{flag}", action="store_true", default=None)
            else:
                sp.add_argument(f"--{flag}", type=typ)

    train_flags = [("mode", str), ("n", int), ("p", int), ("layers", int), ("k", int), ("batch", int),
                   ("samples", int), ("lr", float), ("optimizer", str), ("target-loss", float),
                   ("max-epochs", int), ("seed", int), ("loss-reduction", str), ("activation", str),
                   ("threads", bool), ("beta-includes-loss", bool), ("dtype", str)]
    t = sub.add_parser("train", help="one training run on this GPU: manifest, loss history, cost report")
    common(t, train_flags)
    t.add_argument("--save-model")
    t.set_defaults(fn=cmd_train)
    c = sub.add_parser("compare", help="PP and TP to one target loss, modelled vs measured energy")
    common(c, [f for f in train_flags if f[0] not in ("mode", "beta-includes-loss")])
    c.set_defaults(fn=cmd_compare)
    m = sub.add_parser("costmodel", help="FLOP / comm / energy table over a grid (reference + B200 columns)")
    common(m, [("n", str), ("p", str), ("k", str), ("layers", str), ("batch", int)])
    m.add_argument("--b200-watts", help="busy,idle watts of the B200 columns (default 1000,200)")
    m.set_defaults(fn=cmd_costmodel)
    f = sub.add_parser("fit-comm", help="fit collective timing constants from measurements")
    f.add_argument("--measurements", required=True)
    f.add_argument("--out")
    f.set_defaults(fn=cmd_fit_comm)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except ConfigurationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except PhantomsimError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
