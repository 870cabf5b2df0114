"""The CLI's GPU subcommands against the reference CLI's own output files (tests/golden/cli/,
written by tests/golden/make_cli_golden.py from the unmodified phantomsim CLI):

  train   (C1: n=1024, p=2, k=16, L=4, 1024 samples, B=64, lr 1e-4, mean, 3 epochs, fp32 tier):
          same files and columns; the modelled alpha / beta / energy columns and the cost report
          identical; loss history within the fp32-tier tolerance of test_train_engine_gpu.py;
          measured seconds / joules present.
  compare (the fixed-loss acceptance run, test_acceptance.py:226-250: n=256, p=4, k=8, L=2,
          target 4663.4): both modes converge in the reference's epoch counts (+-2 epochs near the
          threshold) with the reference's modelled energies, plus measured ones.
"""
import csv
import io
import os

import pytest

from paper_2508_00960_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _csv(path):
    return list(csv.DictReader(io.StringIO(open(path).read())))


def _ini(path):
    out = {}
    for ln in open(path):
        if "=" in ln:
            k, v = ln.split("=", 1)
            out[k.strip()] = v.strip()
    return out


def test_cli_train_matches_reference_files(tmp_path):
    out = tmp_path / "train"
    rc = cli.main(["train", "--mode", "pp", "--n", "1024", "--p", "2", "--k", "16", "--layers", "4", "--samples",
                   "1024", "--batch", "64", "--lr", "1e-4", "--max-epochs", "3", "--loss-reduction", "mean",
                   "--seed", "0", "--dtype", "fp32", "--out", str(out)])
    assert rc == 0
    ref, ours = _csv(os.path.join(GOLD, "train_c1", "loss_history.csv")), _csv(out / "loss_history.csv")
    assert len(ours) == len(ref) == 3
    for a, b in zip(ours, ref):
        assert a["epoch"] == b["epoch"]
        assert abs(float(a["global_loss"]) - float(b["global_loss"])) <= 5e-3 * float(b["global_loss"])
        for col in ("alpha_s", "beta_s", "energy_j"):
            assert a[col] == b[col]
        assert float(a["measured_s"]) > 0
    rep_ref, rep = _ini(os.path.join(GOLD, "train_c1", "cost_report.ini")), _ini(out / "cost_report.ini")
    for key, val in rep_ref.items():
        assert rep[key] == val, key
    assert float(rep["measured_s_per_iteration"]) > 0
    man_ref, man = _ini(os.path.join(GOLD, "train_c1", "manifest.ini")), _ini(out / "manifest.ini")
    for key in man_ref:
        if key not in ("package_version", "comm_model_hash", "comm_model_file"):
            assert man[key] == man_ref[key], key


def test_cli_compare_fixed_loss_acceptance(tmp_path):
    out = tmp_path / "cmp"
    rc = cli.main(["compare", "--n", "256", "--p", "4", "--k", "8", "--layers", "2", "--samples", "256", "--lr",
                   "1e-4", "--target-loss", "4663.4", "--max-epochs", "1000", "--loss-reduction", "mean", "--seed",
                   "0", "--dtype", "fp32", "--out", str(out)])
    assert rc == 0
    ref = {r["mode"]: r for r in _csv(os.path.join(GOLD, "compare_acc", "comparison.csv")) if not r["mode"].startswith("#")}
    ours = {r["mode"]: r for r in _csv(out / "comparison.csv") if not r["mode"].startswith("#")}
    for mode in ("pp", "tp"):
        a, b = ours[mode], ref[mode]
        assert a["converged"] == "True" and a["model_size"] == b["model_size"]
        assert abs(int(a["epochs"]) - int(b["epochs"])) <= 2, (mode, a["epochs"], b["epochs"])
        assert a["e_per_iteration_j"] == b["e_per_iteration_j"]
        assert float(a["measured_s_per_iteration"]) > 0
    assert int(ours["pp"]["epochs"]) <= 1.5 * int(ours["tp"]["epochs"])     # acceptance criterion 8
    assert float(ours["pp"]["energy_total_j"]) < float(ours["tp"]["energy_total_j"])
    text = (out / "comparison.csv").read_text()
    assert "# energy_ratio_pp_over_tp" in text
