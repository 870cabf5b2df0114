"""CLI / manifest / cost-report parity (reference cli.py:191-402, energy.py:63-238): the cost
model functions equal phantomsim's, `costmodel` reproduces the reference's table columns
byte for byte (plus the B200 columns), `fit-comm` round-trips, manifests carry the cost-model
hash.  The GPU subcommands (train / compare) are exercised in test_cli_gpu.py."""
import csv
import io
import os
import subprocess
import sys

import pytest

from paper_2508_00960_b200 import cli, costreport as cr
from paper_2508_00960_b200.commmodel import load_comm_model

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")


@needs_ref
def test_cost_functions_match_reference():
    sys.path.insert(0, REF_SRC)
    from phantomsim import energy as ref_e
    from phantomsim import collectives as ref_c
    ours_m = load_comm_model(cli.default_model_path())
    ref_m = ref_c.default_comm_model()
    for n, p, k, L, b in [(256, 2, 4, 2, 1), (1024, 8, 16, 3, 7), (16384, 8, 128, 8, 8192), (64, 4, 16, 1, 3)]:
        assert cr.flops_pp_iteration(n, p, k, L, b) == ref_e.flops_pp_iteration(n, p, k, L, b)
        assert cr.flops_tp_iteration(n, p, L, b) == ref_e.flops_tp_iteration(n, p, L, b)
        assert cr.pp_schedule_beta(k, p, L, b, ours_m) == pytest.approx(ref_e.pp_schedule_beta(k, p, L, b, ref_m),
                                                                          rel=1e-12)
        assert cr.tp_schedule_beta(n, p, L, b, ours_m) == pytest.approx(ref_e.tp_schedule_beta(n, p, L, b, ref_m),
                                                                          rel=1e-12)
        r1, r2 = cr.EnergyRates(), ref_e.EnergyRates()
        a1, a2 = cr.alpha_seconds(cr.flops_pp_iteration(n, p, k, L, b), p, r1), \
            ref_e.alpha_seconds(ref_e.flops_pp_iteration(n, p, k, L, b), p, r2)
        assert a1 == a2
        assert cr.energy_per_iteration(r1, a1, 0.5) == ref_e.energy_per_iteration(r2, a2, 0.5)


@needs_ref
def test_costmodel_table_matches_reference(tmp_path):
    args = ["--n", "256,1024,100", "--p", "2,4,8", "--k", "4,16,300", "--layers", "1,2", "--batch", "3"]
    assert cli.main(["costmodel", *args, "--out", str(tmp_path / "ours")]) == 0
    env = dict(os.environ, PYTHONPATH=REF_SRC, PYTHONDONTWRITEBYTECODE="1")
    subprocess.run([sys.executable, "-m", "phantomsim.cli", "costmodel", *args, "--out", str(tmp_path / "ref")],
                   check=True, env=env, capture_output=True, cwd=tmp_path)
    ours = list(csv.reader(io.StringIO((tmp_path / "ours" / "costmodel.csv").read_text())))
    ref = list(csv.reader(io.StringIO((tmp_path / "ref" / "costmodel.csv").read_text())))
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert a[:len(b)] == b                     # the reference's 17 columns, identical text
    assert ours[0][17:] == ["b200_alpha_pp_s", "b200_alpha_tp_s", "b200_beta_pp_s", "b200_beta_tp_s",
                            "b200_e_pp_j", "b200_e_tp_j"]
    man = (tmp_path / "ours" / "manifest.ini").read_text()
    assert f"comm_model_hash = {cli.blob_hash(cli.default_model_path())}" in man


def test_fit_comm_and_usage_errors(tmp_path):
    from paper_2508_00960_b200.collectives import Collective
    from paper_2508_00960_b200.commmodel import save_measurements
    samples = [(k, m, p, 3.0 * (p.bit_length() - 1) + 1e-4 * m + 2.0) for k in Collective for p in (2, 4, 8)
               for m in (16, 4096, 1 << 20)]
    save_measurements(samples, tmp_path / "s.csv")
    assert cli.main(["fit-comm", "--measurements", str(tmp_path / "s.csv"), "--out", str(tmp_path / "fit")]) == 0
    m = load_comm_model(tmp_path / "fit" / "comm_model.ini")
    assert m.costs[Collective.ALL_GATHER].c1 == pytest.approx(3.0, rel=1e-6)
    assert "measurements_hash" in (tmp_path / "fit" / "manifest.ini").read_text()
    with pytest.raises(SystemExit) as e:
        cli.main(["costmodel", "--no-such-flag"])
    assert e.value.code == cli.EXIT_USAGE
    assert cli.main(["train", "--mode", "pp", "--n", "64", "--p", "4", "--layers", "2", "--k", "99"]) == cli.EXIT_USAGE


def test_cost_report_serialisation():
    rep = cr.build_cost_report("pp", 1024, 2, 16, 4, 64, 48, cr.EnergyRates(), load_comm_model(cli.default_model_path()),
                               measured={"seconds": 1.5, "joules": 30.0, "iterations": 48})
    text = cr.cost_report_text(rep)
    assert text.startswith("[cost_report]\nmode = pp\n")
    assert "measured_j_per_iteration = 0.625" in text
    head, row = cr.cost_report_csv(rep).splitlines()
    assert head.split(",")[:9] == ["mode", "flops_per_iteration_rank", "flops_per_iteration_total", "alpha_s",
                                   "beta_s", "e_per_iteration_j", "nu", "energy_total_j", "bytes_communicated"]
