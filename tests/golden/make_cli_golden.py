"""Run the UNMODIFIED reference CLI (phantomsim, /root/reference/pkg/src) in this container and keep
its output files as golden fixtures for tests/test_cli_gpu.py (the GPU box has no reference tree):

  cli/train_c1/   train --mode pp --n 1024 --p 2 --k 16 --layers 4 --samples 1024 --batch 64
                        --lr 1e-4 --max-epochs 3 --loss-reduction mean --seed 0
  cli/compare_acc/ compare --n 256 --p 4 --k 8 --layers 2 --samples 256 --lr 1e-4
                        --target-loss 4663.4 --max-epochs 1000 --loss-reduction mean --seed 0
                   (the fixed-loss acceptance run, test_acceptance.py:226-250)

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
RUNS = {
    "train_c1": ["train", "--mode", "pp", "--n", "1024", "--p", "2", "--k", "16", "--layers", "4", "--samples",
                 "1024", "--batch", "64", "--lr", "1e-4", "--max-epochs", "3", "--loss-reduction", "mean",
                 "--seed", "0"],
    "compare_acc": ["compare", "--n", "256", "--p", "4", "--k", "8", "--layers", "2", "--samples", "256", "--lr",
                    "1e-4", "--target-loss", "4663.4", "--max-epochs", "1000", "--loss-reduction", "mean",
                    "--seed", "0"],
}


def main():
    env = dict(os.environ, PYTHONPATH=REF_SRC, PYTHONDONTWRITEBYTECODE="1")
    for name, argv in RUNS.items():
        out = os.path.join(HERE, "cli", name)
        shutil.rmtree(out, ignore_errors=True)
        subprocess.run([sys.executable, "-m", "phantomsim.cli", *argv, "--out", out], check=True, env=env)
        for f in os.listdir(out):          # the manifest's comm_model_file path is container-specific
            if f == "manifest.ini":
                p = os.path.join(out, f)
                lines = [ln for ln in open(p) if not ln.startswith("comm_model_file")]
                open(p, "w").writelines(lines)
    print("wrote", os.path.join(HERE, "cli"))


if __name__ == "__main__":
    main()
