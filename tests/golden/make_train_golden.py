"""Per-iteration C1 training losses of the UNMODIFIED reference (phantomsim.train, SURVEY §8c:
n=1024, p=2, k=16, L=4, 1024 samples, B=64, lr=1e-4, mean), first epoch, SGD and Adam.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_train_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import phantomsim as ps
    import phantomsim.training as T

    c1 = np.load(os.path.join(HERE, "c1.npz"))
    n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
    data = ps.gen_dataset(n, 1024, seed)
    rec = []
    orig = T.pp_iteration

    def recording(comm, rank, *a, **kw):
        out = orig(comm, rank, *a, **kw)
        if rank == 0:
            rec.append(out.global_loss)
        return out

    T.pp_iteration = recording
    out = {}
    for opt in ("sgd", "adam"):
        rec.clear()
        cfg = ps.TrainConfig(mode="pp", n=n, p=p, layers=L, k=k, batch=B, lr=1e-4, max_epochs=1, seed=seed,
                             loss_reduction="mean", optimizer=opt, scheduler="lockstep")
        res = ps.train(cfg, data)
        out[f"{opt}_iter_losses"] = np.array(rec)
        out[f"{opt}_epoch_loss"] = np.array(res.loss_history)
    np.savez_compressed(os.path.join(HERE, "c1_train.npz"), **out)
    print({k: v[:4] for k, v in out.items()})


if __name__ == "__main__":
    main()
