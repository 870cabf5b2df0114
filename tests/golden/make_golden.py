"""Generate the golden vectors that pin oracle/phantom_oracle.py to the reference.

Runs the UNMODIFIED reference (phantomsim, imported from /root/reference/pkg/src) in this
container and writes small .npz fixtures next to this script.  The GPU box never runs this (the
reference tree is not there); it only reads the committed .npz files.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import zlib
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (n, p, k, layers, batch, seed, activation, reduction)
TINY_CASES = [
    (4, 2, 1, 1, 1, 6, "identity", "sum"),
    (8, 2, 2, 2, 2, 11, "identity", "sum"),
    (8, 2, 1, 1, 1, 3, "relu", "sum"),
    (16, 4, 2, 2, 3, 0, "relu", "sum"),
    (16, 2, 4, 3, 2, 7, "relu", "mean"),
    (24, 4, 3, 2, 4, 2, "relu", "sum"),
    (64, 4, 8, 3, 4, 5, "relu", "mean"),
    (64, 8, 4, 2, 5, 9, "identity", "sum"),
    (32, 1, 4, 2, 3, 1, "relu", "sum"),
]

N_SAMPLE = 256


def _sample_idx(size, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(size, size=min(N_SAMPLE, size), replace=False))


def main():
    sys.path.insert(0, REF_SRC)
    import phantomsim as ps
    from phantomsim.training import pp_iteration, tp_iteration

    acts = {"relu": ps.Activation.RELU, "identity": ps.Activation.IDENTITY}

    # ---- tiny grid: full tensors ---------------------------------------------------------
    out = {}
    for ci, (n, p, k, L, B, seed, act, red) in enumerate(TINY_CASES):
        pre = f"c{ci}_"
        model = ps.init_phantom_model(n, p, k, L, acts[act], seed)
        rng = np.random.default_rng(100 + ci)
        x = rng.standard_normal((n, B))
        y = rng.standard_normal((n, B))
        s = n // p
        comm = ps.Communicator(p)
        res = comm.run(lambda c, r: pp_iteration(c, r, model.rank_layers[r], model.activations,
                                                 x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], red))
        out[pre + "cfg"] = np.array([n, p, k, L, B, seed])
        out[pre + "act"] = np.array(act)
        out[pre + "red"] = np.array(red)
        out[pre + "x"] = x
        out[pre + "y"] = y
        out[pre + "global_loss"] = np.array(res[0].global_loss)
        for r in range(p):
            out[pre + f"r{r}_local_loss"] = np.array(res[r].local_loss)
            out[pre + f"r{r}_y_out"] = res[r].y_out
            for l in range(L):
                lay = model.rank_layers[r][l]
                g = res[r].grads[l]
                t = res[r].tape[l]
                q = f"{pre}r{r}_l{l}_"
                out[q + "w_local"] = lay.local
                out[q + "w_comp"] = lay.compressor
                out[q + "w_dec"] = (np.stack([lay.decompressors[i] for i in sorted(lay.decompressors)])
                                    if lay.decompressors else np.zeros((0, s, k)))
                out[q + "g_local"] = g.local
                out[q + "g_comp"] = g.compressor
                out[q + "g_dec"] = (np.stack([g.decompressors[i] for i in sorted(g.decompressors)])
                                    if g.decompressors else np.zeros((0, s, k)))
                out[q + "g_bias"] = g.bias
                out[q + "delta"] = res[r].deltas[l]
                out[q + "preact"] = t.preact
                out[q + "phantoms"] = np.stack([t.phantoms[i] for i in range(p)])
                out[q + "received"] = t.phantom_grad
        # forward dense-twin check value
        twin = ps.phantom_dense_twin(model)
        dense_out, _ = ps.dense_forward(twin, x)
        out[pre + "dense_out"] = dense_out
    # TP tiny case vs dense
    n, p, L, B = 16, 4, 2, 3
    tpm = ps.init_tp_model(n, p, L, ps.Activation.RELU, 4)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n, B))
    y = rng.standard_normal((n, B))
    s = n // p
    comm = ps.Communicator(p)
    res = comm.run(lambda c, r: tp_iteration(c, r, tpm.rank_layers[r], tpm.activations,
                                             x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], "sum"))
    out["tp_cfg"] = np.array([n, p, L, B, 4])
    out["tp_x"] = x
    out["tp_y"] = y
    out["tp_global_loss"] = np.array(res[0].global_loss)
    for r in range(p):
        out[f"tp_r{r}_y_out"] = res[r].y_out
        for l in range(L):
            out[f"tp_r{r}_l{l}_g_weight"] = res[r].grads[l].weight
            out[f"tp_r{r}_l{l}_g_bias"] = res[r].grads[l].bias
            out[f"tp_r{r}_l{l}_delta"] = res[r].deltas[l]
    # TP == dense training curve (test_acceptance.py:100-118 shape, shortened)
    dense = ps.init_dense_ffn(n, L, ps.Activation.RELU, 4)
    out["tp_dense_train_hist"] = np.array(ps.dense_train(dense, x, y, 1e-3, 10))
    # sizing goldens (phantom.py:270-296; test_acceptance.py:121-138)
    out["size_cases"] = np.array([[16384, 8, 16, 2], [16384, 16, 6, 2], [16384, 32, 4, 2],
                                  [64, 2, 4, 2], [256, 4, 8, 2]])
    out["size_values"] = np.array([ps.pp_model_size(*c) for c in out["size_cases"]])
    np.savez_compressed(os.path.join(HERE, "tiny.npz"), **out)

    # ---- C1 (n=1024, p=2, k=16, L=4, B=64): checksums + sampled entries --------------------
    n, p, k, L, B, seed = 1024, 2, 16, 4, 64, 0
    data = ps.gen_dataset(n, 1024, seed)
    model = ps.init_phantom_model(n, p, k, L, ps.Activation.RELU, seed)
    s = n // p
    x = data.inputs[:, :B]
    y = data.targets[:, :B]
    comm = ps.Communicator(p)
    res = comm.run(lambda c, r: pp_iteration(c, r, model.rank_layers[r], model.activations,
                                             x[r * s:(r + 1) * s], y[r * s:(r + 1) * s], "mean"))
    c1 = {"cfg": np.array([n, p, k, L, B, seed]),
          "x_sum": np.array(x.sum()), "x_sq": np.array((x * x).sum()),
          "y_sum": np.array(y.sum()), "y_sq": np.array((y * y).sum()),
          "teacher_sum": np.array(data.teacher.sum()),
          "global_loss": np.array(res[0].global_loss)}
    for r in range(p):
        idx = _sample_idx(s * B, 1000 + r)
        c1[f"r{r}_y_idx"] = idx
        c1[f"r{r}_y_val"] = res[r].y_out.ravel()[idx]
        c1[f"r{r}_y_norm"] = np.array(np.linalg.norm(res[r].y_out))
        for l in range(L):
            lay = model.rank_layers[r][l]
            g = res[r].grads[l]
            q = f"r{r}_l{l}_"
            for name, w in (("w_local", lay.local), ("w_comp", lay.compressor),
                            ("w_dec", np.stack([lay.decompressors[i] for i in sorted(lay.decompressors)])),
                            ("g_local", g.local), ("g_comp", g.compressor),
                            ("g_dec", np.stack([g.decompressors[i] for i in sorted(g.decompressors)])),
                            ("g_bias", g.bias), ("delta", res[r].deltas[l]),
                            ("received", res[r].tape[l].phantom_grad),
                            ("preact", res[r].tape[l].preact)):
                idx = _sample_idx(w.size, zlib.crc32(f"{r}:{l}:{name}".encode()) % 10000)
                c1[q + name + "_idx"] = idx
                c1[q + name + "_val"] = w.ravel()[idx]
                c1[q + name + "_norm"] = np.array(np.linalg.norm(w))
    # C1 training curve ([104881.54, 80437.516, 76972.99] in both schedulers)
    cfg = ps.TrainConfig(mode="pp", n=n, p=p, layers=L, k=k, batch=B, lr=1e-4, max_epochs=3,
                         seed=seed, loss_reduction="mean", scheduler="threads")
    c1["train_sgd_hist"] = np.array(ps.train(cfg, data).loss_history)
    cfg = ps.TrainConfig(mode="pp", n=n, p=p, layers=L, k=k, batch=B, lr=1e-4, max_epochs=2,
                         seed=seed, loss_reduction="mean", optimizer="adam", scheduler="threads")
    c1["train_adam_hist"] = np.array(ps.train(cfg, data).loss_history)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **c1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
