"""CPU ORACLE — test infrastructure only, never the product path.

A float64 numpy restatement of the reference algorithm for the phantom-parallel hot path
(phantomsim, /root/reference/pkg/src/phantomsim).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg may import this module, and only as the checker
or the timed CPU baseline.  libppx.so never calls it; the GPU package has no CPU fallback.

Parity is PINNED: tests/test_oracle.py checks every function below against golden vectors the
reference itself produced (tests/golden/make_golden.py imports phantomsim from /root/reference and
writes tests/golden/*.npz), plus the reference tests' hand-worked known answers.

Layout follows the reference: activations are (features x batch) with batch as columns
(core.py:3-4); a model is a list over ranks of lists over layers of dicts
{local (s,s), compressor (k,s), decompressors {src: (s,k)}, bias (s,)}.
All ranks are computed in one process; the collectives are restated inline with the reference's
semantics (concatenate in ascending rank order; sums evaluated in ascending rank order,
collectives.py:337-357).
"""

from __future__ import annotations

import math
import zlib

import numpy as np

RELU = "relu"
IDENTITY = "identity"


# ----------------------------------------------------------------------------------------------
# numerics core (core.py)
# ----------------------------------------------------------------------------------------------
def act_apply(z, act):
    """core.py:70-73 — ReLU = max(z, 0); identity copies."""
    return np.maximum(z, 0.0) if act == RELU else np.array(z, dtype=np.float64, copy=True)


def act_grad(pre, act):
    """core.py:75-78 — ReLU'(x) = 1 iff x > 0 (so ReLU'(0) = 0)."""
    return np.where(pre > 0, 1.0, 0.0) if act == RELU else np.ones_like(np.asarray(pre, dtype=np.float64))


def _key_part(part) -> int:
    """core.py:97-100."""
    if isinstance(part, str):
        return zlib.crc32(part.encode("utf-8"))
    return int(part) & 0xFFFFFFFF


def substream(seed: int, *key) -> np.random.Generator:
    """core.py:103-114 — Philox stream keyed by (seed, *key) through a SeedSequence spawn key."""
    ss = np.random.SeedSequence(entropy=int(seed) & (2**63 - 1),
                                spawn_key=tuple(_key_part(p) for p in key))
    return np.random.Generator(np.random.Philox(key=ss.generate_state(2, dtype=np.uint64)))


def uniform_init(rng, rows, cols, fan_in, fan_out):
    """core.py:117-121 — U[-a, a], a = sqrt(6 / (fan_in + fan_out))."""
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-a, a, size=(rows, cols))


# ----------------------------------------------------------------------------------------------
# model construction (phantom.py:102-132, tensor_parallel.py:67-92)
# ----------------------------------------------------------------------------------------------
def init_phantom_model(n, p, k, layers, seed=0):
    """phantom.py:102-132: per (layer l, rank j) local/compressor/decompressor[i] substreams."""
    s = n // p
    model = []
    for j in range(p):
        own = []
        for l in range(layers):
            own.append({
                "local": uniform_init(substream(seed, "pp", l, j, "local"), s, s, s, s),
                "compressor": uniform_init(substream(seed, "pp", l, j, "compressor"), k, s, s, k),
                "decompressors": {i: uniform_init(substream(seed, "pp", l, j, "decompressor", i),
                                                  s, k, k, s) for i in range(p) if i != j},
                "bias": np.zeros(s),
            })
        model.append(own)
    return model


def full_layer_weight(n, layer, seed):
    """tensor_parallel.py:67-73 — p-independent full weight of one TP layer."""
    return uniform_init(substream(seed, "tp", layer, "weight"), n, n, n, n)


def init_tp_model(n, p, layers, seed=0):
    """tensor_parallel.py:76-92 — rank j owns rows [j s, (j+1) s) of each full weight."""
    s = n // p
    model = [[] for _ in range(p)]
    for l in range(layers):
        full = full_layer_weight(n, l, seed)
        for j in range(p):
            model[j].append({"weight": full[j * s:(j + 1) * s].copy(), "bias": np.zeros(s)})
    return model


def gen_dataset(n, samples, seed):
    """training.py:43-56 — teacher, inputs ~ N(0,1) from substream(seed, "dataset");
    targets = relu(teacher @ relu(inputs))."""
    rng = substream(seed, "dataset")
    teacher = rng.standard_normal((n, n))
    inputs = rng.standard_normal((n, samples))
    return inputs, np.maximum(teacher @ np.maximum(inputs, 0.0), 0.0), teacher


# ----------------------------------------------------------------------------------------------
# phantom-parallel hot path, all ranks at once
# ----------------------------------------------------------------------------------------------
def pp_forward_layer(layers_l, y_prev, act):
    """phantom.py:135-166 for every rank of one layer.

    layers_l[j] is rank j's shard, y_prev[j] its (s, B) input. Returns (outputs, tapes) with
    tape = {inputs, preact, phantoms {src: (k, B)} including the own block}.
    """
    p = len(layers_l)
    own = [layers_l[j]["compressor"] @ y_prev[j] for j in range(p)]          # :153
    gathered = np.concatenate(own, axis=0)                                     # :154, collectives.py:338
    k = own[0].shape[0]
    outs, tapes = [], []
    for j in range(p):
        lay = layers_l[j]
        phantoms = {i: gathered[i * k:(i + 1) * k] for i in range(p)}         # :155
        z = lay["local"] @ y_prev[j]                                           # :152
        for i in sorted(lay["decompressors"]):                                 # :156-159
            z = z + lay["decompressors"][i] @ phantoms[i]
        preact = z + lay["bias"][:, None]                                      # :160
        outs.append(act_apply(preact, act))                                    # :163
        tapes.append({"inputs": y_prev[j], "preact": preact, "phantoms": phantoms})
    return outs, tapes


def pp_output_delta(y_out, y_true, preact, act):
    """phantom.py:169-182 — (y_out - y_true) * act'(preact)."""
    return (y_out - y_true) * act_grad(preact, act)


def pp_exchange_error_phantoms(layers_l, delta):
    """phantom.py:185-207 — slot i of rank r's (p k, B) buffer = D_i^T delta_r (own slot zero);
    reduce-scatter gives rank j the ascending-rank sum of slot j (collectives.py:345-357)."""
    p = len(layers_l)
    k = layers_l[0]["compressor"].shape[0]
    b = delta[0].shape[1]
    contributions = []
    for r in range(p):
        buf = np.zeros((p * k, b))
        for i in sorted(layers_l[r]["decompressors"]):
            buf[i * k:(i + 1) * k] = layers_l[r]["decompressors"][i].T @ delta[r]
        contributions.append(buf)
    received = []
    for j in range(p):
        acc = contributions[0][j * k:(j + 1) * k].copy()
        for r in range(1, p):
            acc += contributions[r][j * k:(j + 1) * k]
        received.append(acc)
    return received


def pp_backward_layer(layer_next, delta_next, preact, act, received):
    """phantom.py:210-236 — (local^T delta + compressor^T r) * act'(preact)."""
    back = layer_next["local"].T @ delta_next + layer_next["compressor"].T @ received
    return back * act_grad(preact, act)


def pp_param_grads(layer, delta, tape, received):
    """phantom.py:239-267."""
    return {
        "bias": delta.sum(axis=1),                                             # :253
        "local": delta @ tape["inputs"].T,                                     # :256
        "compressor": received @ tape["inputs"].T,                             # :257
        "decompressors": {i: delta @ tape["phantoms"][i].T                     # :259-264
                          for i in sorted(layer["decompressors"])},
    }


def mse_loss(y_out, y_true, reduction):
    """training.py:59-71 — per-rank local half-squared error and the ascending-rank global sum."""
    local = []
    for yo, yt in zip(y_out, y_true):
        d = yo - yt
        v = 0.5 * float(np.sum(d * d))
        if reduction == "mean":
            v /= yo.shape[1]
        local.append(v)
    total = local[0]
    for v in local[1:]:
        total += v
    return local, total


def pp_iteration(model, acts, x_shards, y_shards, reduction="sum"):
    """training.py:181-213 for all ranks: forward, loss, delta_L (/B if mean), then per layer
    (descending): exchange (reduce-scatter), param grads, recurrence (if l > 0)."""
    p = len(model)
    L = len(acts)
    out = list(x_shards)
    tapes = [[] for _ in range(p)]
    for l in range(L):
        out, t = pp_forward_layer([model[j][l] for j in range(p)], out, acts[l])
        for j in range(p):
            tapes[j].append(t[j])
    local, glob = mse_loss(out, y_shards, reduction)
    delta = [pp_output_delta(out[j], y_shards[j], tapes[j][-1]["preact"], acts[-1]) for j in range(p)]
    if reduction == "mean":
        delta = [d / x_shards[0].shape[1] for d in delta]
    grads = [[None] * L for _ in range(p)]
    deltas = [[None] * L for _ in range(p)]
    received_all = [[None] * L for _ in range(p)]
    for l in range(L - 1, -1, -1):
        layers_l = [model[j][l] for j in range(p)]
        for j in range(p):
            deltas[j][l] = delta[j]
        received = pp_exchange_error_phantoms(layers_l, delta)
        for j in range(p):
            received_all[j][l] = received[j]
            grads[j][l] = pp_param_grads(layers_l[j], delta[j], tapes[j][l], received[j])
        if l > 0:
            delta = [pp_backward_layer(layers_l[j], delta[j], tapes[j][l - 1]["preact"], acts[l - 1],
                                       received[j]) for j in range(p)]
    return {"y_out": out, "local_loss": local, "global_loss": glob, "grads": grads,
            "deltas": deltas, "tapes": tapes, "received": received_all}


def pp_forward(model, acts, x_shards):
    """Forward-only inference (test_phantom.py:66-71 loop of pp_forward_layer)."""
    out = list(x_shards)
    for l in range(len(acts)):
        out, _ = pp_forward_layer([model[j][l] for j in range(len(model))], out, acts[l])
    return out


# ----------------------------------------------------------------------------------------------
# tensor-parallel comparison (tensor_parallel.py:95-153, training.py:216-244)
# ----------------------------------------------------------------------------------------------
def tp_iteration(model, acts, x_shards, y_shards, reduction="sum"):
    p = len(model)
    L = len(acts)
    s = x_shards[0].shape[0]
    out = list(x_shards)
    tapes = [[] for _ in range(p)]
    for l in range(L):
        y_full = np.concatenate(out, axis=0)                                  # all_gather :111
        new = []
        for j in range(p):
            lay = model[j][l]
            preact = lay["weight"] @ y_full + lay["bias"][:, None]            # :115-116
            tapes[j].append({"y_full": y_full, "preact": preact})
            new.append(act_apply(preact, acts[l]))
        out = new
    local, glob = mse_loss(out, y_shards, reduction)
    delta = [pp_output_delta(out[j], y_shards[j], tapes[j][-1]["preact"], acts[-1]) for j in range(p)]
    if reduction == "mean":
        delta = [d / x_shards[0].shape[1] for d in delta]
    grads = [[None] * L for _ in range(p)]
    deltas = [[None] * L for _ in range(p)]
    for l in range(L - 1, -1, -1):
        for j in range(p):
            deltas[j][l] = delta[j]
            grads[j][l] = {"weight": delta[j] @ tapes[j][l]["y_full"].T, "bias": delta[j].sum(axis=1)}
        if l > 0:
            full = [model[j][l]["weight"].T @ delta[j] for j in range(p)]    # :145
            summed = full[0].copy()
            for f in full[1:]:                                                 # all_reduce asc :146
                summed += f
            delta = [summed[j * s:(j + 1) * s] * act_grad(tapes[j][l - 1]["preact"], acts[l - 1])
                     for j in range(p)]
    return {"y_out": out, "local_loss": local, "global_loss": glob, "grads": grads, "deltas": deltas}


# ----------------------------------------------------------------------------------------------
# dense twin (reference.py:143-172) and optimizers (training.py:74-105)
# ----------------------------------------------------------------------------------------------
def effective_weight(model, l):
    """reference.py:143-157 — diagonal blocks local_j, block (j, i) = D_{i->j} C_i."""
    p = len(model)
    s = model[0][l]["local"].shape[0]
    n = p * s
    w = np.zeros((n, n))
    for j in range(p):
        w[j * s:(j + 1) * s, j * s:(j + 1) * s] = model[j][l]["local"]
        for i, dec in model[j][l]["decompressors"].items():
            w[j * s:(j + 1) * s, i * s:(i + 1) * s] = dec @ model[i][l]["compressor"]
    return w


def dense_forward(weights, biases, acts, x):
    """reference.py:58-79."""
    y = x
    for w, b, a in zip(weights, biases, acts):
        y = act_apply(w @ y + b[:, None], a)
    return y


def sgd_step(params, grads, lr):
    """training.py:74-82 (non-finite check omitted: the GPU path flags it on device)."""
    for theta, g in zip(params, grads):
        theta -= lr * g


def adam_step(params, grads, state, lr, betas=(0.9, 0.999), eps=1e-8):
    """training.py:92-105; state = {"m": [...], "v": [...], "t": int}."""
    state["t"] += 1
    b1, b2 = betas
    for i, (theta, g) in enumerate(zip(params, grads)):
        state["m"][i] = b1 * state["m"][i] + (1 - b1) * g
        state["v"][i] = b2 * state["v"][i] + (1 - b2) * g * g
        m_hat = state["m"][i] / (1 - b1 ** state["t"])
        v_hat = state["v"][i] / (1 - b2 ** state["t"])
        theta -= lr * m_hat / (np.sqrt(v_hat) + eps)


def pp_param_list(model_rank, grads_rank):
    """training.py:251-264 order: per layer local, compressor, decompressors asc, bias."""
    params, gs = [], []
    for lay, g in zip(model_rank, grads_rank):
        params += [lay["local"], lay["compressor"]]
        gs += [g["local"], g["compressor"]]
        for i in sorted(lay["decompressors"]):
            params.append(lay["decompressors"][i])
            gs.append(g["decompressors"][i])
        params.append(lay["bias"])
        gs.append(g["bias"])
    return params, gs


def train_pp(model, acts, inputs, targets, batch, lr, epochs, reduction="sum", optimizer="sgd"):
    """training.py:276-309 loop: contiguous column mini-batches, pre-update losses,
    epoch loss = mean of iteration losses. Mutates `model` in place; returns the history."""
    p = len(model)
    n, samples = inputs.shape
    s = n // p
    iters = samples // batch
    history = []
    states = [None] * p
    for _ in range(epochs):
        losses = []
        for it in range(iters):
            sl = slice(it * batch, (it + 1) * batch)
            xs = [inputs[j * s:(j + 1) * s, sl] for j in range(p)]
            ys = [targets[j * s:(j + 1) * s, sl] for j in range(p)]
            out = pp_iteration(model, acts, xs, ys, reduction)
            for j in range(p):
                params, gs = pp_param_list(model[j], out["grads"][j])
                if optimizer == "adam":
                    if states[j] is None:
                        states[j] = {"m": [np.zeros_like(g) for g in gs],
                                     "v": [np.zeros_like(g) for g in gs], "t": 0}
                    adam_step(params, gs, states[j], lr)
                else:
                    sgd_step(params, gs, lr)
            losses.append(out["global_loss"])
        history.append(float(np.mean(losses)))
    return history


# ----------------------------------------------------------------------------------------------
# sizing and FLOP accounting (phantom.py:270-296)
# ----------------------------------------------------------------------------------------------
def pp_model_size(n, p, k, layers):
    """phantom.py:270-280 — layers * (n^2/p + p k n)."""
    return layers * (n * n // p + p * k * n)


def valid_k(n, p):
    """phantom.py:283-296."""
    s = n // p
    return s, s * (p - 1) / p


def pp_gemm_flops_per_rank(n, p, k, layers, batch):
    """6 L B s (s + p k) - 2 B s (s + k): the GEMM FLOPs one rank executes per training step."""
    s = n // p
    return 6 * layers * batch * s * (s + p * k) - 2 * batch * s * (s + k)
