"""TEACHER-FORCED CHECKER — test infrastructure only, never the product path.

A torch restatement of the per-layer functions of oracle/phantom_oracle.py (itself pinned to the
reference's golden vectors) in the engine's [batch, features] layout, so the GPU path can be
checked kernel by kernel at the BENCHMARKED sizes (C3: n=16384, p=8, k=128, B=8192), where the
float64 CPU oracle would take minutes per step.  Run on the GPU in fp32 with TF32 disabled.

Teacher forcing: every check feeds the teacher the ENGINE's own inputs of that layer
(its bf16 activations, gathered phantoms, deltas, received error phantoms and the bf16 compute
copy of the weights the step read), so each comparison isolates one kernel's arithmetic from the
rounding accumulated upstream and from ReLU-mask flips; what remains is fp32-accumulation order
plus the rounding of the engine's own output (bf16 2^-9 relative per element, fp32 for the raw
weight gradients).  tests/test_teacher.py pins every function here against phantom_oracle in
float64 on the CPU.

Only tests/ and tools/ parity scripts import this module.

Reference semantics (file:line in /root/reference/pkg/src/phantomsim):
  forward_layer        phantom.py:135-166  z = L.y + sum_{i != j asc} D_i.g_i ; pre = z + b
  output_delta / loss  phantom.py:169-182, training.py:59-71, 196-199
  error_phantoms       phantom.py:185-207 + collectives.py:345-357 (ascending-rank sums)
  param_grads          phantom.py:239-267
  backward_delta       phantom.py:210-236  (L^T delta + C^T r) * act'(pre_prev)
"""

from __future__ import annotations

import torch


def _peers(p, j):
    """Source ranks of rank j's decompressors in storage order (ascending, self skipped,
    phantom.py:128-129)."""
    return [i for i in range(p) if i != j]


def engine_weights(eng, jj, l, par, bias=None, dtype=torch.float32):
    """The weights a step of parity `par` READ for local rank jj, layer l: the compute copy
    eng.w[par] (bf16 in the bf16 tier) widened to `dtype`, decompressors stacked [(p-1), s, k]
    in ascending source order.  `bias` overrides eng.bias (pass the pre-step snapshot)."""
    v = eng.layer_views(jj, l, master=eng.w[par][jj, l])
    decs = [v["decompressors"][i].to(dtype) for i in _peers(eng.p, eng.local[jj])]
    return {"local": v["local"].to(dtype), "compressor": v["compressor"].to(dtype),
            "dec": torch.stack(decs) if decs else None,
            "bias": (eng.bias[jj, l] if bias is None else bias).to(dtype)}


def compress(W, y):
    """g = y . C^T  ([B, s] -> [B, k]); phantom.py:153."""
    return y @ W["compressor"].t()


def forward_layer(W, j, y, G, act="relu"):
    """Rank j's layer forward from its input y [B, s] and the gathered phantoms G (list over all
    ranks of [B, k]; slot j unused): returns (pre, out).  phantom.py:152-160."""
    z = y @ W["local"].t()
    for q, i in enumerate(_peers(len(G), j)):
        z = z + G[i] @ W["dec"][q].t()
    pre = z + W["bias"]
    return pre, (torch.clamp_min(pre, 0.0) if act == "relu" else pre)


def phantom_term(W, j, G):
    """sum_{i != j} g_i . D_i^T alone (the part a lost phantom slot would remove)."""
    z = None
    for q, i in enumerate(_peers(len(G), j)):
        t = G[i] @ W["dec"][q].t()
        z = t if z is None else z + t
    return z


def loss_and_delta(y_out, pre, target, reduction, act="relu"):
    """Local half-squared loss and output delta (÷B in mean mode, training.py:66-69, 196-199)."""
    B = y_out.shape[0]
    diff = y_out - target
    scale = 1.0 / B if reduction == "mean" else 1.0
    loss = 0.5 * float((diff.double() ** 2).sum()) * scale
    g = (pre > 0).to(diff.dtype) if act == "relu" else torch.ones_like(diff)
    return loss, diff * g * scale


def error_phantoms(Ws, deltas):
    """received r_i = sum_{j != i, ascending j} delta_j . D_{i->j}  ([B, k] per rank i);
    phantom.py:199-205 then the reduce-scatter's ascending-rank sum (collectives.py:350-356).
    Ws[j] / deltas[j] over ALL p ranks."""
    p = len(Ws)
    out = []
    for i in range(p):
        r = None
        for j in range(p):
            if j == i:
                continue
            q = _peers(p, j).index(i)
            t = deltas[j] @ Ws[j]["dec"][q]
            r = t if r is None else r + t
        out.append(r)
    return out


def param_grads(j, delta, y_prev, G, received):
    """phantom.py:239-267 in [B, .] layout: d local = delta^T y, d compressor = r^T y,
    d decompressor_i = delta^T g_i (s x k, ascending i != j), d bias = sum_batch delta."""
    p = len(G)
    return {"local": delta.t() @ y_prev, "compressor": received.t() @ y_prev,
            "dec": torch.stack([delta.t() @ G[i] for i in _peers(p, j)]) if p > 1 else None,
            "bias": delta.sum(0)}


def backward_delta(W, delta, received, y_prev_out, act="relu"):
    """delta_{l-1} = (delta . L + r . C) * act'(pre_{l-1}); the ReLU mask is y_{l-1} > 0, which
    equals pre_{l-1} > 0 (phantom.py:227-236)."""
    d = delta @ W["local"] + received @ W["compressor"]
    return d * (y_prev_out > 0).to(d.dtype) if act == "relu" else d


def nerr(a, b):
    """Normwise relative error ||a - b|| / ||b|| in float64."""
    a = a.double()
    b = b.double()
    den = float(torch.linalg.vector_norm(b))
    return float(torch.linalg.vector_norm(a - b)) / (den if den > 0 else 1.0)


def rel(a, b):
    """||a|| / ||b||."""
    den = float(torch.linalg.vector_norm(b.double()))
    return float(torch.linalg.vector_norm(a.double())) / (den if den > 0 else 1.0)


def check_engine_step(eng, par, bias0, targets, loss, act="relu"):
    """Teacher-forced check of ONE eager training step of a capture=True PhantomEngine holding
    all p logical ranks (world == 1; any launch plan).  `par` = the parity the step ran,
    `bias0` = eng.bias before the step, `targets[j]` = rank j's [B, s] targets, `loss` = the
    engine's global loss.  Returns {quantity: worst normwise relative error} plus the smallest
    share of the phantom terms (forward: ||sum_i g_i D_i^T|| / ||pre - b||; backward:
    ||r C|| / ||delta L||) — a dropped phantom slot moves the checked tensor by at least
    share / (p - 1), which the tolerance must stay below."""
    assert eng.world == 1 and eng.capture_grads, "needs a capture=True engine with every rank local"
    p, L = eng.p, eng.L
    worst = {k_: 0.0 for k_ in ("phantoms", "activations", "output", "delta_out", "loss", "received",
                                "grad_local", "grad_compressor", "grad_decompressor", "grad_bias", "delta")}
    share = {"forward": float("inf"), "backward": float("inf")}

    def up(key, v):
        worst[key] = max(worst[key], v)

    total = 0.0
    Wl = [None] * L
    for l in range(L):
        Ws = [engine_weights(eng, j, l, par, bias0[j, l]) for j in range(p)]
        Wl[l] = Ws
        Gv = eng.phantoms_view(l)
        G = [Gv[i].float() for i in range(p)]
        for j in range(p):
            Y = eng.Y[par][j][l].float()
            up("phantoms", nerr(G[j], compress(Ws[j], Y)))
            pre, out = forward_layer(Ws[j], j, Y, G, act)
            if p > 1:
                share["forward"] = min(share["forward"], rel(phantom_term(Ws[j], j, G), pre - Ws[j]["bias"]))
            if l < L - 1:
                up("activations", nerr(eng.Y[par][j][l + 1], out))
            else:
                if not eng.skip_output:
                    up("output", nerr(eng.Y[par][j][L], out))
                lj, d = loss_and_delta(out, pre, targets[j].float(), eng.reduction, act)
                total += lj
                up("delta_out", nerr(eng.deltas[L - 1][j], d))
            del pre, out
    worst["loss"] = abs(loss - total) / abs(total)
    for l in range(L - 1, -1, -1):
        Ws = Wl[l]
        D = [eng.deltas[l][j].float() for j in range(p)]
        Rt = error_phantoms(Ws, D)
        Gv = eng.phantoms_view(l)
        G = [Gv[i].float() for i in range(p)]
        for j in range(p):
            Re = eng.received_view(l, j).float()
            if p > 1:
                up("received", nerr(Re, Rt[j]))
            Y = eng.Y[par][j][l].float()
            g = param_grads(j, D[j], Y, G, Re)
            v = eng.layer_views(j, l, master=eng.grad[j, l])
            up("grad_local", nerr(v["local"], g["local"]))
            if p > 1:
                up("grad_compressor", nerr(v["compressor"], g["compressor"]))
                for q, i in enumerate(_peers(p, j)):
                    up("grad_decompressor", nerr(v["decompressors"][i], g["dec"][q]))
            up("grad_bias", nerr(eng.gbias[j, l], g["bias"]))
            if l > 0:
                up("delta", nerr(eng.deltas[l - 1][j], backward_delta(Ws[j], D[j], Re, Y, act)))
                if p > 1:
                    share["backward"] = min(share["backward"], rel(Re @ Ws[j]["compressor"], D[j] @ Ws[j]["local"]))
    return worst, share


def train_sgd_curve(model, x, y, layers, batch, lr, epochs, dtype, reduction="mean", act="relu"):
    """The reference's PP training loop (training.py:276-309: contiguous mini-batches, pre-update
    iteration loss, epoch loss = mean of iteration losses, SGD) restated with this module's
    per-layer functions in `dtype` on the CPU — used to measure how far exact fp32 arithmetic
    drifts from float64 over a training run.  model: oracle-format (list over ranks of lists over
    layers of numpy dicts), x / y: (n, samples) numpy."""
    p = len(model)
    n = x.shape[0]
    s = n // p
    t = lambda a: torch.tensor(a, dtype=dtype)   # noqa: E731  (a copy: updates stay local)
    W = [[{"local": t(lay["local"]), "compressor": t(lay["compressor"]),
           "dec": torch.stack([t(lay["decompressors"][i]) for i in _peers(p, j)]), "bias": t(lay["bias"])}
          for lay in model[j]] for j in range(p)]
    X = [t(x[j * s:(j + 1) * s].T) for j in range(p)]
    Y = [t(y[j * s:(j + 1) * s].T) for j in range(p)]
    iters = x.shape[1] // batch
    hist = []
    for _ in range(epochs):
        losses = []
        for it in range(iters):
            sl = slice(it * batch, (it + 1) * batch)
            acts = [[X[j][sl] for j in range(p)]]
            Gs = []
            for l in range(layers):
                G = [compress(W[j][l], acts[-1][j]) for j in range(p)]
                Gs.append(G)
                acts.append([forward_layer(W[j][l], j, acts[-1][j], G, act)[1] for j in range(p)])
            loss, D = 0.0, []
            for j in range(p):
                out = acts[-1][j]
                lj, d = loss_and_delta(out, out, Y[j][sl], reduction, act)   # ReLU mask: out > 0 == pre > 0
                loss += lj
                D.append(d)
            losses.append(loss)
            grads = [[None] * layers for _ in range(p)]
            for l in range(layers - 1, -1, -1):
                R = error_phantoms([W[j][l] for j in range(p)], D)
                for j in range(p):
                    grads[j][l] = param_grads(j, D[j], acts[l][j], Gs[l], R[j])
                if l > 0:
                    D = [backward_delta(W[j][l], D[j], R[j], acts[l][j], act) for j in range(p)]
            for j in range(p):
                for l in range(layers):
                    g, w = grads[j][l], W[j][l]
                    w["local"] -= lr * g["local"]
                    w["compressor"] -= lr * g["compressor"]
                    w["dec"] -= lr * g["dec"]
                    w["bias"] -= lr * g["bias"]
        hist.append(sum(losses) / len(losses))
    return hist
