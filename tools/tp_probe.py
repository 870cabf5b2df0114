"""TP engine (fp32 tier) step-by-step check: after every step, the compute copy the next step
reads must equal the fp32 master, and the step's update W_t - W_{t-1} must equal -lr * (the
dense oracle's gradient at the engine's own W_{t-1}), so a wrong gradient is pinned to its step."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phantom_oracle as po
from paper_2508_00960_b200.tensor_parallel import TPEngine
n, L, B, lr = 512, 4, 64, 3e-3
graph = len(sys.argv) > 1 and sys.argv[1] == "graph"
rng = np.random.default_rng(5); a = np.sqrt(6.0 / (2 * n))
W = [rng.uniform(-a, a, (n, n)) for _ in range(L)]; b = [0.1 * rng.standard_normal(n) for _ in range(L)]
x = rng.standard_normal((n, B)); y = np.maximum(rng.standard_normal((n, B)), 0.0)
eng = TPEngine(n, L, B, lr=lr, dtype=torch.float32)
eng.load_full_weights(W, b)
for par in (0, 1):
    eng.set_batch(torch.from_numpy(x.T.copy()).cuda(), torch.from_numpy(y.T.copy()).cuda(), par)


def state():
    Ws, bs = [], []
    for m in range(L // 2):
        Ws += [eng.Wa[m].double().cpu().numpy().copy(), eng.Wb[m].double().cpu().numpy().copy()]
        bs += [eng._ba(m).double().cpu().numpy().copy(), eng._bb(m).double().cpu().numpy().copy()]
    return Ws, bs


for step in range(4):
    W0, b0 = state()
    par = eng.parity
    if graph and step == 1:
        eng.capture()
    eng.step(graph=graph and step >= 1)
    loss = eng.read_loss()
    W1, b1 = state()
    out = po.tp_iteration([[{"weight": W0[l], "bias": b0[l]} for l in range(L)]], ["relu"] * L, [x], [y], "mean")
    errs = []
    for l in range(L):
        g = out["grads"][0][l]
        errs.append(np.linalg.norm((W1[l] - W0[l]) + lr * g["weight"]) / np.linalg.norm(lr * g["weight"]))
        errs.append(np.linalg.norm((b1[l] - b0[l]) + lr * g["bias"]) / np.linalg.norm(lr * g["bias"]))
    nxt = 1 - par
    cc = max(max((eng.wa[nxt][m] - eng.Wa[m]).abs().max().item(), (eng.wb[nxt][m] - eng.Wb[m]).abs().max().item())
             for m in range(L // 2))
    print(f"step {step} loss {loss:.6f} oracle {out['global_loss']:.6f} per-step update err max {max(errs):.2e} "
          f"(per tensor {['%.1e' % e for e in errs]}) |copy-master| {cc:.1e}")


# ---- intermediate check of one more (par = parity) step against a float64 restatement --------
def f64(t):
    return t.double()


eng2 = TPEngine(n, L, B, lr=lr, dtype=torch.float32)
eng2.load_full_weights(W, b)
for par in (0, 1):
    eng2.set_batch(torch.from_numpy(x.T.copy()).cuda(), torch.from_numpy(y.T.copy()).cuda(), par)
for step in range(2):
    par = eng2.parity
    Wa = [f64(eng2.Wa[m]).clone() for m in range(L // 2)]
    Wb = [f64(eng2.Wb[m]).clone() for m in range(L // 2)]
    ba = [f64(eng2._ba(m)).clone() for m in range(L // 2)]
    bb = [f64(eng2._bb(m)).clone() for m in range(L // 2)]
    eng2.step(graph=False)
    eng2.read_loss()
    X = f64(eng2.X[par][0])
    T = f64(eng2.Tgt[par])
    Xs, Ys = [X], []
    for m in range(L // 2):
        Ya = torch.clamp_min(Xs[-1] @ Wa[m].t() + ba[m], 0)
        Ys.append(Ya)
        Xs.append(torch.clamp_min(Ya @ Wb[m].t() + bb[m], 0))
    D = (Xs[-1] - T) * (Xs[-1] > 0) / B
    rel = lambda a, b_: float((a.double() - b_).norm() / b_.norm())   # noqa: E731
    msg = [f"Ya{m} {rel(eng2.Ya[m], Ys[m]):.1e} X{m + 1} {rel(eng2.X[par][m + 1], Xs[m + 1]):.1e}" for m in range(L // 2)]
    msg.append(f"Dout {rel(eng2.Dfull[0], D):.1e}")
    for m in range(L // 2 - 1, -1, -1):
        Dya = (D @ Wb[m]) * (Ys[m] > 0)
        if m == 0:
            msg.append(f"Dya0 {rel(eng2.Dya, Dya):.1e}")
        if m > 0:
            D = (Dya @ Wa[m]) * (Xs[m] > 0)
            msg.append(f"D{m - 1 + 1}in {rel(eng2.Dfull[1], D):.1e}")
    print(f"[intermediates] step {step} par {par}: " + "  ".join(msg))
    Xe, Te = f64(eng2.X[par][L // 2]), f64(eng2.Tgt[par])
    De = (Xe - Te) * (Xe > 0) / B
    print(f"   engine-internal: Dout vs (X_P - T) mask / B from the engine's own buffers {rel(eng2.Dfull[0], De):.1e}; "
          f"Tgt vs y {rel(eng2.Tgt[par], torch.from_numpy(y.T.copy()).cuda().double()):.1e}; "
          f"loss {float(eng2.loss.item()):.6f} vs {0.5 * float(((Xe - Te) ** 2).sum()) / B:.6f}")
    Xr = Xs[-1]
    flips = int(((Xr > 0) != (Xe > 0)).sum())
    near = float(Xe[(Xr > 0) != (Xe > 0)].abs().max()) if flips else 0.0
    print(f"   output ReLU mask flips engine vs float64: {flips} of {Xr.numel()} (largest |y| at a flip {near:.2e}); "
          f"|X_P engine - f64| max {float((Xe - Xr).abs().max()):.2e}")
