import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200.training import TrainConfig, gen_dataset, train_engine, train
from paper_2508_00960_b200 import training as T
c1 = np.load("tests/golden/c1.npz")
n, p, k, L, B, seed = (int(v) for v in c1["cfg"])
cfg = TrainConfig(mode="pp", n=n, p=p, layers=L, k=k, batch=B, lr=1e-4, max_epochs=1, seed=seed, loss_reduction="mean", dtype=torch.float32)
data = gen_dataset(n, 1024, seed)
# per-iteration losses of the engine loop
losses = []
orig = T.TrainResult
from paper_2508_00960_b200.engine import PhantomEngine
eng = PhantomEngine(n, p, k, L, B, reduction="mean", optimizer="sgd", lr=1e-4, dtype=torch.float32, seed=seed)
eng.load_params(T._reference_rows(cfg, eng.local))
xs, ys = T._shard_batches(data, n // p, eng.local, torch.float32)
for it in range(16):
    sl = slice(it * B, (it + 1) * B)
    eng.set_batch([x[sl] for x in xs], [y[sl] for y in ys])
    eng.step(graph=False)
    losses.append(eng.read_loss())
print("engine", np.round(losses, 3).tolist(), np.mean(losses))
r = train(cfg, data)
print("api train", r.loss_history)
print("ref", c1["train_sgd_hist"])
# oracle first iterations (f64)
from oracle import phantom_oracle as po
inputs, targets, _ = po.gen_dataset(n, 1024, seed)
model = po.init_phantom_model(n, p, k, L, seed)
ol = []
s = n // p
for it in range(4):
    sl = slice(it * B, (it + 1) * B)
    out = po.pp_iteration(model, ["relu"] * L, [inputs[j*s:(j+1)*s, sl] for j in range(p)], [targets[j*s:(j+1)*s, sl] for j in range(p)], "mean")
    ol.append(out["global_loss"])
    for j in range(p):
        params, grads = po.pp_param_list(model[j], out["grads"][j])
        po.sgd_step(params, grads, 1e-4)
print("oracle", np.round(ol, 3).tolist())
