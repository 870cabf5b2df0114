"""Debug: per-parameter update error of one engine SGD step vs the oracle (small 64-aligned shapes)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import phantom_oracle as po
from test_engine_gpu import _setup
n, p, k, L, B, lr = [int(x) for x in os.environ.get("DBG_CFG", "512,4,64,3,256").split(",")] + [3e-3]
eng, model, x, y = _setup(n, p, k, L, B, torch.bfloat16, "sgd", lr)
import copy
m0 = copy.deepcopy(model)
eng.step(graph=False)
print("loss", eng.read_loss())
s = n // p
out = po.pp_iteration(model, ["relu"] * L, [x[j * s:(j + 1) * s] for j in range(p)], [y[j * s:(j + 1) * s] for j in range(p)], "mean")
print("oracle loss", out["global_loss"])
for j in range(p):
    params, gs = po.pp_param_list(model[j], out["grads"][j])
    po.sgd_step(params, gs, lr)
for jj in range(p):
    for l in range(L):
        v = eng.layer_views(jj, l)
        errs = []
        for name in ("local", "compressor", "bias"):
            a = v[name].double().cpu().numpy() - m0[jj][l][name]
            b = model[jj][l][name] - m0[jj][l][name]
            errs.append(f"{name} {np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.2e}")
        for i, d in v["decompressors"].items():
            a = d.double().cpu().numpy() - m0[jj][l]["decompressors"][i]
            b = model[jj][l]["decompressors"][i] - m0[jj][l]["decompressors"][i]
            errs.append(f"D{i} {np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.2e}")
        print(jj, l, " ".join(errs))
