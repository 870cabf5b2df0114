"""Multi-GPU parity: PhantomEngine on N GPUs (torchrun, one process per GPU) vs the CPU oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mp_parity.py [--dtype fp32|bf16]
        [--p P --k K --B B --width n --lr LR] [--fused auto|0|1] [--nvrs auto|0|1]

Each process owns p/N logical ranks.  Step 1 runs eagerly with the raw fp32 weight gradients
captured and compares them (local, compressor, every decompressor, bias) with the oracle's
step-1 gradients; steps 2..S replay CUDA graphs; then the losses and the weight UPDATES W_S - W_0
of every tensor are compared with the oracle's.  Rank 0 prints one JSON verdict (max over ranks).
Then every process re-runs the same steps with a one-GPU engine holding all p logical ranks (the
launch plan parity-tested kernel by kernel in tests/test_parity_scale_gpu.py) and compares the
same quantities with it: that isolates what the multi-GPU exchange adds.
Tolerances vs the float64 oracle: fp32 tier 1e-4 gradients and losses, 1e-3 updates (the fp32
master's rounding, eps32 * |W|, is ~1e-3 of a 3-step update); bf16 tier 1e-1 gradients and
updates (bf16 activations over 3 ReLU layers), 2e-2 losses.  vs the one-GPU engine: fp32 1e-4,
bf16 2e-2 gradients and losses, 5e-2 updates (the two launch plans round differently, and three
steps amplify that in the updates).
"""
import argparse, copy, json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phantom_oracle as po
from paper_2508_00960_b200 import _lib
from paper_2508_00960_b200.engine import PhantomEngine


def nerr(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def tri(v):
    return None if v == "auto" else v == "1"


def snapshot(eng, master):
    """{(j, l): {local, compressor, bias, decompressors{i}}} as float64 numpy of the flat tensor
    `master` (eng.master or eng.grad; bias from eng.bias / eng.gbias)."""
    out = {}
    for jj, j in enumerate(eng.local):
        for l in range(eng.L):
            v = eng.layer_views(jj, l, master=master[jj, l],
                                bias=(eng.gbias if master is eng.grad else eng.bias)[jj, l])
            out[(j, l)] = {nm: v[nm].double().cpu().numpy().copy() for nm in ("local", "compressor", "bias")}
            out[(j, l)]["decompressors"] = {i: d.double().cpu().numpy().copy() for i, d in v["decompressors"].items()}
    return out


def run_engine(eng, model, x, y, args):
    """load the model + batch, step 1 eager with raw gradients captured, steps 2..S (graphs)."""
    n, p, s = eng.n, eng.p, eng.s
    eng.load_params(model)
    xs = [torch.from_numpy(x[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local]
    ys = [torch.from_numpy(y[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local]
    eng.set_batch(xs, ys, 0)
    eng.set_batch(xs, ys, 1)
    losses = []
    eng.step(graph=False)
    losses.append(eng.read_loss())
    grads = snapshot(eng, eng.grad)
    eng.capture_grads = False
    if args.graph:
        eng.capture()
    for _ in range(args.steps - 1):
        eng.step(graph=bool(args.graph))
        losses.append(eng.read_loss())
    return losses, grads, snapshot(eng, eng.master)


def tensors(d):
    for nm in ("local", "compressor", "bias"):
        yield nm, d[nm]
    for i, t in sorted(d["decompressors"].items()):
        yield f"dec{i}", t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--lr", type=float, default=3e-3)
    ap.add_argument("--fused", default="auto")
    ap.add_argument("--nvrs", default="auto")
    ap.add_argument("--k3", default="auto", help="fused error compression + weight gradients")
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--infer", type=int, default=0, help="forward_only calls back to back instead of training")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [_lib.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    n, p, k, L, B, lr = args.width, args.p, args.k, args.layers, args.B, args.lr
    dtype = torch.float32 if args.dtype == "fp32" else torch.bfloat16
    f32 = args.dtype == "fp32"
    tol_g, tol_u, tol_l = (1e-4, 1e-3, 1e-4) if f32 else (1e-1, 1e-1, 2e-2)
    tol_e = 1e-4 if f32 else 2e-2
    model = po.init_phantom_model(n, p, k, L, 3)
    rng = np.random.default_rng(3)
    for row in model:
        for lay in row:
            lay["bias"] = 0.1 * rng.standard_normal(lay["bias"].shape)
    model0 = copy.deepcopy(model)
    s = n // p
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = PhantomEngine(n, p, k, L, B, world=world, rank=rank, device=local, uid=uid[0], lr=lr, dtype=dtype,
                        fused=tri(args.fused), nvrs=tri(args.nvrs), k3_fused=tri(args.k3), capture=True)
    if args.infer:
        eng.load_params(model)
        return infer(args, eng, model, x, rank, world, s, p, L, tol_l)
    losses, grads, weights = run_engine(eng, model, x, y, args)
    plan = {"fused": bool(eng.fused), "nvrs": bool(eng.nvrs), "bwd_fused": bool(eng.bwd_fused),
            "k3_fused": bool(eng.k3_fused)}
    local_ranks = list(eng.local)
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    # the same steps on ONE GPU holding all p logical ranks
    one = PhantomEngine(n, p, k, L, B, lr=lr, dtype=dtype, device=local, capture=True)
    losses1, grads1, weights1 = run_engine(one, model, x, y, args)
    one.close()
    ref, ref_grads = [], None
    for t in range(args.steps):
        out = po.pp_iteration(model, ["relu"] * L, [x[j * s:(j + 1) * s] for j in range(p)],
                              [y[j * s:(j + 1) * s] for j in range(p)], "mean")
        ref.append(out["global_loss"])
        if t == 0:
            ref_grads = out["grads"]
        for j in range(p):
            params, gs = po.pp_param_list(model[j], out["grads"][j])
            po.sgd_step(params, gs, lr)
    worst = {"loss": max(abs(a - b) / abs(b) for a, b in zip(losses, ref)), "grad": 0.0, "update": 0.0,
             "loss_1gpu": max(abs(a - b) / abs(b) for a, b in zip(losses, losses1)), "grad_1gpu": 0.0,
             "update_1gpu": 0.0}
    for j in local_ranks:
        for l in range(L):
            want_g = dict(tensors({**ref_grads[j][l]}))
            w0 = dict(tensors(model0[j][l]))
            w1 = dict(tensors(model[j][l]))
            g1 = dict(tensors(grads1[(j, l)]))
            u1 = dict(tensors(weights1[(j, l)]))
            for nm, g in tensors(grads[(j, l)]):
                worst["grad"] = max(worst["grad"], nerr(g, want_g[nm]))
                worst["grad_1gpu"] = max(worst["grad_1gpu"], nerr(g, g1[nm]))
            for nm, wt in tensors(weights[(j, l)]):
                worst["update"] = max(worst["update"], nerr(wt - w0[nm], w1[nm] - w0[nm]))
                worst["update_1gpu"] = max(worst["update_1gpu"], nerr(wt - w0[nm], u1[nm] - w0[nm]))
    keys = list(worst)
    w = torch.tensor([worst[k_] for k_ in keys], device="cuda", dtype=torch.float64)
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    worst = dict(zip(keys, (float(v) for v in w)))
    tol = {"loss": tol_l, "grad": tol_g, "update": tol_u, "loss_1gpu": tol_e, "grad_1gpu": tol_e,
           "update_1gpu": tol_e if f32 else 5e-2}
    ok = all(worst[k_] <= tol[k_] for k_ in keys)
    if rank == 0:
        print(json.dumps({"world": world, "dtype": args.dtype, "graph": args.graph, "p": p, "losses": losses,
                          "oracle": ref, "one_gpu": losses1, "worst": worst, "tol": tol, **plan, "pass": bool(ok)}),
              flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    os._exit(0 if ok else 1)


def infer(args, eng, model, x, rank, world, s, p, L, tol):
    """`args.infer` forward_only calls issued back to back (inputs alternate between the two
    parities' buffers: the second holds the input * -0.5), every call's outputs copied out in
    stream order and compared with the oracle's pp_forward.  With L = 1 nothing but the engine's
    inference fence orders call i+1's NVLink phantom stores after the peers' reads of call i."""
    x2 = -0.5 * x
    eng.set_batch([torch.from_numpy(x[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local],
                  [torch.zeros((eng.B, s), device="cuda") for _ in eng.local], 0)
    eng.set_batch([torch.from_numpy(x2[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local],
                  [torch.zeros((eng.B, s), device="cuda") for _ in eng.local], 1)
    outs = []
    for i in range(args.infer):
        outs.append([o.clone() for o in eng.forward_only(i % 2)])
    torch.cuda.synchronize()
    want = [po.pp_forward(model, ["relu"] * L, [xx[j * s:(j + 1) * s] for j in range(p)]) for xx in (x, x2)]
    worst = 0.0
    for i, o in enumerate(outs):
        for jj, j in enumerate(eng.local):
            worst = max(worst, nerr(o[jj].double().cpu().numpy().T, want[i % 2][j]))
    w = torch.tensor([worst], device="cuda", dtype=torch.float64)
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    ok = bool(w[0] <= tol)
    if rank == 0:
        print(json.dumps({"world": world, "dtype": args.dtype, "p": p, "layers": L, "calls": args.infer,
                          "worst": float(w[0]), "tol": tol, "fused": bool(eng.fused), "pass": ok}), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    sys.exit(main())
