#!/usr/bin/env python
"""Phantom-parallel FFN training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c3|c2|c4|c5]

Workload (config C3, the north_star's headline): width n=16384, 8 layers, p=8 logical phantom
ranks, k=128, batch 8192, bf16, ReLU, mean half-squared loss, SGD — the SAME model at every N
(strong scaling): N GPUs each own 8/N logical ranks (N=1 runs all 8 on one GPU and the phantom
all-gather / reduce-scatter stay in HBM; N>1 exchanges phantoms over NVLink inside our kernels).
One step = one pp_iteration + optimizer update over one batch of synthetic teacher data
(reference training.py:181-213, 276-309).  Timed with CUDA events over K CUDA-graph replays,
max over ranks.  The same JSON line also carries:

  roofline    the step's per-kernel table (CUDA events around every launch of an eager step,
              each launch tagged with its algorithmic GEMM FLOPs) and the dominant kernel (largest
              time share) against the measured bf16 peak; `traffic` = that kernel's DRAM bytes
              per launch from the committed ncu capture (profiles/traffic.json, commit-stamped)
  r1_shapes   (N=1) the same step with one logical rank per launch: the per-GPU kernels of the
              8-GPU run, so every 1-GPU bench records their efficiency
  fp32_tier   (N=1) the fp32 parity tier (3xTF32) at C2: samples/s and fraction of that tier's
              tensor ceiling (bf16 peak / 6)
  inference   (C3/C5) forward-only samples/s of the same model (config C5 at k = 128)
  energy      NVML joules per epoch (64 batches) over >= --energy-seconds of steady-state steps
  tp          the same-width Megatron tensor-parallel pipeline on the same GPUs (its energy too)
  e2e         the public API with pinned HOST batches: H2D of inputs+targets and D2H of every
              step's loss inside the timed region (the host reads step i's loss while step i+1
              runs, Engine.loss_async)
  cpu_baseline  the reference algorithm on this box's host cores (bounded sample)

--config c5 runs the inference sweep (k = 32..512) instead of training.  --impl reference times
the UNMODIFIED reference (phantomsim, installed into baseline/_ref from /root/reference) on the
host cores through its own API (Communicator threads + pp_iteration + sgd_step); if that install
is absent it falls back to the pinned oracle port (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FFN train samples/s @1/2/4/8 B200, % TC roofline, J/epoch vs tensor-parallel"
CONFIGS = {
    "c1": dict(n=1024, p=2, k=16, layers=4, batch=64),
    "c2": dict(n=8192, p=4, k=64, layers=8, batch=8192),
    "c3": dict(n=16384, p=8, k=128, layers=8, batch=8192),
    "c4": dict(n=65536, p=8, k=256, layers=16, batch=8192),
    "c5": dict(n=16384, p=8, k=128, layers=8, batch=8192),
}
C5_KS = (32, 64, 128, 256, 512)
STEPS_PER_EPOCH = 64      # epoch = 64 * B samples


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d.get("hbm_gbs", 6546.2), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def refuse_debug_knobs():
    """The bench line is the default launch plan: debug switches (wrong results) and the planner's
    A/B switches (PPX_AB_*, PPX_NO_*, PPX_QBAL) are refused; only PPX_LIB / PPX_NO_NUMA_BIND pass."""
    allowed = {"PPX_LIB", "PPX_NO_NUMA_BIND"}
    bad = sorted(k for k in os.environ if k not in allowed and os.environ[k] != "" and
                 (k.startswith(("PPX_DEBUG", "PPX_AB_", "PPX_NO_")) or k == "PPX_QBAL"))
    if bad:
        sys.exit(f"bench.py: refusing to run with debug / A-B knobs set ({', '.join(bad)}): the bench measures "
                 f"the default plan")


# ---------------------------------------------------------------------------------------------
# clocks / energy
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """NVML polling thread (5 ms period) over the timed region: SM clock + throttle reasons."""

    def __init__(self, cuda_index: int):
        self.idx = cuda_index
        self.ok = False
        self.sm, self.smax, self.reasons = [], None, set()

    def start(self):
        try:
            import pynvml
            from paper_2508_00960_b200.energy import nvml_handle
            h = nvml_handle(self.idx)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "sw_power_cap": 0x4}
            self._stop = threading.Event()

            def poll():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = get_reasons(h)
                        self.reasons.update(nm for nm, b in bits.items() if r & b)
                    except Exception:
                        pass
                    self._stop.wait(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.ok = True
        except Exception as exc:  # pragma: no cover
            self.err = str(exc)

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.t.join(timeout=1)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def energy_mj(cuda_index):
    from paper_2508_00960_b200.energy import energy_mj as e
    return e(cuda_index)


# ---------------------------------------------------------------------------------------------
# CPU baseline / reference arm
# ---------------------------------------------------------------------------------------------
def _phantomsim():
    """The unmodified reference package from baseline/_ref (None if it was not installed)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "phantomsim")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import phantomsim
        return phantomsim
    except Exception:
        return None


def reference_steps(n, p, k, layers, batch, steps, warmup):
    """Time `steps` training iterations of the reference's own CPU implementation: phantomsim's
    Communicator (one thread per rank) running pp_iteration + sgd_step (training.py:276-303) on a
    random model of the configured shape.  Falls back to the pinned oracle port.  Returns
    (seconds per step, kind, threads used)."""
    import numpy as np
    ps = _phantomsim()
    cores = os.cpu_count() or 1
    s = n // p
    rng = np.random.default_rng(0)
    a = (6.0 / (2 * s)) ** 0.5
    xs = [rng.standard_normal((s, batch)) for _ in range(p)]
    ys = [np.maximum(rng.standard_normal((s, batch)), 0) for _ in range(p)]
    if ps is not None:
        acts = [ps.Activation.RELU] * layers
        model = [[ps.PhantomLayer(local=rng.uniform(-a, a, (s, s)), compressor=rng.uniform(-a, a, (k, s)),
                                  decompressors={i: rng.uniform(-a, a, (s, k)) for i in range(p) if i != j},
                                  bias=np.zeros(s)) for _ in range(layers)] for j in range(p)]
        from phantomsim.training import _pp_param_lists

        def worker(comm, rank, nsteps):
            for _ in range(nsteps):
                out = ps.pp_iteration(comm, rank, model[rank], acts, xs[rank], ys[rank], "mean")
                params, grads, names = _pp_param_lists(model[rank], out.grads)
                ps.sgd_step(params, grads, 1e-4, names=names)
        # one host thread per rank (the reference's "threads" scheduler), each BLAS call on
        # cores // p threads: the fastest setting measured for this reference (8-core host, C3:
        # 0.76 s/step vs 1.49 lockstep with all cores per call, 1.77 threads oversubscribed)
        per = max(1, cores // p)
        comm = ps.Communicator(p, mode="threads", timeout=3600.0)
        with _blas_threads(per):
            if warmup:
                comm.run(worker, warmup)
            t0 = time.perf_counter()
            comm.run(worker, steps)
            dt = (time.perf_counter() - t0) / steps
        return dt, "reference", per * p
    from oracle import phantom_oracle as po
    model = [[{"local": rng.uniform(-a, a, (s, s)), "compressor": rng.uniform(-a, a, (k, s)),
               "decompressors": {i: rng.uniform(-a, a, (s, k)) for i in range(p) if i != j}, "bias": np.zeros(s)}
              for _ in range(layers)] for j in range(p)]

    def one():
        out = po.pp_iteration(model, ["relu"] * layers, xs, ys, "mean")
        for j in range(p):
            params, gs = po.pp_param_list(model[j], out["grads"][j])
            po.sgd_step(params, gs, 1e-4)
    with _blas_threads(cores):
        for _ in range(warmup):
            one()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        dt = (time.perf_counter() - t0) / steps
    return dt, "port", cores


def _blas_threads(n):
    """Limit the BLAS pool at run time (numpy may already be loaded, so env vars are too late)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n, user_api="blas")
    except Exception:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, p, k, L = cfg["n"], cfg["p"], cfg["k"], cfg["layers"]
    sample_b = 256
    sample_l = L if n <= 16384 else 1   # C4's float64 weights do not fit host RAM: one layer, x L
    dt, kind, threads = reference_steps(n, p, k, sample_l, sample_b, args.steps, min(args.warmup, 1))
    dt *= L / sample_l
    v = sample_b / dt
    what = "phantomsim (unmodified reference, baseline/_ref)" if kind == "reference" else "oracle port of phantomsim"
    sample = (f"{what}: Communicator(p={p}, threads) pp_iteration + sgd_step, float64, {args.config} model "
              f"(n={n}, p={p}, k={k}, L={sample_l}{f' scaled x{L}' if sample_l != L else ''}) at batch {sample_b} "
              f"per step (samples/s is linear in batch for this GEMM-bound path)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"phantom FFN {args.config}: n={n}, L={L}, p={p}, k={k}, batch {sample_b} (CPU sample)",
                   "global_batch": sample_b, "parallelism": f"pp{p} simulated in one process"},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def cpu_baseline(args, cfg):
    """The reference on this box's host cores, one layer of the model at batch 256, scaled to L."""
    cores = os.cpu_count() or 1
    n, p, k, L = cfg["n"], cfg["p"], cfg["k"], cfg["layers"]
    sample_b = 256
    try:
        dt, kind, threads = reference_steps(n, p, k, 1, sample_b, 2, 1)
        return {"value": sample_b / (dt * L), "unit": "samples/s", "cores": threads, "kind": kind,
                "sample": f"{'phantomsim' if kind == 'reference' else 'oracle port'} pp_iteration + sgd_step "
                          f"(float64, numpy/OpenBLAS, {threads} threads in all) of ONE layer of the {args.config} model "
                          f"(all {p} ranks) at batch {sample_b}, mean of 2 after 1 warm-up, scaled x{L} layers"}
    except Exception as exc:  # pragma: no cover
        return {"value": None, "unit": "samples/s", "cores": cores, "kind": "reference", "sample": f"failed: {exc}"}


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def make_data(eng, seed, cfg):
    """Synthetic teacher data (training.py:43-56 shape): X ~ N(0,1) [B, n]; targets of logical
    rank j = relu(relu(X) . W_j^T) for a fixed N(0,1)/sqrt(n) teacher, computed on the GPU with
    the engine's own GEMM (once, outside the timed region)."""
    import torch
    from paper_2508_00960_b200 import kernels
    B, n, s = eng.B, eng.n, eng.s
    g = torch.Generator(device=eng.dev)
    g.manual_seed(seed)
    X = torch.randn((B, n), generator=g, device=eng.dev).to(torch.bfloat16)
    Xr = torch.empty_like(X)
    eng.ctx.call("ppx_bias_act", 0, B, n, X.data_ptr(), n, None, 0, Xr.data_ptr(), n,
                 torch.cuda.current_stream().cuda_stream)
    xs, ts = [], []
    for jj, j in enumerate(eng.local):
        gt = torch.Generator(device=eng.dev)
        gt.manual_seed(seed * 7919 + j)
        W = (torch.randn((s, n), generator=gt, device=eng.dev) / n ** 0.5).to(torch.bfloat16)
        T = kernels.gemm(Xr, W, transpose_b=True, out_dtype=torch.bfloat16, relu=True, ctx=eng.ctx)
        xs.append(X[:, j * s:(j + 1) * s].to(eng.dtype).contiguous())
        ts.append(T.to(eng.dtype))
        del W
    del X, Xr
    return xs, ts


def bind_to_gpu_cpus(cuda_index):
    """Pin this rank to the host CPUs NVML reports as closest to its GPU, so the pinned host
    batches of the e2e leg are first-touched on that GPU's NUMA node (PPX_NO_NUMA_BIND=1 skips)."""
    try:
        import pynvml
        from paper_2508_00960_b200.energy import nvml_handle
        h = nvml_handle(cuda_index)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1 and 64 * i + b < ncpu}
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception as exc:  # pragma: no cover - best effort, the bench runs unbound
        print(f"[bench] cpu binding skipped: {exc}", file=sys.stderr)


class Dist:
    def __init__(self, world, rank, local_rank):
        self.world, self.rank, self.local = world, rank, local_rank
        if world > 1:
            import torch.distributed as dist
            self.dist = dist

    def barrier(self):
        # drain our own NCCL work first: two communicators' kernels must never interleave
        import torch
        torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        torch.cuda.synchronize()

    def reduce(self, vals, op="max"):
        import torch
        t = torch.tensor(vals, device="cuda", dtype=torch.float64)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return [float(v) for v in t.tolist()]

    def uid(self):
        from paper_2508_00960_b200 import _lib
        if self.world == 1:
            return None
        u = [_lib.Context.unique_id() if self.rank == 0 else None]
        self.dist.broadcast_object_list(u, src=0)
        return u[0]


def timed_steps(eng, D, steps, graph=True):
    """ms per step (CUDA events on the launching stream, max over ranks)."""
    import torch
    S = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    e0.record(S)
    for _ in range(steps):
        eng.step(graph=graph)
    e1.record(S)
    D.barrier()
    return D.reduce([e0.elapsed_time(e1) / steps])[0]


def energy_window(eng, D, ms_per_step, seconds, step=None):
    """NVML joules per step over >= `seconds` of steady-state graph replays (all GPUs summed)."""
    import math as _m
    step = step or (lambda: eng.step())
    steps = max(3, int(_m.ceil(seconds * 1e3 / max(ms_per_step, 1e-3))))
    D.barrier()
    t0 = time.perf_counter()
    e0 = energy_mj(D.local)
    for i in range(steps):
        step()
        if i % 64 == 63:
            import torch
            torch.cuda.synchronize()
    D.barrier()
    e1 = energy_mj(D.local)
    wall = time.perf_counter() - t0
    j = ((e1 - e0) / 1e3 / steps) if (e0 is not None and e1 is not None) else float("nan")
    j_all = D.reduce([j], op="sum")[0]
    return {"j_per_step_all_gpus": j_all, "j_per_epoch": j_all * STEPS_PER_EPOCH,
            "epoch_samples": STEPS_PER_EPOCH * eng.B, "window_s": wall, "window_steps": steps}


def kernel_table(seq, peak, steps=1):
    """Aggregate profile_step output [(call, ms, flops)] -> per-kind rows + dominant kind."""
    rows = {}
    for name, ms, fl in seq:
        r = rows.setdefault(name, {"launches": 0, "ms": 0.0, "flops": 0})
        r["launches"] += 1
        r["ms"] += ms
        r["flops"] += fl
    total = sum(r["ms"] for r in rows.values()) or 1.0
    out = {}
    for name, r in sorted(rows.items(), key=lambda kv: -kv[1]["ms"]):
        tf = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] > 0 and r["flops"] else None
        out[name] = {"launches_per_step": r["launches"] // steps, "ms_per_step": r["ms"] / steps,
                     "share": r["ms"] / total, "flops_per_launch": r["flops"] // max(r["launches"], 1),
                     "ms_per_launch": r["ms"] / max(r["launches"], 1),
                     "tflops": tf, "frac_of_burst": (tf / peak) if tf else None}
    return out, total / steps


def profile(eng, D, reps=3):
    seq = []
    for _ in range(reps):
        seq += eng.profile_step()
    D.barrier()
    return seq


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--optimizer", default="sgd", choices=["sgd", "adam"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"],
                    help="fp32 = the 3xTF32 parity tier (throughput reported separately from the bf16 headline)")
    ap.add_argument("--energy-seconds", type=float, default=20.0)
    ap.add_argument("--k3", default="auto", choices=["auto", "0", "1"],
                    help="A/B of the backward launch plan (k3_fused); default = the engine's choice")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tp", action="store_true")
    ap.add_argument("--no-r1", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    args = ap.parse_args()
    refuse_debug_knobs()
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    from paper_2508_00960_b200.engine import PhantomEngine, pp_step_flops
    from paper_2508_00960_b200.schedule import comm_bytes_per_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1 and not os.environ.get("PPX_NO_NUMA_BIND"):
        bind_to_gpu_cpus(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    D = Dist(world, rank, local_rank)
    uid = D.uid()
    n, p, k, L, B = cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"]
    peak, peak_sus, hbm, peak_kind = peaks()
    use_graph = not args.no_graph
    if args.config == "c5":
        return run_inference_sweep(args, cfg, D, uid, peak)

    dtype = torch.float32 if args.dtype == "fp32" else torch.bfloat16
    eng = PhantomEngine(n, p, k, L, B, world=world, rank=rank, device=local_rank, uid=uid,
                        optimizer=args.optimizer, lr=3e-6, dtype=dtype,
                        k3_fused=None if args.k3 == "auto" else args.k3 == "1")
    xs, ts = make_data(eng, 1234, cfg)
    eng.set_batch(xs, ts, 0)
    eng.set_batch(xs, ts, 1)
    plan = {"fused": eng.fused, "nvrs": eng.nvrs, "k3": eng.k3_fused, "bwd": eng.bwd_fused, "group": eng.group,
            "bits": eng.mask_bits}

    # warm-up: eager step (sets kernel attributes), capture, graph replays
    eng.step(graph=False)
    launches_per_step = eng.launch_count
    if use_graph:
        eng.capture()
    for _ in range(max(args.warmup - 1, 2)):
        eng.step(graph=use_graph)
    loss0 = eng.read_loss()

    sampler = ClockSampler(local_rank)
    sampler.start()
    ms = timed_steps(eng, D, args.steps, use_graph)
    clocks = sampler.stop()
    loss1 = eng.read_loss()
    value = B / (ms / 1e3)
    step_flops = eng.R * pp_step_flops(n, p, k, L, B)
    step_tflops = step_flops / (ms / 1e3) / 1e12

    # ---- per-kernel roofline of the step: CUDA events around every launch of eager steps
    seq = profile(eng, D)
    kernels, kern_ms = kernel_table(seq, peak, steps=3)
    dom_name, dom = next(iter(kernels.items()))
    flops_check = sum(f for _, _, f in seq) / 3
    traffic = stamped_traffic(dom_name)
    roofline = {"bound": "tensor", "kernel": dom_name, "achieved": dom["tflops"], "peak": peak, "unit": "TFLOP/s",
                "frac": dom["tflops"] / peak, "traffic": traffic.get("dram_bytes_per_launch"),
                "traffic_source": traffic.get("source"), "flops_per_launch": dom["flops_per_launch"],
                "ms_per_launch": dom["ms_per_launch"], "peak_kind": f"{peak_kind} burst",
                "step_tflops_per_gpu": step_tflops, "step_frac_of_sustained": step_tflops / peak_sus,
                "step_frac_of_burst": step_tflops / peak, "kernel_sum_ms_per_step": kern_ms,
                "kernel_sum_frac_of_burst": step_flops / (kern_ms / 1e3) / 1e12 / peak,
                "flops_tagged_per_step": flops_check, "flops_algorithmic_per_step": step_flops,
                "kernels": kernels}
    if args.dtype == "fp32":
        roofline["tier_note"] = ("3xTF32 tier: three kind::tf32 MMAs per product at half the bf16 rate, so its "
                                 "tensor ceiling is 1/6 of the bf16 peak (frac_of_tier_ceiling = 6 x frac)")
        roofline["frac_of_tier_ceiling"] = 6 * roofline["frac"]

    # ---- inference (config C5 at this k): forward-only graph replays of the same model
    inference = None
    if args.config in ("c3", "c2") and args.dtype == "bf16":
        inference = time_inference(eng, D, args.steps, use_graph, peak)

    # ---- NVML energy over >= energy_seconds of steady-state training steps
    energy = energy_window(eng, D, ms, args.energy_seconds, step=lambda: eng.step(graph=use_graph))

    # ---- end-to-end through the public API: pinned host batches, H2D + D2H(loss) in the timed region
    e2e = None if args.no_e2e else time_e2e(eng, D, xs, ts, args.steps, use_graph, B)

    r1 = None
    if world == 1 and p > 1 and not args.no_r1 and args.config in ("c3", "c2") and args.dtype == "bf16":
        eng.close()
        del eng
        torch.cuda.empty_cache()
        r1 = time_r1_shapes(cfg, D, xs, ts, args, peak, peak_sus)
        eng = None

    fp32_tier = None
    if world == 1 and args.config == "c3" and args.dtype == "bf16" and not args.no_fp32:
        if eng is not None:
            eng.close()
            del eng
            eng = None
            torch.cuda.empty_cache()
        fp32_tier = time_fp32_tier(D, args, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)

    tp = None
    if not args.no_tp and L % 2 == 0 and args.config != "c4" and args.dtype == "bf16":
        tp = run_tp(args, cfg, D, eng, uid)
    elif eng is not None:
        D.barrier()
        eng.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"phantom FFN {args.config}: n={n}, L={L}, p={p} logical ranks, k={k}, "
                                   f"batch {B}, ReLU, mean loss, {args.optimizer.upper()}; "
                                   f"{p // world} logical rank(s) per GPU",
                       "global_batch": B, "width": n, "layers": L, "p": p, "k": k,
                       "parallelism": f"phantom pp{p} over {world} GPU(s)",
                       "l2": "working set per step (weights + activations) exceeds the 126 MB L2; no flush",
                       "graphs": use_graph,
                       "plan": {"fused_forward": bool(plan["fused"]), "nvlink_reduce_scatter": bool(plan["nvrs"]),
                                "k3_fused": bool(plan["k3"]), "bwd_fused": bool(plan["bwd"]), "group": plan["group"],
                                "mask_bits": bool(plan["bits"])}},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "energy": energy,
            "loss": {"after_warmup": loss0, "after_timed": loss1},
            "comm_bytes_per_step_per_gpu": comm_bytes_per_step(n, p, k, L, B, world),
            "r1_shapes": r1,
            "fp32_tier": fp32_tier,
            "inference": inference,
            "tp": tp,
        }
        if tp and tp.get("value"):
            line["pp_vs_tp"] = {"speedup": value / tp["value"],
                                "comm_bytes_ratio": (line["comm_bytes_per_step_per_gpu"] / tp["comm_bytes_per_step_per_gpu"]
                                                     if tp["comm_bytes_per_step_per_gpu"] else None),
                                "energy_per_epoch_ratio": (energy["j_per_step_all_gpus"] / tp["energy"]["j_per_step_all_gpus"]
                                                           if tp.get("energy") else None)}
        print(json.dumps(line), flush=True)
    finish(D)
    return 0


def finish(D):
    if D.world > 1:
        D.barrier()
        D.dist.destroy_process_group()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


def stamped_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json: {abi_call: {dram_bytes_per_launch, commit, ...}})."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path)).get(kernel)
        if d:
            return {"dram_bytes_per_launch": d["dram_bytes_per_launch"],
                    "source": f"ncu --set full, commit {d.get('commit')}, {d.get('shape', '')}".strip(", ")}
    except Exception:
        pass
    return {"dram_bytes_per_launch": None, "source": "no committed ncu capture for this kernel"}


def time_inference(eng, D, steps, use_graph, peak):
    """Forward-only (config C5 at the engine's k): samples/s over graph replays, max over ranks."""
    import torch
    from paper_2508_00960_b200.engine import pp_forward_flops
    eng.forward_only(0)
    if use_graph:
        eng.capture_inference()
    for _ in range(3):
        eng.forward_only(0, graph=use_graph)
    S = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    e0.record(S)
    for _ in range(steps):
        eng.forward_only(0, graph=use_graph)
    e1.record(S)
    D.barrier()
    ms = D.reduce([e0.elapsed_time(e1) / steps])[0]
    tf = eng.R * pp_forward_flops(eng.n, eng.p, eng.k, eng.L, eng.B) / (ms / 1e3) / 1e12
    return {"config": f"C5: forward-only n={eng.n}, L={eng.L}, p={eng.p}, k={eng.k}, batch {eng.B}",
            "value": eng.B / (ms / 1e3), "unit": "samples/s", "ms_per_batch": ms, "tflops_per_gpu": tf,
            "frac_of_burst": tf / peak, "gpu_launches_per_batch": eng.infer_launch_count}


def run_inference_sweep(args, cfg, D, uid, peak):
    """--config c5: forward-only samples/s for k in 32..512 (BASELINE configs[4])."""
    import torch
    from paper_2508_00960_b200.engine import PhantomEngine
    n, p, L, B = cfg["n"], cfg["p"], cfg["layers"], cfg["batch"]
    rows = []
    for k in C5_KS:
        eng = PhantomEngine(n, p, k, L, B, world=D.world, rank=D.rank, device=D.local, uid=uid if k == C5_KS[0] else
                            D.uid(), lr=3e-6, dtype=torch.bfloat16)
        g = torch.Generator(device="cuda").manual_seed(5)
        xs = [torch.randn((B, eng.s), generator=g, device="cuda").bfloat16() for _ in range(eng.R)]
        eng.set_batch(xs, xs, 0)
        r = time_inference(eng, D, args.steps, not args.no_graph, peak)
        r["k"] = k
        r["fused"] = bool(eng.fused)
        rows.append(r)
        D.barrier()
        eng.close()
        del eng
        torch.cuda.empty_cache()
    if D.rank == 0:
        best = max(rows, key=lambda r: r["value"])
        print(json.dumps({
            "metric": "FFN forward-only inference samples/s (C5 k sweep)", "value": [r["value"] for r in rows],
            "unit": "samples/s", "n_gpus": D.world, "steps": args.steps, "warmup": 3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"phantom FFN c5: n={n}, L={L}, p={p}, batch {B}, k in {list(C5_KS)}",
                       "global_batch": B, "parallelism": f"phantom pp{p} over {D.world} GPU(s)"},
            "sweep": rows, "roofline": {"bound": "tensor", "achieved": best["tflops_per_gpu"], "peak": peak,
                                        "unit": "TFLOP/s", "frac": best["frac_of_burst"], "traffic": None}}), flush=True)
    finish(D)
    return 0


def time_e2e(eng, D, xs, ts, steps, use_graph, B):
    import torch
    xh = torch.stack([x.cpu() for x in xs]).pin_memory()
    th = torch.stack([t_.cpu() for t_ in ts]).pin_memory()
    h2d = 2 * xh.numel() * xh.element_size()
    S = torch.cuda.current_stream()
    D.barrier()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record(S)
    ready = eng.load_batch_async(xh, th, eng.parity)
    prev_done = None
    pending = None
    for i in range(steps):
        S.wait_event(ready)
        par = eng.parity
        eng.step(graph=use_graph)
        loss_i = eng.loss_async()                    # D2H of step i's loss (+ non-finite flag)
        done = torch.cuda.Event()
        done.record(S)
        if i + 1 < steps:
            # the next batch goes into the other parity's buffers, last read by step i-1:
            # its H2D overlaps step i
            if prev_done is not None:
                eng.copy_stream.wait_event(prev_done)
            ready = eng.load_batch_async(xh, th, 1 - par)
        prev_done = done
        if pending is not None:
            pending()                                # the host reads step i-1's loss while step i runs
        pending = loss_i
    pending()
    q1.record(S)
    D.barrier()
    te = D.reduce([q0.elapsed_time(q1) / steps])[0]
    return {"value": B / (te / 1e3), "unit": "samples/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8}


def time_r1_shapes(cfg, D, xs, ts, args, peak, peak_sus):
    """The same C3 step with one logical rank per launch (group=1): the per-GPU kernels of the
    8-GPU run (per-rank forward, per-rank weight-gradient + recurrence LPT launches at s = n/p),
    on this one GPU.  Exchanges stay in HBM, so this is the 8-GPU step's compute bound."""
    import torch
    from paper_2508_00960_b200.engine import PhantomEngine, pp_step_flops
    n, p, k, L, B = cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"]
    eng = PhantomEngine(n, p, k, L, B, lr=3e-6, dtype=torch.bfloat16, group=1)
    eng.set_batch(xs, ts, 0)
    eng.set_batch(xs, ts, 1)
    eng.step(graph=False)
    eng.capture()
    for _ in range(3):
        eng.step()
    ms = timed_steps(eng, D, args.steps)
    seq = profile(eng, D)
    kernels, kern_ms = kernel_table(seq, peak, steps=3)
    flops = p * pp_step_flops(n, p, k, L, B)
    eng.close()
    return {"what": "C3 step with one logical rank per launch (the per-GPU launch shapes of C3 on 8 GPUs), 1 GPU",
            "ms_per_step": ms, "samples_per_s": B / (ms / 1e3), "step_tflops": flops / (ms / 1e3) / 1e12,
            "step_frac_of_sustained": flops / (ms / 1e3) / 1e12 / peak_sus,
            "kernel_sum_ms_per_step": kern_ms,
            "kernel_sum_frac_of_burst": flops / (kern_ms / 1e3) / 1e12 / peak,
            "kernel_sum_frac_of_sustained": flops / (kern_ms / 1e3) / 1e12 / peak_sus,
            "launches_per_step": eng.launch_count, "kernels": kernels}


def time_fp32_tier(D, args, peak):
    """The fp32 parity tier (3xTF32 on kind::tf32, the tier that carries the 1e-4 oracle parity)
    at C2 on this GPU: graph-replayed training steps of the default plan."""
    import torch
    from paper_2508_00960_b200.engine import PhantomEngine, pp_step_flops
    cfg = CONFIGS["c2"]
    n, p, k, L, B = cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"]
    eng = PhantomEngine(n, p, k, L, B, lr=3e-6, dtype=torch.float32)
    xs, ts = make_data(eng, 1234, cfg)
    eng.set_batch(xs, ts, 0)
    eng.set_batch(xs, ts, 1)
    eng.step(graph=False)
    launches = eng.launch_count
    eng.capture()
    for _ in range(3):
        eng.step()
    ms = timed_steps(eng, D, max(5, min(args.steps, 10)))
    eng.close()
    tf = eng.R * pp_step_flops(n, p, k, L, B) / (ms / 1e3) / 1e12
    return {"what": "C2 (n=8192, L=8, p=4, k=64, batch 8192) in the fp32 tier (3xTF32), 1 GPU",
            "samples_per_s": B / (ms / 1e3), "ms_per_step": ms, "step_tflops": tf,
            "frac_of_tier_ceiling": 6 * tf / peak, "launches_per_step": launches,
            "tier_note": "three kind::tf32 MMAs per product at half the bf16 rate: ceiling = bf16 peak / 6"}


def run_tp(args, cfg, D, eng, uid):
    """The same-width Megatron tensor-parallel FFN (TPEngine) on the same GPUs, same batch."""
    import torch
    from paper_2508_00960_b200 import _lib, kernels
    from paper_2508_00960_b200.schedule import tp_comm_bytes_per_step
    from paper_2508_00960_b200.tensor_parallel import TPEngine, tp_step_flops
    n, L, B = cfg["n"], cfg["layers"], cfg["batch"]
    world = D.world
    ctx = eng.ctx if eng is not None else _lib.Context(1, 0, D.local)
    # full replicated input / teacher targets of the dense-width task
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    X = torch.randn((B, n), generator=g, device="cuda").to(torch.bfloat16)
    Xr = torch.empty_like(X)
    ctx.call("ppx_bias_act", _lib.PPX_BF16, B, n, X.data_ptr(), n, None, 0, Xr.data_ptr(), n,
             torch.cuda.current_stream().cuda_stream)
    gt = torch.Generator(device="cuda")
    gt.manual_seed(99)
    W = (torch.randn((n, n), generator=gt, device="cuda") / n ** 0.5).to(torch.bfloat16)
    T = kernels.gemm(Xr, W, transpose_b=True, out_dtype=torch.bfloat16, relu=True, ctx=ctx)
    del W, Xr
    torch.cuda.synchronize()
    if eng is not None:
        D.barrier()
        eng.close()                      # free the phantom engine's graphs + communicator first
    else:
        ctx.close()
    torch.cuda.empty_cache()
    tpe = TPEngine(n, L, B, world=world, rank=D.rank, device=D.local,
                   uid=None if world == 1 else D.uid(), lr=3e-6, dtype=torch.bfloat16)
    tpe.set_batch(X, T, 0)
    tpe.set_batch(X, T, 1)
    del X, T
    tpe.step(graph=False)
    tpe.read_loss()
    tpe.capture()
    for _ in range(2):
        tpe.step()
    tpe.read_loss()
    steps = max(3, min(args.steps, 10))
    ms = timed_steps(tpe, D, steps)
    energy = energy_window(tpe, D, ms, args.energy_seconds)
    loss = tpe.read_loss()
    flops = tp_step_flops(n, world, L, B)
    out = {"pipeline": f"Megatron tensor-parallel FFN n={n}, L={L}, batch {B}, column/row pairs, "
                       f"{world} GPU(s), same kernels, SGD fused", "value": B / (ms / 1e3), "unit": "samples/s",
           "ms_per_step": ms, "steps": steps, "step_tflops_per_gpu": flops / (ms / 1e3) / 1e12,
           "energy": energy, "comm_bytes_per_step_per_gpu": tp_comm_bytes_per_step(n, L, B, world), "loss": loss,
           "gpu_launches": tpe.launch_count * steps}
    D.barrier()
    tpe.close()
    return out


if __name__ == "__main__":
    sys.exit(main())
