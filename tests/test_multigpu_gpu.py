"""N > 1 GPUs (one process per GPU under torchrun): PhantomEngine and TPEngine vs the float64
oracle through tools/mp_parity.py / tools/mp_tp_parity.py — raw step-1 gradients of every tensor,
the losses and the weight UPDATES of every tensor over 3 steps (see those tools for tolerances)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_PORT = [29533]


def _run(nproc, tool, *args):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _PORT[0] += 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_PORT[0]), os.path.join(ROOT, "tools", tool),
           *[str(a) for a in args]]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"pass": true' in r.stdout, r.stdout[-2000:]
    return r.stdout


@pytest.mark.parametrize("dtype,p", [("fp32", 4), ("bf16", 4), ("fp32", 2), ("bf16", 2)])
def test_two_gpus_nccl_exchange(dtype, p):
    """Unfused plan: compression, NCCL all-gather, forward; NCCL reduce-scatter.  p = 4: two
    logical ranks per GPU; p = 2: one per GPU."""
    _run(2, "mp_parity.py", "--dtype", dtype, "--p", p, "--fused", "0", "--nvrs", "0", "--k3", "0")


@pytest.mark.parametrize("nvrs,k3", [("1", "1"), ("1", "0"), ("0", "0")])
@pytest.mark.parametrize("p", [2, 4])
def test_two_gpus_fused_forward(p, nvrs, k3):
    """Fused forward over 2 GPUs: the compression tiles store into the peer's phantom buffer over
    NVLink and bump both GPUs' arrival counters; forward tiles wait in-kernel (bf16, k = 64).
    nvrs=1: the reduce-scatter through NVLink too (error-compression epilogue -> owner staging ->
    in-kernel wait and ascending-rank sum), with k3=1 the error compression inside the
    weight-gradient launch (the default plan); nvrs=0: NCCL reduce-scatter."""
    out = _run(2, "mp_parity.py", "--dtype", "bf16", "--p", p, "--k", 64, "--B", 256, "--fused", "1", "--nvrs", nvrs,
               "--k3", k3)
    assert '"fused": true' in out


@pytest.mark.parametrize("fused", ["1", "0"])
def test_two_gpus_inference_back_to_back(fused):
    """forward_only calls issued back to back with ONE layer: the inference fence keeps
    call i+1's NVLink phantom stores behind the peer's reads of call i."""
    _run(2, "mp_parity.py", "--dtype", "bf16", "--p", 2, "--k", 64, "--B", 256, "--layers", 1, "--fused", fused,
         "--infer", 12)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_two_gpus_tensor_parallel(dtype):
    """The Megatron TP comparison pipeline (NCCL all-reduce pairs) on 2 GPUs vs the dense oracle."""
    _run(2, "mp_tp_parity.py", "--dtype", dtype)


@pytest.mark.parametrize("k3", ["auto", "0"])
def test_two_gpus_default_path_four_ranks(k3):
    """C3's plan on 2 GPUs — four logical ranks per GPU (p = 8): fused compression + NVLink
    all-gather + forward; error compression as slot-pair tiles (4 contributing ranks per pair)
    scattered to the owners over NVLink — inside the weight-gradient launch (k3 default: 4 pair
    problems + 12 weight-gradient problems) or as its own launch (k3 = 0) — in-kernel reduce; vs
    the oracle.  (lr 1e-4: at 3e-3 this bf16 model diverges within 3 steps on every plan.)"""
    out = _run(2, "mp_parity.py", "--dtype", "bf16", "--p", 8, "--width", 1024, "--k", 64, "--B", 256, "--lr", "1e-4",
               "--k3", k3)
    assert '"fused": true' in out


@pytest.mark.parametrize("p,n", [(4, 512), (8, 1024)])
def test_four_gpus_default_path(p, n):
    """The default multi-GPU plan on 4 GPUs (bf16, k = 64): fused compression + NVLink all-gather +
    forward; p = 4 (one logical rank per GPU, the N = p shapes of the scaling run): NCCL
    reduce-scatter + weight gradients and recurrence as one LPT-scheduled launch; p = 8 (two per
    GPU): the NVLink reduce-scatter with 3 peers."""
    out = _run(4, "mp_parity.py", "--dtype", "bf16", "--p", p, "--width", n, "--k", 64, "--B", 256, "--lr", "1e-4")
    assert '"fused": true' in out


def test_four_gpus_tensor_parallel():
    _run(4, "mp_tp_parity.py", "--dtype", "bf16")
