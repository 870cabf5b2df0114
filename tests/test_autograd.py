"""Algorithm 1's autograd pair on the host (CPU tensors): forward all-gather / backward
reduce-scatter is an adjoint pair, <G x, y> = <x, S y> (reference test_acceptance.py:78-97),
over the in-process Communicator (one rank per thread) and over torch.distributed (gloo, 2
processes)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_00960_b200.autograd import all_gather, dist_all_gather
from paper_2508_00960_b200.collectives import Communicator


@pytest.mark.parametrize("p, k, B", [(2, 3, 4), (3, 1, 5), (4, 2, 2)])
def test_in_process_adjoint_pair(p, k, B):
    g = torch.Generator().manual_seed(p * 100 + k)
    xs = [torch.randn(k, B, dtype=torch.float64, generator=g) for _ in range(p)]
    ys = [torch.randn(p * k, B, dtype=torch.float64, generator=g) for _ in range(p)]
    comm = Communicator(p)

    def rank(c, r):
        x = xs[r].clone().requires_grad_(True)
        with torch.autograd.set_multithreading_enabled(False):
            out = all_gather(x, c, r)
            (out * ys[r]).sum().backward()
        return out.detach(), x.grad

    res = comm.run(rank)
    gathered = torch.cat(xs)
    for r in range(p):
        assert torch.equal(res[r][0], gathered)
    lhs = sum(float((gathered * ys[r]).sum()) for r in range(p))
    rhs = sum(float((xs[r] * res[r][1]).sum()) for r in range(p))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    # the backward is the reduce-scatter: rank r receives sum_j ys[j][slot r] in ascending order
    for r in range(p):
        expect = ys[0][r * k:(r + 1) * k].clone()
        for j in range(1, p):
            expect = expect + ys[j][r * k:(r + 1) * k]
        assert torch.equal(res[r][1], expect)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        xs = [torch.randn(3, 4, dtype=torch.float64, generator=g) for _ in range(world)]
        ys = [torch.randn(3 * world, 4, dtype=torch.float64, generator=g) for _ in range(world)]
        x = xs[rank].clone().requires_grad_(True)
        out = dist_all_gather(x)
        (out * ys[rank]).sum().backward()
        ok_fwd = torch.equal(out.detach(), torch.cat(xs))
        expect = sum(ys[j][rank * 3:(rank + 1) * 3] for j in range(world))
        ok_bwd = torch.allclose(x.grad, expect, rtol=0, atol=1e-12)
        q.put((rank, ok_fwd, ok_bwd))
    finally:
        dist.destroy_process_group()


def test_process_group_adjoint_pair_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok_f and ok_b for _, ok_f, ok_b in out), out
