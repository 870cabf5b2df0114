"""The in-process Communicator of the drop-in API (reference collectives.py:87-357) on CPU
tensors, both schedulers: results, record stream and every protocol error the reference's own
collectives tests exercise (test_collectives.py:22-160), plus the lockstep baton's determinism."""
import threading

import pytest
import torch

from paper_2508_00960_b200.collectives import Collective, Communicator, Direction
from paper_2508_00960_b200.errors import ConfigurationError, ProtocolError

MODES = ("lockstep", "threads")
T = lambda *v: torch.tensor(v, dtype=torch.float64)   # noqa: E731


def run(p, fn, mode="lockstep", timeout=10.0):
    c = Communicator(p, mode=mode, timeout=timeout)
    return c.run(fn), c


@pytest.mark.parametrize("mode", MODES)
def test_all_gather_ascending_concat(mode):
    outs, c = run(3, lambda cm, r: cm.all_gather(r, T(float(r), 10.0 + r).reshape(1, 2)), mode)
    for o in outs:
        assert torch.equal(o, torch.tensor([[0.0, 10.0], [1.0, 11.0], [2.0, 12.0]], dtype=torch.float64))
    assert c.records[0].collective is Collective.ALL_GATHER and c.records[0].message_size == 2


@pytest.mark.parametrize("mode", MODES)
def test_reduce_scatter_and_all_reduce(mode):
    contrib = [T(1.0, 2.0), T(10.0, 20.0)]
    outs, c = run(2, lambda cm, r: cm.reduce_scatter(r, contrib[r]), mode)
    assert torch.equal(outs[0], T(11.0)) and torch.equal(outs[1], T(22.0))
    assert c.records[0].message_size == 1
    outs, _ = run(3, lambda cm, r: cm.all_reduce(r, torch.ones(2, dtype=torch.float64)), mode)
    assert all(torch.equal(o, T(3.0, 3.0)) for o in outs)


def test_sums_in_ascending_rank_order_bitwise():
    vals = [T(1e16), T(1.0), T(-1e16), T(1.0)]
    outs, _ = run(4, lambda cm, r: cm.all_reduce(r, vals[r]))
    assert torch.equal(outs[0], ((T(1e16) + T(1.0)) + T(-1e16)) + T(1.0))
    g = torch.Generator().manual_seed(0)
    v = [torch.randn(8, 3, generator=g, dtype=torch.float64) for _ in range(4)]
    red, _ = run(4, lambda cm, r: cm.all_reduce(r, v[r]))
    sc, _ = run(4, lambda cm, r: cm.reduce_scatter(r, v[r]))
    for r in range(4):
        assert torch.equal(sc[r], red[r][2 * r:2 * r + 2])


@pytest.mark.parametrize("mode", MODES)
def test_broadcast_roots(mode):
    outs, c = run(4, lambda cm, r: cm.broadcast(r, 3, T(1.0, 2.0) if r == 3 else None), mode)
    assert all(torch.equal(o, T(1.0, 2.0)) for o in outs) and c.records[0].message_size == 2


def test_world_of_one_is_identity():
    outs, _ = run(1, lambda cm, r: cm.reduce_scatter(r, T(1.0, 2.0).reshape(2, 1)))
    assert torch.equal(outs[0], T(1.0, 2.0).reshape(2, 1))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("fn,match", [
    (lambda cm, r: cm.all_gather(r, torch.ones(r + 1)), "shape disagreement"),
    (lambda cm, r: cm.reduce_scatter(r, torch.ones(3, 1)), "chunk"),
    (lambda cm, r: cm.broadcast(r, r, T(1.0)), "root"),
    (lambda cm, r: cm.all_gather(r, T(1.0)) if r == 0 else cm.all_reduce(r, T(1.0)), "mismatch"),
    (lambda cm, r: cm.all_gather(r, T(1.0), direction=Direction.FORWARD, layer=r), "mismatch"),
    (lambda cm, r: cm.all_gather(r, T(1.0)) if r == 0 else None, "deadlock"),
])
def test_protocol_errors(mode, fn, match):
    with pytest.raises(ProtocolError, match=match):
        run(2, fn, mode)


@pytest.mark.parametrize("mode", MODES)
def test_rank_exception_propagates(mode):
    def fn(cm, r):
        if r == 1:
            raise ValueError("exploded")
        return cm.all_reduce(r, T(1.0))
    with pytest.raises(ValueError, match="exploded"):
        run(3, fn, mode)


def test_timeout_in_threads_mode():
    ev = threading.Event()

    def fn(cm, r):
        if r == 1:
            ev.wait(2.0)           # late, but not finished: only the timeout can catch it
        return cm.all_reduce(r, T(1.0))
    with pytest.raises(ProtocolError, match="timeout"):
        run(2, fn, "threads", timeout=0.3)
    ev.set()


def test_lockstep_is_deterministic_and_matches_threads():
    order = []

    def fn(cm, r):
        order.append((r, "a"))
        x = cm.all_gather(r, T(float(r)), direction=Direction.FORWARD, layer=0)
        order.append((r, "b"))
        y = cm.reduce_scatter(r, torch.arange(4, dtype=torch.float64) * (r + 1), direction=Direction.BACKWARD, layer=0)
        return x, y
    a, ca = run(4, fn, "lockstep")
    first = list(order)
    order.clear()
    run(4, fn, "lockstep")
    assert order == first                        # same interleaving every time
    assert first[:4] == [(r, "a") for r in range(4)]
    assert first[4:8] == [(r, "b") for r in range(4)]
    b, cb = run(4, fn, "threads")
    for (x1, y1), (x2, y2) in zip(a, b):
        assert torch.equal(x1, x2) and torch.equal(y1, y2)
    assert ca.records == cb.records
    assert [r.direction for r in ca.records] == [Direction.FORWARD, Direction.BACKWARD]


def test_bad_arguments():
    with pytest.raises(ConfigurationError):
        Communicator(0)
    with pytest.raises(ConfigurationError):
        Communicator(2, mode="nope")
    with pytest.raises(ConfigurationError):
        run(2, lambda cm, r: cm.broadcast(r, 5, T(1.0)))
