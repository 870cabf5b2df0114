"""Rank groups for the phantom-parallel engine.

Communicator mirrors phantomsim.collectives.Communicator (reference collectives.py:87-357): an
in-process group of `world_size` logical ranks, one host thread per rank (`run`), blocking
rendezvous collectives with the same semantics (all-gather concatenates along axis 0 in
ascending rank order; reductions sum in ascending rank order), the same protocol checks
(kind / tag / shape mismatch, double entry, a rank finishing without entering, timeout) and
the same CommRecord stream.  Payloads are CUDA tensors living on one GPU, so the "exchange" is a
device-side concat / sum; the multi-GPU path (one process per GPU, NCCL over NVLink through
libppx.so) is `engine.PhantomEngine`.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass
from enum import Enum

import torch

from .errors import ConfigurationError, ProtocolError


class Collective(Enum):
    BROADCAST = "broadcast"
    ALL_GATHER = "all_gather"
    ALL_REDUCE = "all_reduce"
    REDUCE_SCATTER = "reduce_scatter"


class Direction(Enum):
    FORWARD = "forward"
    BACKWARD = "backward"
    LOSS = "loss"


@dataclass(frozen=True)
class CommRecord:
    """collectives.py:54-60 — one completed collective; message_size = elements per rank."""

    seq: int
    collective: Collective
    message_size: int
    direction: Direction | None = None
    layer: int | None = None


class _Abort(Exception):
    pass


class _Pending:
    def __init__(self, seq, kind, root, direction, layer, p):
        self.seq, self.kind, self.root, self.direction, self.layer = seq, kind, root, direction, layer
        self.slots = [None] * p
        self.entered = [False] * p
        self.arrived = 0
        self.results = None
        self.done = False
        self.error = None


class Communicator:
    """In-process group of logical ranks with blocking collectives over device tensors."""

    def __init__(self, world_size: int, mode: str = "threads", timeout: float = 120.0):
        if world_size < 1:
            raise ConfigurationError("world_size must be >= 1")
        if mode not in ("lockstep", "threads"):
            raise ConfigurationError(f"unknown scheduler mode: {mode!r}")
        self.world_size = world_size
        self.mode = mode
        self.timeout = timeout
        self.records: list[CommRecord] = []
        self._cv = threading.Condition()
        self._seq = 0
        self._pending: _Pending | None = None
        self._finished = [True] * world_size
        self._failure: BaseException | None = None

    # ---- collectives (collectives.py:115-142) -------------------------------------------------
    def all_gather(self, rank, local, *, direction=None, layer=None):
        return self._collective(rank, Collective.ALL_GATHER, self._payload(local), direction=direction, layer=layer)

    def reduce_scatter(self, rank, contributions, *, direction=None, layer=None):
        return self._collective(rank, Collective.REDUCE_SCATTER, self._payload(contributions),
                                direction=direction, layer=layer)

    def broadcast(self, rank, root, payload=None, *, direction=None, layer=None):
        if not 0 <= root < self.world_size:
            raise ConfigurationError(f"broadcast root {root} out of range")
        data = self._payload(payload) if payload is not None else None
        return self._collective(rank, Collective.BROADCAST, data, root=root, direction=direction, layer=layer)

    def all_reduce(self, rank, local, *, direction=None, layer=None):
        return self._collective(rank, Collective.ALL_REDUCE, self._payload(local), direction=direction, layer=layer)

    # ---- rank programs (collectives.py:147-194) -----------------------------------------------
    def run(self, fn, *args, **kwargs) -> list:
        p = self.world_size
        with self._cv:
            if self._pending is not None:
                raise ProtocolError("a previous run left a collective pending")
            self._finished = [False] * p
            self._failure = None
        results = [None] * p
        errors: list[tuple[int, BaseException]] = []
        device = torch.cuda.current_device() if torch.cuda.is_available() else None
        stream = torch.cuda.current_stream() if torch.cuda.is_available() else None

        def worker(rank):
            failed = False
            try:
                if device is not None:
                    torch.cuda.set_device(device)
                    with torch.cuda.stream(stream):   # one stream: host rendezvous orders the GPU work
                        results[rank] = fn(self, rank, *args, **kwargs)
                else:
                    results[rank] = fn(self, rank, *args, **kwargs)
            except BaseException as exc:  # noqa: BLE001 - re-raised below
                failed = True
                with self._cv:
                    errors.append((rank, exc))
                    if self._failure is None:
                        self._failure = exc
                    if self._pending is not None and self._pending.error is None:
                        self._pending.error = exc
                    self._cv.notify_all()
            finally:
                self._rank_finished(rank, failed)

        if p == 1:
            worker(0)
        else:
            threads = [threading.Thread(target=worker, args=(r,), name=f"rank-{r}", daemon=True) for r in range(p)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        primary = sorted(((r, e) for r, e in errors if not isinstance(e, _Abort)), key=lambda t: t[0])
        if primary:
            raise primary[0][1]
        if errors:
            raise errors[0][1]
        return results

    # ---- internals ------------------------------------------------------------------------------
    @staticmethod
    def _payload(x):
        if not isinstance(x, torch.Tensor):
            raise ConfigurationError("collective payloads must be tensors")
        if x.dim() not in (1, 2):
            raise ConfigurationError("collective payloads must be 1-d or 2-d")
        return x

    def _wait(self, pred, what):
        deadline = time.monotonic() + self.timeout
        while not pred():
            if self._failure is not None:
                raise _Abort(f"aborted while waiting for {what}: {self._failure}")
            remaining = deadline - time.monotonic()
            if remaining <= 0:
                err = ProtocolError(f"timeout after {self.timeout:.0f}s waiting for {what} (possible deadlock)")
                self._fail(err)
                raise err
            self._cv.wait(min(remaining, 0.5))

    def _fail(self, err):
        if self._failure is None:
            self._failure = err
        if self._pending is not None and self._pending.error is None:
            self._pending.error = err
        self._cv.notify_all()

    def _rank_finished(self, rank, failed):
        with self._cv:
            self._finished[rank] = True
            pend = self._pending
            if pend is not None and not pend.entered[rank] and not failed:
                self._fail(ProtocolError(f"deadlock at collective seq {pend.seq} ({pend.kind.value}): "
                                         f"rank {rank} finished without entering"))
            self._cv.notify_all()

    def _collective(self, rank, kind, payload, *, root=None, direction=None, layer=None):
        if not 0 <= rank < self.world_size:
            raise ConfigurationError(f"rank {rank} out of range for world size {self.world_size}")
        with self._cv:
            if self._failure is not None:
                raise _Abort(f"aborted: {self._failure}")
            if self._pending is None:
                self._pending = _Pending(self._seq, kind, root, direction, layer, self.world_size)
            pend = self._pending
            err = None
            if pend.kind is not kind:
                err = ProtocolError(f"collective mismatch at seq {pend.seq}: rank {rank} called {kind.value} "
                                    f"while {pend.kind.value} is in progress")
            elif kind is Collective.BROADCAST and pend.root != root:
                err = ProtocolError(f"broadcast root mismatch at seq {pend.seq}: rank {rank} passed root {root}, "
                                    f"expected {pend.root}")
            elif (pend.direction, pend.layer) != (direction, layer):
                err = ProtocolError(f"record tag mismatch at seq {pend.seq} on rank {rank}")
            elif pend.entered[rank]:
                err = ProtocolError(f"rank {rank} entered seq {pend.seq} twice")
            if err is not None:
                self._fail(err)
                raise err
            pend.entered[rank] = True
            pend.slots[rank] = payload
            pend.arrived += 1
            if pend.arrived == self.world_size:
                try:
                    results, msize = self._combine(pend)
                except ProtocolError as e:
                    self._fail(e)
                    raise
                self.records.append(CommRecord(pend.seq, pend.kind, msize, pend.direction, pend.layer))
                self._seq += 1
                pend.results = results
                pend.done = True
                self._pending = None
                self._cv.notify_all()
            else:
                self._wait(lambda: pend.done or pend.error is not None, f"collective seq {pend.seq} ({kind.value})")
            if pend.error is not None:
                raise pend.error
            return pend.results[rank]

    def _combine(self, pend):
        p = self.world_size
        slots = pend.slots
        if pend.kind is Collective.BROADCAST:
            payload = slots[pend.root]
            if payload is None:
                raise ProtocolError(f"broadcast root {pend.root} passed no payload")
            return [payload.clone() for _ in range(p)], payload.numel()
        shapes = {tuple(s.shape) for s in slots}
        if len(shapes) != 1:
            raise ProtocolError(f"{pend.kind.value} shape disagreement at seq {pend.seq}: {sorted(shapes)}")
        if pend.kind is Collective.ALL_GATHER:
            out = torch.cat(list(slots), dim=0)
            return [out if r == 0 else out.clone() for r in range(p)], slots[0].numel()
        if pend.kind is Collective.ALL_REDUCE:
            acc = slots[0].clone()
            for s in slots[1:]:  # ascending rank order
                acc += s
            return [acc.clone() for _ in range(p)], slots[0].numel()
        rows = slots[0].shape[0]
        if rows % p != 0:
            raise ProtocolError(f"reduce_scatter chunk-count mismatch: {rows} rows not divisible by p={p}")
        chunk = rows // p
        results = []
        for j in range(p):
            acc = slots[0][j * chunk:(j + 1) * chunk].clone()
            for s in slots[1:]:  # ascending rank order
                acc += s[j * chunk:(j + 1) * chunk]
            results.append(acc)
        return results, results[0].numel()
