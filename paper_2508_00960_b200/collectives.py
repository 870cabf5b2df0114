"""In-process rank group for the drop-in API (the reference's Communicator, collectives.py:87-357).

The phantomsim API runs one program per logical rank (`Communicator.run(fn)` calls
fn(comm, rank) on every rank) and exchanges data only through blocking collectives.  Here the
payloads are CUDA tensors of one GPU, so every collective is a device-side concatenate / sum
issued by the last rank to arrive; the multi-GPU engine (one process per GPU, NVLink / NCCL inside
libppx.so) is engine.PhantomEngine.

Semantics kept from the reference (its tests exercise them): all-gather concatenates along axis
0 in ascending rank order; all-reduce and reduce-scatter sum in ascending rank order (so both
schedulers give bit-identical results); every completed collective appends a CommRecord
(seq, kind, elements per rank, direction, layer) in sequence order; misuse raises ProtocolError
on every rank (kind / root / tag mismatch, double entry, shape disagreement, a reduce-scatter
whose rows do not split into p chunks, a rank that finishes while its peers wait = deadlock,
timeout); the first failing rank's exception is re-raised by run().

This module's own design: each rank keeps a private sequence counter, and its i-th collective
joins meeting i (a record of the entrants, created by the first of them); the last entrant
validates and combines, then releases the others.  The two schedulers differ only in who may
run Python between collectives:

  * "threads": every rank thread runs freely; waits are bounded by `timeout`.
  * "lockstep" (the reference default): a baton — exactly one rank runs at a time, and the
    baton always goes to the lowest-numbered rank that is neither finished nor blocked in an
    incomplete meeting, so the interleaving is fully deterministic.  If every unfinished rank
    is blocked, the meeting can never complete: that is reported as a deadlock at once.
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
    """Tag of a collective; LOSS marks the per-iteration scalar loss all-reduce."""
    FORWARD = "forward"
    BACKWARD = "backward"
    LOSS = "loss"


@dataclass(frozen=True)
class CommRecord:
    """One completed collective; message_size = elements per rank (collectives.py:54-60)."""
    seq: int
    collective: Collective
    message_size: int
    direction: Direction | None = None
    layer: int | None = None


class _PeerFailed(ProtocolError):
    """Raised in ranks that were waiting when another rank failed (never the primary error)."""


class _Meeting:
    def __init__(self, seq, kind, root, tag, p):
        self.seq, self.kind, self.root, self.tag = seq, kind, root, tag
        self.inputs = [None] * p
        self.joined = [False] * p
        self.outputs = None

    @property
    def complete(self):
        return self.outputs is not None


def _sum_in_rank_order(parts):
    acc = parts[0].clone()
    for x in parts[1:]:
        acc += x
    return acc


def _combine(m: _Meeting, p: int):
    """(per-rank results, elements per rank) of a full meeting."""
    xs = m.inputs
    if m.kind is Collective.BROADCAST:
        src = xs[m.root]
        if src is None:
            raise ProtocolError(f"broadcast root {m.root} passed no payload (seq {m.seq})")
        return [src.clone() for _ in range(p)], src.numel()
    if len({tuple(x.shape) for x in xs}) != 1:
        raise ProtocolError(f"{m.kind.value} shape disagreement at seq {m.seq}: "
                            f"{[tuple(x.shape) for x in xs]}")
    if m.kind is Collective.ALL_GATHER:
        g = torch.cat(xs, dim=0)
        return [g] + [g.clone() for _ in range(p - 1)], xs[0].numel()
    if m.kind is Collective.ALL_REDUCE:
        s = _sum_in_rank_order(xs)
        return [s] + [s.clone() for _ in range(p - 1)], xs[0].numel()
    rows = xs[0].shape[0]
    if rows % p:
        raise ProtocolError(f"reduce_scatter at seq {m.seq}: {rows} rows do not split into p={p} chunks")
    c = rows // p
    out = [_sum_in_rank_order([x[j * c:(j + 1) * c] for x in xs]) for j in range(p)]
    return out, out[0].numel()


class Communicator:
    """`world_size` logical ranks in one process (one host thread each) with blocking collectives
    over tensors.  mode = "lockstep" (deterministic baton, the reference default) or "threads"."""

    def __init__(self, world_size: int, mode: str = "lockstep", timeout: float = 120.0):
        if world_size < 1:
            raise ConfigurationError("world_size must be >= 1")
        if mode not in ("lockstep", "threads"):
            raise ConfigurationError(f"unknown scheduler mode: {mode!r}")
        self.world_size, self.mode, self.timeout = world_size, mode, timeout
        self.records: list[CommRecord] = []
        self._cond = threading.Condition()
        self._meeting: _Meeting | None = None
        self._next_seq = [0] * world_size
        self._done_seq = 0
        self._finished = [True] * world_size
        self._blocked = [False] * world_size
        self._baton = None
        self._error: BaseException | None = None

    # ---- collectives (collectives.py:115-142) -------------------------------------------------
    def all_gather(self, rank, local, *, direction=None, layer=None):
        return self._enter(rank, Collective.ALL_GATHER, self._tensor(local), None, (direction, layer))

    def reduce_scatter(self, rank, contributions, *, direction=None, layer=None):
        return self._enter(rank, Collective.REDUCE_SCATTER, self._tensor(contributions), None, (direction, layer))

    def broadcast(self, rank, root, payload=None, *, direction=None, layer=None):
        if not 0 <= root < self.world_size:
            raise ConfigurationError(f"broadcast root {root} out of range")
        data = None if payload is None else self._tensor(payload)
        return self._enter(rank, Collective.BROADCAST, data, root, (direction, layer))

    def all_reduce(self, rank, local, *, direction=None, layer=None):
        return self._enter(rank, Collective.ALL_REDUCE, self._tensor(local), None, (direction, layer))

    # ---- rank programs --------------------------------------------------------------------------
    def run(self, fn, *args, **kwargs) -> list:
        """fn(comm, rank, *args, **kwargs) on every rank; returns the per-rank results."""
        p = self.world_size
        with self._cond:
            if self._meeting is not None:
                raise ProtocolError("a previous run left a collective open")
            self._finished = [False] * p
            self._blocked = [False] * p
            self._next_seq = [self._done_seq] * p
            self._error = None
            self._baton = 0 if self.mode == "lockstep" else None
        results = [None] * p
        failures: list[tuple[int, BaseException]] = []
        cuda = torch.cuda.is_available()
        device = torch.cuda.current_device() if cuda else None
        stream = torch.cuda.current_stream() if cuda else None

        def rank_main(rank):
            ok = False
            try:
                with self._cond:
                    self._await(lambda: True, rank, "its first turn")
                if cuda:
                    torch.cuda.set_device(device)
                    with torch.cuda.stream(stream):   # one stream: the rendezvous orders the GPU work
                        results[rank] = fn(self, rank, *args, **kwargs)
                else:
                    results[rank] = fn(self, rank, *args, **kwargs)
                ok = True
            except BaseException as exc:  # noqa: BLE001 - re-raised by run()
                with self._cond:
                    failures.append((rank, exc))
                    self._raise_all(exc)
            finally:
                self._exit(rank, ok)

        if p == 1:
            rank_main(0)
        else:
            threads = [threading.Thread(target=rank_main, args=(r,), name=f"phantom-rank-{r}", daemon=True)
                       for r in range(p)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        primary = sorted(((r, e) for r, e in failures if not isinstance(e, _PeerFailed)), key=lambda t: t[0])
        if primary:
            raise primary[0][1]
        if self._error is not None:      # detected outside any rank's code (deadlock at exit)
            raise self._error
        if failures:
            raise failures[0][1]
        return results

    # ---- internals (caller holds self._cond where noted) ---------------------------------------
    @staticmethod
    def _tensor(x):
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(x)
        if t.dim() not in (1, 2):
            raise ConfigurationError("collective payloads must be 1-d or 2-d")
        return t

    def _raise_all(self, err):
        """(locked) record the first failure and wake everybody."""
        if self._error is None:
            self._error = err
        self._cond.notify_all()

    def _pass_baton(self):
        """(locked, lockstep) hand the baton to the lowest runnable rank; if every unfinished
        rank is blocked on the open meeting, it can never complete."""
        p = self.world_size
        runnable = [r for r in range(p) if not self._finished[r] and not self._blocked[r]]
        self._baton = runnable[0] if runnable else None
        m = self._meeting
        if self._baton is None and m is not None and self._error is None:
            missing = [r for r in range(p) if not m.joined[r]]
            self._raise_all(ProtocolError(f"deadlock at collective seq {m.seq} ({m.kind.value}): "
                                          f"rank(s) {missing} finished without entering"))
        self._cond.notify_all()

    def _await(self, ready, rank, what):
        """(locked) wait until ready() and — in lockstep — this rank holds the baton."""
        deadline = time.monotonic() + self.timeout
        while True:
            if self._error is not None:
                raise _PeerFailed(f"rank {rank} aborted while waiting for {what}: {self._error}")
            if ready() and (self.mode != "lockstep" or self._baton == rank):
                return
            left = deadline - time.monotonic()
            if left <= 0:
                err = ProtocolError(f"timeout after {self.timeout:.0f}s waiting for {what} (possible deadlock)")
                self._raise_all(err)
                raise err
            self._cond.wait(min(left, 0.25))

    def _fail(self, err):
        """(locked) fail the group with a primary error raised in this rank."""
        self._raise_all(err)
        raise err

    def _enter(self, rank, kind, payload, root, tag):
        p = self.world_size
        if not 0 <= rank < p:
            raise ConfigurationError(f"rank {rank} out of range for world size {p}")
        with self._cond:
            if self._error is not None:
                raise _PeerFailed(f"rank {rank} aborted: {self._error}")
            seq = self._next_seq[rank]
            m = self._meeting
            if m is None:
                m = self._meeting = _Meeting(seq, kind, root, tag, p)
            elif m.joined[rank]:
                self._fail(ProtocolError(f"rank {rank} entered seq {m.seq} twice"))
            if m.kind is not kind:
                self._fail(ProtocolError(f"collective mismatch at seq {m.seq}: rank {rank} called {kind.value} "
                                         f"while {m.kind.value} is in progress"))
            if kind is Collective.BROADCAST and m.root != root:
                self._fail(ProtocolError(f"broadcast root mismatch at seq {m.seq}: rank {rank} passed root {root}, "
                                         f"the meeting uses root {m.root}"))
            if m.tag != tag:
                self._fail(ProtocolError(f"record tag mismatch at seq {m.seq} on rank {rank}: {tag} vs {m.tag}"))
            m.joined[rank] = True
            m.inputs[rank] = payload
            self._next_seq[rank] = seq + 1
            if all(m.joined):
                try:
                    m.outputs, size = _combine(m, p)
                except ProtocolError as err:
                    self._fail(err)
                self.records.append(CommRecord(m.seq, kind, size, *tag))
                self._meeting = None
                self._done_seq += 1
                self._blocked = [False] * p
                if self.mode == "lockstep":
                    self._pass_baton()
                self._cond.notify_all()
            else:
                self._blocked[rank] = True
                if self.mode == "lockstep":
                    self._pass_baton()
            self._await(lambda: m.complete, rank, f"collective seq {m.seq} ({kind.value})")
            return m.outputs[rank]

    def _exit(self, rank, ok):
        with self._cond:
            self._finished[rank] = True
            m = self._meeting
            if m is not None and not m.joined[rank] and ok and self._error is None:
                self._raise_all(ProtocolError(f"deadlock at collective seq {m.seq} ({m.kind.value}): "
                                              f"rank {rank} finished without entering"))
            if self.mode == "lockstep":
                self._pass_baton()
            self._cond.notify_all()
