"""Host-side placement and collective schedule of the multi-GPU phantom engine (pure Python).

Logical phantom rank j lives on GPU j // R with R = p / world (contiguous blocks, so every GPU's
slots of a [p, batch, k] phantom buffer are one contiguous chunk and NCCL's in-place all-gather
and reduce-scatter move exactly the reference's rank blocks, collectives.py:337-357).  The
engine and libppx.so (ppx_all_gather / ppx_reduce_scatter) use this arithmetic; the CPU tests
check it with a gloo process group.
"""

from __future__ import annotations

from .errors import ConfigurationError


def local_ranks(p: int, world: int, gpu: int) -> list[int]:
    if world < 1 or p % world:
        raise ConfigurationError(f"p={p} logical ranks do not divide over {world} GPUs")
    if not 0 <= gpu < world:
        raise ConfigurationError(f"gpu {gpu} out of range for world {world}")
    r = p // world
    return list(range(gpu * r, (gpu + 1) * r))


def owner(j: int, p: int, world: int) -> int:
    return j // (p // world)


def slot_chunk(p: int, world: int, gpu: int, slot_elems: int) -> tuple[int, int]:
    """(element offset, element count) of this GPU's contiguous slot range in a [p, ...] buffer:
    the in-place send buffer of the all-gather and receive buffer of the reduce-scatter."""
    r = p // world
    return gpu * r * slot_elems, r * slot_elems


def collective_schedule(layers: int, world: int) -> list[tuple[str, str, int | None]]:
    """Collectives one training step issues, in order (training.py:181-213; Table I of the paper):
    per layer one phantom all-gather forward, one reduce-scatter backward (descending layers),
    one scalar loss all-reduce. With world == 1 the phantom exchange stays in HBM (no NCCL)."""
    if world == 1:
        return []
    sched = [("all_gather", "forward", l) for l in range(layers)]
    sched += [("reduce_scatter", "backward", l) for l in range(layers - 1, -1, -1)]
    sched.append(("all_reduce", "loss", None))
    return sched


def comm_bytes_per_step(n: int, p: int, k: int, layers: int, batch: int, world: int, elem: int = 2) -> int:
    """Bytes one GPU sends per training step (ring all-gather / reduce-scatter: each GPU sends
    (world-1) chunks of R * batch * k elements per layer per direction)."""
    if world == 1:
        return 0
    r = p // world
    return 2 * layers * (world - 1) * r * batch * k * elem


def tp_comm_bytes_per_step(n: int, layers: int, batch: int, world: int, elem: int = 2) -> int:
    """Megatron tensor parallelism: 2 all-reduces of batch x n per column/row pair (forward +
    backward); a ring all-reduce sends 2 (world-1)/world of the buffer per GPU."""
    if world == 1:
        return 0
    pairs = layers // 2
    return int(2 * pairs * 2 * (world - 1) / world * batch * n * elem)


MAX_PROBS = 16   # problems per grouped GEMM launch (csrc/gemm_sm100.cuh)


def wgrad_launch_chunks(R: int, p: int, nprob: int, group: int, with_errors: bool) -> list[tuple[int, int]]:
    """Logical-rank ranges [c0, c1) of one layer's weight-gradient launches (`nprob` problems per
    rank, <= MAX_PROBS per launch, at most `group` ranks per launch, balanced).  with_errors: the
    first launch also carries the layer's error compression as p/2 slot-pair problems (the
    one-GPU default plan, engine.k3_grouped)."""
    per = max(1, min(group, MAX_PROBS // nprob))
    nl = -(-R // per)
    per = -(-R // nl)
    out, c = [], 0
    if with_errors:
        first = min(per, (MAX_PROBS - p // 2) // nprob)
        if first < 1:
            raise ConfigurationError(f"{p // 2} error problems leave no room for weight gradients")
        nl2 = 1 + -(-(R - first) // per)
        first = min(first, -(-R // nl2))          # balance the ranks over the launches
        per = max(1, -(-(R - first) // max(1, nl2 - 1)))
        out.append((0, first))
        c = first
    while c < R:
        out.append((c, min(R, c + per)))
        c += per
    return out


def layer0_split(n_items: int, k: int, s: int, batch: int) -> int:
    """Batch chunks of the layer-0 compressor gradient (ppx_wgrad_splitk, 128 x 256 tiles of the
    1-SM kernel): doubled while the doubled launch still fits one round on the 148 SMs, every
    chunk stays whole 128-row K blocks and the launch holds <= MAX_PROBS problems; 1 = unsplit."""
    tiles = n_items * -(-k // 128) * -(-s // 256)
    nsplit = 1
    while (tiles * nsplit * 2 <= 148 and n_items * nsplit * 2 <= MAX_PROBS and batch % (nsplit * 2) == 0
           and (batch // (nsplit * 2)) % 128 == 0):
        nsplit *= 2
    return nsplit
