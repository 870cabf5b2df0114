"""Multi-process host logic of the N>1 path on CPU (gloo, world size 2): logical-rank placement,
the in-place all-gather / reduce-scatter slot chunks, and the collective schedule, checked against
the reference semantics (collectives.py:337-357: concatenate in ascending rank order; sums in
ascending rank order) by moving real data through torch.distributed with the engine's offsets."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_00960_b200 import schedule


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, p, B, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        slot = B * k
        mine = schedule.local_ranks(p, world, rank)
        off, cnt = schedule.slot_chunk(p, world, rank, slot)
        # all-gather: each logical rank j writes phantom block value 100*j + position
        buf = torch.zeros(p * slot)
        for j in mine:
            buf[j * slot:(j + 1) * slot] = 100.0 * j + torch.arange(slot, dtype=torch.float32)
        chunks = list(buf.view(world, cnt).unbind(0))
        dist.all_gather(chunks, buf[off:off + cnt].clone())
        gathered = torch.cat(chunks)
        expect = torch.cat([100.0 * j + torch.arange(slot, dtype=torch.float32) for j in range(p)])
        ok_ag = torch.equal(gathered, expect)
        # reduce-scatter: logical rank i contributes (i+1) * (slot index + 1) to every peer slot
        contrib = torch.zeros(p * slot)
        for i in mine:
            for j in range(p):
                if j != i:
                    contrib[j * slot:(j + 1) * slot] += (i + 1) * (j + 1)
        total = contrib.clone()
        dist.all_reduce(total)
        mine_sum = total[off:off + cnt]
        exp = torch.cat([torch.full((slot,), float(sum((i + 1) * (j + 1) for i in range(p) if i != j)))
                         for j in mine])
        ok_rs = torch.equal(mine_sum, exp)
        sched = schedule.collective_schedule(3, world)
        objs = [None] * world
        dist.all_gather_object(objs, sched)
        ok_sched = all(o == sched for o in objs)
        q.put((rank, ok_ag, ok_rs, ok_sched, mine))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_slot_chunks_and_schedule_world2(p):
    world, B, k = 2, 3, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, B, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    res.sort()
    assert [r[4] for r in res] == [list(range(0, p // 2)), list(range(p // 2, p))]
    for _, ok_ag, ok_rs, ok_sched, _ in res:
        assert ok_ag and ok_rs and ok_sched


def test_schedule_shapes():
    assert schedule.collective_schedule(2, 1) == []
    s = schedule.collective_schedule(2, 4)
    assert [x[0] for x in s] == ["all_gather", "all_gather", "reduce_scatter", "reduce_scatter", "all_reduce"]
    assert [x[2] for x in s[:4]] == [0, 1, 1, 0]
    # PP sends <= 1/4 of the Megatron TP bytes at the headline shape (north_star target)
    pp = schedule.comm_bytes_per_step(16384, 8, 128, 8, 8192, 8)
    tp = schedule.tp_comm_bytes_per_step(16384, 8, 8192, 8)
    assert pp * 4 <= tp
    with pytest.raises(Exception):
        schedule.local_ranks(6, 4, 0)
