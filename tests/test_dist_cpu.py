"""CPU: the multi-GPU host logic with a world-size-2 gloo process group —
row sharding, NCCL-id exchange, max-over-ranks timing (the data-path
collectives themselves are NCCL inside the library; their schedule is
covered on one GPU by tests/test_gpu_multirank.py)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1804_00462_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = bytes(range(128))
        nid = D.exchange_nccl_id(dist, rank, make_id=lambda: fake)
        t = D.max_over_ranks(dist, 1.5 + rank)
        r0, rows = D.row_partition(10001, world, rank)
        q.put((rank, nid == fake, t, r0, rows))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res)            # every rank received rank 0's id
    assert all(r[2] == 2.5 for r in res)      # max over ranks
    (r0a, na), (r0b, nb) = (res[0][3], res[0][4]), (res[1][3], res[1][4])
    assert r0a == 0 and r0b == na and na + nb == 10001 and na - nb in (0, 1)


@pytest.mark.parametrize("m,world", [(7, 3), (200000, 8), (4000, 1), (5, 5)])
def test_row_partition_covers(m, world):
    from paper_1804_00462_b200 import dist as D
    nxt = 0
    for r in range(world):
        r0, rows = D.row_partition(m, world, r)
        assert r0 == nxt and rows >= m // world
        nxt = r0 + rows
    assert nxt == m
