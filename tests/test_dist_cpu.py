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


def _bench(args, env_extra=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, env=env, cwd=root)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p.returncode, [json.loads(ln) for ln in lines], p.stderr


def test_bench_gpus2_self_launches_two_ranks():
    # `bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (gloo here, NCCL on
    # GPUs); the default C3 workload is strong-scaled: m/2 rows per rank, one JSON line
    rc, out, err = _bench(["--gpus", "2", "--plan-only"])
    assert rc == 0, err[-2000:]
    assert len(out) == 1, out
    line = out[0]
    assert line["n_gpus"] == 2
    assert line["config"]["m"] == 200000 and line["config"]["rows_per_rank"] == 100000
    assert line["rank_rows"] == [[0, 100000], [100000, 100000]]
    assert line["max_over_ranks_check"] == 1.0   # max over ranks of the rank index


def test_bench_world_size_mismatch_fails_loudly():
    rc, out, err = _bench(["--gpus", "4", "--plan-only"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc == 2 and not out and "WORLD_SIZE" in err
