"""CPU, world_size 2 over gloo: the replica plumbing bench.py and the batched-runs layer use
(shard partition, max-over-ranks timing, ordered gather of per-run results)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2505_17430_b200 import dist as D


def test_shard_partition_covers_every_item_once():
    for n in (0, 1, 5, 64, 100, 1023):
        for world in (1, 2, 3, 8):
            owned = []
            for r in range(world):
                a, b = D.shard(n, r, world)
                assert 0 <= a <= b <= n
                owned += list(range(a, b))
            assert owned == list(range(n))
            sizes = [D.shard(n, r, world)[1] - D.shard(n, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    dist = D.init("gloo")
    r, w, _ = D.env()
    t = D.max_over_ranks(1.5 + r, dist)
    a, b = D.shard(64, r, w)
    local = [("run", i) for i in range(a, b)]
    allr = D.gather_ordered(local, 64, dist)
    dist.barrier()
    q.put((r, t, allr))
    dist.destroy_process_group()


def test_gloo_world2_max_and_ordered_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, t, allr in res:
        assert t == 2.5  # the slowest rank's time on every rank
        assert allr == [("run", i) for i in range(64)]
