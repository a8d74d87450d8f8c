"""World-size-2 gloo test of the replica plumbing used by bench.py under torchrun
(barrier, max-over-ranks timing, whole-job aggregation, sharding)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_16675_b200 import dist as D
    r, w, lr = D.rank_info()
    assert (r, w, lr) == (rank, world, rank)
    D.barrier()
    slowest = D.max_over_ranks(10.0 + rank)          # per-rank elapsed ms
    units = D.sum_over_ranks(4096)                   # weak scaling: every rank its own batch
    mine = list(D.shard(10, rank, world))
    q.put((rank, slowest, units, mine))
    dist.destroy_process_group()


def test_replica_plumbing_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [x[1] for x in res] == [11.0, 11.0]        # max over ranks seen by both
    assert [x[2] for x in res] == [8192.0, 8192.0]    # whole-job units
    assert res[0][3] + res[1][3] == list(range(10))   # shards partition the units


def test_shard_balance():
    from paper_2409_16675_b200.dist import shard
    for total in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            parts = [list(shard(total, r, world)) for r in range(world)]
            assert sum(parts, []) == list(range(total))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
