"""Host-side logic of the multi-GPU bench path, run as 2 CPU processes over gloo.

Heads/batch entries are independent, so ranks shard them with no data-path
collective; the only collective is the max-over-ranks of the timings.  Checks: batch shards
(C2/C3) are disjoint and seeded per global batch index, head shards (C4) partition the heads,
and the max reduction returns the slowest rank's time on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        slowest = bench.reduce_max_over_ranks(10.0 + rank, dist, "cpu")
        c2, conf2, sc2 = bench.build_workload("C2", rank, world, bench.rho_oracle)
        c4, conf4, sc4 = bench.build_workload("C4", rank, world, bench.rho_oracle)
        q.put((rank, slowest, [c["batch_ids"] for c in c2], [m.sri.copy() for m in c2[0]["masks"]],
               list(c4[0]["heads"]), sc2, sc4, conf2["global_batch"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_max_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # max over ranks = slowest rank, on every rank
    assert res[0][1] == res[1][1] == 11.0
    # C2: batch entries sharded, different seeds -> different masks (weak scaling)
    assert res[0][2][0] == [0] and res[1][2][0] == [1]
    assert not np.array_equal(res[0][3][0], res[1][3][0])
    assert res[0][5] == "weak" and res[0][7] == 2
    # C4: heads partitioned across ranks (strong scaling)
    assert res[0][4] == list(range(0, 32)) and res[1][4] == list(range(32, 64))
    assert res[0][6] == "strong"
