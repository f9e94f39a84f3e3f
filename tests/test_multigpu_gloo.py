"""Host-side logic of the multi-GPU bench path, run as 2 CPU processes over gloo.

Heads are independent, so ranks shard them with no data-path collective (SURVEY
§8(e)); after the timed region the ranks all_gather their per-rank results.  Checks: every
config is head-sharded over ONE global problem (same masks on every rank, head ranges
partition [0, H)), the per-rank gather returns every rank's vector in rank order, the max
reduction returns the slowest rank's time, and --gpus N without torchrun refuses to run on
fewer GPUs than requested."""
import os
import socket
import subprocess
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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
        gathered = bench.gather_ranks([float(rank), 2.5 * rank, -1.0], dist, "cpu")
        res = {"slowest": slowest, "gathered": gathered}
        for cfg in ("C2", "C3", "C4", "C5:8192:64:causal_document,random_eviction"):
            calls, conf, sc = bench.build_workload(cfg, rank, world, bench.rho_oracle)
            res[cfg] = ([list(c["heads"]) for c in calls], [[m.sri.copy() for m in c["masks"]] for c in calls],
                        sc, conf["global_batch"], [c["B"] for c in calls])
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharding_and_gathers():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, v = q.get(timeout=900)
        res[r] = v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["slowest"] == res[1]["slowest"] == 11.0
    assert res[0]["gathered"] == res[1]["gathered"] == [[0.0, 0.0, -1.0], [1.0, 2.5, -1.0]]
    for cfg, H in (("C2", 32), ("C3", 32), ("C4", 64), ("C5:8192:64:causal_document,random_eviction", 64)):
        h0, m0, sc0, gb0, b0 = res[0][cfg]
        h1, m1, sc1, gb1, b1 = res[1][cfg]
        assert sc0 == sc1 == "strong" and gb0 == gb1 and b0 == b1
        for a, b in zip(h0, h1):          # head ranges partition [0, H)
            assert a == list(range(0, H // 2)) and b == list(range(H // 2, H))
        for ca, cb in zip(m0, m1):        # one global problem: identical masks on both ranks
            assert all(np.array_equal(x, y) for x, y in zip(ca, cb))


def test_gpus_flag_refuses_fewer_gpus():
    """`bench.py --gpus 2` without torchrun re-launches itself as 2 ranks, or fails loudly when
    fewer GPUs are visible (here: none) — it never silently runs on 1 GPU."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "only 0 CUDA device" in r.stderr, r.stderr[-2000:]
