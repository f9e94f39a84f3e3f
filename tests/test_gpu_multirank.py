"""SURVEY §8(e) parity across world sizes, on ONE GPU: bench.py's head-sharded path run as two
ranks (two processes on cuda:0, gloo process group) reproduces the 1-rank run of the same
global problem — per-head O, lse, dK, dV bitwise (atomic-free), dQ to one bf16 ulp (fp32
reduce-add order) — and the per-rank gather carries every rank's checksums."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _outputs(run):
    return [tuple(t.cpu() for t in outs) for outs in run.outs]


def _worker(rank, world, port, cfg, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench
    from paper_2410_01359_b200 import flashmask as fm
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        calls, _, _ = bench.build_workload(cfg, rank, world, bench.rho_gpu(fm))
        run = bench.Runner(fm, calls, torch.device("cuda", 0))
        run.step()
        torch.cuda.synchronize()
        gathered = bench.gather_ranks([float(rank)] + run.checksums(), dist, "cpu")
        torch.save({"heads": [list(c["heads"]) for c in calls], "outs": _outputs(run), "gathered": gathered}, path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["C2", "C5:8192:64:document,random_eviction"])
def test_two_ranks_match_one_rank(tmp_path, cfg):
    import bench
    from paper_2410_01359_b200 import flashmask as fm
    calls, _, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
    ref = bench.Runner(fm, calls, torch.device("cuda", 0))
    ref.step()
    torch.cuda.synchronize()
    ref_outs = _outputs(ref)
    ref.free()
    torch.cuda.empty_cache()

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    paths = [str(tmp_path / f"rank{r}.pt") for r in range(world)]
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, paths[r])) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0
    res = [torch.load(p) for p in paths]
    assert res[0]["gathered"] == res[1]["gathered"] and [g[0] for g in res[0]["gathered"]] == [0.0, 1.0]
    for r in range(world):
        for ci, (heads, outs) in enumerate(zip(res[r]["heads"], res[r]["outs"])):
            h = slice(heads[0], heads[-1] + 1)
            o, lse, dq, dk, dv = ref_outs[ci]
            assert torch.equal(outs[0], o[:, :, h]), ("O", r, ci)
            assert torch.equal(outs[1], lse[:, h]), ("lse", r, ci)
            assert torch.equal(outs[3], dk[:, :, h]), ("dK", r, ci)
            assert torch.equal(outs[4], dv[:, :, h]), ("dV", r, ci)
            a, b = outs[2].float(), dq[:, :, h].float()
            assert ((a - b).abs() <= 2.0 ** -7 * b.abs() + 1e-3).all(), ("dQ", r, ci)
