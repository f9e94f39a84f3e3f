"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The workloads are built by bench.build_workload (C2, C3, C4) with inputs from bench.make_inputs;
the oracle checks what it can compute at that size:
* C2 (N=8192, H=32): two whole heads per mask, every output (O, lse, dQ, dK, dV);
* C3 (N=32768, B=4): 128 sampled rows of one head per batch entry (O, lse, dQ via
  backward_rows), plus the Q=0 closed forms (O, lse, dV) for one batch entry, all heads;
* C4 (N=131072, H=64): 64 sampled rows (O, lse, dQ) of one head per mask, and the Q=0 closed
  forms for two heads.
Bars as in test_gpu_parity (fp32 outputs); bf16 outputs (what bench.py times) are checked
against the same oracle with the bf16 rounding of the output added to the tolerance (R27).
"""
import numpy as np
import pytest
import torch

import bench
from oracle import flashmask_oracle as fo

from gpu_util import TOL_LSE, TOL_MAX, TOL_MEAN, assert_close, assert_lse

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fm():
    assert torch.cuda.is_available()
    from paper_2410_01359_b200 import flashmask
    return flashmask


def _run(fm, c, x, out_dtype):
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out_dtype=out_dtype)
    dq, dk, dv = fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], out_dtype=out_dtype)
    torch.cuda.synchronize()
    return o, lse, dq, dk, dv


def _head(x, name, b, h):
    return x[name][b, :, h, :].float().cpu().double().numpy()


def _check_bf16(name, got, ref):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bound = TOL_MAX + np.abs(ref) * 2.0 ** -8
    assert (err <= bound).all(), f"{name}: worst excess {float((err - bound).max()):.3e}"
    assert err.mean() <= TOL_MEAN, f"{name}: mean {err.mean():.3e}"


def test_c2_full_heads(fm):
    calls, _, _ = bench.build_workload("C2", 0, 1, bench.rho_oracle)
    dev = torch.device("cuda", 0)
    for c in calls:
        x = bench.make_inputs(c, dev)
        r32 = _run(fm, c, x, torch.float32)
        r16 = _run(fm, c, x, torch.bfloat16)
        m = c["masks"][0]
        vec = fo.expand(m.sri, m.causal, m.N)
        for h in (0, 17):
            q, k, v, do = (_head(x, n, 0, h) for n in ("q", "k", "v", "do"))
            O, L = fo.forward(q, k, v, vec)
            gq, gk, gv = fo.backward(q, k, v, do, vec)
            for name, idx, ref in (("O", 0, O), ("dQ", 2, gq), ("dK", 3, gk), ("dV", 4, gv)):
                assert_close(f"{m.family} {name}[h{h}]", r32[idx][0, :, h].cpu().numpy(), ref)
                _check_bf16(f"{m.family} {name}[h{h}] bf16", r16[idx][0, :, h].float().cpu().numpy(), ref)
            assert_lse(r32[1][0, h].cpu().numpy(), L)


def test_c3_sampled_rows_and_q_zero(fm):
    calls, _, _ = bench.build_workload("C3", 0, 1, bench.rho_oracle)
    c = calls[0]
    dev = torch.device("cuda", 0)
    x = bench.make_inputs(c, dev)
    o, lse, dq, dk, dv = _run(fm, c, x, torch.float32)
    rng = np.random.default_rng(0)
    N = c["N"]
    for b, m in enumerate(c["masks"]):
        vec = fo.expand(m.sri, m.causal, N)
        rows = np.sort(rng.choice(N, 128, replace=False))
        q, k, v, do = (_head(x, n, b, 3) for n in ("q", "k", "v", "do"))
        O, L = fo.forward(q, k, v, vec, rows=rows)
        gq, _, _ = fo.backward_rows(q, k, v, do, vec, rows)
        assert_close(f"b{b} O rows", o[b, rows, 3].cpu().numpy(), O)
        assert_lse(lse[b, 3, rows].cpu().numpy(), L)
        assert_close(f"b{b} dQ rows", dq[b, rows, 3].cpu().numpy(), gq)
    # Q = 0 closed forms on batch entry 3 (highest sparsity), all heads
    xz = dict(x)
    xz["q"] = torch.zeros_like(x["q"])
    o, lse, dq, dk, dv = _run(fm, c, xz, torch.float32)
    m = c["masks"][3]
    vec = fo.expand(m.sri, m.causal, N)
    for h in (0, 31):
        O, L = fo.forward_q_zero(_head(x, "v", 3, h), vec)
        assert_close(f"Q=0 O h{h}", o[3, :, h].cpu().numpy(), O)
        assert_lse(lse[3, h].cpu().numpy(), L)
        assert_close(f"Q=0 dV h{h}", dv[3, :, h].cpu().numpy(), fo.dv_q_zero(_head(x, "do", 3, h), vec))


def test_c4_sampled_rows_and_q_zero(fm):
    calls, _, _ = bench.build_workload("C4", 0, 1, bench.rho_oracle)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1)
    for c in calls:
        x = bench.make_inputs(c, dev)
        o, lse, dq, dk, dv = _run(fm, c, x, torch.float32)
        N = c["N"]
        m = c["masks"][0]
        vec = fo.expand(m.sri, m.causal, N)
        rows = np.sort(rng.choice(N, 64, replace=False))
        q, k, v, do = (_head(x, n, 0, 5) for n in ("q", "k", "v", "do"))
        O, L = fo.forward(q, k, v, vec, rows=rows, row_block=16)
        gq, _, _ = fo.backward_rows(q, k, v, do, vec, rows)
        assert_close("C4 O rows", o[0, rows, 5].cpu().numpy(), O)
        assert_lse(lse[0, 5, rows].cpu().numpy(), L)
        assert_close("C4 dQ rows", dq[0, rows, 5].cpu().numpy(), gq)
        del o, lse, dq, dk, dv
        xz = dict(x)
        xz["q"] = torch.zeros_like(x["q"])
        o, lse, dq, dk, dv = _run(fm, c, xz, torch.float32)
        for h in (0, 63):
            O, L = fo.forward_q_zero(_head(x, "v", 0, h), vec)
            assert_close(f"C4 Q=0 O h{h}", o[0, :, h].cpu().numpy(), O)
            assert_lse(lse[0, h].cpu().numpy(), L)
            assert_close(f"C4 Q=0 dV h{h}", dv[0, :, h].cpu().numpy(), fo.dv_q_zero(_head(x, "do", 0, h), vec))
        del x, xz, o, lse, dq, dk, dv
        torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg,fams", [("C5:131072:64", ("causal_document", "share_question")),
                                      ("C5:32768:128", ("random_eviction", "qk_sparse"))])
def test_c5_sampled_rows_and_q_zero(fm, cfg, fams):
    """C5 kernel-sweep shapes the bench does not default to: d=64 at N=128K and the PARTIAL-heavy
    families at N=32K — sampled rows (O, lse, dQ) of one head and the Q=0 closed forms (O, lse,
    dV) of two heads, batch entry 0."""
    calls, _, _ = bench.build_workload(cfg, 0, 1, bench.rho_oracle)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(2)
    for c in calls:
        if c["family"] not in fams:
            continue
        c = dict(c, B=1, masks=c["masks"][:1], batch_ids=c["batch_ids"][:1], heads=range(4))
        x = bench.make_inputs(c, dev)
        o, lse, dq, dk, dv = _run(fm, c, x, torch.float32)
        N = c["N"]
        m = c["masks"][0]
        vec = fo.expand(m.sri, m.causal, N)
        rows = np.sort(rng.choice(N, 48, replace=False))
        q, k, v, do = (_head(x, n, 0, 1) for n in ("q", "k", "v", "do"))
        O, L = fo.forward(q, k, v, vec, rows=rows, row_block=16)
        gq, _, _ = fo.backward_rows(q, k, v, do, vec, rows)
        assert_close(f"{cfg} {m.family} O rows", o[0, rows, 1].cpu().numpy(), O)
        assert_lse(lse[0, 1, rows].cpu().numpy(), L)
        assert_close(f"{cfg} {m.family} dQ rows", dq[0, rows, 1].cpu().numpy(), gq)
        xz = dict(x)
        xz["q"] = torch.zeros_like(x["q"])
        o, lse, dq, dk, dv = _run(fm, c, xz, torch.float32)
        for h in (0, 3):
            O, L = fo.forward_q_zero(_head(x, "v", 0, h), vec)
            assert_close(f"{cfg} Q=0 O h{h}", o[0, :, h].cpu().numpy(), O)
            assert_lse(lse[0, h].cpu().numpy(), L)
            assert_close(f"{cfg} Q=0 dV h{h}", dv[0, :, h].cpu().numpy(), fo.dv_q_zero(_head(x, "do", 0, h), vec))
        del x, xz, o, lse, dq, dk, dv
        torch.cuda.empty_cache()


def test_c3_generic_q_dk_dv_sampled_columns(fm):
    """Generic-Q dK / dV at N = 32K in the C3 bench layout: dK_j, dV_j accumulate in
    fp32 TMEM over up to 512 visited 64-row tiles, a length the small parity cases never reach.
    64 sampled key columns of one head in the lowest- and highest-sparsity batch entries against
    oracle.backward_cols (full forward over all rows, then the columns' gradients)."""
    calls, _, _ = bench.build_workload("C3", 0, 1, bench.rho_oracle)
    c = calls[0]
    x = bench.make_inputs(c, torch.device("cuda", 0))
    o, lse, dq, dk, dv = _run(fm, c, x, torch.float32)
    N = c["N"]
    rng = np.random.default_rng(5)
    for b, h in ((0, 7), (3, 30)):
        m = c["masks"][b]
        vec = fo.expand(m.sri, m.causal, N)
        keys = np.sort(rng.choice(N, 64, replace=False))
        q, k, v, do = (_head(x, n, b, h) for n in ("q", "k", "v", "do"))
        gk, gv = fo.backward_cols(q, k, v, do, vec, keys)
        assert_close(f"C3 b{b} h{h} dK cols", dk[b, keys, h].cpu().numpy(), gk)
        assert_close(f"C3 b{b} h{h} dV cols", dv[b, keys, h].cpu().numpy(), gv)


@pytest.mark.parametrize("N,d,fam", [(262144, 128, "causal_document"), (262144 - 37, 64, "share_question"),
                                     (262144 - 100, 128, "global_sliding_window")])
def test_max_seqlen_sampled_rows_and_q_zero(fm, N, d, fam):
    """The largest supported sequence (2048 column tiles: the forward visit list and the backward
    row-tile list at capacity, include/flashmask.h), exact and ragged: sampled rows (O, lse, dQ) of
    one head against the oracle and the Q = 0 closed forms (O, lse, dV) of both heads."""
    from workloads import masks as wm
    from workloads import tensors as wt
    rng = np.random.default_rng(N + d)
    m = wm.sample_family(fam, N, rng, (5, 9))
    x = {k: t.cuda().to(torch.bfloat16) for k, t in wt.make_qkv(1, N, 2, d, base=11).items()}
    x["sri"] = torch.from_numpy(wm.stack([m])).cuda()
    c = {"causal": m.causal}
    o, lse, dq, dk, dv = _run(fm, c, x, torch.float32)
    vec = fo.expand(m.sri, m.causal, N)
    rows = np.sort(np.concatenate([rng.choice(N, 30, replace=False), [0, N - 1]]))
    q, k, v, do = (_head(x, n, 0, 1) for n in ("q", "k", "v", "do"))
    O, L = fo.forward(q, k, v, vec, rows=rows, row_block=16)
    gq, _, _ = fo.backward_rows(q, k, v, do, vec, rows)
    assert_close(f"N{N} {fam} O rows", o[0, rows, 1].cpu().numpy(), O)
    assert_lse(lse[0, 1, rows].cpu().numpy(), L)
    assert_close(f"N{N} {fam} dQ rows", dq[0, rows, 1].cpu().numpy(), gq)
    del o, lse, dq, dk, dv
    xz = dict(x)
    xz["q"] = torch.zeros_like(x["q"])
    o, lse, dq, dk, dv = _run(fm, c, xz, torch.float32)
    for h in (0, 1):
        O, L = fo.forward_q_zero(_head(x, "v", 0, h), vec)
        assert_close(f"N{N} Q=0 O h{h}", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        assert_close(f"N{N} Q=0 dV h{h}", dv[0, :, h].cpu().numpy(), fo.dv_q_zero(_head(x, "do", 0, h), vec))
