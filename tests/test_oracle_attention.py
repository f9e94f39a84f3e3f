"""Pins for the oracle's attention forward/backward (CPU only).

Each pin is fixed by something other than the oracle itself:
* hand-evaluated worked examples;
* textbook / library reductions: full and causal masks equal torch fp64
  scaled_dot_product_attention; document / causal-document equal per-document SDPA;
  gradients equal torch autograd of fp64 SDPA (full, causal);
* closed forms: Q = 0 gives S = 0 on visible cells, so L_r = ln(count_r),
  O_r = mean of visible V rows, dV_y = sum over rows r that see y of dO_r / count_r;
* invariants: visible rows of P sum to 1, empty rows are 0; dO = 0 => zero grads;
* central finite differences in fp64 (h=1e-6, rel <= 1e-6).
"""
import math

import numpy as np
import pytest
import torch

from oracle import flashmask_oracle as fo
from workloads import masks as wm


def vec(m):
    return fo.expand(m.sri, m.causal, m.N)


def rnd(rng, *shape):
    return rng.standard_normal(shape)


def test_spec_forward_examples():
    # S:249 N=1, d=2, q=k=v=[1,0] -> O=[1,0], L = 1/sqrt(2)
    x = np.array([[1.0, 0.0]])
    O, L = fo.forward(x, x, x, vec(wm.full(1)))
    assert np.allclose(O, [[1, 0]]) and L[0] == pytest.approx(1 / math.sqrt(2), abs=1e-15)
    # S:250 N=2 causal, q=k=v=I, scale=1 -> O[1] = [1/(1+e), e/(1+e)]
    I = np.eye(2)
    O, L = fo.forward(I, I, I, vec(wm.causal(2)), scale=1.0)
    e = math.e
    assert np.allclose(O, [[1, 0], [1 / (1 + e), e / (1 + e)]], atol=1e-15)
    # S:272 1x1, scale 2, q=k=3, v=5 -> O=5, L=18
    O, L = fo.forward(np.array([[3.0]]), np.array([[3.0]]), np.array([[5.0]]), vec(wm.full(1)), scale=2.0)
    assert O[0, 0] == 5.0 and L[0] == 18.0
    # S:271 all masked 2x2 -> O=0, L=-inf (R7)
    sri = np.array([[0, 2], [0, 2]], dtype=np.int32)    # causal C=2: LTS=0, LTE=2
    v = fo.expand(sri, True, 2)
    O, L = fo.forward(rnd(np.random.default_rng(0), 2, 3), rnd(np.random.default_rng(1), 2, 3),
                      rnd(np.random.default_rng(2), 2, 3), v)
    assert (O == 0).all() and np.isneginf(L).all()


def test_spec_backward_example():
    # S:261 N=2 causal, q=k=v=I, scale 1, dO=I: dV = P^T dO with P=[[1,0],[1/(1+e), e/(1+e)]]
    I = np.eye(2)
    e = math.e
    P = np.array([[1, 0], [1 / (1 + e), e / (1 + e)]])
    dq, dk, dv = fo.backward(I, I, I, I, vec(wm.causal(2)), scale=1.0)
    assert np.allclose(dv, P.T @ I, atol=1e-15)
    # dO = 0 -> zero gradients
    rng = np.random.default_rng(3)
    q, k, v_ = rnd(rng, 8, 4), rnd(rng, 8, 4), rnd(rng, 8, 4)
    g = fo.backward(q, k, v_, np.zeros((8, 4)), vec(wm.causal_document([3, 5])))
    assert all((x == 0).all() for x in g)


def _sdpa(q, k, v, causal_):
    t = lambda a: torch.tensor(a, dtype=torch.float64)[None, None]
    return torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v), is_causal=causal_)[0, 0].numpy()


@pytest.mark.parametrize("N,d", [(1, 4), (17, 8), (64, 16), (130, 32)])
def test_forward_full_and_causal_equal_sdpa(N, d):
    rng = np.random.default_rng(N)
    q, k, v_ = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    O, _ = fo.forward(q, k, v_, vec(wm.full(N)))
    assert np.abs(O - _sdpa(q, k, v_, False)).max() < 1e-12
    O, _ = fo.forward(q, k, v_, vec(wm.causal(N)), row_block=7)
    assert np.abs(O - _sdpa(q, k, v_, True)).max() < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_forward_document_masks_equal_per_document_sdpa(seed):
    rng = np.random.default_rng(seed)
    lens = wm.sample_doc_lens(96, 4, rng)
    N, d = 96, 8
    q, k, v_ = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    for builder, is_causal in ((wm.document, False), (wm.causal_document, True)):
        O, L = fo.forward(q, k, v_, vec(builder(lens)))
        s = 0
        for l in lens:
            ref = _sdpa(q[s:s + l], k[s:s + l], v_[s:s + l], is_causal)
            assert np.abs(O[s:s + l] - ref).max() < 1e-12
            s += l


@pytest.mark.parametrize("fam", wm.FAMILIES)
def test_probability_rows_sum_to_one(fam):
    rng = np.random.default_rng(5)
    m = wm.sample_family(fam, 80, rng, (2, 4))
    v = vec(m)
    q, k = rnd(rng, 80, 8), rnd(rng, 80, 8)
    P = fo.probabilities(q, k, v)
    M = fo.to_dense(v)
    live = ~M.all(axis=1)
    assert np.allclose(P[live].sum(axis=1), 1.0, atol=1e-12)
    assert (P[~live] == 0).all()
    assert (P[M] == 0).all()


def _visible_counts(v):
    return (~fo.to_dense(v)).sum(axis=1)


@pytest.mark.parametrize("fam", ["causal_document", "share_question", "global_sliding_window", "qk_sparse",
                                 "prefix_lm_document", "random_eviction"])
def test_q_zero_closed_forms(fam):
    rng = np.random.default_rng(11)
    m = wm.sample_family(fam, 120, rng, (2, 5))
    v = vec(m)
    N, d = m.N, 6
    q = np.zeros((N, d))
    k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    O, L = fo.forward(q, k, v_, v)
    vis = ~fo.to_dense(v)
    cnt = vis.sum(axis=1)
    for r in range(N):
        if cnt[r] == 0:
            assert np.isneginf(L[r]) and (O[r] == 0).all()
        else:
            assert L[r] == pytest.approx(math.log(cnt[r]), abs=1e-12)
            assert np.allclose(O[r], v_[vis[r]].mean(axis=0), atol=1e-12)
    _, _, dv = fo.backward(q, k, v_, do, v)
    w = np.where(cnt > 0, 1.0 / np.maximum(cnt, 1), 0.0)
    ref = vis.T.astype(float) @ (do * w[:, None])
    assert np.abs(dv - ref).max() < 1e-12


@pytest.mark.parametrize("N,d,causal_", [(5, 3, False), (9, 4, True), (24, 8, True)])
def test_backward_equals_torch_autograd(N, d, causal_):
    rng = np.random.default_rng(N * 10 + d)
    q, k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    tq, tk, tv = (torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in (q, k, v_))
    out = torch.nn.functional.scaled_dot_product_attention(tq[None, None], tk[None, None], tv[None, None],
                                                           is_causal=causal_)[0, 0]
    out.backward(torch.tensor(do))
    m = wm.causal(N) if causal_ else wm.full(N)
    dq, dk, dv = fo.backward(q, k, v_, do, vec(m), row_block=4)
    for a, t in ((dq, tq), (dk, tk), (dv, tv)):
        assert np.abs(a - t.grad.numpy()).max() < 1e-12


def _loss(q, k, v_, do, vv, scale):
    O, _ = fo.forward(q, k, v_, vv, scale)
    return float((O * do).sum())


@pytest.mark.parametrize("fam,N,d", [("share_question", 48, 4), ("document", 16, 4), ("global_sliding_window", 20, 3),
                                     ("random_eviction", 24, 4), ("causal_blockwise", 30, 4)])
def test_backward_finite_differences(fam, N, d):
    rng = np.random.default_rng(1 + N)
    m = wm.sample_family(fam, N, rng, (2, 4))
    vv = vec(m)
    N = m.N
    q, k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    scale = 0.7
    grads = fo.backward(q, k, v_, do, vv, scale)
    h = 1e-6
    for which, g in enumerate(grads):
        for _ in range(7):
            i, c = int(rng.integers(0, N)), int(rng.integers(0, d))
            args = [q.copy(), k.copy(), v_.copy()]
            args[which][i, c] += h
            lp = _loss(*args, do, vv, scale)
            args[which][i, c] -= 2 * h
            lm = _loss(*args, do, vv, scale)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[i, c]) <= 1e-6 * max(1.0, abs(g[i, c])), (which, i, c, fd, g[i, c])


def test_masked_key_null_influence():
    """perturbing K/V of a key masked for every row changes nothing."""
    rng = np.random.default_rng(9)
    m = wm.qk_sparse(40, [5, 17], (30, 33))
    vv = vec(m)
    q, k, v_, do = (rnd(rng, 40, 4) for _ in range(4))
    O1, L1 = fo.forward(q, k, v_, vv)
    g1 = fo.backward(q, k, v_, do, vv)
    k2, v2 = k.copy(), v_.copy()
    k2[5] += 3.0
    v2[17] -= 2.0
    O2, L2 = fo.forward(q, k2, v2, vv)
    g2 = fo.backward(q, k2, v2, do, vv)
    assert np.array_equal(O1, O2) and np.array_equal(L1, L2)
    assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[2][np.r_[0:5, 6:17, 18:40]], g2[2][np.r_[0:5, 6:17, 18:40]])
    # dropped query rows [30,33) see nothing: O=0, L=-inf
    assert (O1[30:33] == 0).all() and np.isneginf(L1[30:33]).all()


def test_row_subset_matches_full():
    rng = np.random.default_rng(2)
    m = wm.sample_family("causal_document", 200, rng)
    vv = vec(m)
    q, k, v_ = (rnd(rng, 200, 8) for _ in range(3))
    O, L = fo.forward(q, k, v_, vv)
    rows = np.array([0, 7, 199, 100])
    Os, Ls = fo.forward(q, k, v_, vv, rows=rows)
    assert np.array_equal(Os, O[rows]) and np.array_equal(Ls, L[rows])


def test_backward_rows_partition_sums_to_backward():
    rng = np.random.default_rng(21)
    m = wm.sample_family("document", 90, rng)
    vv = vec(m)
    q, k, v_, do = (rnd(rng, 90, 5) for _ in range(4))
    dq, dk, dv = fo.backward(q, k, v_, do, vv)
    acc_k, acc_v = np.zeros_like(dk), np.zeros_like(dv)
    for s in (range(0, 40), range(40, 90)):
        gq, gk, gv = fo.backward_rows(q, k, v_, do, vv, np.array(list(s)))
        assert np.abs(gq - dq[list(s)]).max() < 1e-13
        acc_k += gk
        acc_v += gv
    assert np.abs(acc_k - dk).max() < 1e-12 and np.abs(acc_v - dv).max() < 1e-12


@pytest.mark.parametrize("fam", wm.FAMILIES)
def test_q_zero_linear_forms_match_dense(fam):
    """The O(N) Q=0 forms used for full-size GPU checks equal the dense oracle."""
    rng = np.random.default_rng(31)
    m = wm.sample_family(fam, 150, rng, (2, 5))
    vv = vec(m)
    N, d = m.N, 5
    q = np.zeros((N, d))
    k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    assert np.array_equal(fo.visible_counts(vv), (~fo.to_dense(vv)).sum(axis=1))
    O, L = fo.forward(q, k, v_, vv)
    O2, L2 = fo.forward_q_zero(v_, vv)
    assert np.abs(O - O2).max() < 1e-12 and np.array_equal(np.isneginf(L), np.isneginf(L2))
    fin = np.isfinite(L)
    assert np.abs(L[fin] - L2[fin]).max() < 1e-12
    _, _, dv = fo.backward(q, k, v_, do, vv)
    assert np.abs(dv - fo.dv_q_zero(do, vv)).max() < 1e-12


@pytest.mark.parametrize("N,d,causal_", [(7, 3, False), (33, 8, True)])
def test_backward_cols_equals_torch_autograd(N, d, causal_):
    """backward_cols (dK, dV of chosen key columns) equals torch autograd of fp64 SDPA."""
    rng = np.random.default_rng(N + 77)
    q, k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    tq, tk, tv = (torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in (q, k, v_))
    out = torch.nn.functional.scaled_dot_product_attention(tq[None, None], tk[None, None], tv[None, None],
                                                           is_causal=causal_)[0, 0]
    out.backward(torch.tensor(do))
    keys = np.array([0, N // 2, N - 1])
    m = wm.causal(N) if causal_ else wm.full(N)
    dk, dv = fo.backward_cols(q, k, v_, do, vec(m), keys, row_block=5)
    assert np.abs(dk - tk.grad.numpy()[keys]).max() < 1e-12
    assert np.abs(dv - tv.grad.numpy()[keys]).max() < 1e-12


@pytest.mark.parametrize("fam,N,d", [("share_question", 40, 4), ("global_sliding_window", 24, 3),
                                     ("qk_sparse", 36, 4), ("random_eviction", 30, 4)])
def test_backward_cols_finite_differences(fam, N, d):
    """backward_cols against central differences of the forward loss, including keys
    masked for every row (zero gradient) and rows masked in every column."""
    rng = np.random.default_rng(5 + N)
    m = wm.sample_family(fam, N, rng, (2, 4))
    vv = vec(m)
    N = m.N
    q, k, v_, do = rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d), rnd(rng, N, d)
    scale = 0.6
    keys = np.unique(rng.integers(0, N, 6))
    dk, dv = fo.backward_cols(q, k, v_, do, vv, keys, scale, row_block=7)
    h = 1e-6
    for which, g in ((1, dk), (2, dv)):
        for ki, y in enumerate(keys):
            for c in range(d):
                args = [q.copy(), k.copy(), v_.copy()]
                args[which][y, c] += h
                lp = _loss(*args, do, vv, scale)
                args[which][y, c] -= 2 * h
                lm = _loss(*args, do, vv, scale)
                fd = (lp - lm) / (2 * h)
                assert abs(fd - g[ki, c]) <= 1e-6 * max(1.0, abs(g[ki, c])), (which, y, c, fd, g[ki, c])


@pytest.mark.parametrize("fam", ["causal_document", "document", "prefix_lm_causal", "hash_sparse"])
def test_backward_cols_matches_backward(fam):
    rng = np.random.default_rng(41)
    m = wm.sample_family(fam, 130, rng, (2, 5))
    vv = vec(m)
    N, d = m.N, 6
    q, k, v_, do = (rnd(rng, N, d) for _ in range(4))
    _, dk, dv = fo.backward(q, k, v_, do, vv)
    keys = np.arange(0, N, 3)
    gk, gv = fo.backward_cols(q, k, v_, do, vv, keys, row_block=32)
    assert np.abs(gk - dk[keys]).max() < 1e-12 and np.abs(gv - dv[keys]).max() < 1e-12
