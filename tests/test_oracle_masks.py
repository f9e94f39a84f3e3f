"""Pins for the mask inputs and the oracle's mask semantics (CPU only).

* Builders vs independent dense predicates, cell for cell (SURVEY c.3b).
* The §4.1 worked example — tests/golden/paper_p127_example.txt.
* SPEC worked examples.
* from_dense round trip and representability.
"""
import os

import numpy as np
import pytest

from oracle import dense_predicates as dp
from oracle import flashmask_oracle as fo
from workloads import masks as wm


def dense_of(m: wm.MaskInput):
    return fo.to_dense(fo.expand(m.sri, m.causal, m.N))


def _rand_lens(rng, N, n):
    return wm.sample_doc_lens(N, n, rng, min_len=1)


@pytest.mark.parametrize("seed", range(40))
def test_builders_match_dense_predicates(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 48))
    n = int(rng.integers(1, 6))
    lens = _rand_lens(rng, N, n)
    w = int(rng.integers(1, N + 1))
    g = int(rng.integers(0, N + 1))
    p = int(rng.integers(0, N + 1))
    cases = [
        (wm.full(N), dp.full(N)),
        (wm.causal(N), dp.causal(N)),
        (wm.sliding_window(N, w), dp.sliding_window(N, w)),
        (wm.causal_document(lens), dp.causal_document(lens)),
        (wm.document(lens), dp.document(lens)),
        (wm.global_sliding_window(N, g, w), dp.global_sliding_window(N, g, w)),
        (wm.causal_blockwise(lens), dp.causal_blockwise(lens)),
        (wm.prefix_lm_causal(N, p), dp.prefix_lm_causal(N, p)),
    ]
    pdocs = [(l, int(rng.integers(0, l + 1))) for l in lens]
    cases.append((wm.prefix_lm_document(pdocs), dp.prefix_lm_document(pdocs)))
    sq = []
    for l in lens:
        k = int(rng.integers(0, 4))
        ans = [1] * min(k, l - 1)
        for _ in range(l - 1 - len(ans)):
            if ans and rng.random() < 0.5:
                ans[int(rng.integers(0, len(ans)))] += 1
        sq.append((l - sum(ans), ans))
    cases.append((wm.share_question(sq), dp.share_question(sq)))
    kd = rng.choice(N, size=int(rng.integers(0, N + 1)), replace=False)
    a = int(rng.integers(0, N + 1))
    b = int(rng.integers(a, N + 1))
    cases.append((wm.qk_sparse(N, kd, (a, b)), dp.qk_sparse(N, kd, (a, b))))
    buckets = np.repeat(np.arange(len(lens)) * 7 % 5, lens)
    try:
        hs = wm.hash_sparse(buckets)
        cases.append((hs, dp.hash_sparse(buckets)))
    except ValueError:
        pass
    span = int(rng.integers(1, N + 1))
    re = wm.random_eviction(N, span, np.random.default_rng(seed + 1000))
    starts = [int(s) if s < N else None for s in re.sri[:, 0]]
    cases.append((re, dp.random_eviction(N, starts, span)))
    for built, ref in cases:
        got = dense_of(built)
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), (built.family, built.params, np.argwhere(got != ref)[:5])


def test_paper_p127_worked_example(golden_dir):
    kv = {}
    for line in open(os.path.join(golden_dir, "paper_p127_example.txt")):
        if line.startswith("#") or not line.strip():
            continue
        key, *vals = line.split()
        kv[key] = [int(x) for x in vals]
    N, y = kv["N"][0], kv["column"][0]
    m = wm.global_sliding_window(N, 2, 3)
    v = fo.expand(m.sri, m.causal, N)
    assert (v.lts[y], v.lte[y], v.uts[y], v.ute[y]) == (kv["LTS"][0], kv["LTE"][0], kv["UTS"][0], kv["UTE"][0])
    assert list(np.nonzero(fo.to_dense(v)[:, y])[0]) == kv["masked_rows"]


def test_spec_builder_examples():
    # S:101 CausalDocument([3,4,3]) -> lts
    m = wm.causal_document([3, 4, 3])
    assert list(m.sri[:, 0]) == [3, 3, 3, 7, 7, 7, 7, 10, 10, 10]
    # S:102 SlidingWindow(2), N=5 -> lts[j] = min(j+2, 5)
    assert list(wm.sliding_window(5, 2).sri[:, 0]) == [2, 3, 4, 5, 5]
    # S:103 Document([2,2]) -> j<2: lts=2, upper empty; j>=2: lts=4 (empty), ute=2
    v = fo.expand(wm.document([2, 2]).sri, False, 4)
    assert list(v.lts) == [2, 2, 4, 4] and list(v.lte) == [4, 4, 4, 4]
    assert list(v.uts) == [0, 0, 0, 0] and list(v.ute) == [0, 0, 2, 2]
    # S:104 ShareQuestion(q=2, answers=[2,2]) -> answer-1 columns lts=4, lte=6
    v = fo.expand(wm.share_question([(2, [2, 2])]).sri, True, 6)
    assert list(v.lts[2:4]) == [4, 4] and list(v.lte[2:4]) == [6, 6]
    # S:446 DPO q=600, answers [200,200] -> answer-1 lts=800
    v = wm.share_question([(600, [200, 200])]).sri[:, 0]
    assert v[600] == 800 and v[799] == 800 and v[800] == 1000 and v[0] == 1000


def test_spec_to_dense_example():
    # S:79 N=6 causal document [3,3]: masked iff i<j or (j<3 and i>=3)
    d = dense_of(wm.causal_document([3, 3]))
    i, j = np.meshgrid(np.arange(6), np.arange(6), indexing="ij")
    assert np.array_equal(d, (i < j) | ((j < 3) & (i >= 3)))


@pytest.mark.parametrize("seed", range(15))
def test_from_dense_round_trip(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 40))
    lens = _rand_lens(rng, N, int(rng.integers(1, 5)))
    for m in [wm.causal_document(lens), wm.sliding_window(N, int(rng.integers(1, N + 1))),
              wm.document(lens), wm.global_sliding_window(N, int(rng.integers(0, N)), 3)]:
        d = dense_of(m)
        sri = fo.from_dense(d, m.causal)
        v2 = fo.expand(sri, m.causal, N)
        assert np.array_equal(fo.to_dense(v2), d)


def test_from_dense_rejects_gaps():
    d = np.zeros((4, 4), dtype=bool)
    d[1, 0] = d[3, 0] = True   # S:90 column 0 masked rows {1,3}
    with pytest.raises(ValueError):
        fo.from_dense(d, causal=False)
    # S:91 QK-sparse kept_q={0,2,3}, kept_k={0,1,3} at N=4 causal is representable
    i, j = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    kept_q = np.isin(np.arange(4), [0, 2, 3])
    kept_k = np.isin(np.arange(4), [0, 1, 3])
    dense = (i < j) | ~kept_q[:, None] | ~kept_k[None, :]
    sri = fo.from_dense(dense, causal=True)
    assert np.array_equal(fo.to_dense(fo.expand(sri, True, 4)), dense)


def test_samplers_sum_and_bounds():
    rng = np.random.default_rng(0)
    for N in (128, 8192, 32768):
        for n in (1, 3, 7, 15):
            lens = wm.sample_doc_lens(N, n, rng, min_len=128 if N >= 128 * n else 1)
            assert sum(lens) == N
    # A.2.1: answers within [0.1L/(1+0.1k), 0.2L/(1+0.2k)]; SPEC S:435 example
    L, k = 1000, 2
    for _ in range(50):
        a = wm.sample_answer_lens(L, k, rng)
        assert all(int(np.ceil(100 / 1.2)) <= x <= int(np.floor(200 / 1.4)) for x in a)
