"""Pins for the oracle's row-wise representation (R32) — CPU only.

* Row-wise builders vs the independent dense predicates of each Figure-1 family, cell for cell,
  and vs the column-wise builders of the same family (two representations, one mask).
* from_dense_rowwise round trip; non-representable rows raise.
* classify_rowwise: brute-force soundness on random (incl. invalid) int32 vectors and ragged
  tiles; the transpose duality with the column-wise classifier ("by transposing the
  attention matrix"); closed forms (causal, full, tile-aligned documents).
"""
import numpy as np
import pytest

from oracle import dense_predicates as dp
from oracle import flashmask_oracle as fo
from workloads import masks as wm


def rdense(m: wm.MaskInput):
    assert m.rowwise
    return fo.to_dense(fo.expand_rowwise(m.sri, m.causal, m.N))


def cdense(m: wm.MaskInput):
    return fo.to_dense(fo.expand(m.sri, m.causal, m.N))


@pytest.mark.parametrize("seed", range(40))
def test_rowwise_builders_match_dense_predicates(seed):
    rng = np.random.default_rng(500 + seed)
    N = int(rng.integers(1, 48))
    lens = wm.sample_doc_lens(N, int(rng.integers(1, 6)), rng, min_len=1)
    w = int(rng.integers(1, N + 1))
    g = int(rng.integers(0, N + 1))
    p = int(rng.integers(0, N + 1))
    pdocs = [(l, int(rng.integers(0, l + 1))) for l in lens]
    cases = [
        (wm.rw_full(N), dp.full(N), wm.full(N)),
        (wm.rw_causal(N), dp.causal(N), wm.causal(N)),
        (wm.rw_sliding_window(N, w), dp.sliding_window(N, w), wm.sliding_window(N, w)),
        (wm.rw_causal_document(lens), dp.causal_document(lens), wm.causal_document(lens)),
        (wm.rw_document(lens), dp.document(lens), wm.document(lens)),
        (wm.rw_global_sliding_window(N, g, w), dp.global_sliding_window(N, g, w), wm.global_sliding_window(N, g, w)),
        (wm.rw_causal_blockwise(lens), dp.causal_blockwise(lens), wm.causal_blockwise(lens)),
        (wm.rw_prefix_lm_document(pdocs), dp.prefix_lm_document(pdocs), wm.prefix_lm_document(pdocs)),
        (wm.rw_prefix_lm_causal(N, p), dp.prefix_lm_causal(N, p), wm.prefix_lm_causal(N, p)),
    ]
    for rw, dense, cw in cases:
        assert np.array_equal(rdense(rw), dense), rw.family
        assert np.array_equal(cdense(cw), dense), cw.family   # the same mask column-wise
    kw = wm.rw_key_window(N, rng, max(1, N // 3))
    assert np.array_equal(rdense(kw), dp.key_window(kw.sri[:, 0], kw.sri[:, 1]))


def test_rowwise_c_table_defaults():
    """Each (causal, C) layout's implicit ends (R32): causal C=1 -> LTS = 0; non-causal C=2 ->
    LTS = 0, UTE = N; causal upper vectors empty."""
    N = 6
    v = fo.expand_rowwise(np.array([[2]] * N), True, N)
    assert (v.lts == 0).all() and (v.lte == 2).all() and (v.uts == v.ute).all() and v.rowwise
    v = fo.expand_rowwise(np.array([[1, 4]] * N), False, N)
    assert (v.lts == 0).all() and (v.lte == 1).all() and (v.uts == 4).all() and (v.ute == N).all()
    # row 3 of a causal C=2 mask [1, 3): keys 1, 2 masked, keys 4, 5 (y > r) masked by causality
    v = fo.expand_rowwise(np.array([[1, 3]] * N), True, N)
    assert fo.to_dense(v)[3].tolist() == [False, True, True, False, True, True]


@pytest.mark.parametrize("seed", range(20))
def test_from_dense_rowwise_round_trip(seed):
    rng = np.random.default_rng(900 + seed)
    N = int(rng.integers(1, 40))
    for causal in (True, False):
        # (rw_key_window is two key intervals that need not split at the diagonal: representable
        # by the vectors, not by the one-interval-per-triangle decomposition of from_dense)
        fam = rng.choice(["causal_document", "global_sliding_window", "prefix_lm_document"] if not causal else
                         ["causal_document", "sliding_window", "causal_blockwise"])
        if causal:
            m = wm.rw_sample_family(str(fam), N, rng, (1, 4))
            if not m.causal:
                continue
        else:
            m = wm.rw_sample_family("document" if fam == "causal_document" else str(fam), N, rng, (1, 4))
            if m.causal:
                continue
        dense = rdense(m)
        sri = fo.from_dense_rowwise(dense, m.causal)
        assert np.array_equal(fo.to_dense(fo.expand_rowwise(sri, m.causal, N)), dense)


def test_from_dense_rowwise_rejects_non_contiguous():
    d = np.zeros((4, 4), dtype=bool)
    d[3, 0] = d[3, 2] = True                      # row 3: keys 0 and 2 masked, 1 visible
    with pytest.raises(ValueError):
        fo.from_dense_rowwise(d, False)
    with pytest.raises(ValueError):
        fo.from_dense_rowwise(np.zeros((3, 3), dtype=bool), True)   # causal must mask y > r


def _random_rowwise(rng, N, causal, C):
    lo, hi = -3, N + 3
    if rng.random() < 0.2:
        lo, hi = -2**31, 2**31 - 1
    sri = rng.integers(lo, hi, size=(N, C), endpoint=True).astype(np.int64)
    return fo.expand_rowwise(np.clip(sri, -2**31, 2**31 - 1), causal, N)


@pytest.mark.parametrize("seed", range(30))
def test_classify_rowwise_sound_bruteforce(seed):
    rng = np.random.default_rng(40 + seed)
    N = int(rng.integers(1, 70))
    causal, C = [(True, 1), (True, 2), (False, 2), (False, 4)][seed % 4]
    v = _random_rowwise(rng, N, causal, C)
    M = fo.to_dense(v)
    for Br, Bc in [(1, 1), (3, 5), (8, 8), (16, 4), (128, 128), (64, 128)]:
        cm, counts, _ = fo.classify_rowwise(v, Br, Bc)
        Tr, Tc = cm.shape
        for i in range(Tr):
            for j in range(Tc):
                blk = M[i * Br:min((i + 1) * Br, N), j * Bc:min((j + 1) * Bc, N)]
                if cm[i, j] == fo.SKIP:
                    assert blk.all(), (Br, Bc, i, j)
                elif cm[i, j] == fo.UNMASKED:
                    assert not blk.any(), (Br, Bc, i, j)
        assert counts.sum() == Tr * Tc


@pytest.mark.parametrize("seed", range(20))
def test_classify_rowwise_is_colwise_of_transpose(seed):
    """the row-wise representation of M is the column-wise representation of M^T (the
    lower / upper intervals trade triangles).  For bidirectional masks the row-wise classifier
    must equal the column-wise classifier run on the transposed problem, transposed back."""
    rng = np.random.default_rng(70 + seed)
    N = int(rng.integers(1, 90))
    v = _random_rowwise(rng, N, False, 4)
    vt = fo.Vectors(v.uts, v.ute, v.lts, v.lte, False, N)     # column-wise vectors of M^T
    assert np.array_equal(fo.to_dense(vt), fo.to_dense(v).T)
    for Br, Bc in [(4, 4), (3, 7), (128, 128), (64, 128)]:
        cm, counts, _ = fo.classify_rowwise(v, Br, Bc)
        cmt, countst, _ = fo.classify_colwise(vt, Bc, Br)
        assert np.array_equal(cm, cmt.T), (Br, Bc)
        assert np.array_equal(counts, countst)


def test_classify_rowwise_closed_forms():
    N = 1000
    cm, counts, _ = fo.classify_rowwise(fo.expand_rowwise(wm.rw_causal(N).sri, True, N), 128, 128)
    cmc, countsc, _ = fo.classify_colwise(fo.expand(wm.causal(N).sri, True, N), 128, 128)
    assert np.array_equal(cm, cmc) and np.array_equal(counts, countsc)   # only the causal triangle
    cm, counts, _ = fo.classify_rowwise(fo.expand_rowwise(wm.rw_full(N).sri, False, N), 128, 128)
    assert (cm == fo.UNMASKED).all()
    # tile-aligned documents of 256: 2x2 diagonal blocks UNMASKED, everything else SKIP
    m = wm.rw_document([256] * 4)
    cm, counts, _ = fo.classify_rowwise(fo.expand_rowwise(m.sri, False, m.N), 128, 128)
    want = np.kron(np.eye(4, dtype=np.uint8), np.ones((2, 2), dtype=np.uint8)) * fo.UNMASKED
    assert np.array_equal(cm, want)
    assert counts.tolist() == [64 - 16, 0, 16]


def test_rowwise_attention_matches_dense_definition():
    """forward/backward take row-wise vectors through the same dense mask: equal to the
    column-wise run of the same family (both represent one mask)."""
    rng = np.random.default_rng(3)
    lens = [40, 25, 31]
    rw, cw = wm.rw_document(lens), wm.document(lens)
    N, d = rw.N, 16
    q, k, v, do = (rng.standard_normal((N, d)) for _ in range(4))
    vr, vc = fo.expand_rowwise(rw.sri, False, N), fo.expand(cw.sri, False, N)
    Or, Lr = fo.forward(q, k, v, vr)
    Oc, Lc = fo.forward(q, k, v, vc)
    assert np.allclose(Or, Oc, atol=1e-12) and np.allclose(Lr, Lc, atol=1e-12)
    gr = fo.backward(q, k, v, do, vr)
    gc = fo.backward(q, k, v, do, vc)
    for a, b in zip(gr, gc):
        assert np.allclose(a, b, atol=1e-12)
