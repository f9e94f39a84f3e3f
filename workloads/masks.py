"""Seeded synthetic FlashMask inputs: the column-interval mask builders.

INPUT GENERATOR ONLY.  This module writes down, for each Figure-1 mask family,
the per-key-column row intervals in the ``startend_row_indices`` layout
(SURVEY.md §8(b) C-table).  It contains none of the method's arithmetic: no
expansion to LTS/LTE/UTS/UTE, no tile classification, no attention.  Both the
oracle tests and the CUDA path consume what it produces; neither imports the
other.

Layout of ``MaskInput.sri`` (int32 ``[N, C]``), column ``y`` = key token ``y``:

    causal  C   col0  col1  col2  col3   implicit
    1       1   LTS   -     -     -      LTE = N, upper = {r < y}
    1       2   LTS   LTE   -     -      upper = {r < y}
    0       2   LTS   UTE   -     -      LTE = N, UTS = 0
    0       4   LTS   LTE   UTS   UTE    -

Rows ``[LTS_y, LTE_y)`` and ``[UTS_y, UTE_y)`` are masked for key ``y``
(§4.1, Eq. 3); 0-based, half-open (DESIGN.md
reading R1).  The family list and the interval formulas follow SURVEY.md
§8(d) d.3 / §8(c) c.3b; each builder cites the passage of PAPER.md §2.1
 describing the family.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

INT32_MAX = np.iinfo(np.int32).max


@dataclass
class MaskInput:
    """One mask in the startend_row_indices layout (one batch entry, one mask head)."""

    N: int
    causal: bool
    C: int
    sri: np.ndarray  # int32 [N, C]
    family: str
    params: dict = field(default_factory=dict)
    rowwise: bool = False  # True: sri rows are query rows holding masked KEY intervals

    def __post_init__(self):
        self.sri = np.ascontiguousarray(self.sri, dtype=np.int32).reshape(self.N, self.C)
        assert (self.causal, self.C) in {(True, 1), (True, 2), (False, 2), (False, 4)}, (self.causal, self.C)


def _mk(N, causal, cols, family, **params):
    sri = np.stack([np.asarray(c, dtype=np.int64) for c in cols], axis=1)
    return MaskInput(N=N, causal=causal, C=len(cols), sri=sri.astype(np.int32), family=family, params=params)


def _doc_bounds(doc_lens: Sequence[int]):
    lens = np.asarray(doc_lens, dtype=np.int64)
    assert (lens > 0).all()
    ends = np.cumsum(lens)
    starts = ends - lens
    N = int(ends[-1])
    doc_of = np.repeat(np.arange(len(lens)), lens)
    return N, starts, ends, doc_of


# ---------------------------------------------------------------- families
def full(N: int) -> MaskInput:
    """No masking (bidirectional, every column empty): LTS=N, UTE=0."""
    return _mk(N, False, [np.full(N, N), np.zeros(N)], "full")


def causal(N: int) -> MaskInput:
    """Fig. 1(a)(1) causal: only the implicit r<y triangle; LTS=N (empty lower)."""
    return _mk(N, True, [np.full(N, N)], "causal")


def sliding_window(N: int, w: int) -> MaskInput:
    """Sliding window: key y visible to rows y..y+w-1; LTS=min(y+w,N)."""
    y = np.arange(N)
    return _mk(N, True, [np.minimum(y + w, N)], "sliding_window", w=w)


def causal_document(doc_lens: Sequence[int]) -> MaskInput:
    """Causal document: causal within a document; LTS = end of y's document."""
    N, starts, ends, doc_of = _doc_bounds(doc_lens)
    return _mk(N, True, [ends[doc_of]], "causal_document", doc_lens=list(map(int, doc_lens)))


def document(doc_lens: Sequence[int]) -> MaskInput:
    """Document (bidirectional within a document): LTS = doc end, UTE = doc start."""
    N, starts, ends, doc_of = _doc_bounds(doc_lens)
    return _mk(N, False, [ends[doc_of], starts[doc_of]], "document", doc_lens=list(map(int, doc_lens)))


def share_question(docs: Sequence[tuple[int, Sequence[int]]]) -> MaskInput:
    """Share question ('multiple answers share a single question').

    ``docs`` = [(question_len, [answer_len, ...]), ...].  Causal; a question
    column is masked from its document's end, an answer column from the end of
    its own answer (later answers never see earlier ones)."""
    lts = []
    for q, answers in docs:
        start = len(lts)
        doc_len = q + sum(answers)
        doc_end = start + doc_len
        lts += [doc_end] * q
        pos = start + q
        for a in answers:
            lts += [pos + a] * a
            pos += a
    N = len(lts)
    return _mk(N, True, [np.asarray(lts)], "share_question",
               docs=[(int(q), list(map(int, a))) for q, a in docs])


def global_sliding_window(N: int, g: int, w: int) -> MaskInput:
    """Global + sliding window: the first g tokens attend to / are attended by all;
    others see a window of w.  Bidirectional global rows (reading R19, pinned
    by the §4.1 example P:127): y<g empty; else LTS=min(y+w,N), LTE=N, UTS=g, UTE=y."""
    y = np.arange(N)
    glob = y < g
    lts = np.where(glob, N, np.minimum(y + w, N))
    lte = np.full(N, N)
    uts = np.where(glob, 0, g)
    ute = np.where(glob, 0, y)
    return _mk(N, False, [lts, lte, uts, ute], "global_sliding_window", g=g, w=w)


def causal_blockwise(block_lens: Sequence[int]) -> MaskInput:
    """Causal blockwise (in-context learning: the last block — the test example —
    attends to all demonstrations; demonstrations only to themselves).
    Non-last block: LTS=end(block), LTE=start(last); last block: empty."""
    N, starts, ends, blk = _doc_bounds(block_lens)
    last = len(block_lens) - 1
    lts = np.where(blk == last, N, ends[blk])
    lte = np.where(blk == last, N, starts[last])
    return _mk(N, True, [lts, lte], "causal_blockwise", block_lens=list(map(int, block_lens)))


def prefix_lm_document(docs: Sequence[tuple[int, int]]) -> MaskInput:
    """Prefix-LM document: per document a bidirectional prefix of length p_D, causal
    after it, no cross-document attention.  ``docs`` = [(len, prefix_len), ...].
    LTS = doc end; UTE = doc start inside the prefix, else y."""
    lens = [int(l) for l, _ in docs]
    N, starts, ends, doc_of = _doc_bounds(lens)
    pre = np.asarray([int(p) for _, p in docs])
    y = np.arange(N)
    in_prefix = (y - starts[doc_of]) < pre[doc_of]
    ute = np.where(in_prefix, starts[doc_of], y)
    return _mk(N, False, [ends[doc_of], ute], "prefix_lm_document", docs=[(l, int(p)) for l, (_, p) in zip(lens, docs)])


def prefix_lm_causal(N: int, p: int) -> MaskInput:
    """Prefix-LM causal / T5-style: bidirectional among the first p tokens,
    causal afterwards.  LTS=N; UTE = 0 for y<p else y."""
    y = np.arange(N)
    return _mk(N, False, [np.full(N, N), np.where(y < p, 0, y)], "prefix_lm_causal", p=p)


def qk_sparse(N: int, dropped_keys: Sequence[int], q_drop: tuple[int, int]) -> MaskInput:
    """QK-sparse (SCFA): causal, a set of dropped keys (whole column masked) and one
    dropped query range [a,b) (those rows see nothing).  DESIGN.md reading R23."""
    a, b = q_drop
    y = np.arange(N)
    drop = np.zeros(N, dtype=bool)
    drop[np.asarray(list(dropped_keys), dtype=np.int64)] = True
    lts_q = np.maximum(a, y)
    has_q = lts_q < b
    lts = np.where(drop, y, np.where(has_q, lts_q, N))
    lte = np.where(drop, N, np.where(has_q, b, N))
    return _mk(N, True, [lts, lte], "qk_sparse", dropped_keys=sorted(map(int, dropped_keys)), q_drop=(int(a), int(b)))


def hash_sparse(buckets: Sequence[int]) -> MaskInput:
    """Hash-sparse (SCFA): causal and r, y must share a hash bucket.  Only instances
    whose masked rows per column form one interval are representable; raises otherwise.
    LTS_y = first row r>y whose bucket differs (every later row is then masked)."""
    bk = np.asarray(buckets, dtype=np.int64)
    N = len(bk)
    lts = np.full(N, N)
    for y in range(N):
        diff = np.nonzero(bk[y:] != bk[y])[0]
        if len(diff):
            s = y + int(diff[0])
            if (bk[s:] == bk[y]).any():
                raise ValueError(f"hash_sparse: column {y} not representable (bucket reappears)")
            lts[y] = s
    return _mk(N, True, [lts, np.full(N, N)], "hash_sparse", buckets=list(map(int, bk)))


def random_eviction(N: int, span: int, rng: np.random.Generator) -> MaskInput:
    """Random eviction (KV-cache eviction): causal plus, per key y, one evicted row span
    [s_y, min(s_y+span,N)) with s_y ~ U{y+1..N-1}; the last key has none (R22)."""
    y = np.arange(N)
    lts = np.full(N, N, dtype=np.int64)
    lte = np.full(N, N, dtype=np.int64)
    for c in range(N - 1):
        s = int(rng.integers(c + 1, N))
        lts[c] = s
        lte[c] = min(s + span, N)
    return _mk(N, True, [lts, lte], "random_eviction", span=span)


def empty_rows_padding(doc_lens: Sequence[int], pad: int) -> MaskInput:
    """Causal document with a trailing padding block whose keys are masked for every row
    (SPEC S:465 convention lts[y]=y): padding rows then see nothing -> O=0, L=-inf."""
    base = causal_document(list(doc_lens) + [pad])
    N = base.N
    lts = base.sri[:, 0].astype(np.int64).copy()
    lts[N - pad:] = np.arange(N - pad, N)
    return _mk(N, True, [lts], "padding_empty_rows", doc_lens=list(doc_lens), pad=pad)


# ---------------------------------------------------------------- row-wise builders
# The row-wise representation (R32): row r of sri holds the masked KEY
# columns of query row r.  C-table (mirror of the column-wise one; an implicit end extends to the
# far edge of its triangle):
#
#     causal  C   col0  col1  col2  col3   implicit
#     1       1   LTE   -     -     -      LTS = 0, upper = {y > r}
#     1       2   LTS   LTE   -     -      upper = {y > r}
#     0       2   LTE   UTS   -     -      LTS = 0, UTE = N
#     0       4   LTS   LTE   UTS   UTE    -
def _mkr(N, causal, cols, family, **params):
    m = _mk(N, causal, cols, family, **params)
    m.rowwise = True
    return m


def rw_full(N: int) -> MaskInput:
    """No masking: LTE = 0, UTS = N (both key intervals empty)."""
    return _mkr(N, False, [np.zeros(N), np.full(N, N)], "rw_full")


def rw_causal(N: int) -> MaskInput:
    """Causal: only the implicit y > r triangle; LTE = 0."""
    return _mkr(N, True, [np.zeros(N)], "rw_causal")


def rw_sliding_window(N: int, w: int) -> MaskInput:
    """Sliding window: row r sees keys r-w+1..r; LTE = max(r-w+1, 0)."""
    r = np.arange(N)
    return _mkr(N, True, [np.maximum(r - w + 1, 0)], "rw_sliding_window", w=w)


def rw_causal_document(doc_lens: Sequence[int]) -> MaskInput:
    """Causal document: row r sees its document's keys up to r; LTE = document start."""
    N, starts, ends, doc_of = _doc_bounds(doc_lens)
    return _mkr(N, True, [starts[doc_of]], "rw_causal_document", doc_lens=list(map(int, doc_lens)))


def rw_document(doc_lens: Sequence[int]) -> MaskInput:
    """Document: row r sees its whole document; LTE = doc start, UTS = doc end."""
    N, starts, ends, doc_of = _doc_bounds(doc_lens)
    return _mkr(N, False, [starts[doc_of], ends[doc_of]], "rw_document", doc_lens=list(map(int, doc_lens)))


def rw_global_sliding_window(N: int, g: int, w: int) -> MaskInput:
    """Global + sliding window (reading R19 as in the column-wise builder): rows r < g see
    every key; a row r >= g sees the global keys y < g and the window y in (r-w, r].
    Masked keys of a row r >= g: [g, max(g, r-w+1)) and [r+1, N)."""
    r = np.arange(N)
    glob = r < g
    lts = np.where(glob, 0, g)
    lte = np.where(glob, 0, np.maximum(g, r - w + 1))
    uts = np.where(glob, N, r + 1)
    ute = np.full(N, N)
    return _mkr(N, False, [lts, lte, uts, ute], "rw_global_sliding_window", g=g, w=w)


def rw_causal_blockwise(block_lens: Sequence[int]) -> MaskInput:
    """Causal blockwise: a row of a demonstration block sees its own block causally; a
    row of the last block sees every earlier key.  LTE = block start (0 in the last block)."""
    N, starts, ends, blk = _doc_bounds(block_lens)
    last = len(block_lens) - 1
    return _mkr(N, True, [np.where(blk == last, 0, starts[blk])], "rw_causal_blockwise",
                block_lens=list(map(int, block_lens)))


def rw_prefix_lm_document(docs: Sequence[tuple[int, int]]) -> MaskInput:
    """Prefix-LM document: row r of document [s, e) with prefix p sees [s, max(s+p, r+1)).
    LTE = s, UTS = max(s + p, r + 1)."""
    lens = [int(l) for l, _ in docs]
    N, starts, ends, doc_of = _doc_bounds(lens)
    pre = np.asarray([int(p) for _, p in docs])
    r = np.arange(N)
    uts = np.maximum(starts[doc_of] + pre[doc_of], r + 1)
    return _mkr(N, False, [starts[doc_of], uts], "rw_prefix_lm_document",
                docs=[(l, int(p)) for l, (_, p) in zip(lens, docs)])


def rw_prefix_lm_causal(N: int, p: int) -> MaskInput:
    """Prefix-LM causal / T5: row r sees [0, max(p, r+1)).  LTE = 0, UTS = max(p, r+1)."""
    r = np.arange(N)
    return _mkr(N, False, [np.zeros(N), np.maximum(p, r + 1)], "rw_prefix_lm_causal", p=p)


def rw_key_window(N: int, rng: np.random.Generator, max_len: int) -> MaskInput:
    """A mask natural only in the row-wise form: every query row r attends to one random key
    window [a_r, b_r) (a per-query retrieval span; b_r - a_r <= max_len).  A column's visible
    rows are then an arbitrary set, so the column-wise form cannot represent it.
    Masked keys [0, a_r) and [b_r, N): LTE = a_r, UTS = b_r."""
    a = rng.integers(0, N, size=N)
    b = np.minimum(a + rng.integers(1, max(2, max_len + 1), size=N), N)
    return _mkr(N, False, [a, b], "rw_key_window", max_len=max_len)


def rw_sample_family(family: str, N: int, rng: np.random.Generator, doc_range=(3, 7)) -> MaskInput:
    """One row-wise instance of a Figure-1 family (those whose masked keys per row form one
    interval per triangle) at the kernel-sweep parameters, or of rw_key_window."""
    lo, hi = doc_range
    if family == "full":
        return rw_full(N)
    if family == "causal":
        return rw_causal(N)
    if family == "sliding_window":
        return rw_sliding_window(N, max(1, N // 16))
    if family == "causal_document":
        return rw_causal_document(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "document":
        return rw_document(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "global_sliding_window":
        return rw_global_sliding_window(N, max(1, N // 16), min(256, N))
    if family == "causal_blockwise":
        return rw_causal_blockwise(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "prefix_lm_document":
        lens = sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng)
        return rw_prefix_lm_document([(l, max(0, int(round(0.1 * l)))) for l in lens])
    if family == "prefix_lm_causal":
        return rw_prefix_lm_causal(N, N // 2)
    if family == "key_window":
        return rw_key_window(N, rng, max(1, N // 8))
    raise KeyError(family)


ROWWISE_FAMILIES = ["full", "causal", "sliding_window", "causal_document", "document", "global_sliding_window",
                    "causal_blockwise", "prefix_lm_document", "prefix_lm_causal", "key_window"]


# ------------------------------------------------------------- sampling
def sample_doc_lens(N: int, n_docs: int, rng: np.random.Generator, min_len: int = 1) -> list[int]:
    """Document lengths summing to N (App. A.5.2 P:588 'sampled the length of each document
    such that the total length equaled').  Normalised-uniform weights with a minimum length;
    the last document takes the remainder (reading R21)."""
    n_docs = max(1, min(n_docs, N // max(min_len, 1), N))
    min_len = max(1, min(min_len, N // n_docs))
    w = rng.uniform(0.0, 1.0, n_docs) + 1e-9
    spare = N - n_docs * min_len
    lens = np.floor(w / w.sum() * spare).astype(np.int64) + min_len
    lens[-1] += N - lens.sum()
    assert lens.sum() == N and (lens >= min_len).all()
    return [int(x) for x in lens]


def sample_answer_lens(L: int, k: int, rng: np.random.Generator) -> list[int]:
    """App. A.2.1: each answer length ~ U[0.1L/(1+0.1k), 0.2L/(1+0.2k)]."""
    lo = int(np.ceil(0.1 * L / (1 + 0.1 * k)))
    hi = int(np.floor(0.2 * L / (1 + 0.2 * k)))
    hi = max(hi, lo)
    return [max(1, int(rng.integers(lo, hi + 1))) for _ in range(k)]


def sample_share_question(N: int, n_docs: int, rng: np.random.Generator, k_range=(2, 6),
                          answer_frac=None, min_len: int = 8) -> MaskInput:
    """Share-question workload: documents split into 1 question + k answers.  By
    default answer lengths follow A.2.1; ``answer_frac=(lo,hi)`` draws each answer as
    that fraction of L instead (used to reach the tables' higher sparsity, SURVEY d.3 row 5)."""
    docs = []
    for L in sample_doc_lens(N, n_docs, rng, min_len=min_len):
        k = int(rng.integers(k_range[0], k_range[1] + 1))
        if answer_frac is None:
            ans = sample_answer_lens(L, k, rng)
        else:
            ans = [max(1, int(rng.uniform(*answer_frac) * L)) for _ in range(k)]
        while sum(ans) >= L and max(ans) > 1:
            i = int(np.argmax(ans))
            ans[i] -= 1
        if sum(ans) >= L:
            ans = ans[: max(0, L - 1)]
        docs.append((L - sum(ans), ans))
    return share_question(docs)


def sample_family(family: str, N: int, rng: np.random.Generator, doc_range=(3, 7)) -> MaskInput:
    """One instance of a Figure-1 family at the kernel-sweep parameters (SURVEY d.3)."""
    lo, hi = doc_range
    if family == "full":
        return full(N)
    if family == "causal":
        return causal(N)
    if family == "sliding_window":
        return sliding_window(N, max(1, N // 16))
    if family == "causal_document":
        return causal_document(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "document":
        return document(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "share_question":
        return sample_share_question(N, int(rng.integers(lo, hi + 1)), rng)
    if family == "global_sliding_window":
        return global_sliding_window(N, max(1, N // 16), min(256, N))
    if family == "causal_blockwise":
        return causal_blockwise(sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng))
    if family == "prefix_lm_document":
        lens = sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng)
        return prefix_lm_document([(l, max(0, int(round(0.1 * l)))) for l in lens])
    if family == "prefix_lm_causal":
        return prefix_lm_causal(N, N // 2)
    if family == "qk_sparse":
        nk = max(1, N // 64)
        keys = rng.choice(N, size=nk, replace=False)
        a = int(rng.integers(0, N))
        b = min(N, a + max(1, N // 64))
        return qk_sparse(N, keys, (a, b))
    if family == "hash_sparse":
        lens = sample_doc_lens(N, int(rng.integers(lo, hi + 1)), rng)
        return hash_sparse(np.repeat(np.arange(len(lens)), lens))
    if family == "random_eviction":
        return random_eviction(N, max(1, N // 16), rng)
    raise KeyError(family)


FAMILIES = ["full", "causal", "sliding_window", "causal_document", "document", "share_question",
            "global_sliding_window", "causal_blockwise", "prefix_lm_document", "prefix_lm_causal",
            "qk_sparse", "hash_sparse", "random_eviction"]


def stack(masks: Sequence[MaskInput], heads: int = 1) -> np.ndarray:
    """Batch masks into the ABI tensor ``[B, Hm, N, C]`` (Hm = heads, broadcast copies)."""
    N, C, causal_ = masks[0].N, masks[0].C, masks[0].causal
    assert all(m.N == N and m.C == C and m.causal == causal_ for m in masks)
    arr = np.stack([m.sri for m in masks])[:, None]
    return np.ascontiguousarray(np.repeat(arr, heads, axis=1))
