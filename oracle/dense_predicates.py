"""Independent dense mask predicates per Figure-1 family — TEST INFRASTRUCTURE ONLY.

masked(r, y) written from the family's definition in PAPER.md §2.1 without
the column-interval vectors, used to pin the input builders in
workloads/masks.py cell for cell on tiny N.
"""
from __future__ import annotations

import numpy as np


def _grid(N):
    r = np.arange(N)[:, None]
    y = np.arange(N)[None, :]
    return r, y


def _doc_index(lens):
    return np.repeat(np.arange(len(lens)), lens)


def full(N):
    return np.zeros((N, N), dtype=bool)


def causal(N):
    r, y = _grid(N)
    return r < y


def sliding_window(N, w):
    r, y = _grid(N)
    return (r < y) | (r - y >= w)


def causal_document(doc_lens):
    N = int(sum(doc_lens))
    r, y = _grid(N)
    doc = _doc_index(doc_lens)
    return (r < y) | (doc[:, None] != doc[None, :])


def document(doc_lens):
    N = int(sum(doc_lens))
    doc = _doc_index(doc_lens)
    return doc[:, None] != doc[None, :]


def share_question(docs):
    """docs = [(q, [a1..ak])]: answer tokens see the question and their own answer."""
    doc, seg = [], []
    for di, (q, answers) in enumerate(docs):
        doc += [di] * q
        seg += [0] * q
        for ai, a in enumerate(answers):
            doc += [di] * a
            seg += [ai + 1] * a
    doc, seg = np.asarray(doc), np.asarray(seg)
    N = len(doc)
    r, y = _grid(N)
    return (r < y) | (doc[:, None] != doc[None, :]) | ((seg[:, None] != seg[None, :]) & (seg[None, :] != 0))


def global_sliding_window(N, g, w):
    r, y = _grid(N)
    visible = (r < g) | (y < g) | ((r - y >= 0) & (r - y < w))
    return ~visible


def causal_blockwise(block_lens):
    N = int(sum(block_lens))
    blk = _doc_index(block_lens)
    last = len(block_lens) - 1
    r, y = _grid(N)
    return (r < y) | ((blk[:, None] != blk[None, :]) & (blk[:, None] != last))


def prefix_lm_document(docs):
    lens = [l for l, _ in docs]
    N = int(sum(lens))
    doc = _doc_index(lens)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    pre = np.asarray([p for _, p in docs])
    r, y = _grid(N)
    ydoc = doc[None, :]
    return (doc[:, None] != ydoc) | ((r < y) & ((y - starts[ydoc]) >= pre[ydoc]))


def prefix_lm_causal(N, p):
    r, y = _grid(N)
    return (r < y) & (y >= p)


def qk_sparse(N, dropped_keys, q_drop):
    a, b = q_drop
    r, y = _grid(N)
    kd = np.zeros(N, dtype=bool)
    kd[list(dropped_keys)] = True
    return (r < y) | kd[None, :] | ((a <= r) & (r < b))


def hash_sparse(buckets):
    bk = np.asarray(buckets)
    N = len(bk)
    r, y = _grid(N)
    return (r < y) | (bk[:, None] != bk[None, :])


def random_eviction(N, starts, span):
    """starts[y] = s_y (or None for no eviction)."""
    r, y = _grid(N)
    s = np.asarray([N if x is None else x for x in starts])
    return (r < y) | ((s[None, :] <= r) & (r < s[None, :] + span))


def key_window(a, b):
    """Row r attends exactly to keys a[r] <= y < b[r] (a per-query key window; row-wise family)."""
    a = np.asarray(a)[:, None]
    b = np.asarray(b)[:, None]
    N = a.shape[0]
    y = np.arange(N)[None, :]
    return ~((a <= y) & (y < b))
