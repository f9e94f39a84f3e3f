"""FlashMask CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_2410_01359_b200``) never imports it and shares no code with it.

Plain, slow, obviously-correct NumPy fp64 implementation of what the FlashMask hot
path computes (PAPER.md arXiv 2410.01359).  FlashMask is exact — skipped tiles
contribute exactly 0 (§4.4) — so attention here is the plain definition
with the dense mask materialised from the column intervals, not a replay of the
tiled Alg. 1/2.  Tile classification is Eq. 4 / Alg. 1 lines 9-14 and 15-21
written out per tile.

Readings of the paper used here are numbered R1..R30 in DESIGN.md §3 (they follow
SURVEY.md §8(c) c.2).  Every function names the passage it follows.
Pins: tests/test_oracle_*.py (-m "not gpu").  Parity unpinned: none of the
functions below (see DESIGN.md §3 for the list of pins per function).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SKIP, PARTIAL, UNMASKED = 0, 1, 2  # tile classes (Eq. 4)


# ------------------------------------------------------------------ mask vectors
@dataclass
class Vectors:
    """LTS/LTE/UTS/UTE of §4.1 for one mask head, int64 length N."""

    lts: np.ndarray
    lte: np.ndarray
    uts: np.ndarray
    ute: np.ndarray
    causal: bool
    N: int
    # False: column-wise (§4.1): index = key column y, values = masked ROW intervals.
    # True: row-wise (R32): index = query row r, values = masked KEY intervals.
    rowwise: bool = False


def expand(sri: np.ndarray, causal: bool, N: int) -> Vectors:
    """startend_row_indices ``[N, C]`` -> the four §4.1 vectors.

    C-table (R17): causal C=1 -> (LTS; LTE=N), causal C=2 ->
    (LTS, LTE); non-causal C=2 -> (LTS, UTE; LTE=N, UTS=0); non-causal C=4 -> all four.
    In causal mode the upper triangle is the implicit r<y region (R8); the upper
    vectors are set to the empty interval [0, 0)."""
    sri = np.asarray(sri, dtype=np.int64).reshape(N, -1)
    C = sri.shape[1]
    zeros = np.zeros(N, dtype=np.int64)
    full_n = np.full(N, N, dtype=np.int64)
    if causal and C == 1:
        return Vectors(sri[:, 0], full_n, zeros, zeros, True, N)
    if causal and C == 2:
        return Vectors(sri[:, 0], sri[:, 1], zeros, zeros, True, N)
    if not causal and C == 2:
        return Vectors(sri[:, 0], full_n, zeros, sri[:, 1], False, N)
    if not causal and C == 4:
        return Vectors(sri[:, 0], sri[:, 1], sri[:, 2], sri[:, 3], False, N)
    raise ValueError(f"unsupported (causal={causal}, C={C})")


def expand_rowwise(sri: np.ndarray, causal: bool, N: int) -> Vectors:
    """Row-wise representation ("by transposing the attention matrix, we can obtain a
    row-wise representation using column index intervals"; R32): row r of
    ``sri [N, C]`` holds the masked KEY intervals of query row r.  The triangles keep their
    meaning — lower = keys left of the diagonal (y <= r), upper = right of it — and the C-table
    is the mirror of the column-wise one: an implicit end extends to the far edge of its
    triangle (column 0 for the lower, column N for the upper):
    causal C=1 -> (LTE; LTS=0), causal C=2 -> (LTS, LTE), non-causal C=2 -> (LTE, UTS;
    LTS=0, UTE=N), non-causal C=4 -> all four.  Causal adds the implicit {y > r} (R8)."""
    sri = np.asarray(sri, dtype=np.int64).reshape(N, -1)
    C = sri.shape[1]
    zeros = np.zeros(N, dtype=np.int64)
    full_n = np.full(N, N, dtype=np.int64)
    if causal and C == 1:
        return Vectors(zeros, sri[:, 0], zeros, zeros, True, N, True)
    if causal and C == 2:
        return Vectors(sri[:, 0], sri[:, 1], zeros, zeros, True, N, True)
    if not causal and C == 2:
        return Vectors(zeros, sri[:, 0], sri[:, 1], full_n, False, N, True)
    if not causal and C == 4:
        return Vectors(sri[:, 0], sri[:, 1], sri[:, 2], sri[:, 3], False, N, True)
    raise ValueError(f"unsupported (causal={causal}, C={C})")


def mask_rows(v: Vectors, r0: int, r1: int) -> np.ndarray:
    """Dense boolean mask rows [r0, r1) x all N columns; True = masked (M = -inf).

    Column-wise: masked(r, y) = LTS_y <= r < LTE_y  or  UTS_y <= r < UTE_y  or  (causal and
    r < y) — Eq. 3 per interval, §4.1 union of both intervals, Eq. 2's
    additive -inf mask, causal as the implicit upper triangle (R8).
    Row-wise (R32): masked(r, y) = LTS_r <= y < LTE_r  or  UTS_r <= y < UTE_r  or
    (causal and r < y)."""
    return _mask_for_rows(v, np.arange(r0, r1, dtype=np.int64))


def to_dense(v: Vectors) -> np.ndarray:
    """The full N x N mask M of Eq. 2 as booleans (O(N^2): small N only)."""
    return mask_rows(v, 0, v.N)


def from_dense(dense: np.ndarray, causal: bool) -> np.ndarray:
    """Dense mask -> startend_row_indices (§3: masked rows of a column are one
    contiguous interval per triangle).  Returns [N, C] int32 in the C-table layout
    (causal -> C=2 (LTS, LTE); bidirectional -> C=4).  Raises ValueError when a column's
    masked rows within a triangle are not contiguous (not representable)."""
    dense = np.asarray(dense, dtype=bool)
    N = dense.shape[0]
    lo = np.full((N, 2), N, dtype=np.int64)      # LTS, LTE (empty = [N, N))
    up = np.zeros((N, 2), dtype=np.int64)        # UTS, UTE (empty = [0, 0))
    for y in range(N):
        col = dense[:, y]
        if causal and not col[:y].all():
            raise ValueError(f"causal mask must mask every r<y (column {y})")
        rows = np.nonzero(col[y:])[0] + y        # lower triangle incl. diagonal (R9)
        if len(rows):
            if rows[-1] - rows[0] + 1 != len(rows):
                raise ValueError(f"column {y} lower triangle not contiguous")
            lo[y] = (rows[0], rows[-1] + 1)
        if not causal:
            rows = np.nonzero(col[:y])[0]
            if len(rows):
                if rows[-1] - rows[0] + 1 != len(rows):
                    raise ValueError(f"column {y} upper triangle not contiguous")
                up[y] = (rows[0], rows[-1] + 1)
    if causal:
        return np.stack([lo[:, 0], lo[:, 1]], 1).astype(np.int32)
    return np.stack([lo[:, 0], lo[:, 1], up[:, 0], up[:, 1]], 1).astype(np.int32)


# ------------------------------------------------------------------ attention
def forward(q, k, v, vec: Vectors, scale: float | None = None, rows=None, row_block: int = 1024):
    """O = Softmax(scale*Q K^T + M) V and L = logsumexp per row (Eq. 1, Eq. 2
    P:68-73; L as in Alg. 1 lines 27-28 P:247-248, natural log of the scaled logits).

    q, k, v: [N, d] (cast to fp64).  ``rows``: optional array of row indices to compute
    (each row is independent).  A row masked in every column has P_r = 0, O_r = 0,
    L_r = -inf (R7).  Returns (O [n_rows, d], L [n_rows])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v_ = np.asarray(v, dtype=np.float64)
    N, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else float(scale)
    rows = np.arange(N) if rows is None else np.asarray(rows, dtype=np.int64)
    O = np.zeros((len(rows), v_.shape[1]))
    L = np.full(len(rows), -np.inf)
    for s in range(0, len(rows), row_block):
        rr = rows[s:s + row_block]
        S = scale * (q[rr] @ k.T)
        M = _mask_for_rows(vec, rr)
        S[M] = -np.inf
        m = S.max(axis=1)
        live = np.isfinite(m)
        P = np.zeros_like(S)
        P[live] = np.exp(S[live] - m[live, None])
        ell = P.sum(axis=1)
        P[live] /= ell[live, None]
        O[s:s + len(rr)] = P @ v_
        L[s:s + len(rr)][live] = m[live] + np.log(ell[live])
    return O, L


def _mask_for_rows(vec: Vectors, rows: np.ndarray) -> np.ndarray:
    r = np.asarray(rows, dtype=np.int64)[:, None]
    y = np.arange(vec.N, dtype=np.int64)[None, :]
    if vec.rowwise:
        rr = r[:, 0]
        m = ((vec.lts[rr, None] <= y) & (y < vec.lte[rr, None])) | ((vec.uts[rr, None] <= y) & (y < vec.ute[rr, None]))
    else:
        m = ((vec.lts[None, :] <= r) & (r < vec.lte[None, :])) | ((vec.uts[None, :] <= r) & (r < vec.ute[None, :]))
    if vec.causal:
        m |= r < y
    return m


def probabilities(q, k, vec: Vectors, scale=None, rows=None):
    """P = Softmax(S + M) rows (Eq. 2); empty rows are all-zero (R7)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    N, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else float(scale)
    rows = np.arange(N) if rows is None else np.asarray(rows)
    S = scale * (q[rows] @ k.T)
    S[_mask_for_rows(vec, rows)] = -np.inf
    m = S.max(axis=1)
    P = np.zeros_like(S)
    live = np.isfinite(m)
    P[live] = np.exp(S[live] - m[live, None])
    P[live] /= P[live].sum(axis=1, keepdims=True)
    return P


def backward(q, k, v, do, vec: Vectors, scale=None, row_block: int = 1024):
    """Gradients of O = Softmax(scale*QK^T + M) V (Alg. 2 P:365-441 restated densely):
    D = rowsum(dO o O) (Alg. 2 line 4 P:379, per row — R5), P from the definition,
    dV = P^T dO, dP = dO V^T, dS = P o (dP - D),
    dQ = scale * dS K, dK = scale * dS^T Q — the scale of Eq. 1 carried
    into dQ/dK (R4).  Row-blocked; returns (dQ, dK, dV) fp64 [N, d]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v_ = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    N, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else float(scale)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v_)
    for s in range(0, N, row_block):
        rr = np.arange(s, min(s + row_block, N))
        P = probabilities(q, k, vec, scale, rr)
        O = P @ v_
        D = (do[rr] * O).sum(axis=1)
        dv += P.T @ do[rr]
        dP = do[rr] @ v_.T
        dS = P * (dP - D[:, None])
        dq[rr] = scale * (dS @ k)
        dk += scale * (dS.T @ q[rr])
    return dq, dk, dv


def backward_rows(q, k, v, do, vec: Vectors, rows, scale=None):
    """One row block of ``backward`` (the same statements, for a given set of query rows):
    returns (dQ[rows], dK contribution, dV contribution).  Summing the contributions over
    a partition of the rows gives ``backward``'s dK, dV.  Used to time the oracle on a
    bounded sample (bench.py cpu_baseline)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v_ = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    d = q.shape[1]
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else float(scale)
    rr = np.asarray(rows, dtype=np.int64)
    P = probabilities(q, k, vec, scale, rr)
    O = P @ v_
    D = (do[rr] * O).sum(axis=1)
    dv = P.T @ do[rr]
    dS = P * (do[rr] @ v_.T - D[:, None])
    return scale * (dS @ k), scale * (dS.T @ q[rr]), dv


def backward_cols(q, k, v, do, vec: Vectors, keys, scale=None, row_block: int = 1024):
    """dK and dV of the key columns ``keys`` only (the column-parallel view of Alg. 2, P:258,
    P:390-438, restated densely): first the forward over ALL rows (L_r and O_r — every row's
    softmax spans all keys), D = rowsum(dO o O) (R5); then for the requested columns
    y: P[:, y] = exp(scale*Q k_y^T - L) on visible cells, 0 on masked cells and on empty rows
    (L = -inf, R7), dV_y = P[:, y]^T dO, dP[:, y] = dO v_y^T,
    dS = P o (dP - D), dK_y = scale * dS[:, y]^T Q.  Cost O(N^2 d) for the
    forward plus O(N |keys| d); used where ``backward`` (O(N^2) memory per block, all
    columns) is too slow: generic-Q dK/dV checks at N = 32K.  Returns (dK [len(keys), d],
    dV [len(keys), d])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v_ = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    N, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else float(scale)
    keys = np.asarray(keys, dtype=np.int64)
    O, L = forward(q, k, v_, vec, scale, row_block=row_block)
    D = (do * O).sum(axis=1)
    dk = np.zeros((len(keys), d))
    dv = np.zeros((len(keys), v_.shape[1]))
    live = np.isfinite(L)
    for s in range(0, N, row_block):
        rr = np.arange(s, min(s + row_block, N))
        S = scale * (q[rr] @ k[keys].T)                       # [rows, |keys|]
        M = _mask_for_rows(vec, rr)[:, keys]
        P = np.zeros_like(S)
        ok = ~M & live[rr, None]
        P[ok] = np.exp((S - np.where(live[rr], L[rr], 0.0)[:, None])[ok])
        dv += P.T @ do[rr]
        dP = do[rr] @ v_[keys].T
        dS = P * (dP - D[rr, None])
        dk += scale * (dS.T @ q[rr])
    return dk, dv


# ------------------------------------------------------------------ classification
def extrema(vec: Vectors, Bc: int) -> np.ndarray:
    """Alg. 1 lines 3-4: per column tile j the min and max of each vector over
    the tile's real columns [j*Bc, min((j+1)*Bc, N)) (R3).  Returns int64 [Tc, 8] in the
    order LTS^min, LTS^max, LTE^min, LTE^max, UTS^min, UTS^max, UTE^min, UTE^max."""
    N = vec.N
    Tc = -(-N // Bc)
    out = np.zeros((Tc, 8), dtype=np.int64)
    for j in range(Tc):
        c0, c1 = j * Bc, min((j + 1) * Bc, N)
        for t, a in enumerate((vec.lts, vec.lte, vec.uts, vec.ute)):
            out[j, 2 * t] = a[c0:c1].min()
            out[j, 2 * t + 1] = a[c0:c1].max()
    return out


def classify(vec: Vectors, Br: int, Bc: int):
    """Dispatch: column-wise vectors -> ``classify_colwise``; row-wise -> ``classify_rowwise``."""
    return classify_rowwise(vec, Br, Bc) if vec.rowwise else classify_colwise(vec, Br, Bc)


def classify_colwise(vec: Vectors, Br: int, Bc: int):
    """Eq. 4 per tile, in Alg. 1's order, 0-based (R2), ragged
    tiles by their real extents (R3), causal region as its own triangle (R13):

      SKIP     iff (r0 >= LTS^max and r1 <= LTE^min)          Alg.1 l.9
               or  (r0 >= UTS^max and r1 <= UTE^min)          Alg.1 l.12
               or  (causal and r1-1 < c0)
      PARTIAL  iff (r1 > LTS^min and r0 < LTE^max)            Alg.1 l.15
               or  (r1 > UTS^min and r0 < UTE^max)            Alg.1 l.18
               or  (causal and r0 < c1-1)
      UNMASKED otherwise.

    Returns (class_map uint8 [Tr, Tc], counts int64 [3] = (skip, partial, unmasked),
    extrema int64 [Tc, 8])."""
    N = vec.N
    Tr, Tc = -(-N // Br), -(-N // Bc)
    ext = extrema(vec, Bc)
    cm = np.zeros((Tr, Tc), dtype=np.uint8)
    # one column tile at a time; the rows of the column are evaluated as a vector,
    # the if/elif chain below is the per-tile rule in the order stated above.
    r0 = np.arange(Tr, dtype=np.int64) * Br
    r1 = np.minimum(r0 + Br, N)
    for j in range(Tc):
        c0, c1 = j * Bc, min((j + 1) * Bc, N)
        ltsmin, ltsmax, ltemin, ltemax, utsmin, utsmax, utemin, utemax = ext[j]
        skip = ((r0 >= ltsmax) & (r1 <= ltemin)) | ((r0 >= utsmax) & (r1 <= utemin))
        if vec.causal:
            skip |= r1 - 1 < c0
        part = ((r1 > ltsmin) & (r0 < ltemax)) | ((r1 > utsmin) & (r0 < utemax))
        if vec.causal:
            part |= r0 < c1 - 1
        cm[:, j] = np.where(skip, SKIP, np.where(part, PARTIAL, UNMASKED))
    counts = np.array([(cm == SKIP).sum(), (cm == PARTIAL).sum(), (cm == UNMASKED).sum()], dtype=np.int64)
    return cm, counts, ext


def classify_rowwise(vec: Vectors, Br: int, Bc: int):
    """Eq. 4 for the row-wise representation ("by transposing the attention matrix";
    DESIGN.md R32): the intervals are KEY ranges of each query row, so Alg. 1 lines 3-4's
    min/max are taken over the real rows of row tile i (R3) and compared with the column
    range [c0, c1) of tile j — Eq. 4 with the roles of rows and columns exchanged; the causal
    triangle (a property of the (r, y) position, not of the vectors) is unchanged:

      SKIP     iff (c0 >= LTS^max and c1 <= LTE^min)
               or  (c0 >= UTS^max and c1 <= UTE^min)
               or  (causal and r1-1 < c0)
      PARTIAL  iff (c1 > LTS^min and c0 < LTE^max)
               or  (c1 > UTS^min and c0 < UTE^max)
               or  (causal and r0 < c1-1)
      UNMASKED otherwise.

    Returns (class_map uint8 [Tr, Tc], counts int64 [3], extrema int64 [Tr, 8] (per row tile))."""
    assert vec.rowwise
    N = vec.N
    Tr, Tc = -(-N // Br), -(-N // Bc)
    ext = extrema(vec, Br)          # index = row: min/max over each row tile's real rows
    cm = np.zeros((Tr, Tc), dtype=np.uint8)
    c0 = np.arange(Tc, dtype=np.int64) * Bc
    c1 = np.minimum(c0 + Bc, N)
    for i in range(Tr):
        r0, r1 = i * Br, min((i + 1) * Br, N)
        ltsmin, ltsmax, ltemin, ltemax, utsmin, utsmax, utemin, utemax = ext[i]
        skip = ((c0 >= ltsmax) & (c1 <= ltemin)) | ((c0 >= utsmax) & (c1 <= utemin))
        if vec.causal:
            skip |= r1 - 1 < c0
        part = ((c1 > ltsmin) & (c0 < ltemax)) | ((c1 > utsmin) & (c0 < utemax))
        if vec.causal:
            part |= r0 < c1 - 1
        cm[i, :] = np.where(skip, SKIP, np.where(part, PARTIAL, UNMASKED))
    counts = np.array([(cm == SKIP).sum(), (cm == PARTIAL).sum(), (cm == UNMASKED).sum()], dtype=np.int64)
    return cm, counts, ext


def from_dense_rowwise(dense: np.ndarray, causal: bool) -> np.ndarray:
    """Dense mask -> row-wise startend indices (R32): the masked keys of row r left of or
    on the diagonal (y <= r) must be one interval, those right of it (y > r) another (for a
    causal mask: all of them).  Returns [N, C] int32: causal -> C=2 (LTS, LTE), bidirectional
    -> C=4 (LTS, LTE, UTS, UTE); empty intervals as [0, 0) / [N, N).  Raises ValueError when
    a row's masked keys within a triangle are not contiguous."""
    dense = np.asarray(dense, dtype=bool)
    N = dense.shape[0]
    lo = np.zeros((N, 2), dtype=np.int64)
    up = np.full((N, 2), N, dtype=np.int64)
    for r in range(N):
        row = dense[r]
        if causal and not row[r + 1:].all():
            raise ValueError(f"causal mask must mask every y>r (row {r})")
        ys = np.nonzero(row[:r + 1])[0]
        if len(ys):
            if ys[-1] - ys[0] + 1 != len(ys):
                raise ValueError(f"row {r} lower triangle not contiguous")
            lo[r] = (ys[0], ys[-1] + 1)
        if not causal:
            ys = np.nonzero(row[r + 1:])[0] + r + 1
            if len(ys):
                if ys[-1] - ys[0] + 1 != len(ys):
                    raise ValueError(f"row {r} upper triangle not contiguous")
                up[r] = (ys[0], ys[-1] + 1)
    if causal:
        return np.stack([lo[:, 0], lo[:, 1]], 1).astype(np.int32)
    return np.stack([lo[:, 0], lo[:, 1], up[:, 0], up[:, 1]], 1).astype(np.int32)


def nonskip_counts(vec: Vectors, Br: int, Bc: int):
    """Per-unit work of the tiled algorithm: the number of non-SKIP tiles in every
    row tile (the forward's unit, Alg. 1's inner loop over j) and in every column
    tile (the backward's unit, Alg. 2's inner loop over i); compute is
    O((1-rho) T_r T_c).  Returns (rows int64 [Tr], cols int64 [Tc])."""
    cm, _, _ = classify(vec, Br, Bc)
    ns = cm != SKIP
    return ns.sum(axis=1).astype(np.int64), ns.sum(axis=0).astype(np.int64)


CHUNK_ROWS, CHUNK_COLS = 32, 16   # refinement sub-blocks of a 128 x 128 tile: 4 x 8 = 32 bits


def refine_chunks(vec: Vectors):
    """Tighter-than-Eq.-4 refinement (R31), rule version 1.

    Eq. 4 classifies a tile from hulls (min/max) of its columns' intervals, so a
    PARTIAL tile may hold large regions with no masked cell (P:232-240 then masks every element
    of it).  Refinement: each 128 x 128 tile (the forward's tile, R14) is cut into 4 row groups
    of 32 rows x 8 column chunks of 16 columns; bit (8 g + c) of the tile's 32-bit word is 1 iff
    the sub-block [r0 + 32 g, r0 + 32 g + 32) x [c0 + 16 c, c0 + 16 c + 16) — real rows and
    columns only (R3) — contains a masked cell: masked(r, y) of Eq. 3 / §4.1 (P:100-104,
    P:127) with the causal triangle (R8).  Written out per column and row group: column y has a
    masked cell in rows [a, b) iff one of its intervals [LTS, LTE), [UTS, UTE) intersects [a, b)
    or (causal) a < y.  Returns uint32 [Tr, Tc]."""
    assert not vec.rowwise, "column-wise representation only"
    N = vec.N
    T = -(-N // 128)
    out = np.zeros((T, T), dtype=np.uint32)
    y = np.arange(N, dtype=np.int64)
    for i in range(T):
        for g in range(4):
            a = i * 128 + g * CHUNK_ROWS
            b = min(a + CHUNK_ROWS, N)
            if a >= N:
                continue
            hit = ((vec.lts < vec.lte) & (vec.lts < b) & (vec.lte > a)) | \
                  ((vec.uts < vec.ute) & (vec.uts < b) & (vec.ute > a))
            if vec.causal:
                hit |= a < y
            for j in range(T):
                for c in range(8):
                    c0 = j * 128 + c * CHUNK_COLS
                    c1 = min(c0 + CHUNK_COLS, N)
                    if c0 < N and hit[c0:c1].any():
                        out[i, j] |= np.uint32(1 << (8 * g + c))
    return out


def alpha_bruteforce(vec: Vectors, Br: int, Bc: int) -> int:
    """alpha of §4.3: number of tiles whose every cell is masked, counted from the
    dense mask (O(N^2): small N only)."""
    M = to_dense(vec)
    N = vec.N
    a = 0
    for r0 in range(0, N, Br):
        for c0 in range(0, N, Bc):
            if M[r0:r0 + Br, c0:c0 + Bc].all():
                a += 1
    return a


def block_sparsity(counts) -> float:
    """rho = alpha / (Tr * Tc) (§4.3) with alpha = the SKIP count of rule R (R11)."""
    return float(counts[0]) / float(np.sum(counts))


def effective_flops(vec: Vectors, d: int, Br: int = 128, Bc: int = 128):
    """Effective FLOPs of one (batch, head) (R15, P:581 'based on the block sparsity ...
    calculate the FLOPs'): forward = 4*d*sum over non-SKIP tiles of rows*cols
    (two GEMMs of 2*rows*cols*d each); backward = 2.5 x forward (five GEMMs)."""
    cm, _, _ = classify(vec, Br, Bc)
    N = vec.N
    Tr, Tc = cm.shape
    rows = np.array([min((i + 1) * Br, N) - i * Br for i in range(Tr)], dtype=np.float64)
    cols = np.array([min((j + 1) * Bc, N) - j * Bc for j in range(Tc)], dtype=np.float64)
    area = (rows[:, None] * cols[None, :])[cm != SKIP].sum()
    fwd = 4.0 * d * area
    return fwd, 2.5 * fwd


# ------------------------------------------------------------------ Q = 0 closed forms (any N)
def visible_counts(vec: Vectors) -> np.ndarray:
    """count_r = number of key columns row r may attend to, in O(N) without the dense mask:
    N minus the columns masked by the lower interval, the upper interval, and (causal) the
    r<y triangle, with inclusion-exclusion done per column on the row axis via difference
    arrays.  Exact for any vectors (each column's masked row set is the union of at most
    three row intervals: [LTS, LTE), [UTS, UTE), and [0, y) if causal)."""
    assert not vec.rowwise, "column-wise representation only"
    N = vec.N
    diff = np.zeros(N + 1, dtype=np.int64)
    y = np.arange(N, dtype=np.int64)
    # represent each column's masked rows as a union of disjoint intervals: sort & merge the
    # (up to) three intervals per column, then add +1/-1 on the difference array.
    ivs = [(np.clip(vec.lts, 0, N), np.clip(vec.lte, 0, N)), (np.clip(vec.uts, 0, N), np.clip(vec.ute, 0, N))]
    if vec.causal:
        ivs.append((np.zeros(N, dtype=np.int64), y))
    starts = np.stack([a for a, _ in ivs], 1)
    ends = np.stack([b for _, b in ivs], 1)
    ends = np.where(ends > starts, ends, starts)          # empty intervals
    order = np.argsort(starts, axis=1, kind="stable")
    starts = np.take_along_axis(starts, order, 1)
    ends = np.take_along_axis(ends, order, 1)
    cur_s, cur_e = starts[:, 0].copy(), ends[:, 0].copy()
    for k in range(1, starts.shape[1]):
        s, e = starts[:, k], ends[:, k]
        merge = s <= cur_e
        # flush the current interval where the next one does not overlap
        flush = ~merge
        np.add.at(diff, cur_s[flush], 1)
        np.add.at(diff, cur_e[flush], -1)
        cur_e = np.where(merge, np.maximum(cur_e, e), e)
        cur_s = np.where(merge, cur_s, s)
    np.add.at(diff, cur_s, 1)
    np.add.at(diff, cur_e, -1)
    masked_cols = np.cumsum(diff)[:N]
    return N - masked_cols


def forward_q_zero(v, vec: Vectors):
    """Q = 0: every visible logit is 0, so L_r = ln(count_r) and O_r = mean of the V rows that
    row r sees (empty rows: O=0, L=-inf) — Eq. 2 with S = 0 on visible cells.  O(N·d): per
    key column the visible rows are the complement of its masked union, accumulated on the
    row axis with difference arrays.  Used only at sizes where the dense oracle is too slow;
    pinned against ``forward`` (tests/test_oracle_attention.py)."""
    v = np.asarray(v, dtype=np.float64)
    N, d = v.shape
    cnt = visible_counts(vec)
    # sum_{y visible to r} V_y = sum over columns y of V_y * [r visible]; the visible rows of
    # column y are the complement of its masked union inside [0, N): accumulate V_y on the
    # row axis with difference arrays over the visible row intervals.
    acc = np.zeros((N + 1, d))
    ivs = [(np.clip(vec.lts, 0, N), np.clip(vec.lte, 0, N)), (np.clip(vec.uts, 0, N), np.clip(vec.ute, 0, N))]
    y = np.arange(N, dtype=np.int64)
    if vec.causal:
        ivs.append((np.zeros(N, dtype=np.int64), y))
    for col in range(N):
        segs = sorted((int(a[col]), int(b[col])) for a, b in ivs if b[col] > a[col])
        pos = 0
        for s, e in segs:
            if s > pos:
                acc[pos] += v[col]
                acc[s] -= v[col]
            pos = max(pos, e)
        if pos < N:
            acc[pos] += v[col]
            acc[N] -= v[col]
    sums = np.cumsum(acc, axis=0)[:N]
    live = cnt > 0
    O = np.zeros((N, d))
    O[live] = sums[live] / cnt[live, None]
    L = np.full(N, -np.inf)
    L[live] = np.log(cnt[live])
    return O, L


def dv_q_zero(do, vec: Vectors):
    """Q = 0: P[r, y] = 1/count_r on visible cells, so dV_y = sum over rows r that see y of
    dO_r / count_r (Alg. 2 line 22, with P written out).  Per column, the visible rows
    are the complement of its masked union: prefix sums of w_r = dO_r / count_r."""
    do = np.asarray(do, dtype=np.float64)
    N, d = do.shape
    cnt = visible_counts(vec)
    w = np.where(cnt[:, None] > 0, do / np.maximum(cnt, 1)[:, None], 0.0)
    pre = np.vstack([np.zeros((1, d)), np.cumsum(w, axis=0)])
    ivs = [(np.clip(vec.lts, 0, N), np.clip(vec.lte, 0, N)), (np.clip(vec.uts, 0, N), np.clip(vec.ute, 0, N))]
    y = np.arange(N, dtype=np.int64)
    if vec.causal:
        ivs.append((np.zeros(N, dtype=np.int64), y))
    dv = np.zeros((N, d))
    for col in range(N):
        segs = sorted((int(a[col]), int(b[col])) for a, b in ivs if b[col] > a[col])
        pos, tot = 0, np.zeros(d)
        for s, e in segs:
            if s > pos:
                tot += pre[s] - pre[pos]
            pos = max(pos, e)
        if pos < N:
            tot += pre[N] - pre[pos]
        dv[col] = tot
    return dv
