"""Pins for the oracle's preprocessing (Alg. 1 lines 3-4) and tile classification (Eq. 4).

* SPEC worked examples (S:166-168 extrema, S:176-178 classes, S:186-188 rho).
* Soundness against brute force on the dense mask: SKIP => every cell masked,
  UNMASKED => no cell masked, #SKIP <= alpha.
* Closed-form class counts — exact integers.
* The paper's own tables: FW/BW TFLOPs of the closed-form masks are reproduced from the
  oracle's SKIP counts at 128x128 tiles and FLOPs = 4 N^2 d B H (1 - rho)
  (tests/golden/paper_kernel_tables_d128.txt).
"""
import os

import numpy as np
import pytest

from oracle import flashmask_oracle as fo
from workloads import masks as wm


def vec(m):
    return fo.expand(m.sri, m.causal, m.N)


def test_spec_extrema_examples():
    v = fo.Vectors(np.array([3, 3, 3, 7, 7, 7, 7, 8]), np.full(8, 8), np.zeros(8, int), np.zeros(8, int), True, 8)
    e = fo.extrema(v, 4)
    assert list(e[:, 0]) == [3, 7] and list(e[:, 1]) == [7, 8]
    assert list(e[:, 2]) == [8, 8] and list(e[:, 3]) == [8, 8]
    e = fo.extrema(vec(wm.causal_document([3, 4, 3])), 5)
    assert list(e[:, 0]) == [3, 7] and list(e[:, 1]) == [7, 10]
    v = fo.Vectors(np.full(8, 8), np.full(8, 8), np.zeros(8, int), np.zeros(8, int), True, 8)
    e = fo.extrema(v, 4)
    assert list(e[:, 0]) == [8, 8] and list(e[:, 1]) == [8, 8]


def _one_col_tile(lts, lte, N=16, causal=False):
    z = np.zeros(N, dtype=np.int64)
    return fo.Vectors(np.asarray(lts, dtype=np.int64), np.asarray(lte, dtype=np.int64), z, z, causal, N)


def test_spec_classification_examples():
    # Rows [4,8) with LTS=4, LTE=8 over the column tile -> SKIP
    v = _one_col_tile(np.full(8, 4), np.full(8, 8), N=8)
    cm, _, _ = fo.classify(v, 4, 8)
    assert cm[1, 0] == fo.SKIP
    # Rows [4,8), LTS min/max 3/7, LTE 10 -> PARTIAL
    lts = np.array([3, 4, 5, 6, 7, 7, 7, 7, 7, 7])
    v = _one_col_tile(lts, np.full(10, 10), N=10)
    cm, _, _ = fo.classify(v, 4, 10)
    assert cm[1, 0] == fo.PARTIAL
    # Rows [0,4), all-empty lower intervals -> UNMASKED
    v = _one_col_tile(np.full(8, 8), np.full(8, 8), N=8)
    cm, _, _ = fo.classify(v, 4, 4)
    assert cm[0, 0] == fo.UNMASKED and cm[0, 1] == fo.UNMASKED


def test_spec_sparsity_examples():
    # S:186 empty bidirectional -> rho 0 ; S:187 causal N=128, 64x64 -> alpha=1, rho=0.25
    _, c, _ = fo.classify(vec(wm.full(64)), 16, 16)
    assert fo.block_sparsity(c) == 0.0
    v = vec(wm.causal(128))
    _, c, _ = fo.classify(v, 64, 64)
    assert c[0] == 1 and fo.block_sparsity(c) == 0.25 and fo.alpha_bruteforce(v, 64, 64) == 1
    # S:188 causal N=8192 at 128x128 -> 0.4922
    _, c, _ = fo.classify(vec(wm.causal(8192)), 128, 128)
    assert round(fo.block_sparsity(c), 4) == 0.4922


def _random_vectors(rng, N, causal):
    """Arbitrary int32-ish vectors, including invalid / inverted intervals (R10)."""
    lo, hi = -3, N + 3
    a = rng.integers(lo, hi, size=(4, N))
    if causal:
        z = np.zeros(N, dtype=np.int64)
        return fo.Vectors(a[0], a[1], z, z, True, N)
    return fo.Vectors(a[0], a[1], a[2], a[3], False, N)


@pytest.mark.parametrize("seed", range(60))
def test_classification_soundness_bruteforce(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 40))
    causal = bool(seed % 2)
    fam = seed % 3
    if fam == 0:
        v = _random_vectors(rng, N, causal)
    else:
        m = wm.sample_family(wm.FAMILIES[seed % len(wm.FAMILIES)], max(N, 4), rng, (1, 4))
        v = vec(m)
        N = v.N
    M = fo.to_dense(v)
    for Br in (1, 2, 3, 4, 8, 16):
        for Bc in (1, 2, 4, 5, 16):
            cm, counts, _ = fo.classify(v, Br, Bc)
            for i in range(cm.shape[0]):
                for j in range(cm.shape[1]):
                    blk = M[i * Br:(i + 1) * Br, j * Bc:(j + 1) * Bc]
                    if cm[i, j] == fo.SKIP:
                        assert blk.all()
                    elif cm[i, j] == fo.UNMASKED:
                        assert not blk.any()
            assert counts[0] <= fo.alpha_bruteforce(v, Br, Bc)
            assert counts.sum() == cm.size


def _closed_form_counts(kind, N, **kw):
    T = N // 128
    if kind == "full":
        return 0, 0, T * T
    if kind == "causal":
        return T * (T - 1) // 2, T, T * (T - 1) // 2
    if kind == "sliding_window":
        W = kw["w"] // 128
        skip = T * (T - 1) // 2 + (T - W - 1) * (T - W) // 2
        part = T + (T - W)
        return skip, part, sum(T - k for k in range(1, W))
    if kind == "prefix_lm_causal":
        P = kw["p"] // 128
        skip = sum(range(P, T))
        part = T - P
        return skip, part, T * T - skip - part
    if kind == "global_sliding":
        W, G = kw["w"] // 128, kw["g"] // 128
        n = T - G
        skip = n * (n - 1) // 2 + (n - W - 1) * (n - W) // 2
        part = n + (n - W)
        return skip, part, T * G + G * n + sum(n - k for k in range(1, W))
    raise KeyError(kind)


def _build(kind, N, rng=None):
    if kind == "full":
        return wm.full(N), {}
    if kind == "causal":
        return wm.causal(N), {}
    if kind == "sliding_window":
        return wm.sliding_window(N, N // 16), {"w": N // 16}
    if kind == "prefix_lm_causal":
        return wm.prefix_lm_causal(N, N // 2), {"p": N // 2}
    if kind == "global_sliding":
        return wm.global_sliding_window(N, N // 16, 256), {"g": N // 16, "w": 256}
    if kind == "random_eviction":
        return wm.random_eviction(N, N // 16, rng), {}
    raise KeyError(kind)


@pytest.mark.parametrize("N", [4096, 8192, 32768])
@pytest.mark.parametrize("kind", ["full", "causal", "sliding_window", "prefix_lm_causal", "global_sliding"])
def test_closed_form_class_counts(kind, N):
    m, kw = _build(kind, N)
    _, counts, _ = fo.classify(vec(m), 128, 128)
    assert tuple(int(x) for x in counts) == _closed_form_counts(kind, N, **kw)


def _table_rows(golden_dir):
    rows = []
    for line in open(os.path.join(golden_dir, "paper_kernel_tables_d128.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, N, fw, bw, sp, src = line.split()
        rows.append((name, int(N), float(fw), float(bw), float(sp), src))
    return rows


def test_paper_table_flops_reproduced(golden_dir):
    rng = np.random.default_rng(7)
    for name, N, fw, bw, sp, src in _table_rows(golden_dir):
        if N > 32768 and name == "random_eviction":
            continue  # O(N) python loop in the generator; 8K/32K rows cover it
        m, _ = _build(name, N, rng)
        v = vec(m)
        _, counts, _ = fo.classify(v, 128, 128)
        rho = fo.block_sparsity(counts)
        d, H, B = 128, 32, 131072 // N
        F = 4.0 * N * N * d * B * H * (1 - rho) / 1e12
        # FW is printed to 2 decimals; at 128K the paper's FW cells sit one unit in the
        # last place above round(F) (281.48 vs 281.475) while BW/TOTAL (703.69, 985.16)
        # round exactly, so FW is checked to +-0.011 and BW to the rounding of 2.5 F.
        assert round(F, 2) == pytest.approx(fw, abs=0.011), (name, N, src, F)
        assert round(2.5 * F, 2) == pytest.approx(bw, abs=0.011), (name, N, src)
        assert round(rho, 2) == pytest.approx(sp, abs=0.006), (name, N, src, rho)
        ef, eb = fo.effective_flops(v, d)
        assert ef * B * H / 1e12 == pytest.approx(F, rel=1e-12)


def test_random_eviction_skip_equals_causal():
    """R22: the bounded-span construction skips exactly the causal tiles (P:613 vs P:623)."""
    rng = np.random.default_rng(3)
    for N in (1024, 8192):
        _, c, _ = fo.classify(vec(wm.random_eviction(N, N // 16, rng)), 128, 128)
        T = N // 128
        assert c[0] == T * (T - 1) // 2


def test_ragged_tiles():
    """R3: ragged last tiles are classified by their real extents (no padding)."""
    for N in (127, 129, 257, 300):
        v = vec(wm.causal_document([N // 3, N // 3, N - 2 * (N // 3)]))
        cm, c, _ = fo.classify(v, 128, 128)
        T = -(-N // 128)
        assert cm.shape == (T, T) and c.sum() == T * T
        M = fo.to_dense(v)
        for i in range(T):
            for j in range(T):
                blk = M[i * 128:(i + 1) * 128, j * 128:(j + 1) * 128]
                if cm[i, j] == fo.SKIP:
                    assert blk.all()
                if cm[i, j] == fo.UNMASKED:
                    assert not blk.any()


@pytest.mark.parametrize("fam", wm.FAMILIES)
def test_rule_r_matches_exact_skip_on_families(fam):
    """SURVEY §8(f) f3 evaluation: an exact (union-coverage) classification cannot skip more
    tiles than rule R on the benchmark mask families — every fully masked 128×128 tile
    (brute force on the dense mask) is already SKIP under Eq. 4 + causal — and it
    would turn only a few per cent of all tiles from PARTIAL into UNMASKED (which saves mask
    ALU work, not MMAs)."""
    N, T = 4096, 32
    rng = np.random.default_rng(11)
    for _ in range(2):
        m = wm.sample_family(fam, N, rng, (3, 7))
        vec = fo.expand(m.sri, m.causal, N)
        _, cnt, _ = fo.classify(vec, 128, 128)
        dense = fo.to_dense(vec).reshape(T, 128, T, 128).transpose(0, 2, 1, 3).reshape(T, T, -1)
        all_masked = int(dense.all(-1).sum())
        none_masked = int((~dense.any(-1)).sum())
        assert cnt[0] == all_masked, (fam, cnt, all_masked)
        assert none_masked - cnt[2] <= 0.03 * T * T, (fam, cnt, none_masked)


@pytest.mark.parametrize("N", [1024, 4096, 8192])
def test_nonskip_counts_closed_forms(N):
    """a2 per-unit work: causal -> row tile i has i+1 non-SKIP tiles, column tile j has T-j;
    sliding window w (multiple of 128, W = w/128) -> row i has min(i, W) + 1; full -> T each;
    both sums equal the non-SKIP count."""
    T = N // 128
    rows, cols = fo.nonskip_counts(vec(wm.causal(N)), 128, 128)
    assert list(rows) == [i + 1 for i in range(T)] and list(cols) == [T - j for j in range(T)]
    w = max(128, N // 16)
    W = w // 128
    rows, cols = fo.nonskip_counts(vec(wm.sliding_window(N, w)), 128, 128)
    assert list(rows) == [min(i, W) + 1 for i in range(T)]
    assert list(cols) == [min(T - j, W + 1) for j in range(T)]
    rows, cols = fo.nonskip_counts(vec(wm.full(N)), 128, 128)
    assert (rows == T).all() and (cols == T).all()
    m = wm.sample_family("causal_document", N, np.random.default_rng(N), (3, 7))
    rows, cols = fo.nonskip_counts(vec(m), 128, 128)
    _, c, _ = fo.classify(vec(m), 128, 128)
    assert rows.sum() == cols.sum() == c[1] + c[2]


@pytest.mark.parametrize("seed", range(6))
def test_refine_chunks_bruteforce(seed):
    """f3 refinement words against brute force on the dense mask (every 32 x 16 sub-block of
    every 128 x 128 tile: bit set iff it holds a masked cell), ragged N, all families, plus the
    class consistency Eq. 4 implies: UNMASKED tiles have word 0, SKIP tiles every real sub-block
    dirty."""
    rng = np.random.default_rng(100 + seed)
    for fam in wm.FAMILIES:
        N = int(rng.integers(1, 420))
        m = wm.sample_family(fam, N, rng, (1, 5))
        v = vec(m)
        words = fo.refine_chunks(v)
        M = fo.to_dense(v)
        cm, _, _ = fo.classify(v, 128, 128)
        T = -(-N // 128)
        for i in range(T):
            for j in range(T):
                want = 0
                full = 0
                for g in range(4):
                    for c in range(8):
                        a, b = i * 128 + 32 * g, min(i * 128 + 32 * g + 32, N)
                        c0, c1 = j * 128 + 16 * c, min(j * 128 + 16 * c + 16, N)
                        if a < N and c0 < N:
                            full |= 1 << (8 * g + c)
                            if M[a:b, c0:c1].any():
                                want |= 1 << (8 * g + c)
                assert int(words[i, j]) == want, (fam, N, i, j)
                if cm[i, j] == fo.UNMASKED:
                    assert want == 0
                if cm[i, j] == fo.SKIP:
                    assert want == full


def test_refine_chunks_qk_sparse_clean_blocks():
    """The case f3 targets: a QK-sparse tile below the diagonal with one dropped key is PARTIAL
    under Eq. 4 but has exactly one dirty column chunk per row group."""
    m = wm.qk_sparse(512, [300], (500, 510))
    v = vec(m)
    cm, _, _ = fo.classify(v, 128, 128)
    w = fo.refine_chunks(v)
    assert cm[3, 2] == fo.PARTIAL           # rows 384..511, keys 256..383 (key 300 dropped)
    chunk = (300 - 256) // 16               # = 2
    rows_hit = 0
    for g in range(4):
        rows_hit |= 1 << (8 * g + chunk)
    # rows 500..509 (dropped query range) are masked for every key: row group 3 is all dirty
    assert int(w[3, 2]) == rows_hit | (0xFF << 24)
