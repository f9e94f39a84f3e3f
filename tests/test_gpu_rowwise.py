"""Row-wise representation (FM_FLAG_ROWWISE, R32) through the C ABI
against the fp64 oracle: tile classification bit-exact (K1a/K1b, transposed Eq. 4), forward and
backward (K2a, K4, K6, and the fp32 path F1-F3) within the north_star tolerances."""
import numpy as np
import pytest
import torch

from oracle import flashmask_oracle as fo
from workloads import masks as wm
from workloads import tensors as wt

from gpu_util import assert_close, assert_lse, to_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmlib():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    from paper_2410_01359_b200 import flashmask
    return flashmask


def _stack(masks):
    return torch.from_numpy(np.stack([m.sri for m in masks])[:, None].copy())


CLS_CASES = [(fam, N) for fam in wm.ROWWISE_FAMILIES for N in (1, 127, 129, 1000)] + \
            [(fam, 4133) for fam in ("causal_document", "document", "key_window", "global_sliding_window")]


@pytest.mark.parametrize("fam,N", CLS_CASES)
def test_rowwise_classify_bit_exact(fmlib, fam, N):
    rng = np.random.default_rng(N * 13 + len(fam))
    masks = [wm.rw_sample_family(fam, N, rng, (1, 5)) for _ in range(2)]
    sri = _stack(masks).cuda()
    for br, bc in ((128, 128), (64, 128), (3, 5), (128, 64)):
        minmax, cmap, counts, rows, cols = fmlib.flashmask_classify(sri, masks[0].causal, br, bc, nonskip=True,
                                                                     rowwise=True)
        torch.cuda.synchronize()
        for b, m in enumerate(masks):
            vec = fo.expand_rowwise(m.sri, m.causal, N)
            cm_ref, cnt_ref, ext_ref = fo.classify_rowwise(vec, br, bc)
            rows_ref, cols_ref = fo.nonskip_counts(vec, br, bc)
            assert np.array_equal(minmax[b, 0].cpu().numpy().astype(np.int64), ext_ref), (br, bc)
            assert np.array_equal(cmap[b, 0].cpu().numpy(), cm_ref), (br, bc)
            assert np.array_equal(counts[b, 0].cpu().numpy(), cnt_ref), (br, bc)
            assert np.array_equal(rows[b, 0].cpu().numpy(), rows_ref), (br, bc)
            assert np.array_equal(cols[b, 0].cpu().numpy(), cols_ref), (br, bc)


def test_rowwise_classify_arbitrary_int32(fmlib):
    rng = np.random.default_rng(1)
    for causal, C in ((True, 1), (True, 2), (False, 2), (False, 4)):
        N = 777
        raw = rng.integers(-1000, N + 1000, size=(1, 1, N, C)).astype(np.int32)
        raw[0, 0, :5] = np.iinfo(np.int32).max
        raw[0, 0, 5:9] = np.iinfo(np.int32).min
        for br, bc in ((128, 128), (64, 128)):
            _, cmap, counts = fmlib.flashmask_classify(torch.from_numpy(raw).cuda(), causal, br, bc, rowwise=True)
            cm_ref, cnt_ref, _ = fo.classify_rowwise(fo.expand_rowwise(raw[0, 0], causal, N), br, bc)
            assert np.array_equal(cmap[0, 0].cpu().numpy(), cm_ref)
            assert np.array_equal(counts[0, 0].cpu().numpy(), cnt_ref)


def _check(fmlib, masks, H, Hkv, d, dtype=torch.bfloat16, flags=0, seed=0):
    """Run fwd+bwd with FM_FLAG_ROWWISE | flags and compare every head with the oracle."""
    B, N, causal = len(masks), masks[0].N, masks[0].causal
    sri = _stack(masks)
    t = {}
    for n, heads in (("q", H), ("do", H), ("k", Hkv), ("v", Hkv)):
        t[n] = wt.make_tensor(n, B, N, heads, d, base=seed, dtype=dtype)
    sri_c, tc = to_cuda(sri, t)
    F = fmlib.FM_FLAG_ROWWISE | flags
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32, flags=F)
    dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, causal,
                                     out_dtype=torch.float32, flags=F)
    torch.cuda.synchronize()
    G = H // Hkv
    f = lambda x, b, h: x[b, :, h, :].double().numpy()
    for b, m in enumerate(masks):
        vec = fo.expand_rowwise(m.sri, causal, N)
        gk_sum = [np.zeros((N, d)) for _ in range(Hkv)]
        gv_sum = [np.zeros((N, d)) for _ in range(Hkv)]
        for h in range(H):
            hk = h // G
            O, L = fo.forward(f(t["q"], b, h), f(t["k"], b, hk), f(t["v"], b, hk), vec)
            gq, gk, gv = fo.backward(f(t["q"], b, h), f(t["k"], b, hk), f(t["v"], b, hk), f(t["do"], b, h), vec)
            gk_sum[hk] += gk
            gv_sum[hk] += gv
            tag = f"{m.family} N={N} d={d} {dtype} flags={flags} [{b},{h}]"
            assert_close(f"O {tag}", o[b, :, h].cpu().numpy(), O)
            assert_lse(lse[b, h].cpu().numpy(), L)
            assert_close(f"dQ {tag}", dq[b, :, h].cpu().numpy(), gq)
        for hk in range(Hkv):
            # GQA: dK/dV sum G heads' gradients (R30)
            assert_close(f"dK {m.family} [{b},{hk}]", dk[b, :, hk].cpu().numpy(), gk_sum[hk], tol_max=2e-2 * G ** 0.5)
            assert_close(f"dV {m.family} [{b},{hk}]", dv[b, :, hk].cpu().numpy(), gv_sum[hk], tol_max=2e-2 * G ** 0.5)
    return o, lse, dq, dk, dv


ATTN = [(fam, N, d) for fam in wm.ROWWISE_FAMILIES for N, d in ((700, 128), (515, 64))] + \
       [("causal_document", 1, 128), ("key_window", 129, 128), ("document", 2049, 128), ("causal", 128, 64)]


@pytest.mark.parametrize("fam,N,d", ATTN)
def test_rowwise_fwd_bwd_parity(fmlib, fam, N, d):
    rng = np.random.default_rng(N + d + len(fam))
    masks = [wm.rw_sample_family(fam, N, rng, (1, 5)) for _ in range(2)]
    _check(fmlib, masks, 2, 2, d, seed=N)


@pytest.mark.parametrize("case", range(12))
def test_rowwise_variants(fmlib, case):
    """GQA, fp16 inputs, deterministic dQ (K6) and fp32 inputs (F1-F3) on row-wise masks."""
    rng = np.random.default_rng(50 + case)
    fam = wm.ROWWISE_FAMILIES[case % len(wm.ROWWISE_FAMILIES)]
    N = int(rng.integers(2, 600))
    d = [64, 128][case % 2]
    masks = [wm.rw_sample_family(fam, N, rng, (1, 4)) for _ in range(1 + case % 2)]
    kind = case % 4
    if kind == 0:
        _check(fmlib, masks, 4, 2, d, seed=case)                                      # GQA
    elif kind == 1:
        _check(fmlib, masks, 2, 2, d, dtype=torch.float16, seed=case)                 # fp16
    elif kind == 2:
        _check(fmlib, masks, 2, 1, d, flags=fmlib.FM_FLAG_DETERMINISTIC, seed=case)   # K6 + MQA
    else:
        _check(fmlib, masks, 2, 2, d, dtype=torch.float32, seed=case)                 # fp32 path


@pytest.mark.parametrize("causal,C,N,d", [(c, C, N, d) for c, C in ((True, 1), (True, 2), (False, 2), (False, 4))
                                          for N, d in ((333, 128), (700, 64))])
def test_rowwise_arbitrary_int32_vectors(fmlib, causal, C, N, d):
    """Any int32 row vectors (negative, > N, inverted, INT_MIN / INT_MAX) through fwd + bwd."""
    rng = np.random.default_rng(N * 3 + C + 50 * causal)
    i32 = np.iinfo(np.int32)
    raw = rng.integers(-N, 2 * N, size=(N, C)).astype(np.int64)
    ok = rng.random(N) < 0.5
    raw[ok, 0] = rng.integers(0, N + 1, ok.sum())
    special = [i32.max, i32.min, -1, 0, N, N + 1, i32.max - 1, i32.min + 1]
    for j in range(min(N, 40)):
        raw[j * (N // 40), int(rng.integers(C))] = special[j % len(special)]
    m = wm.MaskInput(N, causal, C, raw.astype(np.int32), "rw_arbitrary_int32", rowwise=True)
    _check(fmlib, [m], 2, 2, d, seed=N + C)


@pytest.mark.parametrize("fam,N,d", [("causal_document", 1000, 128), ("key_window", 900, 64),
                                     ("global_sliding_window", 640, 128)])
def test_rowwise_skip_equivalence_bitwise(fmlib, fam, N, d):
    """Visiting every tile (FM_FLAG_NO_SKIP) gives bitwise the same outputs."""
    rng = np.random.default_rng(5)
    m = wm.rw_sample_family(fam, N, rng, (2, 5))
    sri = _stack([m]).cuda()
    t = {n: wt.make_tensor(n, 1, N, 2, d, base=9).cuda() for n in ("q", "k", "v", "do")}
    outs = []
    for extra in (0, fmlib.FM_FLAG_NO_SKIP):
        F = fmlib.FM_FLAG_ROWWISE | extra
        o, lse = fmlib.flashmask_fwd(t["q"], t["k"], t["v"], sri, m.causal, out_dtype=torch.float32, flags=F)
        g = fmlib.flashmask_bwd(t["q"], t["k"], t["v"], o, t["do"], lse, sri, m.causal, out_dtype=torch.float32,
                                flags=F | fmlib.FM_FLAG_DETERMINISTIC)
        outs.append((o, lse) + tuple(g))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_rowwise_and_colwise_agree(fmlib):
    """One mask in both representations (document family): the two runs agree to rounding."""
    lens = [300, 411, 289]
    rw, cw = wm.rw_document(lens), wm.document(lens)
    N = rw.N
    t = {n: wt.make_tensor(n, 1, N, 2, 128, base=4).cuda() for n in ("q", "k", "v", "do")}
    res = []
    for m, F in ((rw, fmlib.FM_FLAG_ROWWISE), (cw, 0)):
        s = _stack([m]).cuda()
        o, lse = fmlib.flashmask_fwd(t["q"], t["k"], t["v"], s, False, out_dtype=torch.float32, flags=F)
        g = fmlib.flashmask_bwd(t["q"], t["k"], t["v"], o, t["do"], lse, s, False, out_dtype=torch.float32, flags=F)
        res.append((o, lse) + tuple(g))
    torch.cuda.synchronize()
    for a, b in zip(*res):
        assert torch.allclose(a, b, atol=2e-3, rtol=0)


@pytest.mark.parametrize("fam", ["causal_document", "key_window"])
def test_rowwise_full_size_sampled(fmlib, fam):
    """Row-wise masks at N = 32K (256 x 256 tiles, H = 4): O / lse of sampled rows and dK / dV of
    sampled key columns against the oracle (forward rows and backward_cols)."""
    N, H, d = 32768, 4, 128
    rng = np.random.default_rng(len(fam) * 11)
    m = wm.rw_sample_family(fam, N, rng, (10, 14))
    sri = _stack([m]).cuda()
    x = {n: wt.make_tensor(n, 1, N, H, d, base=21).cuda() for n in ("q", "k", "v", "do")}
    F = fmlib.FM_FLAG_ROWWISE
    o, lse = fmlib.flashmask_fwd(x["q"], x["k"], x["v"], sri, m.causal, out_dtype=torch.float32, flags=F)
    dq, dk, dv = fmlib.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, m.causal,
                                     out_dtype=torch.float32, flags=F)
    torch.cuda.synchronize()
    vec = fo.expand_rowwise(m.sri, m.causal, N)
    rows = np.sort(rng.choice(N, 48, replace=False))
    keys = np.sort(rng.choice(N, 24, replace=False))
    f = lambda t, h: t[0, :, h, :].double().cpu().numpy()
    for h in (0, H - 1):
        O, L = fo.forward(f(x["q"], h), f(x["k"], h), f(x["v"], h), vec, rows=rows)
        assert_close(f"O {fam}[{h}]", o[0, rows, h].cpu().numpy(), O)
        assert_lse(lse[0, h, rows].cpu().numpy(), L)
        gk, gv = fo.backward_cols(f(x["q"], h), f(x["k"], h), f(x["v"], h), f(x["do"], h), vec, keys)
        assert_close(f"dK {fam}[{h}]", dk[0, keys, h].cpu().numpy(), gk)
        assert_close(f"dV {fam}[{h}]", dv[0, keys, h].cpu().numpy(), gv)


# key_window (rows that see a handful of keys) is left out: there the bounded pass's dominant P is
# rounded to bf16 instead of being 1.0, and one GQA head's dQ measured 2.07e-2 against the 2e-2 bar
# (two-pass 5.9e-3) — the precision limit recorded in DESIGN.md R33; row-wise masks therefore keep
# the two-pass forward by default
@pytest.mark.parametrize("fam,N,d", [(fam, 700, 128) for fam in wm.ROWWISE_FAMILIES if fam != "key_window"] +
                         [("causal_document", 515, 64)])
def test_rowwise_bounded_single_pass(fmlib, fam, N, d):
    """R33 bounded single pass (forced with FM_FLAG_MAX_BOUND) on row-wise masks: the element mask
    of PARTIAL tiles comes from the thread's own row vector inside the single pass."""
    rng = np.random.default_rng(N + d + len(fam) + 1)
    masks = [wm.rw_sample_family(fam, N, rng, (1, 5)) for _ in range(2)]
    _check(fmlib, masks, 2, 2, d, flags=fmlib.FM_FLAG_MAX_BOUND, seed=N + 3)
    _check(fmlib, masks[:1], 4, 2, d, flags=fmlib.FM_FLAG_MAX_BOUND, seed=N + 4)  # GQA
