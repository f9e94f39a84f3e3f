"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Bars (BASELINE.json north_star): tile classification bit-exact; O, dQ, dK, dV (bf16 in,
fp32 accumulate, fp32 out — DESIGN.md R27) max abs <= 2e-2 and mean abs <= 2e-3; lse abs
<= 1e-3 with -inf matching exactly.  Exactness: SKIP-as-PARTIAL gives bitwise equal
O / lse / dK / dV.
"""
import numpy as np
import pytest
import torch

from oracle import flashmask_oracle as fo
from workloads import masks as wm
from workloads import tensors as wt

from gpu_util import assert_close, assert_lse, build_case, oracle_head, to_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmlib():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    from paper_2410_01359_b200 import flashmask
    return flashmask


# ------------------------------------------------------------------------- classification
CLS_CASES = [(fam, N) for fam in wm.FAMILIES for N in (1, 127, 128, 129, 300, 1000)] + \
            [(fam, 8192) for fam in wm.FAMILIES if fam != "random_eviction"] + [("random_eviction", 4096)]


@pytest.mark.parametrize("fam,N", CLS_CASES)
def test_classify_bit_exact(fmlib, fam, N):
    rng = np.random.default_rng(N * 31 + len(fam))
    masks = [wm.sample_family(fam, N, rng, (1, 5)) for _ in range(2)]
    m0 = masks[0]
    sri = torch.from_numpy(wm.stack(masks, 1)).cuda()
    for br, bc in ((128, 128), (64, 128), (3, 5), (128, 64)):
        minmax, cmap, counts, rows, cols = fmlib.flashmask_classify(sri, m0.causal, br, bc, nonskip=True)
        torch.cuda.synchronize()
        for b, m in enumerate(masks):
            vec = fo.expand(m.sri, m.causal, N)
            cm_ref, cnt_ref, ext_ref = fo.classify(vec, br, bc)
            rows_ref, cols_ref = fo.nonskip_counts(vec, br, bc)
            assert np.array_equal(minmax[b, 0].cpu().numpy().astype(np.int64), ext_ref), (br, bc)
            assert np.array_equal(cmap[b, 0].cpu().numpy(), cm_ref), (br, bc)
            assert np.array_equal(counts[b, 0].cpu().numpy(), cnt_ref), (br, bc)
            assert np.array_equal(rows[b, 0].cpu().numpy(), rows_ref), (br, bc)   # a2 per-row-tile work
            assert np.array_equal(cols[b, 0].cpu().numpy(), cols_ref), (br, bc)   # a2 per-column-tile work
    # large per-head maps (64 heads x 256 x 256 tiles) take the 64-row-tiles-per-CTA path
    if N == 8192 and fam in ("causal_document", "global_sliding_window"):
        big = [wm.sample_family(fam, 32768, rng, (3, 7)) for _ in range(64)]
        sb = torch.from_numpy(np.stack([m.sri for m in big])[None]).cuda()
        _, cmap, counts, rows, cols = fmlib.flashmask_classify(sb, big[0].causal, 128, 128, nonskip=True)
        torch.cuda.synchronize()
        for h in (0, 21, 42, 63):
            m = big[h]
            vec = fo.expand(m.sri, m.causal, 32768)
            cm_ref, cnt_ref, _ = fo.classify(vec, 128, 128)
            rows_ref, cols_ref = fo.nonskip_counts(vec, 128, 128)
            assert np.array_equal(cmap[0, h].cpu().numpy(), cm_ref)
            assert np.array_equal(counts[0, h].cpu().numpy(), cnt_ref)
            assert np.array_equal(rows[0, h].cpu().numpy(), rows_ref)
            assert np.array_equal(cols[0, h].cpu().numpy(), cols_ref)


@pytest.mark.parametrize("fam,N", [("global_sliding_window", 8192), ("causal_document", 8190), ("share_question", 8192),
                                   ("random_eviction", 8192), ("causal", 8192), ("qk_sparse", 8176)])
def test_classify_uniform_blocks(fmlib, fam, N):
    """K1b's 16-row-tile blocks whose classes are constant (one evaluation, 16 stores): small tiles
    and 8 heads give 16 row tiles per CTA; four column tiles per thread (Tc = 512); structured
    masks with a few columns set to INT_MIN / INT_MAX / out-of-range values (R10)."""
    rng = np.random.default_rng(N + len(fam))
    ms = [wm.sample_family(fam, N, rng, (2, 6)) for _ in range(8)]
    raw = np.stack([m.sri for m in ms])[None].copy()
    for h in range(1, 8, 2):
        cols = rng.choice(N, size=8, replace=False)
        raw[0, h, cols[:3]] = np.iinfo(np.int32).max
        raw[0, h, cols[3:6]] = np.iinfo(np.int32).min
        raw[0, h, cols[6:]] = rng.integers(-N, 2 * N, size=(2, raw.shape[-1]))
    causal = ms[0].causal
    sri = torch.from_numpy(raw).cuda()
    for br, bc in ((16, 16), (64, 16), (16, 64)):
        _, cmap, counts, rows, cols = fmlib.flashmask_classify(sri, causal, br, bc, nonskip=True)
        torch.cuda.synchronize()
        for h in range(8):
            vec = fo.expand(raw[0, h], causal, N)
            cm_ref, cnt_ref, _ = fo.classify(vec, br, bc)
            rows_ref, cols_ref = fo.nonskip_counts(vec, br, bc)
            assert np.array_equal(cmap[0, h].cpu().numpy(), cm_ref), (br, bc, h)
            assert np.array_equal(counts[0, h].cpu().numpy(), cnt_ref), (br, bc, h)
            assert np.array_equal(rows[0, h].cpu().numpy(), rows_ref), (br, bc, h)
            assert np.array_equal(cols[0, h].cpu().numpy(), cols_ref), (br, bc, h)


def test_classify_arbitrary_int32_vectors(fmlib):
    """R10: any int32 values (inverted / out-of-range intervals) classify like the oracle."""
    rng = np.random.default_rng(0)
    for causal, C in ((True, 1), (True, 2), (False, 2), (False, 4)):
        N = 777
        raw = rng.integers(-1000, N + 1000, size=(1, 1, N, C)).astype(np.int32)
        raw[0, 0, :5] = np.iinfo(np.int32).max
        raw[0, 0, 5:9] = np.iinfo(np.int32).min
        _, cmap, counts = fmlib.flashmask_classify(torch.from_numpy(raw).cuda(), causal, 128, 128)
        vec = fo.expand(raw[0, 0], causal, N)
        cm_ref, cnt_ref, _ = fo.classify(vec, 128, 128)
        assert np.array_equal(cmap[0, 0].cpu().numpy(), cm_ref)
        assert np.array_equal(counts[0, 0].cpu().numpy(), cnt_ref)


# ------------------------------------------------------------------------- forward / backward
ATTN_CASES = [
    # (family, N, d, B, H)
    ("causal_document", 128, 64, 1, 1),       # config C1 shape with bf16 inputs (fp32: test_fp32_inputs)
    ("causal", 256, 128, 1, 2),
    ("full", 384, 128, 2, 1),
    ("causal_document", 1000, 128, 2, 2),
    ("document", 640, 128, 1, 2),
    ("share_question", 896, 128, 1, 2),
    ("sliding_window", 1024, 128, 1, 1),
    ("global_sliding_window", 768, 128, 1, 2),
    ("causal_blockwise", 700, 128, 1, 1),
    ("prefix_lm_document", 512, 128, 1, 1),
    ("prefix_lm_causal", 640, 128, 1, 1),
    ("qk_sparse", 513, 128, 1, 1),
    ("hash_sparse", 600, 128, 1, 1),
    ("random_eviction", 512, 128, 1, 1),
    ("causal_document", 1000, 64, 2, 2),
    ("document", 257, 64, 1, 2),
    ("global_sliding_window", 700, 64, 1, 1),
    ("random_eviction", 384, 64, 1, 1),
    ("causal", 129, 128, 1, 1),
    ("full", 1, 128, 1, 1),
    ("full", 127, 64, 1, 1),
]


def _run(fmlib, fam, N, d, B, H, seed=0, flags=0, out_dtype=torch.float32):
    rng = np.random.default_rng(seed + N + d)
    masks = [wm.sample_family(fam, N, rng, (2, 5)) for _ in range(B)]
    sri, t = build_case(masks, H, d, base=seed)
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=out_dtype, flags=flags)
    dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, causal,
                                     out_dtype=out_dtype, flags=flags)
    torch.cuda.synchronize()
    return masks, sri, t, (o, lse, dq, dk, dv)


@pytest.mark.parametrize("fam,N,d,B,H", ATTN_CASES)
def test_fwd_bwd_parity(fmlib, fam, N, d, B, H):
    masks, sri, t, (o, lse, dq, dk, dv) = _run(fmlib, fam, N, d, B, H)
    sri_np = sri.numpy()
    for b in range(B):
        for h in range(H):
            O, L, (gq, gk, gv) = oracle_head(t, masks, sri_np, b, h, 1, masks[0].causal)
            assert_close(f"O[{b},{h}]", o[b, :, h].cpu().numpy(), O)
            assert_lse(lse[b, h].cpu().numpy(), L)
            assert_close(f"dQ[{b},{h}]", dq[b, :, h].cpu().numpy(), gq)
            assert_close(f"dK[{b},{h}]", dk[b, :, h].cpu().numpy(), gk)
            assert_close(f"dV[{b},{h}]", dv[b, :, h].cpu().numpy(), gv)


@pytest.mark.parametrize("fam,N,d", [("causal_document", 1000, 128), ("global_sliding_window", 768, 128),
                                     ("document", 640, 64), ("random_eviction", 512, 128)])
@pytest.mark.parametrize("bounded", [False, True])
def test_skip_equivalence_bitwise(fmlib, fam, N, d, bounded):
    """§4.4: skipping fully masked tiles changes nothing, bit for bit — for the two-pass
    forward and for the bounded single pass (R33, whose reference does not depend on the visit list)."""
    extra = fmlib.FM_FLAG_MAX_BOUND if bounded else 0
    _, _, _, r0 = _run(fmlib, fam, N, d, 1, 2, seed=3, flags=extra)
    _, _, _, r1 = _run(fmlib, fam, N, d, 1, 2, seed=3, flags=fmlib.FM_FLAG_NO_SKIP | extra)
    for name, a, b in zip(("O", "lse", "dK", "dV"), (r0[0], r0[1], r0[3], r0[4]), (r1[0], r1[1], r1[3], r1[4])):
        assert torch.equal(a, b), name


def test_bf16_outputs_close(fmlib):
    """bf16 outputs (the timing configuration) agree with fp32 outputs to bf16 rounding."""
    _, _, _, r32 = _run(fmlib, "causal_document", 1000, 128, 1, 2, seed=5)
    _, _, _, r16 = _run(fmlib, "causal_document", 1000, 128, 1, 2, seed=5, out_dtype=torch.bfloat16)
    for a, b in zip(r32, r16):
        if a.dtype == torch.float32 and b.dtype == torch.bfloat16:
            err = (a - b.float()).abs().max().item()
            assert err <= 0.02 * max(1.0, a.abs().max().item()), err
    assert torch.equal(r32[1], r16[1])


BF16_CASES = [("causal_document", 1000, 128, 2, 2), ("document", 257, 64, 1, 2), ("random_eviction", 129, 128, 1, 1),
              ("full", 127, 64, 1, 1), ("global_sliding_window", 700, 128, 1, 1), ("sliding_window", 384, 64, 1, 2)]


def _check_bf16_vs_fp32(fmlib, tc, sri_c, causal, r32, r16):
    # forward: the bf16 epilogue (shared-memory stage + TMA store) equals RNE(bf16) of the fp32
    # epilogue's values bit for bit — any swizzle / row / clipping error shows up here
    assert torch.equal(r16[0], r32[0].to(torch.bfloat16))
    assert torch.equal(r16[1], r32[1])
    # backward: rerun with fp32 outputs on the SAME (bf16-valued) O, so D = rowsum(dO o O) is
    # identical; dK / dV (atomic-free, deterministic) must then be RNE of the fp32 results bit for
    # bit; dQ (fp32 reduce-add, order-dependent) to within bf16 rounding
    dq32, dk32, dv32 = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], r16[0].float(), tc["do"], r16[1], sri_c, causal,
                                           out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(r16[3], dk32.to(torch.bfloat16)), "dK"
    assert torch.equal(r16[4], dv32.to(torch.bfloat16)), "dV"
    bad = (r16[2].float() - dq32).abs() > 2.0 ** -8 * dq32.abs() + 1e-5
    assert not bad.any(), ("dQ", torch.nonzero(bad)[:5].tolist())


@pytest.mark.parametrize("fam,N,d,B,H", BF16_CASES)
def test_bf16_outputs(fmlib, fam, N, d, B, H):
    """bf16 outputs (the timing configuration): ragged N, odd row-tile counts, d = 64 / 128."""
    _, _, _, r32 = _run(fmlib, fam, N, d, B, H, seed=7)
    masks, sri, t, r16 = _run(fmlib, fam, N, d, B, H, seed=7, out_dtype=torch.bfloat16)
    sri_c, tc = to_cuda(sri, t)
    _check_bf16_vs_fp32(fmlib, tc, sri_c, masks[0].causal, r32, r16)
    O, L, _ = oracle_head(t, masks, sri.numpy(), 0, 0, 1, masks[0].causal, with_grad=False)
    g = r16[0][0, :, 0].float().cpu().numpy()
    assert (np.abs(g - O) <= 2e-2 + 2.0 ** -8 * np.abs(O)).all()   # north_star bar + output rounding


@pytest.mark.parametrize("d", [64, 128])
def test_empty_tiles_bf16(fmlib, d):
    """CTAs with nothing to compute still write their (zero) outputs through the TMA-store
    epilogue: query rows [128, 256) masked for every key (an empty second query tile next to a
    busy first one), keys [256, 384) masked for every row (a key tile with no visited row tile)."""
    N = 640
    sri = np.zeros((N, 4), np.int32)
    sri[:, 0], sri[:, 1] = 128, 256          # lower interval [128, 256): rows 128..255 empty
    sri[:, 2], sri[:, 3] = 0, 0              # no upper interval
    sri[256:384, 0], sri[256:384, 1] = 0, N  # keys 256..383 masked for every row
    m = wm.MaskInput(N, False, 4, sri, "empty_tiles")
    sri_t, t = build_case([m], 2, d, base=11)
    sri_c, tc = to_cuda(sri_t, t)
    res = {}
    for dt in (torch.float32, torch.bfloat16):
        o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, False, out_dtype=dt)
        res[dt] = (o, lse, *fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, False,
                                                out_dtype=dt))
    torch.cuda.synchronize()
    r32, r16 = res[torch.float32], res[torch.bfloat16]
    assert (r16[0][:, 128:256] == 0).all() and torch.isneginf(r16[1][:, :, 128:256]).all()
    assert (r16[3][:, 256:384] == 0).all() and (r16[4][:, 256:384] == 0).all()
    _check_bf16_vs_fp32(fmlib, tc, sri_c, False, r32, r16)
    for h in range(2):
        O, L, (gq, gk, gv) = oracle_head(t, [m], sri_t.numpy(), 0, h, 1, False)
        assert_close("O", r32[0][0, :, h].cpu().numpy(), O)
        assert_lse(r32[1][0, h].cpu().numpy(), L)
        assert_close("dQ", r32[2][0, :, h].cpu().numpy(), gq)
        assert_close("dK", r32[3][0, :, h].cpu().numpy(), gk)
        assert_close("dV", r32[4][0, :, h].cpu().numpy(), gv)


def test_empty_rows(fmlib):
    """Rows masked in every column: O = 0, lse = -inf, zero dQ; padding keys get zero dK/dV."""
    m = wm.empty_rows_padding([100, 150], 50)
    sri, t = build_case([m], 2, 128)
    sri_c, tc = to_cuda(sri, t)
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, True, out_dtype=torch.float32)
    dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, True, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.isneginf(lse[:, :, 250:]).all() and (o[:, 250:] == 0).all() and (dq[:, 250:] == 0).all()
    for h in range(2):
        O, L, (gq, gk, gv) = oracle_head(t, [m], sri.numpy(), 0, h, 1, True)
        assert_close("O", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        assert_close("dK", dk[0, :, h].cpu().numpy(), gk)
        assert_close("dV", dv[0, :, h].cpu().numpy(), gv)


def test_masked_key_null_influence(fmlib):
    """perturbing K/V of keys masked for every row leaves every output bitwise unchanged."""
    m = wm.qk_sparse(512, [3, 200, 201, 450], (300, 310))
    sri, t = build_case([m], 2, 128)
    sri_c, tc = to_cuda(sri, t)
    run = lambda tt: (lambda o, l: (o, l, *fmlib.flashmask_bwd(tt["q"], tt["k"], tt["v"], o, tt["do"], l, sri_c, True)))(
        *fmlib.flashmask_fwd(tt["q"], tt["k"], tt["v"], sri_c, True))
    r0 = run(tc)
    tc2 = {k: v.clone() for k, v in tc.items()}
    tc2["k"][:, [3, 200, 201, 450]] += 1.5
    tc2["v"][:, [3, 200, 201, 450]] -= 2.0
    r1 = run(tc2)
    torch.cuda.synchronize()
    for a, b in zip(r0[:3], r1[:3]):
        assert torch.equal(a, b)
    keep = [i for i in range(512) if i not in (3, 200, 201, 450)]
    assert torch.equal(r0[3][:, keep], r1[3][:, keep]) and torch.equal(r0[4][:, keep], r1[4][:, keep])


def test_abi_errors(fmlib):
    q = torch.zeros(1, 128, 1, 96, dtype=torch.bfloat16, device="cuda")
    sri = torch.zeros(1, 1, 128, 1, dtype=torch.int32, device="cuda")
    with pytest.raises(fmlib.FlashMaskError) as e:
        fmlib.flashmask_fwd(q, q, q, sri, True)
    assert e.value.status == fmlib.FM_ERR_INVALID_ARGUMENT
    q = torch.zeros(1, 128, 1, 128, dtype=torch.bfloat16, device="cuda")
    sri4 = torch.zeros(1, 1, 128, 4, dtype=torch.int32, device="cuda")
    with pytest.raises(fmlib.FlashMaskError) as e:
        fmlib.flashmask_fwd(q, q, q, sri4, True)   # causal with C=4 is not in the C-table
    assert e.value.status == fmlib.FM_ERR_INVALID_ARGUMENT


# ------------------------------------------------------------------------- grouped-query attention
GQA_CASES = [("causal_document", 700, 128, 4, 2), ("document", 513, 128, 4, 1), ("share_question", 640, 64, 6, 3),
             ("global_sliding_window", 384, 64, 2, 1)]


@pytest.mark.parametrize("fam,N,d,H,Hkv", GQA_CASES)
def test_gqa_parity(fmlib, fam, N, d, H, Hkv):
    """query head h attends with key/value head h // (H/Hkv); dK/dV of a
    key/value head are the sums over its query heads (accumulated atomic-free in one CTA)."""
    from workloads import tensors as wt
    rng = np.random.default_rng(N + H)
    masks = [wm.sample_family(fam, N, rng, (2, 5))]
    sri = torch.from_numpy(wm.stack(masks, 1))
    q = wt.make_tensor("q", 1, N, H, d, base=9)
    do = wt.make_tensor("do", 1, N, H, d, base=9)
    k = wt.make_tensor("k", 1, N, Hkv, d, base=9)
    v = wt.make_tensor("v", 1, N, Hkv, d, base=9)
    causal = masks[0].causal
    qc, kc, vc, doc, sc = q.cuda(), k.cuda(), v.cuda(), do.cuda(), sri.cuda()
    o, lse = fmlib.flashmask_fwd(qc, kc, vc, sc, causal, out_dtype=torch.float32)
    dq, dk, dv = fmlib.flashmask_bwd(qc, kc, vc, o, doc, lse, sc, causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert dk.shape == (1, N, Hkv, d) and dq.shape == (1, N, H, d)
    vec = fo.expand(masks[0].sri, causal, N)
    G = H // Hkv
    f = lambda t, hh: t[0, :, hh, :].double().numpy()
    gk_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    gv_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    for h in range(H):
        hk = h // G
        O, L = fo.forward(f(q, h), f(k, hk), f(v, hk), vec)
        gq, gk, gv = fo.backward(f(q, h), f(k, hk), f(v, hk), f(do, h), vec)
        gk_sum[hk] += gk
        gv_sum[hk] += gv
        assert_close(f"O[{h}]", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        assert_close(f"dQ[{h}]", dq[0, :, h].cpu().numpy(), gq)
    for hk in range(Hkv):
        assert_close(f"dK[{hk}]", dk[0, :, hk].cpu().numpy(), gk_sum[hk], tol_max=2e-2 * G ** 0.5)
        assert_close(f"dV[{hk}]", dv[0, :, hk].cpu().numpy(), gv_sum[hk], tol_max=2e-2 * G ** 0.5)


# ------------------------------------------------------------------------- deterministic dQ
@pytest.mark.parametrize("fam,N,d,B,H", [("causal_document", 1000, 128, 2, 2), ("document", 640, 64, 1, 2),
                                         ("random_eviction", 513, 128, 1, 1), ("global_sliding_window", 384, 64, 1, 1),
                                         ("causal", 129, 128, 1, 1), ("full", 1, 128, 1, 1)])
def test_deterministic_dq(fmlib, fam, N, d, B, H):
    """SURVEY f1 / P:300: FM_FLAG_DETERMINISTIC gives bitwise reproducible dQ (two runs equal),
    within tolerance of the oracle; dK and dV are bitwise those of the default mode."""
    masks, sri, t, r0 = _run(fmlib, fam, N, d, B, H, seed=7, flags=fmlib.FM_FLAG_DETERMINISTIC)
    _, _, _, r1 = _run(fmlib, fam, N, d, B, H, seed=7, flags=fmlib.FM_FLAG_DETERMINISTIC)
    _, _, _, rd = _run(fmlib, fam, N, d, B, H, seed=7)
    assert torch.equal(r0[2], r1[2])
    assert torch.equal(r0[3], rd[3]) and torch.equal(r0[4], rd[4])
    for b in range(B):
        for h in range(H):
            _, _, (gq, _, _) = oracle_head(t, masks, sri.numpy(), b, h, 1, masks[0].causal)
            assert_close(f"det dQ[{b},{h}]", r0[2][b, :, h].cpu().numpy(), gq)


# ------------------------------------------------------------------------- fp32 inputs (config C1)
# The fp32 path computes in fp32 throughout (reading R26), so its bar is far tighter than the
# bf16 north_star bar: fp32 rounding over <= 1000-term sums of O(1) values stays below 1e-4
# (this would fail for any path that rounded the inputs to bf16: |x|·2^-9 ~ 4e-3).
TOL32 = dict(tol_max=1e-4, tol_mean=1e-5)
F32_CASES = [
    # (mask builder, d, H, Hkv, out dtype)
    (lambda: wm.causal_document([40, 48, 40]), 64, 1, 1, torch.float32),     # config C1 exactly
    (lambda: wm.causal_document([1, 126, 1]), 64, 1, 1, torch.float32),      # C1 seeded variant
    (lambda: wm.global_sliding_window(257, 16, 40), 128, 2, 1, torch.float32),
    (lambda: wm.document([100, 200, 33]), 64, 3, 3, torch.float32),
    (lambda: wm.random_eviction(300, 19, np.random.default_rng(3)), 128, 2, 2, torch.float32),
    (lambda: wm.empty_rows_padding([60, 70], 20), 64, 1, 1, torch.float32),
    (lambda: wm.causal(200), 128, 1, 1, torch.bfloat16),
]


@pytest.mark.parametrize("case", range(len(F32_CASES)))
def test_fp32_inputs(fmlib, case):
    from workloads import tensors as wt
    build, d, H, Hkv, out_dtype = F32_CASES[case]
    m = build()
    N = m.N
    sri = torch.from_numpy(wm.stack([m], 1))
    q = wt.make_tensor("q", 1, N, H, d, base=5, dtype=torch.float32)
    do = wt.make_tensor("do", 1, N, H, d, base=5, dtype=torch.float32)
    k = wt.make_tensor("k", 1, N, Hkv, d, base=5, dtype=torch.float32)
    v = wt.make_tensor("v", 1, N, Hkv, d, base=5, dtype=torch.float32)
    qc, kc, vc, doc, sc = q.cuda(), k.cuda(), v.cuda(), do.cuda(), sri.cuda()
    o, lse = fmlib.flashmask_fwd(qc, kc, vc, sc, m.causal, out_dtype=out_dtype)
    dq, dk, dv = fmlib.flashmask_bwd(qc, kc, vc, o, doc, lse, sc, m.causal, out_dtype=out_dtype)
    dq2, dk2, dv2 = fmlib.flashmask_bwd(qc, kc, vc, o, doc, lse, sc, m.causal, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)  # no atomics
    vec = fo.expand(m.sri, m.causal, N)
    G = H // Hkv
    f = lambda t, hh: t[0, :, hh, :].double().numpy()
    tol = TOL32 if out_dtype == torch.float32 else {}
    gk_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    gv_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    for h in range(H):
        hk = h // G
        O, L = fo.forward(f(q, h), f(k, hk), f(v, hk), vec)
        gq, gk, gv = fo.backward(f(q, h), f(k, hk), f(v, hk), f(do, h), vec)
        gk_sum[hk] += gk
        gv_sum[hk] += gv
        assert_close(f"fp32 O[{h}]", o[0, :, h].float().cpu().numpy(), O, **tol)
        assert_lse(lse[0, h].cpu().numpy(), L, tol=1e-5)
        assert_close(f"fp32 dQ[{h}]", dq[0, :, h].float().cpu().numpy(), gq, **tol)
    for hk in range(Hkv):
        assert_close(f"fp32 dK[{hk}]", dk[0, :, hk].float().cpu().numpy(), gk_sum[hk], **tol)
        assert_close(f"fp32 dV[{hk}]", dv[0, :, hk].float().cpu().numpy(), gv_sum[hk], **tol)


def test_back_to_back_shared_workspace(fmlib):
    """Programmatic dependent launch (fm_ptx.cuh pdl_wait): consecutive calls on one stream that
    reuse ONE workspace and consume each other's outputs give exactly the results of isolated,
    synchronised calls (no kernel may touch the workspace or a predecessor's output early)."""
    masks_a = [wm.sample_family("causal_document", 1000, np.random.default_rng(1), (2, 5))]
    masks_b = [wm.sample_family("sliding_window", 1000, np.random.default_rng(2), (2, 5))]
    sri_a, t_a = build_case(masks_a, 4, 128, base=21)
    sri_b, t_b = build_case(masks_b, 4, 128, base=22)
    (sa, ta), (sb, tb) = to_cuda(sri_a, t_a), to_cuda(sri_b, t_b)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")

    def chain(sync):
        res = []
        for s, t in ((sa, ta), (sb, tb), (sa, ta)):
            o, lse = fmlib.flashmask_fwd(t["q"], t["k"], t["v"], s, True, workspace=ws)
            if sync:
                torch.cuda.synchronize()
            g = fmlib.flashmask_bwd(t["q"], t["k"], t["v"], o, t["do"], lse, s, True, workspace=ws)
            if sync:
                torch.cuda.synchronize()
            res.append((o, lse, *g))
        torch.cuda.synchronize()
        return res

    ref, got = chain(True), chain(False)
    for r, g in zip(ref, got):
        for name, a, b in zip(("O", "lse", "dQ", "dK", "dV"), r, g):
            if name == "dQ":   # fp32 reduce-add order may differ between runs: one bf16 ulp
                assert ((a.float() - b.float()).abs() <= 2.0 ** -7 * a.float().abs() + 1e-3).all(), name
            else:
                assert torch.equal(a, b), name


def test_chunked_calls_match_full_call(fmlib):
    """bench.py's e2e leg splits a step into one call per (batch entry, head group) — heads and
    batch entries are independent.  The chunked calls reproduce the full call: O, lse, dK,
    dV bitwise (atomic-free), dQ to one bf16 ulp (fp32 reduce-add order)."""
    masks = [wm.sample_family("document", 900, np.random.default_rng(s), (2, 5)) for s in (7, 8)]
    causal = masks[0].causal
    sri, t = build_case(masks, 8, 128, base=31)
    s, t = to_cuda(sri, t)
    o, lse = fmlib.flashmask_fwd(t["q"], t["k"], t["v"], s, causal)
    dq, dk, dv = fmlib.flashmask_bwd(t["q"], t["k"], t["v"], o, t["do"], lse, s, causal)
    HG = 2
    for b in range(2):
        for h0 in range(0, 8, HG):
            c = {k: v[b:b + 1, :, h0:h0 + HG].contiguous() for k, v in t.items()}
            sc = s[b:b + 1].contiguous()
            oc, lc = fmlib.flashmask_fwd(c["q"], c["k"], c["v"], sc, causal)
            gq, gk, gv = fmlib.flashmask_bwd(c["q"], c["k"], c["v"], oc, c["do"], lc, sc, causal)
            assert torch.equal(oc, o[b:b + 1, :, h0:h0 + HG])
            assert torch.equal(lc, lse[b:b + 1, h0:h0 + HG])
            assert torch.equal(gk, dk[b:b + 1, :, h0:h0 + HG])
            assert torch.equal(gv, dv[b:b + 1, :, h0:h0 + HG])
            ref = dq[b:b + 1, :, h0:h0 + HG].float()
            assert ((gq.float() - ref).abs() <= 2.0 ** -7 * ref.abs() + 1e-3).all()
    torch.cuda.synchronize()


# ------------------------------------------------------------------------- fp16 inputs
FP16_CASES = [("causal_document", 1000, 128, 1, 2), ("document", 257, 64, 1, 2), ("random_eviction", 384, 128, 1, 1),
              ("global_sliding_window", 700, 64, 1, 1)]


@pytest.mark.parametrize("fam,N,d,B,H", FP16_CASES)
def test_fp16_inputs(fmlib, fam, N, d, B, H):
    """fp16 q/k/v/dO run the same tcgen05 kernels with fp16 operands (P, dS packed as fp16):
    fp32 outputs within the north_star bars of the fp64 oracle on the same fp16 values; fp16
    outputs bit-equal to RNE(fp16) of the fp32 outputs (forward) / of the fp32-output backward
    on the same fp16 O (dK, dV), dQ within fp16 rounding."""
    from workloads import tensors as wt
    rng = np.random.default_rng(N + d)
    masks = [wm.sample_family(fam, N, rng, (2, 5)) for _ in range(B)]
    sri = torch.from_numpy(wm.stack(masks, 1))
    t = {n: wt.make_tensor(n, B, N, H, d, base=13, dtype=torch.float16) for n in ("q", "k", "v", "do")}
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    o32, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32)
    g32 = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o32, tc["do"], lse, sri_c, causal, out_dtype=torch.float32)
    o16, lse16 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal)
    g16 = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o16, tc["do"], lse16, sri_c, causal)
    h32 = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o16.float(), tc["do"], lse16, sri_c, causal,
                              out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert o16.dtype == torch.float16 and g16[0].dtype == torch.float16
    assert torch.equal(o16, o32.to(torch.float16)) and torch.equal(lse16, lse)
    assert torch.equal(g16[1], h32[1].to(torch.float16)) and torch.equal(g16[2], h32[2].to(torch.float16))
    assert ((g16[0].float() - h32[0]).abs() <= 2.0 ** -10 * h32[0].abs() + 1e-4).all()
    sri_np = sri.numpy()
    for b in range(B):
        for h in range(H):
            O, L, (gq, gk, gv) = oracle_head(t, masks, sri_np, b, h, 1, causal)
            assert_close(f"O[{b},{h}]", o32[b, :, h].cpu().numpy(), O)
            assert_lse(lse[b, h].cpu().numpy(), L)
            assert_close(f"dQ[{b},{h}]", g32[0][b, :, h].cpu().numpy(), gq)
            assert_close(f"dK[{b},{h}]", g32[1][b, :, h].cpu().numpy(), gk)
            assert_close(f"dV[{b},{h}]", g32[2][b, :, h].cpu().numpy(), gv)


def test_fp16_dtype_errors(fmlib):
    q = torch.zeros(1, 128, 1, 128, dtype=torch.float16, device="cuda")
    sri = torch.full((1, 1, 128, 1), 128, dtype=torch.int32, device="cuda")
    with pytest.raises(fmlib.FlashMaskError) as e:
        fmlib.flashmask_fwd(q, q, q, sri, True, out_dtype=torch.bfloat16)   # fp16 in, bf16 out
    assert e.value.status == fmlib.FM_ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("d", [64, 128])
def test_fp16_deterministic_dq(fmlib, d):
    """fp16 inputs with FM_FLAG_DETERMINISTIC (row-parallel dQ kernel K6 with fp16 operands):
    bitwise reproducible dQ, dK/dV bitwise those of the default fp16 run, dQ vs the oracle."""
    from workloads import tensors as wt
    N, H = 700, 2
    masks = [wm.sample_family("causal_document", N, np.random.default_rng(d), (2, 5))]
    sri = torch.from_numpy(wm.stack(masks, 1))
    t = {n: wt.make_tensor(n, 1, N, H, d, base=17, dtype=torch.float16) for n in ("q", "k", "v", "do")}
    sri_c, tc = to_cuda(sri, t)
    outs = []
    for flags in (fmlib.FM_FLAG_DETERMINISTIC, fmlib.FM_FLAG_DETERMINISTIC, 0):
        o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, True, out_dtype=torch.float32, flags=flags)
        outs.append(fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, True,
                                        out_dtype=torch.float32, flags=flags))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[2][1]) and torch.equal(outs[0][2], outs[2][2])
    for h in range(H):
        _, _, (gq, _, _) = oracle_head(t, masks, sri.numpy(), 0, h, 1, True)
        assert_close(f"fp16 det dQ[{h}]", outs[0][0][0, :, h].cpu().numpy(), gq)


@pytest.mark.parametrize("d", [64, 128])
def test_gqa_per_kv_head_masks(fmlib, d):
    """one mask per key/value head (mask_heads = num_kv_heads): query head h uses the
    mask of its key/value head h // G; different families per kv head."""
    from workloads import tensors as wt
    N, H, Hkv = 520, 4, 2
    rng = np.random.default_rng(d)
    masks = [wm.sample_family("causal_document", N, rng, (2, 5)), wm.sample_family("sliding_window", N, rng, (2, 5))]
    assert masks[0].causal == masks[1].causal and masks[0].C == masks[1].C
    sri = torch.from_numpy(np.stack([m.sri for m in masks])[None].copy())  # [1, Hkv, N, C]
    q = wt.make_tensor("q", 1, N, H, d, base=23)
    do = wt.make_tensor("do", 1, N, H, d, base=23)
    k = wt.make_tensor("k", 1, N, Hkv, d, base=23)
    v = wt.make_tensor("v", 1, N, Hkv, d, base=23)
    qc, kc, vc, doc, sc = q.cuda(), k.cuda(), v.cuda(), do.cuda(), sri.cuda()
    o, lse = fmlib.flashmask_fwd(qc, kc, vc, sc, True, out_dtype=torch.float32)
    dq, dk, dv = fmlib.flashmask_bwd(qc, kc, vc, o, doc, lse, sc, True, out_dtype=torch.float32)
    torch.cuda.synchronize()
    G = H // Hkv
    f = lambda t, hh: t[0, :, hh, :].double().numpy()
    gk_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    gv_sum = [np.zeros((N, d)) for _ in range(Hkv)]
    for h in range(H):
        hk = h // G
        vec = fo.expand(masks[hk].sri, True, N)
        O, L = fo.forward(f(q, h), f(k, hk), f(v, hk), vec)
        gq, gk, gv = fo.backward(f(q, h), f(k, hk), f(v, hk), f(do, h), vec)
        gk_sum[hk] += gk
        gv_sum[hk] += gv
        assert_close(f"O[{h}]", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        assert_close(f"dQ[{h}]", dq[0, :, h].cpu().numpy(), gq)
    for hk in range(Hkv):
        assert_close(f"dK[{hk}]", dk[0, :, hk].cpu().numpy(), gk_sum[hk], tol_max=2e-2 * G ** 0.5)
        assert_close(f"dV[{hk}]", dv[0, :, hk].cpu().numpy(), gv_sum[hk], tol_max=2e-2 * G ** 0.5)


RANDOM_CASES = list(range(48))


@pytest.mark.parametrize("seed", RANDOM_CASES)
def test_random_configurations(fmlib, seed):
    """Seeded random configurations (family, ragged N, d, B, H / Hkv, input and output dtype,
    deterministic flag) against the oracle — catches combinations the fixed cases miss."""
    from workloads import tensors as wt
    rng = np.random.default_rng(1000 + seed)
    fam = wm.FAMILIES[int(rng.integers(len(wm.FAMILIES)))]
    N = int(rng.integers(1, 600))
    d = int(rng.choice([64, 128]))
    Hkv = int(rng.integers(1, 3))
    G = int(rng.integers(1, 3))
    H = Hkv * G
    B = int(rng.integers(1, 3))
    in_dt = [torch.bfloat16, torch.float16][int(rng.integers(2))]
    flags = fmlib.FM_FLAG_DETERMINISTIC if rng.random() < 0.3 else 0
    masks = [wm.sample_family(fam, N, rng, (1, 4)) for _ in range(B)]
    sri = torch.from_numpy(wm.stack(masks, 1))
    t = {}
    for n, heads in (("q", H), ("do", H), ("k", Hkv), ("v", Hkv)):
        t[n] = wt.make_tensor(n, B, N, heads, d, base=seed, dtype=in_dt)
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32, flags=flags)
    dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, causal,
                                     out_dtype=torch.float32, flags=flags)
    torch.cuda.synchronize()
    f = lambda x, b, hh: x[b, :, hh, :].double().numpy()
    for b in range(B):
        vec = fo.expand(masks[b].sri, causal, N)
        gk_sum = [np.zeros((N, d)) for _ in range(Hkv)]
        gv_sum = [np.zeros((N, d)) for _ in range(Hkv)]
        for h in range(H):
            hk = h // G
            O, L = fo.forward(f(t["q"], b, h), f(t["k"], b, hk), f(t["v"], b, hk), vec)
            gq, gk, gv = fo.backward(f(t["q"], b, h), f(t["k"], b, hk), f(t["v"], b, hk), f(t["do"], b, h), vec)
            gk_sum[hk] += gk
            gv_sum[hk] += gv
            tag = f"{fam} N={N} d={d} B={B} H={H}/{Hkv} {in_dt} flags={flags} [{b},{h}]"
            assert_close(f"O {tag}", o[b, :, h].cpu().numpy(), O)
            assert_lse(lse[b, h].cpu().numpy(), L)
            assert_close(f"dQ {tag}", dq[b, :, h].cpu().numpy(), gq)
        for hk in range(Hkv):
            assert_close(f"dK {fam} [{b},{hk}]", dk[b, :, hk].cpu().numpy(), gk_sum[hk], tol_max=2e-2 * G ** 0.5)
            assert_close(f"dV {fam} [{b},{hk}]", dv[b, :, hk].cpu().numpy(), gv_sum[hk], tol_max=2e-2 * G ** 0.5)


@pytest.mark.parametrize("causal", [True, False])
def test_sliding_window_indices(fmlib, causal):
    """SURVEY f4 sliding-window shortcut: the device-generated startend_row_indices expand (oracle)
    to exactly the window predicate — causal: visible iff 0 <= r - y < w; bidirectional: |r - y| < w —
    and drive the attention kernels to the oracle's result."""
    N, w, B = 777, 100, 2
    sri = fmlib.flashmask_sliding_window_indices(B, N, w, causal)
    torch.cuda.synchronize()
    s = sri.cpu().numpy()
    r = np.arange(N)[:, None]
    y = np.arange(N)[None, :]
    want = ~((r - y >= 0) & (r - y < w)) if causal else ~(np.abs(r - y) < w)
    for b in range(B):
        vec = fo.expand(s[b, 0], causal, N)
        assert np.array_equal(fo.to_dense(vec), want)
    if causal:
        assert np.array_equal(s[0, 0, :, 0], wm.sliding_window(N, w).sri[:, 0])
    m = wm.MaskInput(N, causal, s.shape[-1], s[0, 0], "sliding_window_api")
    sri_t, t = build_case([m], 2, 128, base=31)
    sri_c, tc = to_cuda(sri_t, t)
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    O, L, _ = oracle_head(t, [m], sri_t.numpy(), 0, 1, 1, causal, with_grad=False)
    assert_close("O", o[0, :, 1].cpu().numpy(), O)
    assert_lse(lse[0, 1].cpu().numpy(), L)
    with pytest.raises(fmlib.FlashMaskError):
        fmlib.flashmask_sliding_window_indices(1, 16, 0, causal)


# ------------------------------------------------------------------ arbitrary int32 intervals (R10)
INT32_CASES = [(causal, C, N, d) for causal, C in ((True, 1), (True, 2), (False, 2), (False, 4))
               for N, d in ((333, 128), (700, 64))]


@pytest.mark.parametrize("causal,C,N,d", INT32_CASES)
def test_fwd_bwd_arbitrary_int32_vectors(fmlib, causal, C, N, d):
    """R10 / flashmask.h: ANY int32 startend_row_indices has defined semantics through the
    masked(r, y) predicate (Eq. 3): negative, > N, inverted (start >= end),
    INT_MIN / INT_MAX.  The attention kernels (clamp + (start, length) normalisation in K1a)
    must give the oracle's O / lse / dQ / dK / dV on such vectors, ragged N, both head dims."""
    rng = np.random.default_rng(N * 7 + C + 100 * causal)
    i32 = np.iinfo(np.int32)
    raw = rng.integers(-N, 2 * N, size=(N, C)).astype(np.int64)
    # a share of ordinary well-formed columns so most rows keep visible keys
    ok = rng.random(N) < 0.5
    raw[ok, 0] = rng.integers(0, N + 1, ok.sum())
    if C >= 2:
        raw[ok, 1] = np.maximum(raw[ok, 0], rng.integers(0, N + 1, ok.sum())) if causal or C == 4 else \
            rng.integers(0, N + 1, ok.sum())
    special = [i32.max, i32.min, -1, 0, N, N + 1, i32.max - 1, i32.min + 1]
    for j in range(min(N, 40)):
        raw[j * (N // 40), int(rng.integers(C))] = special[j % len(special)]
    raw = raw.astype(np.int32)
    m = wm.MaskInput(N, causal, C, raw, "arbitrary_int32")
    sri_t, t = build_case([m], 2, d, base=N + C)
    sri_c, tc = to_cuda(sri_t, t)
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32)
    dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, causal,
                                     out_dtype=torch.float32)
    torch.cuda.synchronize()
    for h in range(2):
        O, L, (gq, gk, gv) = oracle_head(t, [m], sri_t.numpy(), 0, h, 1, causal)
        assert_close(f"O[{h}]", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        assert_close(f"dQ[{h}]", dq[0, :, h].cpu().numpy(), gq)
        assert_close(f"dK[{h}]", dk[0, :, h].cpu().numpy(), gk)
        assert_close(f"dV[{h}]", dv[0, :, h].cpu().numpy(), gv)


# ------------------------------------------------------------------ binding argument checks
def test_binding_rejects_bad_tensors(fmlib):
    """The binding passes raw pointers to the C ABI, so it refuses what the kernels would
    misread: non-contiguous views, non-int32 masks, mixed dtypes, and a backward whose o has a
    different dtype than the requested gradients."""
    N, H, d = 256, 2, 128
    qkv = torch.randn(1, N, 3, H, d, device="cuda").to(torch.bfloat16)
    q, k, v = qkv.unbind(2)                      # strided views
    sri = torch.full((1, 1, N, 1), N, dtype=torch.int32, device="cuda")
    E = fmlib.FlashMaskError
    with pytest.raises(E, match="contiguous"):
        fmlib.flashmask_fwd(q, k, v, sri, True)
    q, k, v = (x.contiguous() for x in (q, k, v))
    with pytest.raises(E, match="int32"):
        fmlib.flashmask_fwd(q, k, v, sri.long(), True)
    with pytest.raises(E, match="dtype"):
        fmlib.flashmask_fwd(q, k.half(), v, sri, True)
    o32, lse = fmlib.flashmask_fwd(q, k, v, sri, True, out_dtype=torch.float32)
    do = torch.randn_like(q)
    with pytest.raises(E, match="out_dtype"):
        fmlib.flashmask_bwd(q, k, v, o32, do, lse, sri, True, out_dtype=torch.bfloat16)
    # o.dtype decides the gradient dtype: the fp32 O of the forward gives fp32 gradients
    dq, dk, dv = fmlib.flashmask_bwd(q, k, v, o32, do, lse, sri, True)
    ref = fmlib.flashmask_bwd(q, k, v, o32, do, lse, sri, True, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert dq.dtype == torch.float32 and torch.equal(dk, ref[1]) and torch.equal(dv, ref[2])
    with pytest.raises(E, match="shape"):
        fmlib.flashmask_bwd(q, k, v, o32, do, lse[:, :1], sri, True)



# ------------------------------------------------------------------ f3 refinement (K1c)
REFINE_CASES = [(fam, N) for fam in wm.FAMILIES for N in (129, 700)] + \
               [("qk_sparse", 4096), ("random_eviction", 4096), ("causal_blockwise", 4096), ("document", 4096)]


@pytest.mark.parametrize("fam,N", REFINE_CASES)
def test_refine_words_bit_exact(fmlib, fam, N):
    """f3 (R31): the refinement words of every tile equal the oracle's refine_chunks bit for
    bit, and the counts (PARTIAL tiles without a masked cell, dirty sub-blocks) follow."""
    rng = np.random.default_rng(N + 7 * len(fam))
    masks = [wm.sample_family(fam, N, rng, (2, 6)) for _ in range(2)]
    sri = torch.from_numpy(wm.stack(masks, 1)).cuda()
    words, counts = fmlib.flashmask_refine(sri, masks[0].causal)
    torch.cuda.synchronize()
    for b, m in enumerate(masks):
        vec = fo.expand(m.sri, m.causal, N)
        ref = fo.refine_chunks(vec)
        cm, _, _ = fo.classify(vec, 128, 128)
        got = words[b, 0].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, ref), np.argwhere(got != ref)[:5]
        part = cm == fo.PARTIAL
        clean = int((ref[part] == 0).sum())
        dirty = int(sum(bin(int(w)).count("1") for w in ref[part]))
        assert counts[b, 0].tolist() == [clean, dirty]


@pytest.mark.parametrize("fam,N,d", [("qk_sparse", 1000, 128), ("random_eviction", 777, 64), ("causal_document", 900, 128),
                                     ("global_sliding_window", 640, 64), ("hash_sparse", 513, 128)])
def test_refine_forward_bitwise(fmlib, fam, N, d):
    """Masking only the dirty sub-blocks of PARTIAL tiles is exact: O and lse are bitwise those
    of the unrefined forward (FM_FLAG_NO_REFINE), both vs the oracle."""
    _, _, _, r0 = _run(fmlib, fam, N, d, 1, 2, seed=9)
    masks, sri, t, r1 = _run(fmlib, fam, N, d, 1, 2, seed=9, flags=fmlib.FM_FLAG_NO_REFINE)
    assert torch.equal(r0[0], r1[0]) and torch.equal(r0[1], r1[1])
    for h in range(2):
        O, L, _ = oracle_head(t, masks, sri.numpy(), 0, h, 1, masks[0].causal, with_grad=False)
        assert_close(f"O[{h}]", r0[0][0, :, h].cpu().numpy(), O)
        assert_lse(r0[1][0, h].cpu().numpy(), L)


# ------------------------------------------------ R33 bounded single pass (K1e + K2a BND + fixup)
def _aligned(N, H, d, seed):
    """Q rows and keys along one direction with small noise: Cauchy-Schwarz is nearly tight, so
    the fixed reference sits ~64 above the true row maximum (P up to ~2^64 before normalising)."""
    g = torch.Generator().manual_seed(seed)
    q = 0.05 * torch.randn(1, N, H, d, generator=g)
    q[..., 0] = 12.0
    k = 0.05 * torch.randn(1, N, H, d, generator=g)
    k[..., 0] = 1.0 + torch.rand(1, N, H, generator=g)
    v = torch.randn(1, N, H, d, generator=g)
    do = torch.randn(1, N, H, d, generator=g)
    return {n: x.to(torch.bfloat16) for n, x in (("q", q), ("k", k), ("v", v), ("do", do))}


@pytest.mark.parametrize("fam,N,d", [("full", 1024, 128), ("full", 1000, 64), ("causal_document", 1024, 128),
                                     ("document", 896, 64), ("qk_sparse", 1024, 128), ("random_eviction", 640, 128)])
@pytest.mark.parametrize("inputs", ["unit", "aligned", "large_norm"])
def test_bounded_single_pass(fmlib, fam, N, d, inputs):
    """R33 (forced at small N with FM_FLAG_MAX_BOUND; the default from N = 16K, covered by
    test_gpu_fullsize): with bf16 operands the forward computes every P of a row against one fixed reference
    (the Cauchy-Schwarz bound of its logits minus 64) in a single pass per tile, and rows whose sum
    ends below 2^-60 are recomputed by the two-pass kernel.  Against the oracle and against
    FM_FLAG_NO_MAX_BOUND: unit-normal inputs (single pass), Q and K aligned (tight bound, P near
    2^64), large norms (bound far too loose: every unit recomputed, so the result equals the
    two-pass run bit for bit); qk_sparse has fully masked rows (recomputed: O = 0, lse = -inf)."""
    rng = np.random.default_rng(N + d)
    m = wm.sample_family(fam, N, rng, (2, 5))
    H = 2
    if inputs == "aligned":
        t = _aligned(N, H, d, seed=d)
    else:
        t = wt.make_qkv(1, N, H, d, base=7)
        if inputs == "large_norm":
            t = {n: (x.float() * (4.0 if n in ("q", "k") else 1.0)).to(torch.bfloat16) for n, x in t.items()}
    sri = torch.from_numpy(wm.stack([m]))
    sri_c, tc = to_cuda(sri, t)
    res = {}
    for flags in (fmlib.FM_FLAG_MAX_BOUND, fmlib.FM_FLAG_NO_MAX_BOUND):
        o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, m.causal, out_dtype=torch.float32, flags=flags)
        dq, dk, dv = fmlib.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, m.causal,
                                         out_dtype=torch.float32)
        torch.cuda.synchronize()
        res[flags] = (o, lse, dq, dk, dv)
    vec = fo.expand(m.sri, m.causal, N)
    for h in range(H):
        f = lambda n: t[n][0, :, h, :].double().numpy()
        O, L = fo.forward(f("q"), f("k"), f("v"), vec)
        _, _, gv = fo.backward(f("q"), f("k"), f("v"), f("do"), vec)
        for flags, (o, lse, dq, dk, dv) in res.items():
            assert_close(f"{inputs} O[h{h}] flags={flags}", o[0, :, h].cpu().numpy(), O)
            assert_lse(lse[0, h].cpu().numpy(), L)
            assert_close(f"{inputs} dV[h{h}] flags={flags}", dv[0, :, h].cpu().numpy(), gv)
    a, b = res[fmlib.FM_FLAG_MAX_BOUND], res[fmlib.FM_FLAG_NO_MAX_BOUND]
    if inputs == "large_norm":
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])  # every unit went through the fixup
    elif fam != "qk_sparse":
        assert not torch.equal(a[0], b[0])  # the single pass ran (another reference, other rounding)


def test_bounded_fixup_many_units_bitwise(fmlib):
    """R33 persistent fixup: with norms far too large for the bound every unit is flagged, and the
    one-wave fixup launch (one CTA per SM) runs 512 units, several per CTA with its mbarriers
    re-initialised between units — O and lse equal the two-pass forward bit for bit."""
    rng = np.random.default_rng(11)
    N, H, d = 4096, 32, 128
    m = wm.sample_family("causal_document", N, rng, (3, 7))
    t = wt.make_qkv(1, N, H, d, base=13, with_do=False)
    t = {n: (x.float() * 4.0 if n in ("q", "k") else x.float()).to(torch.bfloat16) for n, x in t.items()}
    sri_c, tc = to_cuda(torch.from_numpy(wm.stack([m])), t)
    res = []
    for flags in (fmlib.FM_FLAG_MAX_BOUND, fmlib.FM_FLAG_NO_MAX_BOUND):
        for out_dtype in (torch.float32, torch.bfloat16):
            res.append(fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, m.causal, out_dtype=out_dtype, flags=flags))
    torch.cuda.synchronize()
    for a, b in ((res[0], res[2]), (res[1], res[3])):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("d,H,Hkv", [(128, 8, 2), (64, 4, 1)])
def test_bounded_gqa_bf16_out(fmlib, d, H, Hkv):
    """R33 with GQA (the key-norm bound of the shared kv head) and bf16 outputs, against the oracle
    (bf16 output rounding added to the bar, R27)."""
    rng = np.random.default_rng(d + H)
    N = 1000
    m = wm.sample_family("causal_document", N, rng, (2, 5))
    q = wt.make_tensor("q", 1, N, H, d, base=3)
    k = wt.make_tensor("k", 1, N, Hkv, d, base=3)
    v = wt.make_tensor("v", 1, N, Hkv, d, base=3)
    sri_c = torch.from_numpy(wm.stack([m])).cuda()
    o, lse = fmlib.flashmask_fwd(q.cuda(), k.cuda(), v.cuda(), sri_c, m.causal, out_dtype=torch.bfloat16,
                                 flags=fmlib.FM_FLAG_MAX_BOUND)
    torch.cuda.synchronize()
    vec = fo.expand(m.sri, m.causal, N)
    G = H // Hkv
    for h in range(H):
        O, L = fo.forward(q[0, :, h].double().numpy(), k[0, :, h // G].double().numpy(),
                          v[0, :, h // G].double().numpy(), vec)
        got = o[0, :, h].float().cpu().double().numpy()
        err = np.abs(got - O)
        assert (err <= 2e-2 + np.abs(O) * 2.0 ** -8).all() and err.mean() <= 2e-3, (h, err.max(), err.mean())
        assert_lse(lse[0, h].cpu().numpy(), L)
