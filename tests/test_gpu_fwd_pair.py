"""K2b (CTA-pair forward, FM_FLAG_FWD_PAIR, fm_fwd2.cu) against the fp64 oracle and against the
single-SM forward K2a on the same inputs.  Alg. 1; exactness P:273-275."""
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
    from paper_2410_01359_b200 import flashmask
    return flashmask


def _inputs(fam, N, B, H, Hkv, seed, dtype=torch.bfloat16, heads_per_mask=1):
    rng = np.random.default_rng(7000 + seed + N)
    masks = [wm.sample_family(fam, N, rng, (1, 5)) for _ in range(B)]
    sri = torch.from_numpy(wm.stack(masks, heads_per_mask))
    t = {}
    for n, heads in (("q", H), ("k", Hkv), ("v", Hkv)):
        t[n] = wt.make_tensor(n, B, N, heads, 128, base=seed, dtype=dtype)
    return masks, sri, t


CASES = [(fam, N) for fam in wm.FAMILIES for N in (129, 700)] + [
    ("causal_document", 1), ("full", 1), ("document", 127), ("causal", 128), ("causal", 255), ("causal", 256),
    ("random_eviction", 1000), ("qk_sparse", 1536), ("global_sliding_window", 2100), ("share_question", 1333),
]


@pytest.mark.parametrize("fam,N", CASES)
def test_pair_forward_vs_oracle_and_single(fmlib, fam, N):
    B, H = 2, 2
    masks, sri, t = _inputs(fam, N, B, H, H, seed=len(fam))
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    o2, l2 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32,
                                 flags=fmlib.FM_FLAG_FWD_PAIR)
    o1, l1 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    # same running-max decisions and PV order; the two kernels split exp2 differently between MUFU
    # and the polynomial (1 vs 3 pairs of 8), so some P values round to a neighbouring bf16 — up to
    # ~5e-3 in O where few keys are visible (P near 1); both are checked against the oracle below
    assert torch.allclose(o2, o1, atol=1e-2, rtol=0), (o2 - o1).abs().max().item()
    fin = torch.isfinite(l1)
    assert torch.equal(fin, torch.isfinite(l2))
    assert torch.allclose(l2[fin], l1[fin], atol=1e-4, rtol=0)
    f = lambda x, b, h: x[b, :, h, :].double().numpy()
    for b in range(B):
        vec = fo.expand(masks[b].sri, causal, N)
        for h in range(H):
            O, L = fo.forward(f(t["q"], b, h), f(t["k"], b, h), f(t["v"], b, h), vec)
            assert_close(f"O {fam} N={N} [{b},{h}]", o2[b, :, h].cpu().numpy(), O)
            assert_lse(l2[b, h].cpu().numpy(), L)


@pytest.mark.parametrize("fam,N", [("causal_document", 1000), ("document", 900), ("qk_sparse", 777),
                                   ("global_sliding_window", 640)])
def test_pair_forward_skip_equivalence(fmlib, fam, N):
    """Visiting every tile (FM_FLAG_NO_SKIP) gives the same O and lse.  Not bitwise for
    K2b: the two softmax warpsets take alternate visit-list entries and keep separate row-sum
    shares, so extra (all-zero) tiles change which share a tile's row sum joins — the rounding of
    the final l, nothing else (P, the running maxima and the PV sum are identical)."""
    masks, sri, t = _inputs(fam, N, 1, 2, 2, seed=3)
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    F = fmlib.FM_FLAG_FWD_PAIR
    oa, la = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32, flags=F)
    ob, lb = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32,
                                 flags=F | fmlib.FM_FLAG_NO_SKIP)
    torch.cuda.synchronize()
    assert torch.allclose(oa, ob, rtol=1e-6, atol=1e-7), (oa - ob).abs().max().item()
    assert torch.allclose(la, lb, rtol=0, atol=1e-6)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("fam,N", [("causal_document", 1000), ("sliding_window", 515), ("prefix_lm_document", 640)])
def test_pair_forward_16bit_outputs(fmlib, fam, N, dtype):
    """16-bit O through the TMA-store epilogue equals the fp32-output kernel rounded (RNE)."""
    masks, sri, t = _inputs(fam, N, 2, 2, 2, seed=5, dtype=dtype)
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    F = fmlib.FM_FLAG_FWD_PAIR
    o16, l16 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, flags=F)
    o32, l32 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32, flags=F)
    torch.cuda.synchronize()
    assert o16.dtype == dtype
    assert torch.equal(o16, o32.to(dtype))
    assert torch.equal(l16, l32)


@pytest.mark.parametrize("fam,N,H,Hkv,per_kv", [("causal_document", 900, 4, 2, False), ("share_question", 700, 4, 1, False),
                                                ("document", 640, 4, 2, True)])
def test_pair_forward_gqa(fmlib, fam, N, H, Hkv, per_kv):
    masks, sri, t = _inputs(fam, N, 1, H, Hkv, seed=11, heads_per_mask=Hkv if per_kv else 1)
    if per_kv:  # a different mask per key/value head
        rng = np.random.default_rng(99)
        ms = [wm.sample_family(fam, N, rng, (1, 5)) for _ in range(Hkv)]
        sri = torch.from_numpy(np.stack([m.sri for m in ms])[None])
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    o2, l2 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32,
                                 flags=fmlib.FM_FLAG_FWD_PAIR)
    torch.cuda.synchronize()
    G = H // Hkv
    f = lambda x, h: x[0, :, h, :].double().numpy()
    for h in range(H):
        hk = h // G
        vec = fo.expand(sri[0, hk if per_kv else 0].numpy(), causal, N)
        O, L = fo.forward(f(t["q"], h), f(t["k"], hk), f(t["v"], hk), vec)
        assert_close(f"O {fam} [{h}]", o2[0, :, h].cpu().numpy(), O)
        assert_lse(l2[0, h].cpu().numpy(), L)


@pytest.mark.parametrize("fam,N", [("causal_document", 1000), ("document", 700), ("random_eviction", 1000),
                                   ("qk_sparse", 1536), ("full", 129)])
@pytest.mark.parametrize("scale_qk", [1.0, 4.0])
def test_pair_bounded_single_pass(fmlib, fam, N, scale_qk):
    """R33 on the CTA pair (FM_FLAG_FWD_PAIR | FM_FLAG_MAX_BOUND): against the oracle; with Q, K
    scaled by 4 the bound is far too loose, every unit goes through K2a's two-pass fixup and the
    result equals the single-SM two-pass forward bit for bit."""
    masks, sri, t = _inputs(fam, N, 2, 2, 2, seed=5)
    if scale_qk != 1.0:
        t = {n: (x.float() * (scale_qk if n in ("q", "k") else 1.0)).to(torch.bfloat16) for n, x in t.items()}
    sri_c, tc = to_cuda(sri, t)
    causal = masks[0].causal
    flags = fmlib.FM_FLAG_FWD_PAIR | fmlib.FM_FLAG_MAX_BOUND
    o, lse = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32, flags=flags)
    o2, lse2 = fmlib.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32,
                                   flags=fmlib.FM_FLAG_NO_MAX_BOUND)
    torch.cuda.synchronize()
    if scale_qk != 1.0:
        assert torch.equal(o, o2) and torch.equal(lse, lse2)
    sri_np = sri.numpy()
    for b in range(2):
        vec = fo.expand(sri_np[b, 0], causal, N)
        for h in range(2):
            f = lambda n: t[n][b, :, h, :].double().numpy()
            O, L = fo.forward(f("q"), f("k"), f("v"), vec)
            assert_close(f"O[{b},{h}]", o[b, :, h].cpu().numpy(), O)
            assert_lse(lse[b, h].cpu().numpy(), L)
