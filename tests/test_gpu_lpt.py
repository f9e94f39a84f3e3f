"""LPT scheduling (K1d, small grids: a few waves of 148 SMs) — the attention kernels read the
unit order before griddepcontrol.wait, so back-to-back calls under programmatic dependent launch
are the case to cover.  SURVEY a2 (per-unit work O((1-rho) T_r T_c))."""
import numpy as np
import pytest
import torch

from oracle import flashmask_oracle as fo
from workloads import masks as wm
from workloads import tensors as wt

from gpu_util import assert_close, assert_lse

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmlib():
    from paper_2410_01359_b200 import flashmask
    return flashmask


# (family, N, H, Hkv): forward grids of 256-1024 CTAs, backward 512-2048 (LPT on)
CASES = [("causal_document", 8192, 32, 32), ("share_question", 8192, 16, 16), ("document", 4096, 64, 64),
         ("causal_document", 4096, 64, 16)]


@pytest.mark.parametrize("fam,N,H,Hkv", CASES)
def test_lpt_back_to_back(fmlib, fam, N, H, Hkv):
    rng = np.random.default_rng(N + H + len(fam))
    m = wm.sample_family(fam, N, rng, (3, 7))
    sri = torch.from_numpy(wm.stack([m])).cuda()
    x = {}
    for n, heads in (("q", H), ("do", H), ("k", Hkv), ("v", Hkv)):
        x[n] = wt.make_tensor(n, 1, N, heads, 128, base=5).cuda()
    runs = []
    for _ in range(3):   # no synchronisation between the calls: PDL chains across them
        o, lse = fmlib.flashmask_fwd(x["q"], x["k"], x["v"], sri, m.causal, out_dtype=torch.float32)
        g = fmlib.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, m.causal, out_dtype=torch.float32)
        runs.append((o, lse) + tuple(g))
    torch.cuda.synchronize()
    for r in runs[1:]:
        for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), runs[0], r):
            if name == "dq":   # fp32 hardware reduce-add order (R25)
                assert torch.allclose(a, b, atol=1e-5, rtol=0), name
            else:
                assert torch.equal(a, b), name
    o, lse, dq, dk, dv = runs[0]
    vec = fo.expand(m.sri, m.causal, N)
    G = H // Hkv
    f = lambda t, h: t[0, :, h, :].double().cpu().numpy()
    for h in (0, H - 1):
        hk = h // G
        O, L = fo.forward(f(x["q"], h), f(x["k"], hk), f(x["v"], hk), vec)
        assert_close(f"O[{h}]", o[0, :, h].cpu().numpy(), O)
        assert_lse(lse[0, h].cpu().numpy(), L)
        if G == 1:
            gq, gk, gv = fo.backward(f(x["q"], h), f(x["k"], h), f(x["v"], h), f(x["do"], h), vec)
            assert_close(f"dQ[{h}]", dq[0, :, h].cpu().numpy(), gq)
            assert_close(f"dK[{h}]", dk[0, :, h].cpu().numpy(), gk)
            assert_close(f"dV[{h}]", dv[0, :, h].cpu().numpy(), gv)


# split-G backward: MQA / GQA with fewer key-tile units than SMs (K4 over gsplit CTAs + K7)
SPLIT_CASES = [("causal_document", 2048, 8, 1, 128, torch.bfloat16, 0), ("document", 1500, 16, 2, 64, torch.float16, 0),
               ("sliding_window", 4096, 8, 1, 128, torch.bfloat16, 2), ("random_eviction", 777, 4, 1, 128, torch.bfloat16, 0)]


@pytest.mark.parametrize("fam,N,H,Hkv,d,dtype,flags", SPLIT_CASES)
def test_split_g_backward(fmlib, fam, N, H, Hkv, d, dtype, flags):
    rng = np.random.default_rng(N + H)
    m = wm.sample_family(fam, N, rng, (2, 5))
    sri = torch.from_numpy(wm.stack([m])).cuda()
    x = {}
    for n, heads in (("q", H), ("do", H), ("k", Hkv), ("v", Hkv)):
        x[n] = wt.make_tensor(n, 1, N, heads, d, base=7, dtype=dtype).cuda()
    outs = []
    for od in (torch.float32, None):
        o, lse = fmlib.flashmask_fwd(x["q"], x["k"], x["v"], sri, m.causal, out_dtype=od, flags=flags)
        g = fmlib.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, m.causal, out_dtype=od, flags=flags)
        outs.append(g)
    g2 = fmlib.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, m.causal, flags=flags)
    torch.cuda.synchronize()
    dq, dk, dv = outs[0]
    # K7 sums the slices in a fixed order: dK / dV reproducible bit for bit (16-bit run repeated);
    # the 16-bit run (whose O, hence D, is itself rounded) agrees with the fp32 run to bf16 rounding
    assert torch.equal(outs[1][1], g2[1]) and torch.equal(outs[1][2], g2[2])
    for a16, a32 in ((outs[1][1], dk), (outs[1][2], dv)):
        assert torch.allclose(a16.float(), a32, atol=2e-2, rtol=1e-2)
    G = H // Hkv
    vec = fo.expand(m.sri, m.causal, N)
    f = lambda t, h: t[0, :, h, :].double().cpu().numpy()
    for hk in range(Hkv):
        gk = np.zeros((N, d))
        gv = np.zeros((N, d))
        for h in range(hk * G, (hk + 1) * G):
            gq, k_, v_ = fo.backward(f(x["q"], h), f(x["k"], hk), f(x["v"], hk), f(x["do"], h), vec)
            gk += k_
            gv += v_
            if h in (hk * G, (hk + 1) * G - 1):
                assert_close(f"dQ[{h}]", dq[0, :, h].cpu().numpy(), gq)
        assert_close(f"dK[{hk}]", dk[0, :, hk].cpu().numpy(), gk, tol_max=2e-2 * G ** 0.5)
        assert_close(f"dV[{hk}]", dv[0, :, hk].cpu().numpy(), gv, tol_max=2e-2 * G ** 0.5)


def test_per_head_masks_uniform_blocks(fmlib):
    """32 distinct masks (Hm = H = 32) at N = 32K: the class maps take K1b's 16-row-tile uniform
    blocks (forward row map and the backward's transposed map).  Each head must equal the same
    head run alone (Hm = 1, per-row path) — bitwise for O / lse / dK / dV, dQ to fp32 reduce order."""
    N, H = 32768, 32
    rng = np.random.default_rng(7)
    fams = ("causal_document", "share_question", "causal", "causal_blockwise")
    ms = [wm.sample_family(fams[h % 4], N, rng, (3, 9)) for h in range(H)]
    C = max(m.C for m in ms)
    raw = np.stack([np.pad(m.sri, ((0, 0), (0, C - m.C)), constant_values=0) if m.C < C else m.sri for m in ms])
    # causal masks of C = 1 (LTS) and C = 2 (LTS, LTE): pad C = 1 with LTE = N (R-causal layout)
    for h, m in enumerate(ms):
        if m.C < C:
            raw[h, :, 1] = N
    sri = torch.from_numpy(raw[None].astype(np.int32)).cuda()
    x = {n: wt.make_tensor(n, 1, N, H, 128, base=11).cuda() for n in ("q", "k", "v", "do")}
    o, lse = fmlib.flashmask_fwd(x["q"], x["k"], x["v"], sri, True, out_dtype=torch.float32)
    dq, dk, dv = fmlib.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, True, out_dtype=torch.float32)
    for h in (0, 5, 18, 31):
        xs = {n: t[:, :, h:h + 1].contiguous() for n, t in x.items()}
        s1 = sri[:, h:h + 1].contiguous()
        o1, l1 = fmlib.flashmask_fwd(xs["q"], xs["k"], xs["v"], s1, True, out_dtype=torch.float32)
        g1 = fmlib.flashmask_bwd(xs["q"], xs["k"], xs["v"], o1, xs["do"], l1, s1, True, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(o[:, :, h:h + 1], o1) and torch.equal(lse[:, h:h + 1], l1), h
        assert torch.allclose(dq[:, :, h:h + 1], g1[0], atol=1e-5, rtol=0), h
        assert torch.equal(dk[:, :, h:h + 1], g1[1]) and torch.equal(dv[:, :, h:h + 1], g1[2]), h
