"""Helpers for the -m gpu parity tests: seeded inputs -> CUDA path via the C ABI, and the
same inputs -> the fp64 oracle (which never sees a CUDA result)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import flashmask_oracle as fo
from workloads import masks as wm
from workloads import tensors as wt

TOL_MAX, TOL_MEAN, TOL_LSE = 2e-2, 2e-3, 1e-3   # BASELINE.json north_star thresholds


def build_case(masks, H, d, base=0, heads_per_mask=1):
    """masks: list of B MaskInput (one per batch entry).  Returns CPU inputs."""
    B, N = len(masks), masks[0].N
    sri = torch.from_numpy(wm.stack(masks, heads_per_mask))
    t = wt.make_qkv(B, N, H, d, base=base)
    return sri, t


def to_cuda(sri, t):
    return sri.cuda(), {k: v.cuda() for k, v in t.items()}


def oracle_head(t, masks, sri_np, b, h, Hm, causal, scale=None, with_grad=True, rows=None):
    m = masks[b]
    hm = 0 if Hm == 1 else h
    vec = fo.expand(sri_np[b, hm], causal, m.N)
    f = lambda n: t[n][b, :, h, :].double().numpy()
    O, L = fo.forward(f("q"), f("k"), f("v"), vec, scale, rows=rows)
    if not with_grad:
        return O, L, None
    g = fo.backward(f("q"), f("k"), f("v"), f("do"), vec, scale)
    return O, L, g


def assert_close(name, got, ref, tol_max=TOL_MAX, tol_mean=TOL_MEAN):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{name}: non-finite values"
    err = np.abs(got - ref)
    mx, mean = float(err.max()) if err.size else 0.0, float(err.mean()) if err.size else 0.0
    assert mx <= tol_max and mean <= tol_mean, f"{name}: max abs {mx:.3e} (tol {tol_max}), mean {mean:.3e} (tol {tol_mean})"
    return mx, mean


def assert_lse(got, ref, tol=TOL_LSE):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    ninf_g, ninf_r = np.isneginf(got), np.isneginf(ref)
    assert np.array_equal(ninf_g, ninf_r), f"lse -inf pattern differs at {np.argwhere(ninf_g != ninf_r)[:5]}"
    fin = ~ninf_r
    if fin.any():
        e = np.abs(got[fin] - ref[fin]).max()
        assert e <= tol, f"lse max abs {e:.3e} > {tol}"
