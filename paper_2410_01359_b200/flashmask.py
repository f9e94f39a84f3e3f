"""Thin ctypes binding over libflashmask.so (include/flashmask.h).

Argument marshalling only: every step of the path runs in the library's CUDA kernels.
PyTorch provides device memory and the current stream.  There is no CPU or eager
fallback: if the shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLASHMASK_LIB", os.path.join(_PKG, "libflashmask.so"))

FM_OK, FM_ERR_INVALID_ARGUMENT, FM_ERR_UNSUPPORTED, FM_ERR_WORKSPACE_TOO_SMALL, FM_ERR_CUDA = range(5)
FM_BF16, FM_FP32, FM_FP16 = 0, 1, 2
FM_TILE_SKIP, FM_TILE_PARTIAL, FM_TILE_UNMASKED = 0, 1, 2
FM_FLAG_NO_SKIP = 1
FM_FLAG_DETERMINISTIC = 2
FM_FLAG_NO_REFINE = 4
FM_FLAG_FWD_PAIR = 8
FM_FLAG_ROWWISE = 16
FM_FLAG_NO_MAX_BOUND = 32
FM_FLAG_MAX_BOUND = 64
FM_PASS_FWD, FM_PASS_BWD = 0, 1

EXPORTED = ["flashmask_workspace_size", "flashmask_classify", "flashmask_refine", "flashmask_fwd", "flashmask_bwd",
            "flashmask_status_string", "flashmask_last_error", "flashmask_timing_enable", "flashmask_timing_collect",
            "flashmask_sliding_window_indices"]
KERNEL_NAMES = ["expand", "classify", "fwd", "bwd_pre", "bwd", "dq_convert", "dq", "refine", "keynorm"]
(FM_KERNEL_EXPAND, FM_KERNEL_CLASSIFY, FM_KERNEL_FWD, FM_KERNEL_BWD_PRE, FM_KERNEL_BWD, FM_KERNEL_DQ_CONVERT,
 FM_KERNEL_DQ, FM_KERNEL_REFINE) = range(8)


class FmParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("seqlen", ctypes.c_int64), ("num_heads", ctypes.c_int64),
                ("head_dim", ctypes.c_int64), ("mask_heads", ctypes.c_int64), ("mask_cols", ctypes.c_int64),
                ("causal", ctypes.c_int32), ("scale", ctypes.c_float), ("in_dtype", ctypes.c_int32),
                ("out_dtype", ctypes.c_int32), ("flags", ctypes.c_int32), ("num_kv_heads", ctypes.c_int64)]


class FlashMaskError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str):
        super().__init__(f"{what}: {detail}")
        self.status = status


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_2410_01359_b200.build` (no fallback path exists)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER(FmParams)
    vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
    lib.flashmask_workspace_size.argtypes = [P, ctypes.c_int]
    lib.flashmask_workspace_size.restype = sz
    lib.flashmask_classify.argtypes = [P, vp, i32, i32, vp, vp, vp, vp, vp, vp]
    lib.flashmask_classify.restype = ctypes.c_int
    lib.flashmask_refine.argtypes = [P, vp, vp, vp, vp, vp]
    lib.flashmask_refine.restype = ctypes.c_int
    lib.flashmask_fwd.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.flashmask_fwd.restype = ctypes.c_int
    lib.flashmask_bwd.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.flashmask_bwd.restype = ctypes.c_int
    lib.flashmask_status_string.argtypes = [ctypes.c_int]
    lib.flashmask_status_string.restype = ctypes.c_char_p
    lib.flashmask_last_error.argtypes = []
    lib.flashmask_last_error.restype = ctypes.c_char_p
    lib.flashmask_timing_enable.argtypes = [ctypes.c_int]
    lib.flashmask_sliding_window_indices.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                     vp, vp]
    lib.flashmask_sliding_window_indices.restype = ctypes.c_int
    lib.flashmask_timing_enable.restype = ctypes.c_int
    lib.flashmask_timing_collect.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    lib.flashmask_timing_collect.restype = ctypes.c_int
    return lib


_lib = load_library()


def _check(status: int, what: str):
    if status != FM_OK:
        raise FlashMaskError(status, what, f"{_lib.flashmask_status_string(status).decode()}: "
                                           f"{_lib.flashmask_last_error().decode()}")


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream, device=None):
    """The caller's stream, by default the current stream of the tensors' device."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _require(cond: bool, what: str, msg: str):
    if not cond:
        raise FlashMaskError(FM_ERR_INVALID_ARGUMENT, what, msg)


def _check_tensor(t, name: str, what: str, shape, dtypes, device):
    """The C ABI takes raw pointers to packed row-major tensors: refuse anything else here
    (non-contiguous views, wrong dtype, wrong device) instead of letting the kernels read the
    wrong bytes."""
    _require(isinstance(t, torch.Tensor), what, f"{name} must be a torch.Tensor")
    _require(t.is_cuda, what, f"{name} must be a CUDA tensor")
    _require(t.device == device, what, f"{name} is on {t.device}, expected {device}")
    _require(t.is_contiguous(), what, f"{name} must be contiguous (got strides {tuple(t.stride())})")
    _require(t.dtype in dtypes, what, f"{name} has dtype {t.dtype}, expected one of {sorted(map(str, dtypes))}")
    if shape is not None:
        _require(tuple(t.shape) == tuple(shape), what, f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _check_sri(sri, B, N, what, device):
    _check_tensor(sri, "startend_row_indices", what, None, (torch.int32,), device)
    _require(sri.dim() == 4 and sri.shape[0] == B and sri.shape[2] == N, what,
             f"startend_row_indices must be [B={B}, Hm, N={N}, C], got {tuple(sri.shape)}")


_DTYPES = {torch.bfloat16: FM_BF16, torch.float32: FM_FP32, torch.float16: FM_FP16}


def _in_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return FM_BF16
    if t.dtype == torch.float16:
        return FM_FP16
    if t.dtype == torch.float32:
        return FM_FP32
    raise TypeError(f"flashmask inputs must be bfloat16, float16 or float32, got {t.dtype}")


def make_params(B, N, H, d, sri: torch.Tensor, causal: bool, scale=None, out_dtype=torch.bfloat16,
                flags: int = 0, num_kv_heads: int = 0, in_dtype: int = FM_BF16) -> FmParams:
    assert sri.dim() == 4 and sri.shape[0] == B and sri.shape[2] == N, sri.shape
    return FmParams(batch=B, seqlen=N, num_heads=H, head_dim=d, mask_heads=sri.shape[1], mask_cols=sri.shape[3],
                    causal=int(bool(causal)), scale=float(scale) if scale else 0.0, in_dtype=in_dtype,
                    out_dtype=_DTYPES[out_dtype], flags=int(flags),
                    num_kv_heads=int(num_kv_heads))


def flashmask_workspace_size(params: FmParams, pass_: int) -> int:
    n = _lib.flashmask_workspace_size(ctypes.byref(params), pass_)
    if n == 0:
        _check(FM_ERR_INVALID_ARGUMENT, "flashmask_workspace_size")
    return int(n)


def flashmask_classify(sri: torch.Tensor, causal: bool, br: int = 128, bc: int = 128, num_heads: int | None = None,
                       class_map: bool = True, stream=None, nonskip: bool = False, rowwise: bool = False):
    """Tile classification (K1).  sri: int32 cuda [B, Hm, N, C].  Returns
    (minmax int32 [B,Hm,Tc,8], class_map uint8 [B,Hm,Tr,Tc] or None, counts int64 [B,Hm,3]);
    with nonskip=True also (row_nonskip int32 [B,Hm,Tr], col_nonskip int32 [B,Hm,Tc]): the
    number of non-SKIP tiles per row tile / per column tile.  rowwise=True
    (FM_FLAG_ROWWISE): sri is the row-wise representation and minmax is per row tile
    [B,Hm,Tr,8]."""
    _require(isinstance(sri, torch.Tensor) and sri.dim() == 4, "flashmask_classify",
             "startend_row_indices must be a 4-D tensor [B, Hm, N, C]")
    B, Hm, N, C = sri.shape
    _check_sri(sri, B, N, "flashmask_classify", sri.device)
    p = FmParams(batch=B, seqlen=N, num_heads=num_heads or Hm, head_dim=128, mask_heads=Hm, mask_cols=C,
                 causal=int(bool(causal)), scale=0.0, in_dtype=FM_BF16, out_dtype=FM_BF16,
                 flags=FM_FLAG_ROWWISE if rowwise else 0)
    Tr, Tc = -(-N // br), -(-N // bc)
    dev = sri.device
    minmax = torch.empty(B, Hm, Tr if rowwise else Tc, 8, dtype=torch.int32, device=dev)
    cmap = torch.empty(B, Hm, Tr, Tc, dtype=torch.uint8, device=dev) if class_map else None
    counts = torch.empty(B, Hm, 3, dtype=torch.int64, device=dev)
    rows = torch.empty(B, Hm, Tr, dtype=torch.int32, device=dev) if nonskip else None
    cols = torch.empty(B, Hm, Tc, dtype=torch.int32, device=dev) if nonskip else None
    with torch.cuda.device(dev):
        _check(_lib.flashmask_classify(ctypes.byref(p), _ptr(sri), br, bc, _ptr(minmax), _ptr(cmap), _ptr(counts),
                                       _ptr(rows), _ptr(cols), _stream(stream, dev)), "flashmask_classify")
    if nonskip:
        return minmax, cmap, counts, rows, cols
    return minmax, cmap, counts


def flashmask_refine(sri: torch.Tensor, causal: bool, class_map: torch.Tensor | None = None, stream=None):
    """f3 refinement (K1c): uint32 [B, Hm, Tr, Tc] words, bit 8g+c set iff the 32-row group g x
    16-column chunk c of the 128 x 128 tile holds a masked cell; and int64 [B, Hm, 2] counts
    (PARTIAL tiles without any masked cell, dirty sub-blocks of PARTIAL tiles).  class_map: the
    128 x 128 map of flashmask_classify (computed here when None)."""
    B, Hm, N, C = sri.shape
    _check_sri(sri, B, N, "flashmask_refine", sri.device)
    if class_map is None:
        _, class_map, _ = flashmask_classify(sri, causal, 128, 128, stream=stream)
    T = -(-N // 128)
    _check_tensor(class_map, "class_map", "flashmask_refine", (B, Hm, T, T), (torch.uint8,), sri.device)
    p = FmParams(batch=B, seqlen=N, num_heads=Hm, head_dim=128, mask_heads=Hm, mask_cols=C,
                 causal=int(bool(causal)), scale=0.0, in_dtype=FM_BF16, out_dtype=FM_BF16, flags=0)
    words = torch.empty(B, Hm, T, T, dtype=torch.int32, device=sri.device)   # uint32 bit patterns
    counts = torch.empty(B, Hm, 2, dtype=torch.int64, device=sri.device)
    with torch.cuda.device(sri.device):
        _check(_lib.flashmask_refine(ctypes.byref(p), _ptr(sri), _ptr(class_map), _ptr(words), _ptr(counts),
                                     _stream(stream, sri.device)), "flashmask_refine")
    return words, counts


def flashmask_sliding_window_indices(batch: int, seqlen: int, window: int, causal: bool = True, device="cuda",
                                     stream=None) -> torch.Tensor:
    """startend_row_indices of a sliding window of `window` keys, generated on the device:
    causal -> int32 [batch, 1, seqlen, 1]; bidirectional -> int32 [batch, 1, seqlen, 2]."""
    out = torch.empty(batch, 1, seqlen, 1 if causal else 2, dtype=torch.int32, device=device)
    with torch.cuda.device(out.device):
        _check(_lib.flashmask_sliding_window_indices(batch, seqlen, window, int(bool(causal)), _ptr(out),
                                                     _stream(stream, out.device)), "flashmask_sliding_window_indices")
    return out


def _workspace(params, pass_, workspace, dev):
    need = flashmask_workspace_size(params, pass_)
    if workspace is not None:
        _check_tensor(workspace, "workspace", "workspace", None, (torch.uint8,), dev)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    return workspace, need


def _out_dtype(q, out_dtype):
    """Default output type: the 16-bit type of the inputs (bf16 for fp32 inputs)."""
    if out_dtype is not None:
        return out_dtype
    return torch.float16 if q.dtype == torch.float16 else torch.bfloat16


def _check_qkv(q, k, v, what):
    _require(isinstance(q, torch.Tensor) and q.dim() == 4, what, "q must be a 4-D tensor [B, N, H, d]")
    B, N, H, d = q.shape
    dev = q.device
    _check_tensor(q, "q", what, None, tuple(_DTYPES), dev)
    _require(isinstance(k, torch.Tensor) and k.dim() == 4, what, "k must be a 4-D tensor [B, N, Hkv, d]")
    Hkv = k.shape[2]
    _check_tensor(k, "k", what, (B, N, Hkv, d), (q.dtype,), dev)
    _check_tensor(v, "v", what, (B, N, Hkv, d), (q.dtype,), dev)
    return B, N, H, d, Hkv, dev


def flashmask_fwd(q, k, v, sri, causal: bool, scale=None, out_dtype=None, flags: int = 0,
                  out=None, lse=None, workspace=None, stream=None):
    """o, lse = FlashMask forward.  q: bf16/fp16 (tcgen05 path) or fp32 (fp32 path) cuda [B, N, H, d];
    k/v: [B, N, Hkv, d] of the same dtype (Hkv divides H, grouped-query attention);
    sri: int32 [B, Hm, N, C] with Hm in {1, Hkv}.  All tensors contiguous on one device."""
    what = "flashmask_fwd"
    B, N, H, d, Hkv, dev = _check_qkv(q, k, v, what)
    _check_sri(sri, B, N, what, dev)
    if out is not None and out_dtype is None:
        out_dtype = out.dtype
    out_dtype = _out_dtype(q, out_dtype)
    _require(out_dtype in _DTYPES, what, f"unsupported out_dtype {out_dtype}")
    p = make_params(B, N, H, d, sri, causal, scale, out_dtype, flags, num_kv_heads=Hkv, in_dtype=_in_dtype(q))
    if out is not None:
        _check_tensor(out, "out", what, (B, N, H, d), (out_dtype,), dev)
    if lse is not None:
        _check_tensor(lse, "lse", what, (B, H, N), (torch.float32,), dev)
    o = out if out is not None else torch.empty(B, N, H, d, dtype=out_dtype, device=dev)
    lse = lse if lse is not None else torch.empty(B, H, N, dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        ws, need = _workspace(p, FM_PASS_FWD, workspace, dev)
        _check(_lib.flashmask_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(sri), _ptr(o), _ptr(lse), _ptr(ws),
                                  ws.numel(), _stream(stream, dev)), what)
    return o, lse


def flashmask_bwd(q, k, v, o, do, lse, sri, causal: bool, scale=None, out_dtype=None, flags: int = 0,
                  dq=None, dk=None, dv=None, workspace=None, stream=None, deterministic: bool = False):
    """dq, dk, dv = FlashMask backward.  o and lse come from flashmask_fwd on the same inputs; the
    gradients take o's dtype (out_dtype, if given, must equal it).  dk, dv have the key/value head
    count of k, v.  dQ is reduced with fp32 hardware reduce-adds whose order is not fixed, so dq may
    differ in the last bits run to run; `deterministic=True` (FM_FLAG_DETERMINISTIC) computes dq
    row-parallel in ascending key-tile order instead — bitwise reproducible, ~1.6x the backward time."""
    what = "flashmask_bwd"
    B, N, H, d, Hkv, dev = _check_qkv(q, k, v, what)
    _check_sri(sri, B, N, what, dev)
    _require(isinstance(o, torch.Tensor), what, "o must be a torch.Tensor")
    _require(out_dtype is None or out_dtype == o.dtype, what,
             f"out_dtype {out_dtype} differs from o.dtype {o.dtype}: the gradients take the forward output's dtype")
    out_dtype = o.dtype
    _require(out_dtype in (torch.float32, torch.float16 if q.dtype == torch.float16 else torch.bfloat16), what,
             f"o has dtype {o.dtype}; expected float32 or the 16-bit type of the inputs")
    _check_tensor(o, "o", what, (B, N, H, d), (out_dtype,), dev)
    _check_tensor(do, "do", what, (B, N, H, d), (q.dtype,), dev)
    _check_tensor(lse, "lse", what, (B, H, N), (torch.float32,), dev)
    if deterministic:
        flags |= FM_FLAG_DETERMINISTIC
    p = make_params(B, N, H, d, sri, causal, scale, out_dtype, flags, num_kv_heads=Hkv, in_dtype=_in_dtype(q))
    for t, name, h in ((dq, "dq", H), (dk, "dk", Hkv), (dv, "dv", Hkv)):
        if t is not None:
            _check_tensor(t, name, what, (B, N, h, d), (out_dtype,), dev)
    mk = lambda t, h: t if t is not None else torch.empty(B, N, h, d, dtype=out_dtype, device=dev)
    dq, dk, dv = mk(dq, H), mk(dk, Hkv), mk(dv, Hkv)
    with torch.cuda.device(dev):
        ws, need = _workspace(p, FM_PASS_BWD, workspace, dev)
        _check(_lib.flashmask_bwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(do), _ptr(lse),
                                  _ptr(sri), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream(stream, dev)),
               what)
    return dq, dk, dv


FM_TIMING_SELECT = 0x10000


def flashmask_timing_enable(enable: bool = True, kernels=None):
    """Per-kernel CUDA-event timing; `kernels` = iterable of FM_KERNEL_* ids (default: all)."""
    if enable and kernels is not None:
        code = FM_TIMING_SELECT | sum(1 << k for k in set(kernels))
    else:
        code = int(bool(enable))
    _check(_lib.flashmask_timing_enable(code), "flashmask_timing_enable")


def flashmask_timing_collect():
    """{kernel name: (total ms, launches)} of the launches recorded since the last collect."""
    n = len(KERNEL_NAMES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    _check(_lib.flashmask_timing_collect(ms, cnt), "flashmask_timing_collect")
    return {KERNEL_NAMES[i]: (ms[i], cnt[i]) for i in range(n)}


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
