"""CPU checks of the C-ABI library: it builds for sm_100a, exports every symbol that
include/flashmask.h declares, and validates arguments on the host (no GPU needed —
argument errors return before any CUDA call)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2410_01359_b200 import build
    return build.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "flashmask.h")).read()
    return sorted(set(re.findall(r"FM_API\s+[\w\s\*]+?\b(flashmask_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("flashmask_fwd", "flashmask_bwd", "flashmask_classify", "flashmask_workspace_size",
              "flashmask_status_string", "flashmask_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_sass_contains_tcgen05_and_tma(lib_path):
    """The kernels are sm_100a tcgen05/TMA code (B200_PROFILING.md SASS mnemonics)."""
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "no tcgen05.mma in SASS"
    assert "UTMALDG" in sass, "no TMA tensor loads in SASS"
    assert "LDTM" in sass and "STTM" in sass, "no tcgen05.ld/st in SASS"
    assert "HMMA" not in re.sub(r"UTC\w*HMMA", "", sass), "legacy mma.sync path present"


def test_host_validation_without_gpu(lib_path):
    from paper_2410_01359_b200 import flashmask as fm
    lib = fm._lib
    p = fm.FmParams(batch=1, seqlen=128, num_heads=1, head_dim=96, mask_heads=1, mask_cols=1, causal=1, scale=0.0,
                    in_dtype=0, out_dtype=0, flags=0, num_kv_heads=0)
    st = lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None)
    assert st == fm.FM_ERR_INVALID_ARGUMENT
    assert b"head_dim" in lib.flashmask_last_error()
    p.head_dim = 128
    p.mask_cols = 4   # causal with C=4 is not in the C-table
    assert lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == \
        fm.FM_ERR_INVALID_ARGUMENT
    p.mask_cols = 1
    assert lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == \
        fm.FM_ERR_INVALID_ARGUMENT  # NULL pointers
    p.in_dtype = 7
    assert lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == \
        fm.FM_ERR_INVALID_ARGUMENT
    p.in_dtype = 0
    p.batch = 70000
    assert lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == \
        fm.FM_ERR_UNSUPPORTED
    p.batch = 1
    p.seqlen = 262144 + 1  # beyond the largest supported N (2048 column tiles)
    assert lib.flashmask_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == \
        fm.FM_ERR_UNSUPPORTED
    assert b"262144" in lib.flashmask_last_error()
    p.seqlen = 128
    assert lib.flashmask_status_string(fm.FM_ERR_WORKSPACE_TOO_SMALL) == b"FM_ERR_WORKSPACE_TOO_SMALL"


def test_workspace_size_is_linear_in_n(lib_path):
    from paper_2410_01359_b200 import flashmask as fm
    sizes = {}
    for N in (8192, 16384):
        p = fm.FmParams(batch=1, seqlen=N, num_heads=32, head_dim=128, mask_heads=1, mask_cols=1, causal=1,
                        scale=0.0, in_dtype=0, out_dtype=0, flags=0, num_kv_heads=0)
        sizes[N] = (fm.flashmask_workspace_size(p, fm.FM_PASS_FWD), fm.flashmask_workspace_size(p, fm.FM_PASS_BWD))
    # forward: O(N) vectors + O(T^2) bytes of class map; backward dominated by the O(N H d) dQ accumulator
    assert sizes[8192][0] < 2 * 1024 * 1024
    assert 1.9 < sizes[16384][1] / sizes[8192][1] < 2.1
    assert sizes[8192][1] >= 8192 * 32 * 128 * 4


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU or eager fallback: with the shared library absent, importing the binding raises."""
    code = "import paper_2410_01359_b200.flashmask"
    env = dict(os.environ, FLASHMASK_LIB=str(tmp_path / "absent" / "libflashmask.so"), PYTHONPATH=ROOT)
    r = subprocess.run(["python", "-c", code], cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0, r.stdout
    assert "libflashmask" in r.stderr or "absent" in r.stderr, r.stderr[-2000:]


def test_product_package_never_references_the_oracle():
    """The oracle is test infrastructure: nothing in the product package imports or calls it."""
    pkg = os.path.join(ROOT, "paper_2410_01359_b200")
    hits = []
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                if re.search(r"^\s*(from|import)\s+oracle\b|oracle[./]", src, re.M):
                    hits.append(f)
    assert hits == []


def test_batch_times_mask_heads_limit(lib_path):
    """K1 grids hold B * mask_heads in one dimension: > 65535 is refused on the host."""
    from paper_2410_01359_b200 import flashmask as fm
    p = fm.FmParams(batch=2048, seqlen=128, num_heads=64, head_dim=128, mask_heads=64, mask_cols=1, causal=1,
                    scale=0.0, in_dtype=0, out_dtype=0, flags=0, num_kv_heads=0)
    assert fm._lib.flashmask_workspace_size(ctypes.byref(p), 0) == 0
    assert b"mask_heads" in fm._lib.flashmask_last_error()
    p.mask_heads = 1
    assert fm._lib.flashmask_workspace_size(ctypes.byref(p), 0) > 0


def test_binding_rejects_host_tensors(lib_path):
    """The binding refuses non-CUDA tensors before any call (no CPU fallback exists)."""
    import torch
    from paper_2410_01359_b200 import flashmask as fm
    q = torch.zeros(1, 128, 1, 128, dtype=torch.bfloat16)
    sri = torch.full((1, 1, 128, 1), 128, dtype=torch.int32)
    with pytest.raises(fm.FlashMaskError, match="CUDA"):
        fm.flashmask_fwd(q, q, q, sri, True)


def test_classify_row_tile_grid_limit(lib_path):
    """K1b holds <= 64 row tiles per CTA and <= 65535 CTAs along that grid dimension: a classify
    call with more than 4194240 row tiles is refused on the host, before any launch."""
    from paper_2410_01359_b200 import flashmask as fm
    p = fm.FmParams(batch=1, seqlen=1 << 27, num_heads=1, head_dim=128, mask_heads=1, mask_cols=1, causal=1,
                    scale=0.0, in_dtype=0, out_dtype=0, flags=0, num_kv_heads=0)
    dummy = ctypes.c_void_p(256)   # aligned, never dereferenced: the call fails in host validation
    st = fm._lib.flashmask_classify(ctypes.byref(p), dummy, 16, 128, dummy, None, None, None, None, None)
    assert st == fm.FM_ERR_UNSUPPORTED
    assert b"row tiles" in fm._lib.flashmask_last_error()
