"""B200-native (sm_100a) FlashMask hot path: C-ABI libflashmask.so + a thin ctypes binding.

    from paper_2410_01359_b200 import flashmask
    o, lse = flashmask.flashmask_fwd(q, k, v, startend_row_indices, causal=True)
    dq, dk, dv = flashmask.flashmask_bwd(q, k, v, o, do, lse, startend_row_indices, causal=True)

Importing ``flashmask`` raises if the library is not built (no fallback).
"""
__all__ = ["flashmask", "build"]
