"""Seeded synthetic input generators shared by the oracle tests, the CUDA parity tests and
bench.py.  Holds none of FlashMask's arithmetic (see masks.py / tensors.py headers)."""
from . import masks, tensors  # noqa: F401
