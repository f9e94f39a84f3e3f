"""FlashMask oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import anything under oracle/.  The product package never does.
"""
from . import dense_predicates, flashmask_oracle  # noqa: F401
