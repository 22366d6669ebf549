"""Harness: SHA-256 of the reproducible CPU-built config matrices (compare across hosts)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11843_b200 import inputs  # noqa: E402

for name, kw in (("cfg3", {"d": 2048}), ("cfg3", {})):
    t = time.time()
    A = inputs.cpu_reproducible(name, **kw)
    print(name, kw, inputs.sha256(A), f"{time.time() - t:.1f}s", flush=True)
