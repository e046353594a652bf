"""B200-native MRAB / SBP-SAT overset hot path (arXiv 1805.06607): libmrab.so + ctypes binding.

The product path is `paper_1805_06607_b200.mrab` over `lib/libmrab.so` (built by
`paper_1805_06607_b200/build.py`).  It never imports `oracle/` and has no CPU fallback.
"""
from . import mrab  # noqa: F401
