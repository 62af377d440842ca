"""paper_math_9809043_b200 — B200-native recursive multi-scale PCG (Lackner & Menikoff,
arXiv math/9809043) for -div(K grad p) = f.

The product is the C-ABI library ``libmss.so`` (include/mss.h, sources in csrc/);
``mss.Solver`` is a thin ctypes binding over it.  Importing the package does not load
the library; ``mss.load_library()`` (called by ``Solver``) does, and raises if it is
missing — there is no CPU fallback.
"""
__all__ = ["mss", "build"]
