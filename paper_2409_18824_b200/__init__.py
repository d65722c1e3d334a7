"""B200 (sm_100a) implementation of the Fortran array path of arXiv 2409.18824.

The product is ``libftn.so`` (C ABI in ``include/ftn.h``); ``ftn`` is its thin
ctypes binding.  ``from paper_2409_18824_b200 import ftn`` loads the library and
raises if it is not built -- there is no fallback.
"""
__all__ = ["ftn"]
