"""paper_1410_0986_b200 -- B200-native Born assembly -> low-rank compression ->
low-rank matvec path of arXiv 1410.0986 ("hydot").

Python mirror of the reference's hydot::born / hydot::lowrank interfaces over
the C ABI in include/hydot_b200.h (libhydot_b200.so, sm_100a).  Importing
this package loads the library; there is no CPU fallback.
"""
from ._lib import LIB_PATH, HydotError, Ledger, lib  # noqa: F401
from .core import Context, default_context, dgemm, gaussian, mt19937_64, rng_selftest  # noqa: F401
from . import born, lowrank, configs  # noqa: F401

lib()  # fail loudly when the CUDA extension is missing
