"""B200-native Smolyak sparse-grid quadrature hot path (arXiv 2210.14313, MDI-SG).

The compute lives in ``libsg_b200.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/sg_b200.h``); ``paper_2210_14313_b200.api`` only marshals arguments.  Importing the package
does not load CUDA, so CPU-only tools (the build, the ABI symbol check) work without a GPU.
"""
from ._lib import LIB_PATH, SGError, lib  # noqa: F401

__all__ = ["LIB_PATH", "SGError", "lib"]
