"""paper_2210_00882_b200: B200-native engine for fraglow's GPU-only distribution policy (DP-D).

The product is the C-ABI library libfraglow_b200.so (include/fraglow_b200.h, sources in csrc/);
this package only binds it (`_native`) and mirrors the reference API (`api`).
"""
from .api import DpdEngine, Program  # noqa: F401
from ._native import FlwError  # noqa: F401

__all__ = ["Program", "DpdEngine", "FlwError"]
