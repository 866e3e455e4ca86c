"""paper_2004_04049_b200 -- B200-native hot path of arXiv 2004.04049.

LUT phase randomisation for One-Step Phase-Retrieval (OSPR) and
Gerchberg-Saxton (GS) holography: libholo.so (hand-written sm_100a CUDA behind
the C ABI of include/holo.h) plus this thin binding.  Importing the package
does not touch CUDA; the first call loads libholo.so and fails loudly if it is
missing.
"""
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from ._lib import HoloError, lib  # noqa: F401
from .stream import OsprStream  # noqa: F401

__all__ = list(_api_all) + ["HoloError", "lib", "OsprStream"]
