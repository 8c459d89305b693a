"""B200-native CO2 outer-step hot path (arXiv 2401.16265).

The product is libco2b200.so (sm_100a kernels + C ABI, include/co2_b200.h);
`co2` is the Python mirror of the reference's operator API over it.
"""
from . import _lib  # noqa: F401
from ._lib import NumericError, ValidationError  # noqa: F401

__all__ = ["co2", "NumericError", "ValidationError"]
