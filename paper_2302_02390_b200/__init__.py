"""paper_2302_02390_b200 -- B200-native QSDP communication hot path.

Quantized weight all-gather and quantized gradient reduce-scatter of QSDP
(arXiv 2302.02390) as hand-written sm_100a kernels behind a C ABI
(include/qsdp_b200.h), bit-exact with the reference implementation's codes,
scales and dequantized values.
"""

from ._lib import LIB_PATH, build  # noqa: F401

__version__ = "0.1.0"
