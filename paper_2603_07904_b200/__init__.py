"""paper_2603_07904_b200 -- B200-native (sm_100a) hot path of DyQ-VLA (arXiv 2603.07904).

The runtime-switchable low-bit quantized linear layer, its weight packer, the
dynamic activation quantizer and the kinematic bit-selection kernel, behind the
C ABI declared in include/dyq.h (libdyq.so).  `dyq` is the thin Python binding.
"""
from . import dyq  # noqa: F401

__all__ = ["dyq"]
