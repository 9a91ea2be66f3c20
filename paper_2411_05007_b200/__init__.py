"""B200-native (sm_100a) SVDQuant W4A4 + low-rank linear (arXiv 2411.05007).

The hot path lives in libsvdq.so (csrc/, C ABI in include/svdq.h); this
package is the thin binding around it (abi.py) plus the tensor-parallel glue
(tp.py).  PyTorch supplies device memory, streams and process groups only.
"""
from .abi import *  # noqa: F401,F403
from .abi import QuantizedLinear, SvdqError, EXPORTS  # noqa: F401

__all__ = [n for n in dir() if n.startswith("svdq_")] + ["QuantizedLinear", "SvdqError", "EXPORTS"]
