"""B200-native label-looping greedy decoding for RNN-T and TDT (arXiv 2406.06220).

The product is the C-ABI library `libll.so` (include/ll.h), built in-tree for
sm_100a from `csrc/`.  `ll` is the thin ctypes binding with the C names;
`decoder` wraps it with device-resident weights and buffers (PyTorch is used
only for device memory and streams).
"""
from . import ll  # noqa: F401

__version__ = "0.1.0"
