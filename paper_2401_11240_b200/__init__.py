"""B200-native batched multi-adapter heterogeneous-rank LoRA delta (CaraServe hot path).

The product is the C-ABI library ``lib/liblora.so`` (include/lora_delta.h) built from
``csrc/`` for sm_100a; ``binding`` is a thin ctypes layer over it.  Importing this
package never falls back to a CPU path: if the library is missing, import fails.
"""
from .binding import LIB, LoraError, LoraPool, apply_multi, header_symbols  # noqa: F401

__all__ = ["LIB", "LoraError", "LoraPool", "apply_multi", "header_symbols"]
