"""paper_2603_08743_b200 — B200-native compression step of Compressed PagedAttention (Zipage).

The product is the C-ABI library ``lib/libzipc.so`` (include/zipc.h, hand-written sm_100a CUDA);
``zipc`` is its thin ctypes binding. Importing this package loads nothing; the library is loaded
on first use and there is no CPU fallback.
"""
__all__ = ["zipc"]
