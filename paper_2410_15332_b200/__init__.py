"""B200-native (sm_100a) KVLink / LegoLink linked prefill — arXiv 2410.15332 (Epic).

The product is the C-ABI library ``libpic.so`` (include/pic.h); ``pic`` is its ctypes binding.
"""
from .pic import Engine, LinkOutput, PicError, lib, parse_alg  # noqa: F401
