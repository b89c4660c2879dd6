"""B200-native (sm_100a) FreeKV decode-step KV-retrieval path (arXiv 2505.13109).

The compute lives in ``libfreekv.so`` (hand-written CUDA behind the C ABI of
``include/freekv.h``); ``freekv`` is a thin ctypes binding with the same names.
"""
from .freekv import (FreeKV, FreeKVConfig, FreeKVError, MODE_ALWAYS_CORRECT, MODE_NEVER_CORRECT,
                     MODE_SPECULATIVE, load_library, query_sizes)

__all__ = ["FreeKV", "FreeKVConfig", "FreeKVError", "MODE_SPECULATIVE", "MODE_ALWAYS_CORRECT",
           "MODE_NEVER_CORRECT", "load_library", "query_sizes"]
