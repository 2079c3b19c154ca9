"""B200-native sparse persistent RNN hot path (arXiv 1804.10223).

The product is the C-ABI library ``libsrnn.so`` (include/srnn.h) built from
``csrc/`` for sm_100a; ``SparseRNN`` is its thin ctypes binding.
"""
from ._lib import (FLAG_DEBUG_JITTER, FLAG_DENSE_TC, FLAG_FP32_STAGING, FLAG_GRID_SYNC, FLAG_HOST_ONLY, FLAG_NAIVE_LAYOUT, FLAG_PROFILE, FLAG_RESERVE_SMS,
                   FLAG_CLASS_BALANCE, FLAG_COLUMN_SPLIT, FLAG_STAGED, FLAG_SIMT_GEMM, FLAG_Y_BATCH_MAJOR, SparseRNN, SrnnError, from_problem, load_library)

__all__ = ["SparseRNN", "SrnnError", "from_problem", "load_library", "FLAG_GRID_SYNC", "FLAG_NAIVE_LAYOUT",
           "FLAG_HOST_ONLY", "FLAG_SIMT_GEMM", "FLAG_DEBUG_JITTER", "FLAG_FP32_STAGING", "FLAG_PROFILE", "FLAG_RESERVE_SMS",
           "FLAG_DENSE_TC", "FLAG_Y_BATCH_MAJOR", "FLAG_CLASS_BALANCE", "FLAG_COLUMN_SPLIT", "FLAG_STAGED"]
