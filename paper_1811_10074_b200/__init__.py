"""B200-native (sm_100a) hot path of arxiv 1811.10074 "Parallel sliding window sums":
sliding window sums by the block suffix/prefix decomposition, and minimizer extraction
+ seed tables built on it.  The compute runs in libmzslsum.so (hand-written CUDA);
`_lib` is a thin ctypes binding, `dist` the multi-GPU shard/exchange planner.
"""
from . import _lib  # noqa: F401  (raises ImportError if the CUDA library is missing)
from ._lib import *  # noqa: F401,F403
