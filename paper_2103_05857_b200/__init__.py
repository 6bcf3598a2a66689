"""B200-native hot path of block-coordinate Frank-Wolfe for convex semi-relaxed OT
(arXiv 2103.05857). The compute lives in libsro.so (CUDA, sm_100a) behind the
C-ABI of include/sro.h; `sro` is the thin ctypes binding with the same names."""
from .sro import *  # noqa: F401,F403
