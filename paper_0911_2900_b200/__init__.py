"""B200-native F.A.S.T. pedestrian simulator: planning + motion hot path on sm_100a.

``paper_0911_2900_b200.fastped`` mirrors the reference's ``namespace fastped`` API; the compute
runs in the CUDA library libfastped_b200.so behind the C ABI in include/fastped_b200.h.
"""
from . import fastped  # noqa: F401
from .fastped import *  # noqa: F401,F403
