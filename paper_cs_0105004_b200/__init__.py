"""B200-native TRANSIMS cellular-automaton step (arxiv cs/0105004).

The hot path lives in csrc/ (sm_100a CUDA behind the C-ABI of
include/tsim.h); ``tsim`` is the ctypes binding.
"""
from .tsim import (ACTIVE, ARRIVED, FLAG_FUSED, FLAG_GENERAL, FLAG_GRAPH, FLAG_HASH,  # noqa: F401
                   FLAG_LINK_WORK,
                   PENDING, Sim, TsError, load_library, orb_partition)
