"""B200-native TRANSIMS cellular-automaton step (arxiv cs/0105004).

The hot path lives in csrc/ (sm_100a CUDA behind the C-ABI of
include/tsim.h); ``tsim`` is the ctypes binding.
"""
from .tsim import (ABSENT, ACTIVE, ARRIVED, FLAG_FUSED, FLAG_GENERAL, FLAG_GRAPH,  # noqa: F401
                   FLAG_HASH, FLAG_LINK_WORK, PENDING, Sim, TsError, debug_checks, domain_plan,
                   exchange_local,
                   load_library, load_times, multilevel_partition, nccl_unique_id,
                   orb_partition, rebalance, strip_bytes)
