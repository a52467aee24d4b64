"""paper_2412_20501_b200: B200-native TokenRing sequence-parallel attention.

A drop-in for the attention path of the reference ``ringsim`` package
(arxiv 2412.20501, "TokenRing"), with the same public names:

* core:       MaskKind, MaskSpec, Partial, block_attention, merge_partial,
              dense_attention (alias dense_attention_oracle), max_relative_error
* partition:  Partition, split_contiguous, split_zigzag, causal_work_count,
              gather_local, global_reorder
* engine:     MsgKind, Schedule, build_ring_attention, build_token_ring,
              build_zigzag_token_ring (route="ring"|"direct"), build_hybrid,
              execute, trace_from_schedule, comm_volume
* ring:       TokenRingAttention / token_ring_attention (one process per GPU)
* errors:     RingsimError, DimensionError, InputError, ConfigError,
              ScheduleError, TopologyError

Compute runs in libtokenring.so (hand-written sm_100a kernels behind a C
ABI, include/tokenring.h); there is no CPU fallback.
"""

from .errors import (ConfigError, DimensionError, InputError, RingsimError,  # noqa: F401
                     ScheduleError, TopologyError)
from .partition import (Partition, causal_work_count, gather_local,  # noqa: F401
                        global_reorder, split_contiguous, split_zigzag)

from .kernels import BACKEND as KERNEL_BACKEND  # noqa: F401,E402
from .core import (MaskKind, MaskSpec, Partial, block_attention,  # noqa: F401,E402
                   dense_attention, dense_attention_oracle, max_relative_error,
                   merge_partial)
from .engine import (MessageTrace, MsgKind, Schedule, build_ring_attention,  # noqa: F401,E402
                     build_hybrid, build_schedule, build_token_ring, build_zigzag_token_ring,
                     comm_volume,
                     execute, trace_from_schedule)
from .ring import TokenRingAttention, token_ring_attention  # noqa: F401,E402
from . import core, engine, kernels, partition, ring, rng  # noqa: F401,E402

__version__ = "0.2.0"
