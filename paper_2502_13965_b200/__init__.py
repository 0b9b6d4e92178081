"""B200-native Autellix scheduler hot path (arXiv 2502.13965): PLAS/ATLAS per-step scheduling,
paged KV swap and Alg. 2 routing as hand-written sm_100a CUDA behind the C ABI in
include/autx.h.  This package is the thin Python side: the ctypes binding and a trace driver."""
from .autx import (Scheduler, load_library, AutxError, CALL_DESC, CALL_STATE, INF,  # noqa: F401
                   ORDER_SELECT, ORDER_RADIX, SWAP_SM, SWAP_PER_CHUNK_MEMCPY, SWAP_STAGED_DMA,
                   exported_symbols)
from .driver import TraceDriver  # noqa: F401
