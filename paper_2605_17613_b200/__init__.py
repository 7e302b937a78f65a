"""VeriCache decode loop on B200 (arxiv 2605.17613) -- the lossless
compressed-KV drafting / full-KV verification path, as sm_100a kernels and a
C++ engine behind the C-ABI in include/vc_api.h.  See DESIGN.md."""
from ._lib import ConfigError, ContractError, CudaError, VcError, load  # noqa: F401
from .engine import (LLAMA3_8B, LLAMA3_70B, TINY, Engine, ModelShape, SpecRoundResult,  # noqa: F401
                     TpLoopback, accept, drop_indices, nccl_unique_id, reload_span, tp_shard)
