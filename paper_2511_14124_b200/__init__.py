"""b200-tencache: a B200-native tensor cache & migration engine with the
decision API of 10Cache (arXiv 2511.14124).

* ``policy``   — the reference's decision API (IPolicy, run, decisions) over
                 our C++ host core.
* ``traces``   — trace files and machine configs (reference JSONL format),
                 chunk-level traces for the BASELINE configs.
* ``engine``   — the per-GPU CUDA migration engine (pinned pools, copy-engine
                 streams, fused AdamW) through the C-ABI.
* ``kernels``  — direct access to the sm_100a data-plane kernels.
* ``zero3``    — ZeRO-3 sharding of traces and the NCCL exchange steps.
"""
from ._native import (ConfigError, CudaError, OomError, PoolError, TencacheError, TraceError, LIB_PATH)  # noqa: F401

__all__ = ["ConfigError", "CudaError", "OomError", "PoolError", "TencacheError", "TraceError", "LIB_PATH"]
