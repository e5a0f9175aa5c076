"""B200-native GENIE match-count engine (arXiv 1603.08390), drop-in for the
`mcx` batched query path.  See DESIGN.md.

Layers:
  _native  ctypes bindings of the C ABI (include/genie/genie.h)
  engine   array-level API: DeviceIndex, DeviceGroup, QueryBatch, Results, Encoder
  mcx      object-level mirror of the reference API (namespace mcx)
  synth    seeded synthetic workloads of the five BASELINE configs
  dist     multi-GPU sharding + all-gather merge over torch.distributed
"""
from .engine import (CSR, ContractError, CudaError, DataError, DeviceGroup, DeviceIndex, Encoder, InvariantError, McxError,
                     QueryBatch, Results, config, hash_results, lsh_config, merge_lists, point_queries)

__all__ = ["CSR", "ContractError", "CudaError", "DataError", "DeviceGroup", "DeviceIndex", "Encoder", "InvariantError", "McxError",
           "QueryBatch", "Results", "config", "hash_results", "lsh_config", "merge_lists", "point_queries"]
