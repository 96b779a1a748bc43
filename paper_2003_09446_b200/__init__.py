"""B200-native DetNet layer-stack engine (arXiv 2003.09446 hot path).

The product is the CUDA library lib/libdetnet_b200.so behind the C-ABI in
include/detnet_b200.h; this package is its ctypes host binding plus seeded
workload builders. Importing it fails loudly if the library is not built.
"""
from .detnet import (BatchEval, ConfigError, Context, ContractError, CudaError, DetnetError,
                     DivergenceError, Model,
                     SingularMatrixError, UnsupportedError, lib_path, record_size, rng_seed,
                     rng_split, rng_stream, stream_wait_event)

__all__ = ["BatchEval", "ConfigError", "Context", "ContractError", "CudaError", "DetnetError",
           "DivergenceError",
           "Model", "SingularMatrixError", "UnsupportedError", "lib_path", "record_size",
           "rng_seed", "rng_split", "rng_stream", "stream_wait_event"]
