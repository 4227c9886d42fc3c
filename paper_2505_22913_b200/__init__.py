"""B200-native (sm_100a) Mustafar hot path: per-token magnitude pruning of the KV cache,
bitmap compression, and decode attention over the compressed cache (arXiv 2505.22913).

The compute path is the C-ABI library lib/libmustafar.so (include/mustafar.h); this
package is its thin binding plus the build script. See DESIGN.md.
"""
from .mustafar import (  # noqa: F401
    BUFFERS, EXPORTS, LIB_PATH, OUT_F16, OUT_F32, DenseAttention, MustafarCache, MustafarError,
    buffer_bytes, k_pad, keep_from_sparsity, lib, shard_units,
)
