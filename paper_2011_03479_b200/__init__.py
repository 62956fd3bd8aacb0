"""B200-native GEMPE hot path: one Jacobi round of the predictive-entropy graph embedding
(reference: entropy-embed, /root/reference/proj) behind the C-ABI of include/gempe.h."""
from .engine import (ConfigError, Context, CudaError, DataError, DivergenceError, EmbeddingEngine, EmbedResult,
                     Graph, Group, IterationConfig, IterationStats, NearCompleteGraphError, alloc_host, embed, free_host,
                     trim_device_cache)
from ._capi import (INIT_NORMAL, INIT_REFERENCE, INIT_UNIFORM_PM1, MATH_EXACT, MATH_TABLES, NEG_PER_EDGE_2,
                    NEG_PER_VERTEX_K, RNG_PHILOX, RNG_REFERENCE)

__all__ = ["ConfigError", "Context", "CudaError", "DataError", "DivergenceError", "EmbeddingEngine", "EmbedResult",
           "Graph", "Group", "IterationConfig", "IterationStats", "NearCompleteGraphError", "embed", "trim_device_cache", "alloc_host", "free_host",
           "INIT_NORMAL",
           "INIT_REFERENCE", "INIT_UNIFORM_PM1", "MATH_EXACT", "MATH_TABLES", "NEG_PER_EDGE_2", "NEG_PER_VERTEX_K",
           "RNG_PHILOX", "RNG_REFERENCE"]
