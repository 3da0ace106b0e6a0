"""B200-native PAG (Projection-Augmented Graph, arXiv 2603.06660) query path.

The compute path is the hand-written sm_100a library libpag_gpu.so (C ABI in
include/pag_gpu.h); this package mirrors the reference's host API over it.

The library is loaded on first use of the API (PEP 562 module __getattr__),
not at package import: the data helpers (fvecs, shard) import without it, so
a process that only needs them (the reference arm of bench.py) never maps
libpag_gpu.so. The first API access raises ImportError when the library is
missing (no CPU fallback exists).
"""
from __future__ import annotations

import importlib

__all__ = ["BatchResult", "ConstructionResult", "IndexArrays", "PagIndex", "PendingBatch", "SearchParams", "SearchResult",
           "SearchStats", "ground_truth", "load_index", "mean_recall", "recall_at_k", "search"]


def __getattr__(name):
    if name in ("mean_recall", "recall_at_k"):  # plain numpy (recall.py)
        return getattr(importlib.import_module(".recall", __name__), name)
    if name in __all__:
        return getattr(importlib.import_module(".pag", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return sorted(list(globals()) + __all__)
