"""B200-native PAG (Projection-Augmented Graph, arXiv 2603.06660) query path.

The compute path is the hand-written sm_100a library libpag_gpu.so (C ABI in
include/pag_gpu.h); this package mirrors the reference's host API over it.
"""
from .pag import (BatchResult, ConstructionResult, PagIndex, PendingBatch, SearchParams, SearchResult,
                  SearchStats, ground_truth, load_index, mean_recall, recall_at_k, search)

__all__ = ["BatchResult", "ConstructionResult", "PagIndex", "PendingBatch", "SearchParams", "SearchResult",
           "SearchStats", "ground_truth", "load_index", "mean_recall", "recall_at_k", "search"]
