"""recall_at_k (proj/src/bench.cpp:55-71) and its batch mean. Plain numpy,
no native library: the evaluation metric, shared by the GPU API (pag.py) and
the measurement code's reference arm, which must not load libpag_gpu.so."""
from __future__ import annotations

import numpy as np


def recall_at_k(result_ids, truth_ids, truth_sq, K: int) -> float:
    """bench.cpp:55-71: |result[0..K) ∩ truth| / K, ids distance-tied with
    the K-th true neighbour count as hits."""
    truth_ids = np.asarray(truth_ids)
    truth_sq = np.asarray(truth_sq, np.float32)
    k = min(K, len(truth_ids))
    if k == 0:
        return 0.0
    tie = truth_sq[k - 1]
    first = {}
    for i, t in enumerate(truth_ids.tolist()):
        first.setdefault(t, truth_sq[i])
    hits = 0
    for r in list(result_ids)[:K]:
        s = first.get(int(r))
        if s is not None and s <= tie:
            hits += 1
    return hits / K


def mean_recall(ids: np.ndarray, n_out: np.ndarray, truth_ids: np.ndarray, truth_sq: np.ndarray,
                K: int) -> float:
    """Vectorised recall_at_k averaged over a batch (same tie policy)."""
    nq = ids.shape[0]
    k = min(K, truth_ids.shape[1])
    if k == 0 or nq == 0:
        return 0.0
    total = 0.0
    step = max(1, int(2e7 // max(1, K * truth_ids.shape[1])))
    for s in range(0, nq, step):
        e = min(nq, s + step)
        tie = truth_sq[s:e, k - 1:k]
        ok = truth_sq[s:e] <= tie                                  # q x kt
        res = ids[s:e, :K].astype(np.int64)
        valid = np.arange(res.shape[1])[None, :] < n_out[s:e, None]
        res = np.where(valid, res, -1)
        hit = (res[:, :, None] == truth_ids[s:e, None, :].astype(np.int64)) & ok[:, None, :]
        total += float(hit.any(axis=2).sum())
    return total / (nq * K)
