"""Regenerates the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/pag_ref, compiled from /root/reference/proj/src). Run in the
build container (where /root/reference exists):

    python tests/golden/make_golden.py

Outputs (small, committed):
  golden_index.pagidx   PAGIDX01 v1 index built single-threaded by the reference
  golden_queries.fvecs  16 raw queries
  golden_expected.npz   reference search results for each (K, efS) in CASES
                        plus exact ground truth (k = 32) from the reference
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2603_06660_b200.fvecs import gaussian_mixture, write_fvecs  # noqa: E402

CASES = [(10, 10), (10, 30), (10, 100), (1, 1), (5, 40), (32, 64), (40, 160)]


def main():
    base = gaussian_mixture(800, 24, 12, 0.5, seed=31, centre_seed=7)
    queries = gaussian_mixture(16, 24, 12, 0.5, seed=32, centre_seed=7)
    b = os.path.join(HERE, "golden_base.fvecs")
    q = os.path.join(HERE, "golden_queries.fvecs")
    idx = os.path.join(HERE, "golden_index.pagidx")
    write_fvecs(b, base)
    write_fvecs(q, queries)
    O.ref_build(b, idx, threads=1, M=8, efC=60, seed=11)
    out = {}
    for K, efS in CASES:
        ids, sq, n_out, st, _ = O.ref_search(idx, q, K, efS, os.path.join(HERE, "_tmp.bin"), no_warm=True)
        out[f"ids_{K}_{efS}"] = ids
        out[f"sq_{K}_{efS}"] = sq
        out[f"n_{K}_{efS}"] = n_out
        out[f"stats_{K}_{efS}"] = st
    gi, gs = O.ref_gt(b, q, 32, os.path.join(HERE, "_tmp.bin"))
    out["gt_ids"], out["gt_sq"] = gi, gs
    np.savez_compressed(os.path.join(HERE, "golden_expected.npz"), cases=np.array(CASES), **out)
    os.remove(os.path.join(HERE, "_tmp.bin"))
    os.remove(b)  # the index carries the rows
    print("golden fixtures written:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
