"""The reference's acceptance criterion 7 (proj/tests/acceptance.cpp:360-426,
"search-state invariants under fuzz") on the GPU: the same index recipe
(gen_synthetic(gaussian, 2000, 32, 700), BuildParams{M = 12, efC = 120,
seed = 31}, built by the reference binary), 10,000 N(0, 1) queries, each with
its own K in [1, 64] and efS = K + U[0, 128). Run through the invariant-
checking build (PAG_GPU_LIB=build/lib_validate.so: capacity, z_max, single
residence, result order after every expansion and end_round, reported as the
reference's logic_error texts) in both distance modes; every result is also
compared bit for bit with the oracle (reference order, and the warp-tree
order), and the conservation rule exact = seeds + passes is checked.
usage: PAG_GPU_LIB=build/lib_validate.so python tests/fuzz_criterion7.py [queries] > fuzz_criterion7.json"""
import collections
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_06660_b200 as pag  # noqa: E402
from oracle import oracle as O  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
with tempfile.TemporaryDirectory() as td:
    b, i = os.path.join(td, "c7.fvecs"), os.path.join(td, "c7.pagidx")
    O.ref_gen_synthetic("gaussian", 2000, 32, 700, b)
    O.ref_build(b, i, threads=1, M=12, efC=120, seed=31)
    ix, oix = pag.load_index(i), O.OracleIndex(i)
    rng = np.random.default_rng(701)
    q = rng.standard_normal((nq, 32)).astype(np.float32)
    K = rng.integers(1, 65, nq)
    efS = K + rng.integers(0, 128, nq)
    groups = collections.defaultdict(list)
    for j in range(nq):
        groups[(int(K[j]), int(efS[j]))].append(j)
    n_seeds = min(32, len(oix.entry_nodes()))
    out = {"queries": nq, "distinct_K_efS": len(groups), "library": os.environ.get("PAG_GPU_LIB", "default"),
           "invariant_violations": 0, "first_violation": None}
    for mode, exact in (("reference_order", True), ("warp_tree", False)):
        equal = conserved = 0
        for (k, e), idx in groups.items():
            qs = q[idx]
            try:
                got = ix.search_batch(qs, pag.SearchParams(K=k, efS=e, exact_dist=exact))
            except AssertionError as err:  # the reference's logic_error texts (PAG_VALIDATE)
                out["invariant_violations"] += len(idx)
                out["first_violation"] = out["first_violation"] or str(err)
                continue
            ids, sq, n_out, st = oix.search(qs, k, e, warp_tree=not exact)
            for r in range(len(idx)):
                n = int(n_out[r])
                equal += int(got.n_out[r] == n and np.array_equal(got.ids[r, :n], ids[r, :n])
                             and np.array_equal(got.sq[r, :n].view(np.uint32), sq[r, :n].view(np.uint32))
                             and np.array_equal(got.stats[r], st[r]))
                conserved += int(got.stats[r][0] == min(max(10, k), n_seeds) + got.stats[r][2])
        out[mode] = {"bit_identical_to_oracle": equal, "exact_equals_seeds_plus_passes": conserved}
    ix.close()
print(json.dumps(out))
