"""Driver for tests/test_validate.py, run in its own process with
PAG_GPU_LIB pointing at the invariant-checking build (build/lib_validate.so,
-DPAG_VALIDATE): searches and construction searches over the given indexes;
any violated TfbState invariant raises the reference's logic_error text
(AssertionError here); results must also stay bit-identical to the oracle.
usage: python tests/validate_run.py index.pagidx queries.fvecs [...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_06660_b200 as pag  # noqa: E402
from conftest import assert_same_results  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

assert os.environ.get("PAG_GPU_LIB", "").endswith("lib_validate.so")
checked = 0
args = sys.argv[1:]
for i in range(0, len(args), 2):
    ipath, qpath = args[i], args[i + 1]
    q = read_fvecs(qpath)
    ix = pag.load_index(ipath)
    oix = O.OracleIndex(ipath)
    for K, efS, b in ((10, 10, 0), (10, 80, 0), (1, 1, 0), (32, 96, 0), (10, 300, 7), (50, 120, 0), (100, 300, 0),
                      (150, 400, 160)):
        for exact in (True, False):
            got = ix.search_batch(q, pag.SearchParams(K=K, efS=efS, b_override=b, exact_dist=exact))
            if exact:
                assert_same_results((got.ids, got.sq, got.n_out, got.stats), oix.search(q, K, efS, b_override=b),
                                    f"{ipath} {K}/{efS}/{b}")
            checked += len(q)
    nodes = np.arange(0, ix.n, 17, dtype=np.uint32)
    got = ix.construction_search(nodes)
    want = oix.construction_search(nodes)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats), want[:4], f"{ipath} construction")
    checked += len(nodes)
    ix.close()
print(f"validated {checked} searches")
