"""Time the tensor-core ground truth against the exact SIMT path on a cached
bench config and check bit-equality; one JSON line per k.
usage: python tools/gt_tc_bench.py cfg2 10 100 1000 [--lists]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_06660_b200 as pag  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
lists = "--lists" in sys.argv  # the per-split candidate-list path for k <= 32
ks = [int(x) for x in sys.argv[2:] if x != "--lists"] or [10]
cfg, p = bench.prepare(cfg_name, os.environ.get("PAG_CACHE", "/tmp/pag_b200_cache"), os.cpu_count())
ix = pag.load_index(p["index"])
q = read_fvecs(p["queries"])
for k in ks:
    os.environ.pop("PAG_GPU_GT_EXACT", None)
    if lists:
        os.environ["PAG_GPU_GT_LISTS"] = "1"
    ix.ground_truth(q[:256], k)  # warm
    u0 = ix.gt_uncertified()
    t = time.time()
    gi, gs = ix.ground_truth(q, k)
    t1 = time.time() - t
    unc = ix.gt_uncertified() - u0
    os.environ.pop("PAG_GPU_GT_LISTS", None)
    os.environ["PAG_GPU_GT_EXACT"] = "1"
    t = time.time()
    ei, es = ix.ground_truth(q, k)
    t2 = time.time() - t
    flop = 2.0 * len(q) * ix.n * ix.padded_dim
    print(json.dumps({"config": cfg_name, "k": k, "nq": len(q), "n": ix.n, "d": ix.padded_dim,
                      "path": ("tc-lists" if (k <= 32 and lists) else "tc-pool") if k <= 1000 else "exact",
                      "tc_s": round(t1, 4), "exact_s": round(t2, 4), "speedup": round(t2 / t1, 2),
                      "tc_gemm_equiv_tflops": round(flop / t1 / 1e12, 1),
                      "identical": bool(np.array_equal(gi, ei) and np.array_equal(gs.view(np.uint32),
                                                                                  es.view(np.uint32))),
                      "uncertified": int(unc)}), flush=True)
