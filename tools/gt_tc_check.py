"""Tensor-core ground truth vs the exact path (and the oracle) on a small index."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06660_b200 as pag
from oracle import oracle as O
from paper_2603_06660_b200.fvecs import gaussian_mixture, write_fvecs
import tempfile
td = tempfile.mkdtemp()
base = gaussian_mixture(20000, 96, 50, 0.5, seed=5, unit=True)
qs = gaussian_mixture(300, 96, 50, 0.5, seed=6, unit=True)
write_fvecs(os.path.join(td, "b.fvecs"), base)
O.ref_build(os.path.join(td, "b.fvecs"), os.path.join(td, "i.pagidx"), threads=16, M=8, efC=40)
ix = pag.load_index(os.path.join(td, "i.pagidx"))
for k in (1, 10, 32):
    t = time.time(); gi, gs = ix.ground_truth(qs, k); t1 = time.time() - t
    os.environ["PAG_GPU_GT_EXACT"] = "1"
    t = time.time(); ei, es = ix.ground_truth(qs, k); t2 = time.time() - t
    del os.environ["PAG_GPU_GT_EXACT"]
    oi, os_ = O.ground_truth(base, qs, k)
    print("k", k, "tc==exact", np.array_equal(gi, ei) and np.array_equal(gs, es), "exact==oracle",
          np.array_equal(ei, oi), "tc %.3fs exact %.3fs" % (t1, t2))
info = np.zeros(13, np.uint64)
pag._lib.lib.pag_gpu_info(ix.handle, info, 13)
print("uncertified total", int(info[12]))
