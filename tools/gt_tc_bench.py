"""Time tensor-core vs exact ground truth on a cached bench config; check equality."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2603_06660_b200 as pag
from paper_2603_06660_b200.fvecs import read_fvecs
cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg, p = bench.prepare(cfg_name, os.environ.get("PAG_CACHE", "/tmp/pag_b200_cache"), os.cpu_count())
ix = pag.load_index(p["index"])
q = read_fvecs(p["queries"])
ix.ground_truth(q[:256], k)  # warm
t = time.time(); gi, gs = ix.ground_truth(q, k); t1 = time.time() - t
info = np.zeros(13, np.uint64); pag._lib.lib.pag_gpu_info(ix.handle, info, 13)
os.environ["PAG_GPU_GT_EXACT"] = "1"
t = time.time(); ei, es = ix.ground_truth(q, k); t2 = time.time() - t
print(f"{cfg_name} k={k} nq={len(q)}: tensor-core {t1:.3f}s exact {t2:.3f}s speedup {t2/t1:.1f}x "
      f"identical={np.array_equal(gi, ei) and np.array_equal(gs.view(np.uint32), es.view(np.uint32))} "
      f"uncertified={int(info[12])}")
