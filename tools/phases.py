"""Per-phase cycle accounting of the search kernel (diagnostic build
build/lib_phase.so, -DPAG_PHASE_TIMING) on a cached bench config."""
import ctypes as C
import os
import sys

import numpy as np

os.environ.setdefault("PAG_GPU_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "build", "lib_phase.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_06660_b200 as pag  # noqa: E402
from paper_2603_06660_b200 import _lib  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
efs = int(sys.argv[2]) if len(sys.argv) > 2 else 70
exact = (sys.argv[3] != "fast") if len(sys.argv) > 3 else True
cfg, p = bench.prepare(cfg_name, os.environ.get("PAG_CACHE", "/tmp/pag_b200_cache"), os.cpu_count())
ix = pag.load_index(p["index"])
q = read_fvecs(p["queries"])
fn = _lib.lib.pag_gpu_phase_cycles
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 8)()
params = pag.SearchParams(K=cfg["K"], efS=efs, exact_dist=exact)
ix.search_batch(q, params)
fn(buf, 1)
r = ix.search_batch(q, params)
fn(buf, 1)
buf = list(buf)
names = ["setup+T+seeds", "marks", "argmin/entry/adj-issue", "adjacency wait+visited", "PRT+codes",
         "distances", "replay", "end_round/flush/out"]
tot = sum(buf)
exp = r.stats[:, 3].sum()
import torch  # noqa: E402
nq = q.shape[0]
qd = torch.from_numpy(q).cuda()
outs = [torch.empty((nq, cfg["K"]), dtype=torch.int32, device="cuda"),
        torch.empty((nq, cfg["K"]), dtype=torch.float32, device="cuda"),
        torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), 0)
torch.cuda.synchronize()
fn((C.c_ulonglong * 8)(), 1)  # (phase counters of this extra run are discarded)
raw = outs[3].cpu().numpy().view(np.uint32)
spec = float((raw[:, 7] >> 16).sum())
print(f"speculative survivors {spec / nq:.1f} per query vs exact distances (passes + seeds) "
      f"{r.stats[:, 0].mean():.1f}: {spec / r.stats[:, 2].sum():.3f} rows per pass")
print(f"{cfg_name} efS={efs} exact={exact}: total warp-cycles {tot:.3e}; per expansion {tot / exp:.0f} cycles")
for k in range(8):
    if buf[k]:
        print(f"  {names[k]:28s} {100 * buf[k] / tot:5.1f}%  {buf[k] / exp:8.0f} cyc/expansion")
