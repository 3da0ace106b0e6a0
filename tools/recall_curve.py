"""QPS-recall curve on a cached bench config (one B200): for each efS of the
config's sweep (plus larger ones), recall@K of the warp-tree search against
the exact GPU ground truth and the device-resident QPS of 10 back-to-back
10k-query launches, for both distance modes.
usage: python tools/recall_curve.py cfg2 [efS ...]  -> JSON on stdout"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_06660_b200 as pag  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg, p = bench.prepare(cfg_name, os.environ.get("PAG_CACHE", "/tmp/pag_b200_cache"), os.cpu_count())
K = cfg["K"]
efs_list = [int(x) for x in sys.argv[2:]] or [e for e in cfg["efs"] if e >= K]
ix = pag.load_index(p["index"])
q = read_fvecs(p["queries"])
nq = q.shape[0]
gt_ids, gt_sq = ix.ground_truth(q, K)
qd = torch.from_numpy(q).cuda()
outs = [torch.empty((nq, K), dtype=torch.int32, device="cuda"), torch.empty((nq, K), dtype=torch.float32, device="cuda"),
        torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
s = torch.cuda.Stream()
rows = []
for efs in efs_list:
    row = {"efS": efs}
    for mode in ("warp-tree", "exact"):
        params = pag.SearchParams(K=K, efS=efs, exact_dist=mode == "exact")
        for _ in range(3):
            ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(10):
            ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
        ev[1].record(s)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 10
        ids = outs[0].cpu().numpy().view(np.uint32)
        n = outs[2].cpu().numpy().view(np.uint32)
        st = outs[3].cpu().numpy().view(np.uint32).astype(np.float64)
        row[mode] = {"qps": round(nq / ms * 1e3, 1), "recall": round(pag.mean_recall(ids, n, gt_ids, gt_sq, K), 4),
                     "exact_per_query": round(float(st[:, 0].mean()), 1)}
    print(f"efS={efs}: {row}", file=sys.stderr, flush=True)
    rows.append(row)
print(json.dumps({"workload": cfg_name, "n": cfg["n"], "d": cfg["d"], "K": K, "queries": nq,
                  "timing": "device-resident batch, 10 back-to-back launches after 3 warm-up, CUDA events",
                  "curve": rows}))
