"""Kernel QPS versus batch size on the cached cfg2 index (tail effect of the
persistent grid), and back-to-back launches with / without overlap."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_06660_b200 as pag  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

cfg, p = bench.prepare("cfg2", "/tmp/pag_b200_cache", os.cpu_count())
ix = pag.load_index(p["index"])
q0 = read_fvecs(p["queries"])
params = pag.SearchParams(K=10, efS=70, exact_dist=False)
s = torch.cuda.Stream()
for mult in (1, 2, 4):
    q = np.concatenate([q0] * mult)
    nq = q.shape[0]
    qd = torch.from_numpy(q).cuda()
    outs = [torch.empty((nq, 10), dtype=torch.int32, device="cuda"),
            torch.empty((nq, 10), dtype=torch.float32, device="cuda"),
            torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
    for _ in range(3):
        ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(s)
    for _ in range(10):
        ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
    ev[1].record(s)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 10
    print(f"batch {nq}: {ms:.3f} ms/launch, {nq / ms * 1e3 / 1e6:.3f} M QPS")
