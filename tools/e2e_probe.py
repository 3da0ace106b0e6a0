"""Where the end-to-end (host buffers) time goes on the cached cfg2 index:
search_batch wall time vs the device-resident kernel time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_06660_b200 as pag  # noqa: E402
from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

cfg, p = bench.prepare("cfg2", "/tmp/pag_b200_cache", os.cpu_count())
ix = pag.load_index(p["index"])
q = read_fvecs(p["queries"])
nq = q.shape[0]
qp = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
qp.numpy()[:] = q
params = pag.SearchParams(K=10, efS=70, exact_dist=False)
for _ in range(3):
    ix.search_batch(qp.numpy(), params)
ts = []
for _ in range(10):
    t = time.perf_counter()
    ix.search_batch(qp.numpy(), params)
    ts.append(time.perf_counter() - t)
print(f"search_batch pinned: median {1e3 * np.median(ts):.3f} ms")
ts = []
for _ in range(10):
    t = time.perf_counter()
    ix.search_batch(q, params)
    ts.append(time.perf_counter() - t)
print(f"search_batch pageable: median {1e3 * np.median(ts):.3f} ms")
qd = qp.cuda()
outs = [torch.empty((nq, 10), dtype=torch.int32, device="cuda"), torch.empty((nq, 10), dtype=torch.float32, device="cuda"),
        torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
s = torch.cuda.Stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
ev[0].record(s)
for _ in range(10):
    ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
ev[1].record(s)
torch.cuda.synchronize()
print(f"device kernel: {ev[0].elapsed_time(ev[1]) / 10:.3f} ms")
ts = []
for _ in range(10):
    t = time.perf_counter()
    ix.search_device(qd.data_ptr(), nq, params, *(t_.data_ptr() for t_ in outs), s.cuda_stream)
    s.synchronize()
    ts.append(time.perf_counter() - t)
print(f"device call + sync wall: median {1e3 * np.median(ts):.3f} ms")
# zero-copy query reads inside the kernel: kernel fed from pinned host memory
ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev2[0].record(s)
for _ in range(10):
    ix.search_device(qp.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
ev2[1].record(s)
torch.cuda.synchronize()
print(f"device kernel reading pinned host queries: {ev2[0].elapsed_time(ev2[1]) / 10:.3f} ms")
