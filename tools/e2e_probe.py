"""Where the end-to-end (host buffers) time goes on the cached cfg2 index."""
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
S = 10


def timeit(label, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(S):
        fn()
    torch.cuda.synchronize()
    print(f"{label:48s} {1e3 * (time.perf_counter() - t) / S:.3f} ms/batch")


timeit("search_batch (sync, pinned q)", lambda: ix.search_batch(qp.numpy(), params))
qd = qp.cuda()
outs = [torch.empty((nq, 10), dtype=torch.int32, device="cuda"), torch.empty((nq, 10), dtype=torch.float32, device="cuda"),
        torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
s = torch.cuda.Stream()
timeit("device q, device out (back to back)",
       lambda: ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream))
timeit("pinned host q, device out (back to back)",
       lambda: ix.search_device(qp.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream))
hout = [torch.empty((nq, 10), dtype=torch.int32, pin_memory=True), torch.empty((nq, 10), dtype=torch.float32, pin_memory=True),
        torch.empty((nq,), dtype=torch.int32, pin_memory=True), torch.empty((nq, 8), dtype=torch.int32, pin_memory=True)]
timeit("device q, pinned host out (back to back)",
       lambda: ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in hout), s.cuda_stream))
timeit("pinned q, pinned out (back to back)",
       lambda: ix.search_device(qp.data_ptr(), nq, params, *(t.data_ptr() for t in hout), s.cuda_stream))
pend = []


def async_step():
    pend.append(ix.search_submit(qp.numpy(), params))
    if len(pend) == 3:
        pend.pop(0).wait()


timeit("async submit/wait, depth 3", async_step)
while pend:
    pend.pop(0).wait()
bufs = [pag.BatchResult(np.zeros((nq, 10), np.uint32), np.zeros((nq, 10), np.float32), np.zeros(nq, np.uint32),
                        np.zeros((nq, 5), np.uint64)) for _ in range(4)]
k = [0]


def async_step2():
    pend.append(ix.search_submit(qp.numpy(), params, out=bufs[k[0] % 4]))
    k[0] += 1
    if len(pend) == 3:
        pend.pop(0).wait()


timeit("async submit/wait, depth 3, reused outputs", async_step2)
while pend:
    pend.pop(0).wait()
ts, tw = [], []
for i in range(20):
    t = time.perf_counter()
    pb = ix.search_submit(qp.numpy(), params, out=bufs[i % 4])
    ts.append(time.perf_counter() - t)
    t = time.perf_counter()
    pb.wait()
    tw.append(time.perf_counter() - t)
print(f"submit {1e3 * np.median(ts):.3f} ms, wait (incl. kernel) {1e3 * np.median(tw):.3f} ms")
