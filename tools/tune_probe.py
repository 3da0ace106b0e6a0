"""A/B of PAG_GPU_TUNE settings on a cached bench index: kernel time per
10k/20k-query launch (device-resident, 10 back-to-back launches) and a hash
of the returned ids (must not change). TUNES="a b c" lists the settings.
usage: python tools/tune_probe.py [cfg] [efS]"""
import os
import subprocess
import sys

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
efs = int(sys.argv[2]) if len(sys.argv) > 2 else 70

if os.environ.get("PF_CHILD"):
    import numpy as np
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench  # noqa: E402
    import paper_2603_06660_b200 as pag  # noqa: E402
    from paper_2603_06660_b200.fvecs import read_fvecs  # noqa: E402

    cfg, p = bench.prepare(cfg_name, "/tmp/pag_b200_cache", os.cpu_count())
    K = cfg["K"]
    ix = pag.load_index(p["index"])
    q = read_fvecs(p["queries"])
    nq = q.shape[0]
    params = pag.SearchParams(K=K, efS=efs, exact_dist=bool(int(os.environ.get("EXACT", "0"))))
    s = torch.cuda.Stream()
    qd = torch.from_numpy(q).cuda()
    outs = [torch.empty((nq, K), dtype=torch.int32, device="cuda"),
            torch.empty((nq, K), dtype=torch.float32, device="cuda"),
            torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq, 8), dtype=torch.int32, device="cuda")]
    for _ in range(3):
        ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    steps = 10
    ev[0].record(s)
    for _ in range(steps):
        ix.search_device(qd.data_ptr(), nq, params, *(t.data_ptr() for t in outs), s.cuda_stream)
    ev[1].record(s)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    st = outs[3].cpu().numpy().view(np.uint32).astype(np.float64)
    ids = outs[0].cpu().numpy()
    line = f"tune={os.environ.get('PAG_GPU_TUNE', '0'):>4} {ms:.3f} ms/launch {nq / ms / 1e3:.3f} M QPS"
    line += f"  ids-hash {int(np.bitwise_xor.reduce(ids.astype(np.int64).ravel() * 2654435761 % (1 << 31)))}"
    print(line, flush=True)
else:
    for t in os.environ.get("TUNES", "0 1024 0 1024").split():
        subprocess.run([sys.executable, __file__, cfg_name, str(efs)],
                       env=dict(os.environ, PF_CHILD="1", PAG_GPU_TUNE=t), check=False)
