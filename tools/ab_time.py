"""A/B timing of two builds of the library on a cached bench config, same
process order alternated (device-resident batches, K launches, CUDA events).
usage: PAG_CACHE=... python tools/ab_time.py cfg efs dist libA libB [reps]"""
import json
import os
import subprocess
import sys

cfg, efs, dist, la, lb = sys.argv[1:6]
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
res = {la: [], lb: []}
for r in range(reps):
    for lib in (la, lb) if r % 2 == 0 else (lb, la):
        env = dict(os.environ, PAG_GPU_LIB=lib)
        out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--efs", efs, "--dist", dist, "--steps", "10",
                              "--warmup", "3", "--no-cpu-baseline", "--no-e2e"], env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib].append(d["ms_per_step"])
        except Exception:
            print(out.stderr[-2000:], file=sys.stderr)
for lib, v in res.items():
    print(json.dumps({"lib": lib, "config": cfg, "efS": efs, "dist": dist, "ms_per_step": v,
                      "best": min(v) if v else None}))
