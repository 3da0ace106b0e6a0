"""A/B timing of two library builds on the construction-search bench (cfg-2
index, bit-exact distances), alternating order.
usage: python tools/ab_cons.py libA libB [reps]"""
import json
import os
import subprocess
import sys

la, lb = sys.argv[1:3]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {la: [], lb: []}
for r in range(reps):
    for lib in (la, lb) if r % 2 == 0 else (lb, la):
        out = subprocess.run([sys.executable, "bench.py", "--mode", "construction", "--steps", "5", "--warmup", "3",
                              "--no-cpu-baseline", "--no-e2e"], env=dict(os.environ, PAG_GPU_LIB=lib),
                             capture_output=True, text=True)
        try:
            res[lib].append(json.loads(out.stdout.strip().splitlines()[-1])["ms_per_step"])
        except Exception:
            print(out.stderr[-2000:], file=sys.stderr)
for lib, v in res.items():
    print(json.dumps({"lib": lib, "mode": "construction", "ms_per_step": v, "best": min(v) if v else None}))
