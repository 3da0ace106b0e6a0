"""Record the search kernel's DRAM bytes per launch from ncu CSV captures
into profiles/ncu_traffic.json, keyed by workload, distance mode, efS, batch
size and the library's source hash (bench.source_sha), which bench.py checks
before reporting roofline.traffic.
usage: python tools/ncu_traffic.py CAPTURE.csv CONFIG DIST EFS NQ [more quintuples...]
The CSV comes from `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum
--csv -k regex:pag_search -c 1 ...` (or --set full --csv)."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

out = os.path.join(bench.ROOT, "profiles", "ncu_traffic.json")
try:
    data = json.load(open(out))
except (OSError, ValueError):
    data = {}
data = {"_comment": "DRAM bytes per launch of pag_search_kernel (dram__bytes_read.sum + dram__bytes_write.sum) "
                    "from one ncu capture each; bench.py reports it as roofline.traffic only when config, distance "
                    "mode, efS, batch size and the library's source hash all match.",
        "captures": [c for c in data.get("captures", []) if c.get("source_sha") == bench.source_sha()]}
args = sys.argv[1:]
for i in range(0, len(args), 5):
    path, cfg, dist, efs, nq = args[i:i + 5]
    rd = wr = None
    for row in csv.reader(l for l in open(path) if l.startswith('"')):
        if len(row) < 3:
            continue
        if row[-3] == "dram__bytes_read.sum" or (len(row) > 12 and "dram__bytes_read.sum" in row):
            rd = float(row[-1].replace(",", ""))
        if row[-3] == "dram__bytes_write.sum" or (len(row) > 12 and "dram__bytes_write.sum" in row):
            wr = float(row[-1].replace(",", ""))
    if rd is None or wr is None:
        sys.exit(f"no dram byte metrics in {path}")
    unit_scale = 1.0
    data["captures"] = [c for c in data["captures"] if not (c["config"] == cfg and c["dist"] == dist
                                                            and c["efS"] == int(efs))]
    data["captures"].append({"config": cfg, "dist": dist, "efS": int(efs), "queries_per_launch": int(nq),
                             "dram_bytes_read": rd * unit_scale, "dram_bytes_write": wr * unit_scale,
                             "bytes_per_launch": (rd + wr) * unit_scale, "source_sha": bench.source_sha(),
                             "capture": os.path.relpath(path, bench.ROOT)})
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(data, indent=1))
