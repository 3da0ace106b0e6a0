"""Aggregate ncu source-page instruction counts and stall samples by the
function (line range) they belong to in pag_search.cu."""
import csv
import re
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
nq = float(sys.argv[3]) if len(sys.argv) > 3 else 1e4
lines = open(src).read().splitlines()
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"\s*(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\(", l)
    if m and not l.strip().endswith(";"):
        starts.append((i, m.group(1)))
starts.sort()


def fn_of(ln):
    name = "top"
    for s, n in starts:
        if s <= ln:
            name = n
    return name


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, aggs = {}, {}
fname = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if len(r) < 8 or r[2] != "-":
        continue
    try:
        ln, n, s = int(r[0]), int(r[7]), int(r[4])
    except ValueError:
        continue
    key = fn_of(ln) if fname and fname.endswith(src.split("/")[-1]) else f"hdr:{fname.split('/')[-1] if fname else '?'}"
    agg[key] = agg.get(key, 0) + n
    aggs[key] = aggs.get(key, 0) + s
t, ts = sum(agg.values()) or 1, sum(aggs.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:25]:
    print(f"{k:28s} {100 * v / t:5.1f}% instr {100 * aggs[k] / ts:5.1f}% stall {v / nq:9.0f} instr/query")
