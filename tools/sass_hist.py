"""Per-kernel SASS instruction histograms of the built library (cuobjdump
-sass), the evidence that the hot kernels use the Blackwell instructions the
design names (UTCHMMA / UTMALDG / LDTM for tcgen05 + TMA, UBLKPF for bulk L2
prefetch, FFMA2 / FADD2 / FMNMX3, CREDUX). Writes a text summary.
usage: python tools/sass_hist.py [lib.so] > profiles/r02/sass_histograms.txt"""
import collections
import hashlib
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2603_06660_b200", "libpag_gpu.so")
KEY = ["UTCHMMA", "UTCBAR", "UTMALDG", "LDTM", "UBLKPF", "UBLKCP", "FFMA2", "FADD2", "FMUL2", "FMNMX3", "CREDUX",
       "REDUX", "VOTE", "SHFL", "MATCH", "LDG", "STG", "LDS", "STS", "ATOMS", "ATOMG", "RED", "BAR", "SYNCS"]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
sha = hashlib.sha256(open(lib, "rb").read()).hexdigest()[:16]
kernels = {}
cur = None
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        kernels[cur][m.group(1)] += 1
demangle = {}
try:
    out = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
    demangle = dict(zip(kernels, out))
except OSError:
    pass
print(f"# SASS histograms of {os.path.relpath(lib, ROOT)} (sha256 {sha}), {len(kernels)} kernels")
for k, c in sorted(kernels.items(), key=lambda kv: -sum(kv[1].values())):
    name = demangle.get(k, k)
    short = re.sub(r"pagdev::\(anonymous namespace\)::", "", name)[:150]
    print(f"\n## {short}\n   total {sum(c.values())}; " +
          ", ".join(f"{x} {c[x]}" for x in KEY if c[x]))
    print("   top: " + ", ".join(f"{x} {n}" for x, n in c.most_common(12)))
