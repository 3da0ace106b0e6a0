"""Per-kernel registers / spills from a csrc/build/*.ptxas.log (nvcc -Xptxas -v)."""
import re
import subprocess
import sys

log = open(sys.argv[1]).read()
for e in re.split(r"ptxas info    : Compiling entry function '", log)[1:]:
    name = e.split("'")[0]
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", e)
    r = re.search(r"Used (\d+) registers", e)
    short = dem.replace("pagdev::(anonymous namespace)::", "").replace("void ", "")
    short = re.sub(r"\(pagdev::SearchLaunch\)", "", short)
    print(f"{short[:100]:100s} regs {r.group(1):>3s} stack/spill-st/spill-ld {m.groups() if m else None}")
