"""Summarise an ncu report: key SOL/occupancy metrics, stall reasons, top source lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM", "Theoretical Active Warps per SM",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Executed Instructions",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Block Limit Registers",
        "Block Limit Shared Mem"]
rows = list(csv.reader(run("--page", "details", "--csv").splitlines()))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
hdr, vals = raw[0], raw[2]
st = [(float(v), k) for k, v in zip(hdr, vals) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued") and v.replace('.', '', 1).isdigit()]
tot = sum(x for x, _ in st)
print("stall reasons (share of samples):")
for x, k in sorted(st, reverse=True)[:8]:
    print(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * x / tot:5.1f}%")
for k, v in zip(hdr, vals):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        print(k, v, raw[1][hdr.index(k)])
src = list(csv.reader(run("--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
out = []
for r in src[3:]:
    if len(r) < 8 or r[2] != '-':
        continue
    try:
        out.append((int(r[4]), int(r[7]), r[0], r[1][:88]))
    except ValueError:
        pass
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"source lines: samples {ts} instructions {ti}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:7d} {100 * o[0] / ts:5.1f}%  {100 * o[1] / ti:5.1f}%i  L{o[2]:<5s} {o[3]}")
