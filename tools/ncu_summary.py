"""Key ncu 'details' metrics per kernel launch: python tools/ncu_summary.py report.ncu-rep [name-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ni, mi, ui, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Memory Throughput",
        "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Block Limit Shared Mem", "Block Limit Registers"]
by = {}
for r in rows[1:]:
    if len(r) <= vi or (pat and not pat.search(r[ni])):
        continue
    if r[mi] in want:
        by.setdefault((r[ki], r[ni][:40]), {})[r[mi]] = r[vi] + " " + r[ui]
for (k, n), m in by.items():
    print(k, n)
    for w in want:
        if w in m:
            print(f"   {w:36s} {m[w]}")
