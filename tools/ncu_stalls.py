"""Top SASS lines by warp-stall samples: python tools/ncu_stalls.py report.ncu-rep kernel-regex [n]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
si, src, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
rows = [x for x in r[2:] if len(x) > si and x[si].isdigit()]
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print("samples", sum(int(x[si]) for x in rows), "warp instructions", sum(int(x[ie]) for x in rows))
agg = {c: sum(int(x[h.index(c)]) for x in rows) for c in stalls}
print(sorted(agg.items(), key=lambda a: -a[1])[:8])
for x in sorted(rows, key=lambda x: -int(x[si]))[:top_n]:
    print(x[si], x[ie], x[src][:60], [(c[6:], x[h.index(c)]) for c in stalls if int(x[h.index(c)]) > int(x[si]) // 4])
