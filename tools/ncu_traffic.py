"""Extract per-launch DRAM traffic of the fused MVM from an ncu --set full report into
profiles/mvm_traffic.json (read by bench.py for roofline.traffic).
python tools/ncu_traffic.py report.ncu-rep WORKLOAD VARIANT"""
import csv
import io
import json
import os
import subprocess
import sys

rep, workload, variant = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
get = {k: (x, u) for k, u, x in zip(h, units, v)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(k):
    x, u = get[k]
    return float(x.replace(",", "")) * scale.get(u, 1.0)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
out = {"workload": workload, "variant": variant, "kernel": get["Kernel Name"][0],
       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
       "duration_us": val("gpu__time_duration.sum") / 1e3 if get["gpu__time_duration.sum"][1] == "nsecond"
       else float(get["gpu__time_duration.sum"][0]),
       "source": f"ncu --set full --clock-control none ({os.path.basename(rep)}), dram__bytes_read.sum + "
                 f"dram__bytes_write.sum"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "mvm_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
