"""Extract dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture into
profiles/verify_dram_bytes.json (the roofline "traffic" field bench.py reports).
  python tools/ncu_traffic.py gpurun_out/prof_verify.ncu-rep config2"""
import csv
import json
import os
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(name):
    i = hdr.index(name)
    return float(vals[i].replace(",", "")) * scale[units[i]]


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
out = {"workload": workload, "bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
       "kernel": vals[hdr.index("Kernel Name")], "source": os.path.basename(rep)}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "verify_dram_bytes.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out)
