"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the hop kernels from an ncu
--set full report, averaged per kernel family as bench.py's roofline uses them:
  feature_hop = hop_kernel<0|1|2|5,...> (feature kinds), gcn_hop = hop_kernel<3|6,...> (GCN, paired GCN).
Usage: python tools/traffic_from_ncu.py <report.ncu-rep> <config> [out.json]"""
import csv
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
fam = {}
for d in data:
    name = d[hdr.index("Kernel Name")]
    if "hop_kernel<" not in name:
        continue
    kind = int(name.split("hop_kernel<")[1].split(",")[0])
    key = "gcn_hop" if kind in (3, 6) else ("transform" if kind == 4 else "feature_hop")
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[hdr.index(m)].replace(",", "")) * mul[units[hdr.index(m)]]
    fam.setdefault(key, []).append(b)
try:
    js = json.load(open(out))
except Exception:
    js = {}
js[cfg] = {k: sum(v) / len(v) for k, v in fam.items()}
js[cfg]["_source"] = rep
json.dump(js, open(out, "w"), indent=1)
print(js[cfg])
