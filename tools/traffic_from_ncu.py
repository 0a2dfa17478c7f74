"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the hop kernels from an ncu
--set full report, averaged per kernel family as bench.py's roofline uses them:
  feature_hop = hop_kernel<0|1|2|5,...> (feature kinds), gcn_hop = hop_kernel<3|6,...> (GCN, paired GCN).
Usage: python tools/traffic_from_ncu.py <report.ncu-rep | raw-page.csv> <config> [out.json]"""
import csv
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
fam, extra = {}, {}
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

    def val(m):
        return float(d[hdr.index(m)].replace(",", "")) if m in hdr and d[hdr.index(m)] else None
    sec, req = val("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"), val("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
    extra.setdefault(key, []).append({"l2_hit_rate_pct": val("lts__t_sector_hit_rate.pct"),
                                      "sectors_per_request": (sec / req) if sec and req else None,
                                      "dram_pct_of_nominal_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")})
try:
    js = json.load(open(out))
except Exception:
    js = {}
js[cfg] = {k: sum(v) / len(v) for k, v in fam.items()}
for k, lst in extra.items():   # per-launch counters averaged per family
    js[cfg][k + "_ncu"] = {m: (sum(e[m] for e in lst if e[m] is not None) / max(1, sum(e[m] is not None for e in lst)))
                           for m in lst[0]}
js[cfg]["_source"] = rep
json.dump(js, open(out, "w"), indent=1)
print(js[cfg])
