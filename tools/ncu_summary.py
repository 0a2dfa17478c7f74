"""Summarise ncu output for profiles/: per-kernel launch shares (from a --metrics gpu__time_duration.sum
CSV log) and the key counters of a --set full report (raw page CSV)."""
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in data:
        name = r[ki].split("(")[0].replace("unnamed>::", "")
        tot.setdefault(name, [0.0, 0])
        tot[name][0] += float(r[vi].replace(",", ""))
        tot[name][1] += 1
    s = sum(v[0] for v in tot.values())
    out = ["kernel | launches | total ms | share", "---|---|---|---"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
        out.append(f"{k} | {v[1]} | {v[0] / 1e6:.3f} | {100 * v[0] / s:.1f}%")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        name = d[hdr.index("Kernel Name")].split("(")[0].replace("unnamed>::", "")
        out.append(f"### {name}")
        vals = {k: d[hdr.index(k)] for k in KEYS if k in hdr}
        for k in KEYS:
            if k in vals:
                out.append(f"- {k}: {vals[k]} {units[hdr.index(k)]}")
        try:
            t = float(vals["gpu__time_duration.sum"].replace(",", ""))
            tu = units[hdr.index("gpu__time_duration.sum")]
            t_s = t * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}[tu]
            rb = float(vals["dram__bytes_read.sum"].replace(",", ""))
            wb = float(vals["dram__bytes_write.sum"].replace(",", ""))
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= mul[units[hdr.index("dram__bytes_read.sum")]]
            wb *= mul[units[hdr.index("dram__bytes_write.sum")]]
            out.append(f"- DRAM traffic per launch: {(rb + wb) / 1e9:.3f} GB -> {(rb + wb) / t_s / 1e9:.0f} GB/s")
        except Exception as e:  # noqa: BLE001
            out.append(f"- (traffic not computed: {e})")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
