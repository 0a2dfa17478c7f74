"""Summarise `ncu --page raw --csv` exports (one row per profiled launch) into markdown for profiles/: time, DRAM
bytes and throughput, L2 hit rate, SM / issue / pipe utilisation, occupancy, and for the tensor-core kernels the
tensor-pipe and shared-memory wavefront activity.

usage: python tools/ncu_raw_summary.py RAW.csv [title] > profiles/r02/ncu_xxx.md"""
import csv
import sys

COLS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def fmt(name, unit, v):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if name.startswith("dram__bytes"):
        x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        return f"{x / 1e9:.3f} GB"
    if name == "gpu__time_duration.sum":
        x = x * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1)
        return f"{x:.3f} ms"
    return f"{x:.1f}" if abs(x) < 1e4 else f"{x:.0f}"


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# {title}\n")
    print("Source: `ncu --set full --clock-control none` (serialised, cold-cache launches; times are per launch).\n")
    present = [(c, lab) for c, lab in COLS if c in idx]
    print("| kernel | " + " | ".join(lab for _, lab in present) + " |")
    print("|---" * (len(present) + 1) + "|")
    for d in data:
        name = d[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")
        print(f"| `{name[:70]}` | " + " | ".join(fmt(c, units[idx[c]], d[idx[c]]) for c, _ in present) + " |")


if __name__ == "__main__":
    main()
